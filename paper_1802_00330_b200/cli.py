"""Run the reference's CLI (rootbox.cli) with the B200 engine as its solver.

    python -m paper_1802_00330_b200.cli solve katsura6 --format json

Rebinds ``rootbox.bnb.solve`` / ``rootbox.cli.solve`` / ``rootbox.solve`` (the
three import-time bindings: __init__.py:12, cli.py:26-34) to
``paper_1802_00330_b200.solve``, ``rootbox.cli.run_pipeline`` to the native
pipeline (B200 solve + exact native backtracking merge, pipeline.py) and the
report writers RunReport.to_json / to_csv to the native ones (byte-identical),
then calls ``rootbox.cli.main``.  Report formats and exit codes are the reference's own.
Requires the reference package to be importable.
"""
from __future__ import annotations

import sys


def install():
    """Make the reference package use the B200 engine; returns the rootbox module."""
    import rootbox
    import rootbox.bnb
    import rootbox.cli

    from .bnb import solve
    from .pipeline import report_to_csv, report_to_json, run_pipeline
    rootbox.bnb.solve = solve
    rootbox.cli.solve = solve
    rootbox.solve = solve
    rootbox.cli.run_pipeline = run_pipeline
    # the report writers: same bytes, roots section written natively (rb_format_boxes)
    rootbox.cli.RunReport.to_json = report_to_json
    rootbox.cli.RunReport.to_csv = report_to_csv
    return rootbox


def main(argv=None) -> int:
    rootbox = install()
    return rootbox.cli.main(argv)


if __name__ == "__main__":
    sys.exit(main())
