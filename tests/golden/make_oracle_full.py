"""Full-solve fixtures for the BASELINE configs the Python reference cannot finish.

TEST INFRASTRUCTURE ONLY.  The oracle (oracle/rootbox_oracle.c, the C
restatement of rootbox.bnb.solve, bnb.py:224-354) is pinned bit-exact against the
unmodified reference by tests/golden/make_golden.py on 25 complete solves and on
the first rounds of these very configs (solve_katsura6_r3, solve_eco8_r2,
solve_brown8_r2, solve_broyden_banded12_r1).  This script runs the same oracle
to completion on the BASELINE configs 3-5 (all host threads; the result is
independent of the thread count, see rootbox_oracle.c's header) and records:

  per round  (round, boxes_in, boxes_after_filter, boxes_after_hs, width as hex,
              children, hs_calls, dups)                      -- RoundStats, bnb.py:89-96
  final set  status, counts, SHA-256 of the canonical rows (_batch.py:244-266,
             same digest as make_golden.box_digest) and, up to 4096 rows, the rows
             themselves as float hex

    python tests/golden/make_oracle_full.py [--threads T] [NAME ...]

Output: tests/golden/full_<NAME>.json.  The -m gpu test
tests/test_full_solves.py solves each config on the device (graph and host round
loops) and asserts equality with these files.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

# name: (system in systems.json, SolverConfig kwargs) -- the same as bench.py CONFIGS
FULL = {
    "katsura6": ("katsura6", dict()),
    "eco8": ("eco8", dict()),
    "brown8": ("brown8", dict(target_width=1e-8)),
    "broyden_banded12": ("broyden_banded12", dict(target_width=1e-8)),
}
KEEP_ROWS = 4096


def box_digest(lo, hi, cert, unsplit):
    h = hashlib.sha256()
    lo = np.where(lo == 0.0, 0.0, lo)  # canonical +0
    hi = np.where(hi == 0.0, 0.0, hi)
    h.update(np.ascontiguousarray(lo, dtype="<f8").tobytes())
    h.update(np.ascontiguousarray(hi, dtype="<f8").tobytes())
    h.update(np.ascontiguousarray(cert, dtype=np.uint8).tobytes())
    h.update(np.ascontiguousarray(unsplit, dtype=np.uint8).tobytes())
    return h.hexdigest()


def load_system(name):
    with open(os.path.join(HERE, "systems.json")) as f:
        d = json.load(f)["systems"][name]
    eqs = [[(float.fromhex(c), tuple(e)) for c, e in p] for p in d["eqs"]]
    jac = [[[(float.fromhex(c), tuple(e)) for c, e in q] for q in row] for row in d["jac"]]
    ilo = [float.fromhex(v) if isinstance(v, str) else float(v) for v in d["init_lo"]]
    ihi = [float.fromhex(v) if isinstance(v, str) else float(v) for v in d["init_hi"]]
    return d["n"], eqs, jac, ilo, ihi


def run(name, threads):
    sysname, kw = FULL[name]
    n, eqs, jac, ilo, ihi = load_system(sysname)
    osys = O.OSystem(n, eqs, jac)
    t0 = time.time()
    r = osys.solve(ilo, ihi, threads=threads, **kw)
    wall = time.time() - t0
    st = r["stats"]
    rounds = [[int(x[0]), int(x[1]), int(x[2]), int(x[3]), float(x[4]).hex(), int(x[6]), int(x[7]), int(x[8])]
              for x in st]
    N = r["lo"].shape[0]
    out = {
        "case": name, "system": sysname, "config": kw, "status": r["status"],
        "generator": "tests/golden/make_oracle_full.py (oracle/rootbox_oracle.c, pinned by make_golden.py)",
        "oracle_wall_seconds": wall, "oracle_threads": threads,
        "rounds": rounds, "nboxes": int(N), "ncert": int(r["cert"].sum()), "nunsplit": int(r["unsplit"].sum()),
        "digest": box_digest(r["lo"], r["hi"], r["cert"], r["unsplit"]),
        "children_total": int(st[:, 6].sum()), "hs_calls_total": int(st[:, 7].sum()),
    }
    if N <= KEEP_ROWS:
        out["lo"] = [[float(v).hex() for v in row] for row in np.where(r["lo"] == 0.0, 0.0, r["lo"])]
        out["hi"] = [[float(v).hex() for v in row] for row in np.where(r["hi"] == 0.0, 0.0, r["hi"])]
        out["cert"] = [int(v) for v in r["cert"]]
        out["unsplit"] = [int(v) for v in r["unsplit"]]
    else:  # a few rows at both ends pin the order and give a readable failure
        sel = list(range(8)) + list(range(N - 8, N))
        out["sample_rows"] = sel
        out["sample_lo"] = [[float(v).hex() for v in r["lo"][i]] for i in sel]
        out["sample_hi"] = [[float(v).hex() for v in r["hi"][i]] for i in sel]
    path = os.path.join(HERE, f"full_{name}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(f"{name}: {r['status']} {len(rounds)} rounds {N} boxes ({out['ncert']} certified) "
          f"in {wall:.1f} s with {threads} threads -> {path}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("names", nargs="*", default=list(FULL))
    a = ap.parse_args()
    for name in a.names:
        run(name, a.threads)


if __name__ == "__main__":
    main()
