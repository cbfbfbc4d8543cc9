"""One host-driven solve of a BASELINE config (for ncu launch lists / captures):
    RB_CODEGEN=2 ncu ... python tools/prof_solve.py brown8 [--opt key=value ...]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS, load_spec  # noqa: E402
from paper_1802_00330_b200 import SolverConfig, bnb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("name")
ap.add_argument("--opt", nargs="*", default=[])
ap.add_argument("--graph", type=int, default=0)
a = ap.parse_args()
sysname, kw, _ = CONFIGS[a.name]
eng = bnb.engine_for(load_spec(sysname))
eng.set_option("codegen_wait", 1)
eng.set_option("graph", a.graph)
for o in a.opt:
    k, v = o.split("=")
    eng.set_option(k, int(v))
out = eng.solve(bnb.native_config(SolverConfig(**kw)))
print(a.name, out["status"], len(out["stats"]), out["lo"].shape[0], out["device_ms"])
