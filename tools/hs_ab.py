"""Per-round HS time, fused vs three-kernel, against the round's HS row count (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, load_spec
from paper_1802_00330_b200 import SolverConfig, bnb
names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["broyden_tri6", "katsura6", "eco8", "brown8", "broyden_banded12"]
for name in names:
    sysname, kw, _ = CONFIGS[name]
    spec = load_spec(sysname)
    eng = bnb.engine_for(spec)
    cfg = bnb.native_config(SolverConfig(**kw))
    eng.set_option("graph", 0)
    res = {}
    for fused in (0, 2, 1):
        eng.set_option("hs_fused", fused)
        eng.solve(cfg)
        runs = [eng.solve(cfg) for _ in range(3)]
        res[fused] = [min(r["stats"][i]["hs_ms"] for r in runs) for i in range(len(runs[0]["stats"]))]
        st = runs[0]["stats"]
    print(f"== {name} n={spec.n}")
    for i, s in enumerate(st):
        print(f"  r{s['round']:2d} hs_rows={s['boxes_after_filter']:9d} three={res[0][i]*1e3:9.1f}us fused={res[2][i]*1e3:9.1f}us auto={res[1][i]*1e3:9.1f}us")
    eng.set_option("graph", 1); eng.set_option("hs_fused", 1)
