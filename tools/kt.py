"""Kernel-time totals per config with host-driven rounds (dev tool): python tools/kt.py [configs]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, load_spec
from paper_1802_00330_b200 import SolverConfig, bnb
names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["broyden_tri6", "katsura6", "eco8", "brown8", "broyden_banded12"]
fused = int(os.environ.get("RB_HS_FUSED", "1"))
for name in names:
    sysname, kw, _ = CONFIGS[name]
    spec = load_spec(sysname)
    eng = bnb.engine_for(spec)
    eng.set_option("hs_fused", fused)
    cfg = bnb.native_config(SolverConfig(**kw))
    eng.solve(cfg)
    g = min((eng.solve(cfg) for _ in range(3)), key=lambda o: o["device_ms"])
    eng.set_option("graph", 0)
    o = min((eng.solve(cfg) for _ in range(3)), key=lambda o: o["device_ms"])
    eng.set_option("graph", 1)
    st = o["stats"]
    f = sum(s["filter_ms"] for s in st); h = sum(s["hs_ms"] for s in st); c = sum(s["classify_ms"] for s in st)
    print(f"fused={fused} {name:18s} graph={g['device_ms']:8.3f}ms host={o['device_ms']:8.3f}ms filter={f:7.3f} hs={h:7.3f} classify={c:6.3f} status={o['status']} boxes={o['lo'].shape[0]}")
