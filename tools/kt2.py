"""Filter variants for one config (dev tool): python tools/kt2.py eco8"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, load_spec
from paper_1802_00330_b200 import SolverConfig, bnb
for name in sys.argv[1].split(","):
    sysname, kw, _ = CONFIGS[name]
    spec = load_spec(sysname)
    eng = bnb.engine_for(spec)
    cfg = bnb.native_config(SolverConfig(**kw))
    eng.set_option("graph", 0)
    for tab in (0, 1):
        eng.set_option("filter_tab", tab)
        eng.solve(cfg)
        o = min((eng.solve(cfg) for _ in range(3)), key=lambda o: o["device_ms"])
        f = sum(s["filter_ms"] for s in o["stats"])
        print(f"{name} filter_tab={tab} total={o['device_ms']:.3f}ms filter={f:.3f}ms")
