"""Per-round phase timeline from device timestamps (dev tool).
RB_TRACE=1 python tools/trace_run.py CONFIG [graph] [hs_fused] [hs_cond]"""
import os, sys
os.environ.setdefault("RB_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, load_spec
from paper_1802_00330_b200 import SolverConfig, bnb
name = sys.argv[1]
graph, fused, cond = (int(sys.argv[i]) if len(sys.argv) > i else 1 for i in (2, 3, 4))
sysname, kw, _ = CONFIGS[name]
eng = bnb.engine_for(load_spec(sysname))
eng.set_option("graph", graph); eng.set_option("hs_fused", fused); eng.set_option("hs_cond", cond)
cfg = bnb.native_config(SolverConfig(**kw))
for _ in range(3):
    out = eng.solve(cfg)
print(f"{name} graph={graph} hs_fused={fused} hs_cond={cond}: device {out['device_ms']:.3f} ms", file=sys.stderr)
