import os, sys
sys.path.insert(0, "/root/repo")
from bench import CONFIGS, load_spec
from paper_1802_00330_b200 import SolverConfig, bnb
name = sys.argv[1]
sysname, kw, _ = CONFIGS[name]
eng = bnb.engine_for(load_spec(sysname))
cfg = bnb.native_config(SolverConfig(**kw))
for fused, cond in ((0, 1), (2, 1), (1, 1), (1, 0)):
    eng.set_option("hs_fused", fused); eng.set_option("hs_cond", cond)
    ts = sorted(eng.solve(cfg)["device_ms"] for _ in range(50))
    print(f"{name} hs_fused={fused} hs_cond={cond}: median {ts[25]:.3f} min {ts[0]:.3f} ms")
