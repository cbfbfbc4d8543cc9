"""Short solve used as the ncu target (dev tool): python tools/prof_run.py CONFIG MAX_ROUNDS"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, load_spec
from paper_1802_00330_b200 import SolverConfig, solve_arrays
name, rounds = sys.argv[1], int(sys.argv[2])
sysname, kw, _ = CONFIGS[name]
kw = dict(kw); kw["max_rounds"] = rounds
from paper_1802_00330_b200 import bnb
spec = load_spec(sysname)
eng = bnb.engine_for(spec)
eng.set_option("graph", int(os.environ.get("RB_GRAPH", "1")))
eng.set_option("hs_fused", int(os.environ.get("RB_HS_FUSED", "1")))
out = solve_arrays(spec, SolverConfig(**kw))
print(name, out["status"], out["lo"].shape[0], f"{out['device_ms']:.2f} ms")
