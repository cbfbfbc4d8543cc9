"""Where the end-to-end solve() time goes beyond the device time (dev tool)."""
import os, sys, time, cProfile, pstats
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, load_spec
from paper_1802_00330_b200 import SolverConfig, bnb, solve
sysname, kw, _ = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "broyden_tri6"]
spec = load_spec(sysname)
cfg = SolverConfig(**kw)
eng = bnb.engine_for(spec)
ncfg = bnb.native_config(cfg)
for _ in range(20):
    solve(spec, cfg)
N = 200
t0 = time.perf_counter()
for _ in range(N):
    o = eng.solve(ncfg)
t1 = time.perf_counter()
for _ in range(N):
    r = solve(spec, cfg)
t2 = time.perf_counter()
print(f"engine.solve wall {1e3*(t1-t0)/N:.3f} ms (device {o['device_ms']:.3f}), public solve {1e3*(t2-t1)/N:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    solve(spec, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
