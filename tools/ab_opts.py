"""A/B device time of engine options on one config (dev tool):
python tools/ab_opts.py CONFIG 'opt=v,opt=v' 'opt=v' ..."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, load_spec
from paper_1802_00330_b200 import SolverConfig, bnb
name = sys.argv[1]
sysname, kw, _ = CONFIGS[name]
eng = bnb.engine_for(load_spec(sysname))
cfg = bnb.native_config(SolverConfig(**kw))
reps = int(os.environ.get("REPS", "40"))
for variant in sys.argv[2:]:
    opts = [kv.split("=") for kv in variant.split(",") if kv]
    for k, v in opts:
        eng.set_option(k, int(v))
    eng.solve(cfg)
    ts, ws = [], []
    for _ in range(reps):
        t0 = time.perf_counter()
        ts.append(eng.solve(cfg)["device_ms"])
        ws.append(1e3 * (time.perf_counter() - t0))
    ts.sort(); ws.sort()
    print(f"{name:16s} {variant:28s} device median {ts[len(ts)//2]:8.3f} min {ts[0]:8.3f} ms, "
          f"host wall median {ws[len(ws)//2]:8.3f} min {ws[0]:8.3f} ms", flush=True)
