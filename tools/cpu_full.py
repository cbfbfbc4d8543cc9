"""Time the oracle (C restatement of the reference algorithm) on full solves (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, load_spec
from oracle import oracle as O
threads = int(sys.argv[2]) if len(sys.argv) > 2 else os.cpu_count()
for name in sys.argv[1].split(","):
    sysname, kw, _ = CONFIGS[name]
    spec = load_spec(sysname)
    osys = O.OSystem(spec.n, spec.eqs, spec.jac)
    t0 = time.perf_counter()
    r = osys.solve(spec.init_lo, spec.init_hi, threads=threads, **kw)
    dt = time.perf_counter() - t0
    boxes = int(r["stats"][:, 6].sum() + r["stats"][:, 7].sum())
    print(f"{name}: {r['status']} rounds={len(r['stats'])} final={r['lo'].shape[0]} cert={int(r['cert'].sum())} "
          f"threads={threads} wall={dt:.2f}s boxes={boxes} boxes/s={boxes/dt:.3e}", flush=True)
