"""Backtracking merge of a BASELINE result: host (rb_merge) vs device (rb_merge_device).
    python tools/merge_bench.py [katsura6]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS, load_spec  # noqa: E402
from paper_1802_00330_b200 import SolverConfig, solve_arrays  # noqa: E402
from paper_1802_00330_b200.pipeline import merge_arrays  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "katsura6"
sysname, kw, _ = CONFIGS[name]
spec = load_spec(sysname)
out = solve_arrays(spec, SolverConfig(**kw))
for dev in (None, 0, 0, 0):
    t = time.perf_counter()
    r = merge_arrays(spec.init_lo, spec.init_hi, out["lo"], out["hi"], out["cert"], device=dev)
    print(f"{name}: {out['lo'].shape[0]} boxes -> {r[0].shape[0]} merged, levels {len(r[3])}, "
          f"{'host' if dev is None else 'device'} {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
