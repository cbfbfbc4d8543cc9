"""Solve a BASELINE config on the GPU with a round cap and print per-round stats (dev tool).
The solve runs twice in one process; the second (warm memory pool) is reported."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, load_spec
from paper_1802_00330_b200 import SolverConfig, solve_arrays

name = sys.argv[1]
max_rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 24
max_seconds = float(sys.argv[3]) if len(sys.argv) > 3 else None
sysname, kw, desc = CONFIGS[name]
spec = load_spec(sysname)
kw = dict(kw)
kw["max_rounds"] = max_rounds
if max_seconds:
    kw["max_seconds"] = max_seconds
for rep in range(2):
    t0 = time.time()
    out = solve_arrays(spec, SolverConfig(**kw))
    wall = time.time() - t0
print(f"{name}: {out['status']} final={out['lo'].shape[0]} cert={int(out['cert'].sum())} "
      f"uns={int(out['unsplit'].sum())} wall={wall:.3f}s dev={out['device_ms']:.2f}ms launches={out['kernel_launches']}")
for s in out["stats"]:
    print("  r{round:2d} in={boxes_in:>11d} filt={boxes_after_filter:>11d} hs={boxes_after_hs:>11d} w={width:.3g} "
          "ch={children:>12d} hsc={hs_calls:>10d} ex={exact_boxes} dup={dups} att={attempts} "
          "cls={classify_ms:.3f} filt={filter_ms:.3f} hs={hs_ms:.3f}ms el={elapsed_seconds:.3f}s".format(**s))
