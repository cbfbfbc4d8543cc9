"""Where the end-to-end time of solve() goes beyond the device time (headline config)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import load_spec  # noqa: E402
from paper_1802_00330_b200 import SolverConfig, bnb, solve  # noqa: E402
from paper_1802_00330_b200 import _native  # noqa: E402

spec = load_spec("broyden_tri6")
cfg = SolverConfig(target_width=1e-8)
for _ in range(50):
    solve(spec, cfg)
R = 2000


def timeit(f):
    t = time.perf_counter()
    for _ in range(R):
        f()
    return 1e6 * (time.perf_counter() - t) / R


eng = bnb.engine_for(spec)
ncfg = bnb.native_config(cfg)
print(f"solve()                         {timeit(lambda: solve(spec, cfg)):8.1f} us")
print(f"engine_for + native_config      {timeit(lambda: (bnb.engine_for(spec), bnb.native_config(cfg))):8.1f} us")
print(f"validate_config                 {timeit(lambda: bnb.validate_config(cfg)):8.1f} us")
print(f"Engine.solve (no device timing) {timeit(lambda: eng.solve(ncfg, stats_rows=True, device_timing=False)):8.1f} us")
out = eng.solve(ncfg, stats_rows=True, device_timing=False)
print(f"_own_result                     {timeit(lambda: bnb._own_result(out)):8.1f} us")
info = _native.RbResultInfo()
L = _native.lib()
import ctypes as C  # noqa: E402
print(f"rb_solve alone                  {timeit(lambda: L.rb_solve(eng.h, C.byref(ncfg), C.byref(info))):8.1f} us")
