"""Cold vs warm instruction cache for k_hs_fused (dev tool): the same HS batch three
times in a row; run under ncu --cache-control none to compare launch durations."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import load_spec
from paper_1802_00330_b200 import bnb
spec = load_spec("broyden_tri6")
eng = bnb.engine_for(spec)
eng.set_option("codegen_wait", 1)
eng.set_option("hs_fused", 2)
rng = np.random.default_rng(0)
k = rng.integers(0, 2 ** 3, (2446, 6))
lo = spec.init_lo + k * (spec.init_hi - spec.init_lo) / 8
hi = lo + (spec.init_hi - spec.init_lo) / 8
for _ in range(3):
    eng.filter(lo[:8], hi[:8])  # another kernel in between (evicts nothing much: small)
    eng.hs(lo, hi, True)
    eng.hs(lo, hi, True)
