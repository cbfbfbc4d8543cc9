"""paper_1802_00330_b200: B200-native (sm_100a) engine for the data-parallel hot
path of arXiv 1802.00330 -- global interval branch-and-bound with
Hansen-Sengupta contraction -- behind the reference ``rootbox`` solver entry
point ``solve(PolySystem, SolverConfig) -> SolveResult`` (rootbox/bnb.py:224).

The compute path is librootbox_b200.so (CUDA, sm_100a) behind the C ABI in
include/rootbox_b200.h; there is no CPU fallback.
"""
__version__ = "0.1.0"

from .system import SystemSpec, compile_tables, as_spec  # noqa: F401
from .hansen import krawczyk, krawczyk_arrays  # noqa: F401, E402
from .bnb import (  # noqa: F401
    BUDGET_EXHAUSTED, NO_REAL_SOLUTION, WIDTH_REACHED, Box, Interval, RootBox, RootBoxes, RoundStats, SolveResult,
    SolverConfig, solve, solve_arrays,
)
