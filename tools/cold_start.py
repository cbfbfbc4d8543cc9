import sys, time
sys.path.insert(0, "/root/repo")
from bench import CONFIGS, load_spec
from paper_1802_00330_b200 import SolverConfig, bnb, _native
from paper_1802_00330_b200.system import compile_tables
sysname, kw, _ = CONFIGS["broyden_tri6"]
spec = load_spec(sysname)
cfg = bnb.native_config(SolverConfig(**kw))
t0 = time.perf_counter(); _native.lib(); t1 = time.perf_counter()
print(f"lib load {1e3*(t1-t0):.1f} ms")
for trial in range(3):
    t0 = time.perf_counter(); eng = _native.Engine(compile_tables(spec), 0); t1 = time.perf_counter()
    o = eng.solve(cfg); t2 = time.perf_counter(); o = eng.solve(cfg); t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms, first solve {1e3*(t2-t1):.1f} ms, second {1e3*(t3-t2):.2f} ms")
    eng.close()
