"""Per-phase device times of the large BASELINE configs (host-driven rounds, CUDA
events around each phase): the A/B harness for filter / HS kernel changes.

    python tools/hs_bench.py [katsura6 brown8 broyden_banded12 eco8] [--reps 3] [--opt key=value ...]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS, load_spec  # noqa: E402
from paper_1802_00330_b200 import SolverConfig, bnb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=["katsura6", "brown8", "broyden_banded12", "eco8"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--opt", nargs="*", default=[])
    a = ap.parse_args()
    for name in a.names:
        sysname, kw, _ = CONFIGS[name]
        eng = bnb.engine_for(load_spec(sysname))
        eng.set_option("codegen_wait", 1)
        for o in a.opt:
            k, v = o.split("=")
            eng.set_option(k, int(v))
        cfg = bnb.native_config(SolverConfig(**kw))
        graph_ms = min(eng.solve(cfg)["device_ms"] for _ in range(a.reps))
        eng.set_option("graph", 0)
        best = None
        for _ in range(a.reps):
            o = eng.solve(cfg)
            f = sum(s["filter_ms"] for s in o["stats"]); h = sum(s["hs_ms"] for s in o["stats"])
            c = sum(s["classify_ms"] for s in o["stats"])
            if best is None or o["device_ms"] < best[0]:
                best = (o["device_ms"], f, h, c, o)
        eng.set_option("graph", 1)
        dev, f, h, c, o = best
        hs_ops = sum(s["hs_ops"] for s in o["stats"]); f_ops = sum(s["filter_ops"] for s in o["stats"])
        print(f"{name:18s} solve {graph_ms:8.2f} ms (host rounds {dev:8.2f}): filter {f:7.2f} ms "
              f"({f_ops / f / 1e9 if f else 0:6.2f} Gop/s)  hs {h:7.2f} ms ({hs_ops / h / 1e9 if h else 0:6.2f} Gop/s)"
              f"  classify {c:6.2f} ms  rounds {len(o['stats'])} boxes {o['lo'].shape[0]}", flush=True)
        per = [(s["round"], round(s["filter_ms"], 3), round(s["hs_ms"], 3), s["hs_calls"]) for s in o["stats"]]
        print("   per round (round, filter_ms, hs_ms, hs_calls):", per, flush=True)


if __name__ == "__main__":
    main()
