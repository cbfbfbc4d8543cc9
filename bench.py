#!/usr/bin/env python
"""Benchmark: boxes/s and time-to-all-solutions of the interval B&B + HS solve on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl ours|reference]

A step is one complete solve (rootbox.bnb.solve semantics, bnb.py:224-354) of
the configured system to its target width.  Default workload: BASELINE.json
configs[1], Broyden tridiagonal n=6 on [-2,2]^6, eps=1e-8.

boxes = children evaluated by the filter (active parents x 2^n, every round)
      + boxes contracted by Hansen-Sengupta.
value = boxes of all ranks / max over ranks of the device time of the K steps
        (CUDA events on the engine's stream, first to last op of each solve).
e2e   = the same metric through the public API ``paper_1802_00330_b200.solve``
        from host buffers: engine creation (table upload H2D), solve, result
        fetch (D2H) and Python SolveResult construction, timed on the host.

Multi-GPU (--gpus N > 1; re-launched under torch.distributed.run when WORLD_SIZE
is unset, one rank per GPU): the line is BASELINE config 4, Brown n=8, solved with
its frontier sharded across the ranks (strong scaling, dist.solve_sharded).  The
N = 1 line carries the same solve on one GPU under "sharded", the curve's first
point.

--impl reference times the reference algorithm's CPU implementation (the C
restatement in oracle/, all host threads) on the same workload and metric;
rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (system, SolverConfig kwargs, description)
    "circle_line": ("circle_line", dict(target_width=1e-6), "circle-line x^2+y^2-1, x-y on [-2,2]^2, eps=1e-6"),
    "broyden_tri6": ("broyden_tri6", dict(target_width=1e-8), "Broyden tridiagonal n=6 on [-2,2]^6, eps=1e-8"),
    "katsura6": ("katsura6", dict(), "Katsura-6 (7 vars) on [-1,1]^7, default eps 2^-9, HS width 1.0"),
    "eco8": ("eco8", dict(), "eco8 on [-8,8]^8, default eps 2^-6, HS width 1.0"),
    "brown8": ("brown8", dict(target_width=1e-8), "Brown almost-linear n=8 on [-2,2]^8, eps=1e-8"),
    "broyden_banded12": ("broyden_banded12", dict(target_width=1e-8),
                         "Broyden banded n=12 on [-1,1]^12, eps=1e-8"),
}


def load_spec(name):
    from paper_1802_00330_b200 import SystemSpec
    with open(os.path.join(ROOT, "tests", "golden", "systems.json")) as f:
        d = json.load(f)["systems"][name]
    return SystemSpec.from_json(d, name=name)


def boxes_of(stats):
    return int(sum(s["children"] + s["hs_calls"] for s in stats))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()  # nvidia-smi takes a while to start: wait for its first sample
            while not self.lines and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.skip = len(self.lines)  # idle samples before the measured work
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines[getattr(self, "skip", 0):]:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax = float(p[2])
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def l2_flush(buf):
    if buf is not None:
        buf.add_(1.0)  # 512 MiB read+write > 126 MB L2


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.impl == "ours":
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(world, v, local):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v)], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(world, v, local):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v)], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def cpu_baseline(spec, kw, budget_s=10.0, threads=None):
    """The oracle (C restatement of the reference algorithm) on the host cores:
    repeated full solves of the same workload for ~budget_s seconds.  Run in a
    child process (cpu_baseline_subprocess) so the GPU arm's process never maps
    the oracle library."""
    from oracle import oracle as O
    threads = threads or os.cpu_count() or 1
    osys = O.OSystem(spec.n, spec.eqs, spec.jac)
    reps, boxes, t_total = 0, 0, 0.0
    status = None
    while t_total < budget_s and reps < 1000:
        t0 = time.perf_counter()
        r = osys.solve(spec.init_lo, spec.init_hi, threads=threads, **kw)
        t_total += time.perf_counter() - t0
        boxes += int(r["stats"][:, 6].sum() + r["stats"][:, 7].sum())
        status = r["status"]
        reps += 1
    return {"value": boxes / t_total, "unit": "boxes/s", "cores": threads, "kind": "port",
            "sample": f"{reps} complete solve(s) of the same workload ({status}), "
                      f"{t_total:.2f} s of CPU wall time, oracle/rootbox_oracle.c with {threads} threads",
            "time_to_solution_s": t_total / reps}


def cpu_baseline_subprocess(config, budget_s):
    """cpu_baseline of a CONFIGS entry in a child interpreter (prints one JSON object)."""
    out = subprocess.run([sys.executable, os.path.abspath(__file__), "--cpu-baseline-child", config,
                          "--cpu-seconds", str(budget_s)], capture_output=True, text=True, timeout=600)
    if out.returncode != 0:
        return {"unavailable": out.stderr.strip().splitlines()[-1:] or ["cpu baseline child failed"]}
    return json.loads(out.stdout.strip().splitlines()[-1])


def cpu_baseline_child(config, budget_s):
    sysname, kw, desc = CONFIGS[config]
    print(json.dumps(cpu_baseline(load_spec(sysname), kw, budget_s=budget_s)), flush=True)


def other_configs(args, device, peak):
    """The throughput-bound BASELINE configs solved completely on this GPU (not the
    headline line; evidence for the kernels' rooflines at scale)."""
    from paper_1802_00330_b200 import SolverConfig, bnb
    res = {}
    for name in ("katsura6", "eco8", "brown8", "broyden_banded12"):
        if name == args.config:
            continue
        sysname, kw, desc = CONFIGS[name]
        spec = load_spec(sysname)
        eng = bnb.engine_for(spec, device)
        eng.set_option("codegen_wait", 1)
        ncfg = bnb.native_config(SolverConfig(**kw))
        eng.solve(ncfg)  # warm: buffers sized, memory pool populated
        best = None
        for _ in range(2):
            o = eng.solve(ncfg)
            if best is None or o["device_ms"] < best["device_ms"]:
                best = o
        st = best["stats"]
        eng.set_option("graph", 0)  # kernel times need host-driven rounds
        prof = eng.solve(ncfg)["stats"]
        eng.set_option("graph", 1)
        f_ms = sum(x["filter_ms"] for x in prof); h_ms = sum(x["hs_ms"] for x in prof)
        f_ops = sum(x["filter_ops"] for x in st); h_ops = sum(x["hs_ops"] for x in st)
        boxes = boxes_of(st)
        # end to end through the public API from host buffers (drop-in solve(): result
        # rows D2H, lazy SolveResult for large sets)
        from paper_1802_00330_b200 import solve as public_solve
        public_solve(spec, SolverConfig(**kw))  # warm: the round graph is re-captured after the graph=0 pass
        e2e = []
        for _ in range(3):
            t0 = time.perf_counter()
            public_solve(spec, SolverConfig(**kw))
            e2e.append(time.perf_counter() - t0)
        dom = ("k_hs_eval+k_hs_lin+k_hs_sweep", h_ops, h_ms) if h_ms >= f_ms else ("k_filter", f_ops, f_ms)
        ach = dom[1] / (dom[2] * 1e-3) if dom[2] > 0 else 0.0
        res[name] = {"workload": desc, "status": best["status"], "rounds": len(st),
                     "final_boxes": int(best["lo"].shape[0]), "certified": int(best["cert"].sum()),
                     "time_to_solution_ms": best["device_ms"], "e2e_time_to_solution_ms": 1e3 * min(e2e),
                     "boxes": boxes,
                     "boxes_per_s": boxes / (best["device_ms"] * 1e-3),
                     "filter_ms": f_ms, "hs_ms": h_ms,
                     "roofline": {"bound": "fp64", "kernel": dom[0], "achieved": ach / 1e12, "peak": peak / 1e12,
                                  "unit": "TFLOP/s", "frac": ach / peak if peak else None}}
    return res


def run_reference(args, world, rank):
    if rank != 0:
        return
    config = args.config if world == 1 else "brown8"  # N > 1: the workload of run_scaling
    sysname, kw, desc = CONFIGS[config]
    spec = load_spec(sysname)
    from oracle import oracle as O
    threads = os.cpu_count() or 1
    osys = O.OSystem(spec.n, spec.eqs, spec.jac)
    sample = "complete solves"
    if world > 1:
        # a complete Brown-8 solve takes minutes on the host: each step is its first 4
        # rounds (4.4M children, 0.71M HS boxes), a bounded sample of the same workload
        kw = dict(kw, max_rounds=4)
        sample = "rounds 1-4 of the solve per step (bounded sample; boxes/s over those rounds)"
    for _ in range(args.warmup if world == 1 else 0):
        osys.solve(spec.init_lo, spec.init_hi, threads=threads, **kw)
    times, boxes = [], 0
    budget = 150.0 if world > 1 else float("inf")
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r = osys.solve(spec.init_lo, spec.init_hi, threads=threads, **kw)
        times.append(time.perf_counter() - t0)
        boxes += int(r["stats"][:, 6].sum() + r["stats"][:, 7].sum())
        if sum(times) > budget:
            break
    args.steps = len(times)
    total = sum(times)
    value = boxes / total
    thr = None
    if world == 1 and args.config == "broyden_tri6" and not args.no_other_configs:
        # the throughput-bound BASELINE config 4 (Brown n=8), one complete solve on all host
        # threads, so the same run holds a CPU time-to-solution for the large-frontier case
        tname, tkw, tdesc = CONFIGS["brown8"]
        tspec = load_spec(tname)
        tsys = O.OSystem(tspec.n, tspec.eqs, tspec.jac)
        t0 = time.perf_counter()
        r = tsys.solve(tspec.init_lo, tspec.init_hi, threads=threads, **tkw)
        tt = time.perf_counter() - t0
        tb = int(r["stats"][:, 6].sum() + r["stats"][:, 7].sum())
        thr = {"workload": tdesc, "system": tname, "status": r["status"], "final_boxes": int(r["lo"].shape[0]),
               "time_to_solution_s": tt, "boxes": tb, "boxes_per_s": tb / tt, "cores": threads,
               "kind": "port", "sample": "1 complete solve, oracle/rootbox_oracle.c"}
    line = {
        "impl": "reference", "metric": "boxes/s (children evaluated + HS boxes contracted) per complete solve",
        "value": value, "unit": "boxes/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic benchmark system)",
        "config": {"workload": desc, "system": sysname, "time_to_solution_s": total / args.steps},
        "cpu_baseline": {"value": value, "unit": "boxes/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} steps ({sample}), oracle/rootbox_oracle.c with {threads} threads"},
        "e2e": {"value": value, "unit": "boxes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if thr:
        line["throughput_config"] = thr
    print(json.dumps(line), flush=True)


def run_ours(args, world, rank, local):
    import torch
    from paper_1802_00330_b200 import SolverConfig, _native, bnb
    sysname, kw, desc = CONFIGS[args.config]
    spec = load_spec(sysname)
    cfg = SolverConfig(**kw)
    torch.cuda.set_device(local)
    flush = torch.zeros(128 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")  # 512 MiB
    eng = bnb.engine_for(spec, local)
    eng.set_option("codegen_wait", 1)  # steady state: the system-specialised kernels (compiled once, cached)
    kernels_active, kernels_why = eng.codegen_active()
    ncfg = bnb.native_config(cfg)
    sampler = ClockSampler(local)
    sampler.start()  # clocks sampled through warm-up and the timed region
    for _ in range(max(3, args.warmup)):
        out = eng.solve(ncfg)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    dev_ms, boxes, launches = [], 0, 0
    t_wall0 = time.perf_counter()
    for _ in range(args.steps):
        l2_flush(flush)
        torch.cuda.synchronize()
        out = eng.solve(ncfg)
        dev_ms.append(out["device_ms"])
        boxes += boxes_of(out["stats"])
        launches += out["kernel_launches"]
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_wall0
    # nvidia-smi samples every 50 ms, longer than a K-step timed region of sub-ms solves:
    # the same solves continue untimed for 0.6 s so the sampler sees the clocks under
    # this load (the samples span warm-up, the timed region and this window)
    t_win = time.perf_counter() + 0.6
    while time.perf_counter() < t_win:
        eng.solve(ncfg)
    torch.cuda.synchronize()
    barrier(world)
    clocks = sampler.stop()
    clocks["window"] = "warm-up + timed steps + 0.6 s of the same solves right after"
    # per-kernel device times (CUDA events around each kernel) need host-driven
    # rounds: a separate pass with the device round loop switched off
    filt_ms = hs_ms = cls_ms = 0.0
    filt_ops = hs_ops = cls_bytes = 0
    prof_steps = max(3, min(args.steps, 50))
    eng.set_option("graph", 0)
    host_ms = []
    for _ in range(prof_steps):
        l2_flush(flush)
        torch.cuda.synchronize()
        o = eng.solve(ncfg)
        host_ms.append(o["device_ms"])
        for s_ in o["stats"]:
            filt_ms += s_["filter_ms"]; hs_ms += s_["hs_ms"]; cls_ms += s_["classify_ms"]
            filt_ops += s_["filter_ops"]; hs_ops += s_["hs_ops"]; cls_bytes += s_["classify_bytes"]
    eng.set_option("graph", 1)
    t_dev = sum(dev_ms) * 1e-3
    t_max = allreduce_max(world, t_dev, local)
    boxes_all = allreduce_sum(world, boxes, local)
    value = boxes_all / t_max
    status = out["status"]
    nrounds = len(out["stats"])
    nfinal = out["lo"].shape[0]

    # ---- e2e through the public API from host buffers.  Serving semantics: the
    # compiled system stays resident (engine cache, like model weights); every
    # step sends the step's input (initial box + config) H2D, solves, reads the
    # result (boxes, flags, round stats) D2H and builds the SolveResult objects.
    from paper_1802_00330_b200 import solve as public_solve
    from paper_1802_00330_b200 import _native as nat
    import ctypes
    e2e_steps = max(3, min(args.steps, 500))
    public_solve(spec, cfg)
    e2e_t = []
    for _ in range(e2e_steps):
        l2_flush(flush)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = public_solve(spec, cfg)
        e2e_t.append(time.perf_counter() - t0)
    assert len(res.boxes) == nfinal and res.status == status
    e2e_value = allreduce_sum(world, boxes_of(out["stats"]) * e2e_steps, local) / allreduce_max(world, sum(e2e_t), local)
    h2d = spec.n * 16 + ctypes.sizeof(nat.RbConfig)
    d2h = nfinal * spec.n * 16 + 2 * nfinal + nrounds * ctypes.sizeof(nat.RbRoundStats)
    # cold start: first solve of a system in a process (engine creation + table upload + buffers)
    cold_t = []
    for _ in range(3):
        bnb._ENGINES.clear()
        t0 = time.perf_counter()
        public_solve(spec, cfg)
        cold_t.append(time.perf_counter() - t0)

    # ---- roofline of the dominant kernel (FP64 directed-op pipe)
    peak = _native.fp64_peak(local)
    if hs_ms >= filt_ms:
        dom, ops, ms = "k_hs (Hansen-Sengupta)", hs_ops, hs_ms
    else:
        dom, ops, ms = "k_filter (bisect+inclusion filter+compaction)", filt_ops, filt_ms
    achieved = ops / (ms * 1e-3) if ms > 0 else 0.0
    # DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture
    traffic = None
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        kname = (f"k_hs_fused<{spec.n}>" if dom.startswith("k_hs") else f"k_filter<{spec.n}>")
        t = json.load(open(tpath)).get(kname)
        if t:
            traffic = {"kernel": kname, "dram_bytes_per_launch": t["dram_bytes_per_launch"], "source": t["source"], "kernel_name": t.get("kernel_name", kname)}
    roofline = {"bound": "fp64", "kernel": dom, "achieved": achieved / 1e12, "peak": peak / 1e12,
                "unit": "TFLOP/s", "frac": achieved / peak if peak else None, "traffic": traffic,
                "note": "1 directed FP64 op (DMUL/DADD.RM/RP) = 1 FLOP; peak = measured directed-op throughput "
                        "of this B200 (rb_fp64_peak microbenchmark); algorithmic ops per SURVEY §8(d)",
                "share_of_step": {"filter_ms": filt_ms / prof_steps, "hs_ms": hs_ms / prof_steps,
                                  "classify_ms": cls_ms / prof_steps,
                                  "device_ms_host_driven_rounds": statistics.mean(host_ms),
                                  "device_ms_graph_rounds": sum(dev_ms) / args.steps},
                "classify_hbm_gbs": (cls_bytes / (cls_ms * 1e-3) / 1e9) if cls_ms > 0 else None}

    line = {
        "metric": "boxes/s (children evaluated + HS boxes contracted) per complete solve",
        "value": value, "unit": "boxes/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sum(dev_ms) / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic benchmark system)",
        "config": {"workload": desc, "system": sysname, "status": status, "rounds": nrounds,
                   "final_boxes": nfinal, "boxes_per_step": boxes // args.steps,
                   "time_to_solution_ms": sum(dev_ms) / args.steps,
                   "l2": "flushed between steps (512 MiB write)", "parallelism": f"replicas x{world}",
                   "kernels": "system-specialised (NVRTC)" if kernels_active else f"table kernels ({kernels_why})",
                   "host_wall_ms_per_step": 1e3 * wall / args.steps},
        "e2e": {"value": e2e_value, "unit": "boxes/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "time_to_solution_ms": 1e3 * statistics.mean(e2e_t),
                "path": "paper_1802_00330_b200.solve(spec, cfg) -> SolveResult objects; compiled system resident, "
                        "initial box + config H2D and boxes + flags + round stats D2H every step",
                "cold_start_ms": 1e3 * statistics.mean(cold_t)},
        "gpu_launches": int(launches),
        "roofline": roofline,
        "clocks": clocks,
    }
    if not args.no_other_configs:
        # the N > 1 lines are the strong-scaled brown8 solve (run_scaling); this is its
        # single-GPU point, so the scaling curve has a same-workload N = 1 value
        line["sharded"] = sharded_solve(args, world, rank, local, config=args.sharded or "brown8")
    if rank == 0 and world == 1 and not args.no_other_configs:
        line["other_configs"] = other_configs(args, local, peak)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_subprocess(args.config, args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)


def sharded_solve(args, world, rank, local, config="brown8", steps=None):
    """BASELINE config 4 (Brown n=8, large frontier) solved with its frontier sharded
    across the ranks (dist.solve_sharded: two all_gathers per round, thin-row owner
    routing and surplus rebalancing over one all_to_all).  The protocol synchronises
    with the host every round, so a step is timed by the host clock bracketed by a
    barrier and torch.cuda.synchronize() on every rank, max over ranks.  At world size 1
    the solve is the engine's own (nothing to exchange)."""
    import torch
    from paper_1802_00330_b200 import SolverConfig
    from paper_1802_00330_b200.dist import CudaShardBackend, solve_sharded
    sysname, kw, desc = CONFIGS[config]
    spec = load_spec(sysname)
    cfg = SolverConfig(**kw)
    backend = CudaShardBackend(spec, local, device_exchange=True)
    backend.eng.set_option("codegen_wait", 1)
    steps = steps or args.sharded_steps
    for _ in range(max(1, min(args.warmup, 3))):
        out = solve_sharded(spec, cfg, backend=backend, arrays=True)  # warm: buffers, kernels
    ts = []
    from paper_1802_00330_b200 import _native
    launches = 0
    for _ in range(steps):
        barrier(world)
        torch.cuda.synchronize()
        l0 = _native.lib().rb_kernel_launches(backend.eng.h)
        t0 = time.perf_counter()
        out = solve_sharded(spec, cfg, backend=backend, arrays=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        # world 1 runs rb_solve (its own count); otherwise the protocol's calls accumulate
        launches += int(out["kernel_launches"]) if world == 1 else \
            int(_native.lib().rb_kernel_launches(backend.eng.h) - l0)
    barrier(world)
    t = allreduce_max(world, sum(ts), local)
    launches = int(allreduce_sum(world, launches, local))
    boxes = None
    if rank == 0:
        boxes = int(sum(st["children"] + st["hs_calls"] for st in out["stats"]))
    # end to end through the public API: solve_sharded(spec, cfg) -> SolveResult on rank 0
    solve_sharded(spec, cfg)  # warm: the public path's cached engine
    e2e_t = []
    for _ in range(max(1, min(steps, 5))):
        barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = solve_sharded(spec, cfg)
        torch.cuda.synchronize()
        e2e_t.append(time.perf_counter() - t0)
    barrier(world)
    te = allreduce_max(world, sum(e2e_t), local)
    if rank != 0:
        return None
    return {"workload": desc, "system": sysname, "n_gpus": world, "steps": steps, "status": out["status"],
            "rounds": len(out["stats"]), "final_boxes": int(out["lo"].shape[0]), "boxes_per_step": boxes,
            "time_to_solution_ms": 1e3 * t / steps, "boxes_per_s": boxes * steps / t,
            "e2e_time_to_solution_ms": 1e3 * te / len(e2e_t), "e2e_boxes_per_s": boxes * len(e2e_t) / te,
            "gpu_launches": launches,
            "timing": "host clock between barrier+synchronize, max over ranks",
            "path": "dist.solve_sharded (world 1: the engine's own solve)",
            "final_result_type": type(res.boxes).__name__}


def run_scaling(args, world, rank, local):
    """N > 1: the headline line is BASELINE config 4 (Brown n=8) strong-scaled over
    the N ranks: fixed total work, value = boxes of the whole solve / time."""
    import torch
    torch.cuda.set_device(local)
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    sh = sharded_solve(args, world, rank, local, config="brown8", steps=args.steps)
    clocks = sampler.stop() if sampler else None
    if rank != 0:
        return
    spec = load_spec("brown8")
    line = {
        "metric": "boxes/s (children evaluated + HS boxes contracted) per complete solve",
        "value": sh["boxes_per_s"], "unit": "boxes/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sh["time_to_solution_ms"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (deterministic benchmark system)",
        "config": {"workload": sh["workload"], "system": "brown8", "status": sh["status"], "rounds": sh["rounds"],
                   "final_boxes": sh["final_boxes"], "boxes_per_step": sh["boxes_per_step"],
                   "time_to_solution_ms": sh["time_to_solution_ms"], "parallelism": f"frontier sharded x{world}",
                   "l2": "inputs (frontiers of 10^5-10^6 rows x 128 B) exceed L2 in the large rounds"},
        "e2e": {"value": sh["e2e_boxes_per_s"], "unit": "boxes/s", "h2d_bytes_per_step": int(spec.n * 16),
                "d2h_bytes_per_step": int(sh["final_boxes"] * (16 * spec.n + 2)),
                "time_to_solution_ms": sh["e2e_time_to_solution_ms"],
                "path": "paper_1802_00330_b200.dist.solve_sharded(spec, cfg) -> SolveResult on rank 0"},
        "gpu_launches": sh["gpu_launches"],
        "clocks": clocks,
        "timing": sh["timing"],
    }
    print(json.dumps(line), flush=True)


def self_launch(args):
    """bench.py --gpus N without torchrun: re-run under torch.distributed.run with one
    process per GPU (127.0.0.1 rendezvous)."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if args.gpus > have:
        print(json.dumps({"error": f"--gpus {args.gpus} but only {have} CUDA device(s) visible"}), flush=True)
        sys.exit(2)
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="broyden_tri6")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--sharded", choices=sorted(CONFIGS), default=None,
                    help="config of the single-GPU sharded-solve object (default brown8)")
    ap.add_argument("--sharded-steps", type=int, default=5)
    ap.add_argument("--cpu-baseline-child", default=None, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.cpu_baseline_child:
        cpu_baseline_child(args.cpu_baseline_child, args.cpu_seconds)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)
    world, rank, local = dist_setup(args)
    if world != args.gpus and rank == 0:
        print(f"bench: WORLD_SIZE={world} but --gpus {args.gpus}; measuring {world} rank(s)", file=sys.stderr)
    try:
        if args.impl == "reference":
            run_reference(args, world, rank)
        elif world > 1:
            run_scaling(args, world, rank, local)
        else:
            run_ours(args, world, rank, local)
    finally:
        if world > 1 and args.impl == "ours":
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
