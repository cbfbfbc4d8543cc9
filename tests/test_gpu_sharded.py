"""The sharded solve protocol (dist.solve_sharded) with two ranks on the GPU.

Two processes over gloo on cuda:0, each with its own engine handle
(CudaShardBackend, rows exchanged through host memory): the device routing
kernels (rb_shard_route_count / rb_shard_route), the packed export/import, the
per-shard dedup and the final gather + device canonical order all run with
world size 2 -- no rank's kernel waits on the other's, so one GPU is a valid
stand-in for two.  Results must equal the reference goldens and the oracle's
full solve of brown8 (BASELINE config 4), bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu

CASES = ["circle_line", "broyden_tri6", "katsura3", "quirk17b", "rediff3_rounds3", "brown5", "katsura6_r3",
         "mickey_maxboxes", "broyden_tri4_nocontract", "conform1", "full:brown8"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from conftest import golden_spec, load_solve
    from test_full_solves import load_full
    from paper_1802_00330_b200 import SolverConfig
    from paper_1802_00330_b200.dist import CudaShardBackend, solve_sharded
    out = {}
    try:
        for case in CASES:
            meta = load_full(case[5:]) if case.startswith("full:") else load_solve(case)
            spec = golden_spec(meta["system"])
            be = CudaShardBackend(spec, 0, device_exchange=False)
            res = solve_sharded(spec, SolverConfig(**meta["config"]), backend=be)
            if rank == 0:
                b = res.boxes
                lo = np.array([[iv.lo for iv in rb.box] for rb in b]).reshape(-1, spec.n)
                hi = np.array([[iv.hi for iv in rb.box] for rb in b]).reshape(-1, spec.n)
                out[case] = {"status": res.status, "lo": lo, "hi": hi,
                             "cert": np.array([rb.certified for rb in b], bool),
                             "unsplit": np.array([rb.unsplittable for rb in b], bool),
                             "stats": [dict(round=s.round, boxes_in=s.boxes_in,
                                            boxes_after_filter=s.boxes_after_filter,
                                            boxes_after_hs=s.boxes_after_hs, width=s.width) for s in res.stats]}
        if rank == 0:
            q.put(out)
    except Exception as e:  # surface the worker's error in the test
        q.put({"error": repr(e)})
        raise
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_vs_goldens():
    from conftest import load_solve
    from test_full_solves import load_full
    from test_gpu_parity import check_against_golden
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=1200)
    for p in procs:
        p.join(timeout=120)
    assert "error" not in out, out.get("error")
    for p in procs:
        assert p.exitcode == 0
    for case in CASES:
        got = out[case]
        if case.startswith("full:"):
            meta = load_full(case[5:])
            assert got["status"] == meta["status"]
            assert [[s["round"], s["boxes_in"], s["boxes_after_filter"], s["boxes_after_hs"]] for s in got["stats"]] \
                == [r[:4] for r in meta["rounds"]]
            from test_full_solves import digest
            assert digest(got["lo"], got["hi"], got["cert"], got["unsplit"]) == meta["digest"]
        else:
            check_against_golden(case, got, load_solve(case))
