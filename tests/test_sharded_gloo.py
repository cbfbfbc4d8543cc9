"""Multi-rank driver (dist.solve_sharded) on CPU: world_size 2 over gloo with the
oracle shard backend; results must equal the reference's own single-process
solve (golden fixtures) -- statistics and boxes, bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT, assert_bits_equal, golden_jac, golden_spec, load_solve

CASES = ["circle_line", "broyden_tri4", "mickey", "rediff3", "noon3", "katsura3", "conform1", "quirk17b",
         "broyden_tri4_nocontract", "circle_line_nohs", "mickey_maxboxes", "rediff3_rounds3"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from shard_backends import OracleShardBackend
    from paper_1802_00330_b200 import SolverConfig
    from paper_1802_00330_b200.dist import solve_sharded
    out = {}
    try:
        for case in cases:
            meta = load_solve(case)
            spec = golden_spec(meta["system"])
            be = OracleShardBackend(spec, golden_jac(meta["system"]))
            res = solve_sharded(spec, SolverConfig(**meta["config"]), backend=be)
            if rank == 0:
                lo = np.array([[iv.lo for iv in rb.box] for rb in res.boxes]).reshape(-1, spec.n)
                hi = np.array([[iv.hi for iv in rb.box] for rb in res.boxes]).reshape(-1, spec.n)
                out[case] = (res.status, [(s.round, s.boxes_in, s.boxes_after_filter, s.boxes_after_hs, s.width)
                                          for s in res.stats], lo, hi,
                             [rb.certified for rb in res.boxes], [rb.unsplittable for rb in res.boxes])
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_driver_matches_reference(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for case in CASES:
        meta = load_solve(case)
        status, stats, lo, hi, cert, uns = out[case]
        assert status == meta["status"], case
        assert [list(s[:4]) for s in stats] == [w[:4] for w in meta["stats"]], case
        for s, w in zip(stats, meta["stats"]):
            assert float(s[4]).hex() == w[4] or float(s[4]) == float.fromhex(w[4]), case
        assert lo.shape[0] == meta["nboxes"], case
        if "lo" in meta:
            want_lo = np.array([[float.fromhex(v) for v in r] for r in meta["lo"]]).reshape(lo.shape)
            want_hi = np.array([[float.fromhex(v) for v in r] for r in meta["hi"]]).reshape(hi.shape)
            assert_bits_equal(lo, want_lo, case)
            assert_bits_equal(hi, want_hi, case)
            assert [int(v) for v in cert] == meta["cert"] and [int(v) for v in uns] == meta["unsplit"], case


def test_rebalance_plan():
    from paper_1802_00330_b200.dist import rebalance_plan
    assert rebalance_plan([100, 100], [100, 100]) == [[0, 0], [0, 0]]       # balanced: nothing moves
    assert rebalance_plan([110, 100], [110, 100]) == [[0, 0], [0, 0]]       # within 1.25x
    mv = rebalance_plan([300, 0, 100], [300, 0, 100])
    assert mv[0][1] == 133 and mv[0][2] == 33 and sum(map(sum, mv)) == 166  # -> 134/133/133
    assert rebalance_plan([300, 0], [10, 0]) == [[0, 10], [0, 0]]           # only movable rows move
    assert rebalance_plan([1, 0, 0], [1, 0, 0]) == [[0, 0, 0]] * 3           # fewer rows than ranks
    for sizes in ([7, 0, 0, 0], [1000, 3, 500, 2], [5, 9, 1, 0]):
        mv = rebalance_plan(sizes, sizes)
        after = [sizes[r] - sum(mv[r]) + sum(mv[s][r] for s in range(len(sizes))) for r in range(len(sizes))]
        assert sum(after) == sum(sizes) and max(after) - min(after) <= 1, (sizes, after)


def test_thin_rows_host_twin():
    from paper_1802_00330_b200.dist import thin_rows
    lo = np.array([[0.0, 1.0], [0.0, 1.0], [-1e-300, 0.5]])
    hi = np.array([[1.0, 2.0], [0.0, 2.0], [1e-300, 0.5 + 2 ** -52]])
    assert thin_rows(lo, hi).tolist() == [False, True, True]


def test_row_owner_is_balanced_and_deterministic():
    from paper_1802_00330_b200.dist import row_owner
    rng = np.random.default_rng(0)
    lo = rng.uniform(-1, 1, (20000, 6)); hi = lo + rng.uniform(0, 1e-3, lo.shape)
    own = row_owner(lo, hi, 8)
    counts = np.bincount(own, minlength=8)
    assert counts.min() > 0.9 * 2500 and counts.max() < 1.1 * 2500
    assert np.array_equal(own, row_owner(lo.copy(), hi.copy(), 8))
    # -0.0 and +0.0 rows hash alike (they are equal rows for the dedup)
    z = np.zeros((1, 3)); nz = -np.zeros((1, 3))
    assert row_owner(z, z + 1, 7)[0] == row_owner(nz, nz + 1, 7)[0]
