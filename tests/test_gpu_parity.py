"""CUDA engine parity against the oracle and the reference's golden outputs.

Every test here calls the product path through the C ABI
(paper_1802_00330_b200/librootbox_b200.so); the oracle (oracle/) and the
golden fixtures (tests/golden/) are only the checkers.  Bit-exact throughout:
float64 endpoints compared as bit patterns (signed zero canonicalised)."""
import os

import numpy as np
import pytest

from conftest import (GOLDEN, assert_bits_equal, bits, canonical_sort, golden_jac, golden_spec,
                      load_solve, solve_cases)
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def native():
    from paper_1802_00330_b200 import _native
    assert _native.device_count() >= 1, "no CUDA device visible"
    return _native


def engine(name):
    from paper_1802_00330_b200 import bnb
    return bnb.engine_for(golden_spec(name))


def oracle_sys(name):
    spec = golden_spec(name)
    return O.OSystem(spec.n, spec.eqs, golden_jac(name))


def test_device_and_version(native):
    assert "sm_100a" in native.version()


# ------------------------------------------------------------------ K1 filter


def _round_files():
    return sorted(f for f in os.listdir(GOLDEN) if f.startswith("rounds_"))


@pytest.mark.parametrize("fn", _round_files())
def test_filter_and_hs_vs_reference_rounds(native, fn):
    """rb_filter == bnb._chunk_batch and rb_hs == bnb._hs_pass on the exact
    arrays the reference saw in its own rounds (same order)."""
    case = fn[len("rounds_"):-4]
    meta = load_solve(case)
    eng = engine(meta["system"])
    d = np.load(os.path.join(GOLDEN, fn))
    checked = 0
    for k in d.files:
        if k.endswith("_plo"):
            r = k[:-4]
            off_p = np.concatenate([[0], np.cumsum(d[f"{r}_pcount"])])
            off_o = np.concatenate([[0], np.cumsum(d[f"{r}_ocount"])])
            for c in range(len(off_p) - 1):
                glo, ghi = eng.filter(d[f"{r}_plo"][off_p[c]:off_p[c + 1]], d[f"{r}_phi"][off_p[c]:off_p[c + 1]])
                assert_bits_equal(glo, d[f"{r}_olo"][off_o[c]:off_o[c + 1]], f"{case} {r} filter lo")
                assert_bits_equal(ghi, d[f"{r}_ohi"][off_o[c]:off_o[c + 1]], f"{case} {r} filter hi")
                checked += 1
        if k.endswith("_ocert"):
            r = k[:-6]
            olo, ohi, oc = eng.hs(d[f"{r}_lo"], d[f"{r}_hi"], bool(d["contract"]))
            assert_bits_equal(olo, d[f"{r}_olo"], f"{case} {r} hs lo")
            assert_bits_equal(ohi, d[f"{r}_ohi"], f"{case} {r} hs hi")
            assert np.array_equal(oc, d[f"{r}_ocert"]), f"{case} {r} cert"
            checked += 1
    assert checked


def random_cells(spec, P, depth, seed):
    rng = np.random.default_rng(seed)
    L, H = spec.init_lo, spec.init_hi
    k = rng.integers(0, 2 ** depth, (P, spec.n))
    return L + k * (H - L) / 2 ** depth, L + (k + 1) * (H - L) / 2 ** depth


FILTER_SYSTEMS = ["circle_line", "broyden_tri6", "katsura6", "eco8", "brown8", "broyden_banded12", "cyclic5",
                  "reimer5", "noon5", "kinema", "caprasse", "katsura4", "trinks1", "redeco8"]


def _set_codegen(eng, on):
    """Select the system-specialised (NVRTC) kernels or the table kernels."""
    if on:
        eng.set_option("codegen_wait", 1)
        active, why = eng.codegen_active()
        assert active, f"specialised kernels unavailable: {why}"
    eng.set_option("codegen", int(on))


@pytest.mark.parametrize("mode,codegen", [(1, 0), (0, 0), (0, 1), (1, 1), (2, 0), (2, 1)],
                         ids=["tabulated", "direct_tables", "direct_specialised", "tabulated_specialised",
                              "warp_tabulated", "warp_tabulated_specialised"])
@pytest.mark.parametrize("name", FILTER_SYSTEMS)
def test_filter_random_cells_vs_oracle(native, name, mode, codegen):
    spec = golden_spec(name)
    from paper_1802_00330_b200 import _native
    from paper_1802_00330_b200.system import compile_tables
    eng = _native.Engine(compile_tables(spec), 0)
    _set_codegen(eng, codegen)
    eng.set_option("filter_tab", int(mode == 1))
    eng.set_option("filter_wt", int(mode == 2))  # k_filter_wt where 5 <= n <= 16, else the direct filter
    osys = oracle_sys(name)
    for depth, seed in ((1, 1), (3, 2), (7, 3), (30, 4)):
        P = max(1, min(2048, (1 << 16) >> spec.n))
        plo, phi = random_cells(spec, P, depth, seed)
        glo, ghi = eng.filter(plo, phi)
        olo, ohi = osys.chunk_filter(plo, phi)
        assert glo.shape == olo.shape, (name, depth)
        assert_bits_equal(glo, olo, f"{name} d={depth} lo")
        assert_bits_equal(ghi, ohi, f"{name} d={depth} hi")


# ------------------------------------------------------------------ K2 Hansen-Sengupta


def test_hs_kat_vs_reference(native):
    d = np.load(os.path.join(GOLDEN, "kat_hs.npz"))
    names = sorted({k.rsplit("_", 1)[0] for k in d.files if k.endswith("_kind")})
    for name in names:
        eng = engine(name)
        lo, hi = d[f"{name}_lo"], d[f"{name}_hi"]
        kind, olo_ref, ohi_ref, cert_ref = (d[f"{name}_kind"], d[f"{name}_olo"], d[f"{name}_ohi"],
                                            d[f"{name}_cert"])
        # reference _hs_pass semantics from the per-box outcomes
        exp_lo, exp_hi, exp_c = [], [], []
        for r in range(lo.shape[0]):
            k = int(kind[r])
            if k == 0:
                continue
            if k == 3:
                exp_lo.append(lo[r]); exp_hi.append(hi[r]); exp_c.append(False)
                continue
            for q in range(k):
                exp_lo.append(olo_ref[r, q]); exp_hi.append(ohi_ref[r, q]); exp_c.append(bool(cert_ref[r]))
        glo, ghi, gc = eng.hs(lo, hi, True)
        assert glo.shape[0] == len(exp_lo), name
        if exp_lo:
            assert_bits_equal(glo, np.array(exp_lo), f"{name} hs lo")
            assert_bits_equal(ghi, np.array(exp_hi), f"{name} hs hi")
            assert gc.tolist() == exp_c, name


HS_SYSTEMS = ["circle_line", "broyden_tri6", "katsura6", "eco8", "brown8", "broyden_banded12", "cyclic5",
              "noon5", "kinema", "caprasse", "reimer5", "katsura8", "cyclic9", "noon9"]


@pytest.mark.parametrize("codegen", [1, 0], ids=["specialised", "tables"])
@pytest.mark.parametrize("fused", [2, 0], ids=["fused", "three_kernel"])
@pytest.mark.parametrize("name", HS_SYSTEMS)
def test_hs_random_cells_vs_oracle(native, name, fused, codegen):
    spec = golden_spec(name)
    from paper_1802_00330_b200.system import compile_tables
    eng = native.Engine(compile_tables(spec), 0)
    _set_codegen(eng, codegen)
    eng.set_option("hs_fused", fused)
    osys = oracle_sys(name)
    for depth, seed in ((2, 5), (6, 6), (12, 7), (24, 8), (40, 9)):
        plo, phi = random_cells(spec, 512, depth, seed)
        for contract in (True, False):
            glo, ghi, gc = eng.hs(plo, phi, contract)
            olo, ohi, oc = osys.hs_pass(plo, phi, contract)
            assert glo.shape == olo.shape, (name, depth, contract)
            assert_bits_equal(glo, olo, f"{name} d={depth} lo")
            assert_bits_equal(ghi, ohi, f"{name} d={depth} hi")
            assert np.array_equal(gc, oc), (name, depth)


# ------------------------------------------------------------------ Krawczyk


def test_krawczyk_kat_vs_reference(native):
    """rb_krawczyk == hansen.krawczyk (hansen.py:141-170) on the reference's own outputs."""
    d = np.load(os.path.join(GOLDEN, "kat_krawczyk.npz"))
    names = sorted({k.rsplit("_", 1)[0] for k in d.files if k.endswith("_ok")})
    assert names
    for name in names:
        ok, olo, ohi = engine(name).krawczyk(d[f"{name}_lo"], d[f"{name}_hi"])
        assert np.array_equal(ok, d[f"{name}_ok"]), name
        assert_bits_equal(olo[ok], d[f"{name}_olo"][ok], f"{name} krawczyk lo")
        assert_bits_equal(ohi[ok], d[f"{name}_ohi"][ok], f"{name} krawczyk hi")
        assert np.isnan(olo[~ok]).all()


@pytest.mark.parametrize("name", HS_SYSTEMS)
def test_krawczyk_random_cells_vs_oracle(native, name):
    spec = golden_spec(name)
    eng = engine(name)
    osys = oracle_sys(name)
    for depth, seed in ((2, 15), (8, 16), (20, 17), (45, 18)):
        plo, phi = random_cells(spec, 700, depth, seed)
        ok, glo, ghi = eng.krawczyk(plo, phi)
        ook, olo, ohi = osys.krawczyk(plo, phi)
        assert np.array_equal(ok, ook), (name, depth)
        assert_bits_equal(glo[ok], olo[ok], f"{name} d={depth} lo")
        assert_bits_equal(ghi[ok], ohi[ok], f"{name} d={depth} hi")


def test_krawczyk_public_api(native):
    import math
    from paper_1802_00330_b200 import Box, krawczyk
    spec = golden_spec("circle_line")
    b = Box.from_bounds([0.5, 0.5], [0.9, 0.9])
    out = krawczyk(spec, None, b)
    ook, olo, ohi = oracle_sys("circle_line").krawczyk(np.array([[0.5, 0.5]]), np.array([[0.9, 0.9]]))
    if ook[0]:
        assert [iv.lo for iv in out] == olo[0].tolist() and [iv.hi for iv in out] == ohi[0].tolist()
    else:
        assert out is None
    with pytest.raises(ValueError):
        krawczyk(spec, None, Box.from_bounds([0.0, -math.inf], [1.0, 1.0]))


# ------------------------------------------------------------------ whole solves


def check_against_golden(case, out, meta):
    assert out["status"] == meta["status"], case
    assert len(out["stats"]) == len(meta["stats"]), case
    for st, want in zip(out["stats"], meta["stats"]):
        got = [st["round"], st["boxes_in"], st["boxes_after_filter"], st["boxes_after_hs"]]
        assert got == want[:4], (case, got, want)
        assert bits(st["width"]) == bits(float.fromhex(want[4])), (case, st["width"], want[4])
    lo, hi = out["lo"], out["hi"]
    assert lo.shape[0] == meta["nboxes"], case
    # the engine returns canonical order already
    order = canonical_sort(lo, hi)
    assert np.array_equal(order, np.arange(lo.shape[0])), "engine output not in canonical order"
    assert int(out["cert"].sum()) == meta["ncert"] and int(out["unsplit"].sum()) == meta["nunsplit"], case
    if "lo" in meta:
        want_lo = np.array([[float.fromhex(v) for v in r] for r in meta["lo"]]).reshape(lo.shape)
        want_hi = np.array([[float.fromhex(v) for v in r] for r in meta["hi"]]).reshape(hi.shape)
        assert_bits_equal(lo, want_lo, f"{case} lo")
        assert_bits_equal(hi, want_hi, f"{case} hi")
        assert out["cert"].astype(int).tolist() == meta["cert"], case
        assert out["unsplit"].astype(int).tolist() == meta["unsplit"], case
    import hashlib
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(lo, "<f8").tobytes())
    h.update(np.ascontiguousarray(hi, "<f8").tobytes())
    h.update(out["cert"].astype(np.uint8).tobytes())
    h.update(out["unsplit"].astype(np.uint8).tobytes())
    assert h.hexdigest() == meta["digest"], case
    # signed zeros never escape (the reference never emits -0.0)
    assert not np.any(np.signbit(lo) & (lo == 0)) and not np.any(np.signbit(hi) & (hi == 0))


@pytest.mark.parametrize("graph,fused,codegen,pingpong",
                         [(1, 1, 1, 1), (1, 1, 1, 0), (0, 1, 1, 1), (0, 0, 1, 1), (1, 2, 1, 1), (1, 1, 0, 1),
                          (0, 0, 0, 1)],
                         ids=["device_loop", "device_loop_round_tail", "host_loop", "host_loop_three_kernel_hs",
                              "device_loop_fused_hs", "device_loop_tables", "host_loop_three_kernel_hs_tables"])
@pytest.mark.parametrize("case", solve_cases())
def test_solve_vs_reference_golden(native, case, graph, fused, codegen, pingpong):
    """Whole solves, with the round loop on the device (CUDA graph WHILE node)
    and host-driven, with the system-specialised and the table kernels, against
    the reference's recorded results."""
    from paper_1802_00330_b200 import bnb
    meta = load_solve(case)
    spec = golden_spec(meta["system"])
    eng = bnb.engine_for(spec)
    _set_codegen(eng, codegen)
    eng.set_option("graph", graph)
    eng.set_option("hs_fused", fused)
    eng.set_option("pingpong", pingpong)
    try:
        out = eng.solve(bnb.native_config(bnb.SolverConfig(**meta["config"])))
    finally:
        eng.set_option("graph", 1)
        eng.set_option("hs_fused", 1)
        eng.set_option("codegen", 1)
        eng.set_option("pingpong", 1)
    check_against_golden(case, out, meta)


@pytest.mark.parametrize("case", solve_cases())
def test_solve_host_loop_tabulated_specialised_filter(native, case):
    """Host-driven rounds with the tabulated filter on the specialised table sums."""
    from paper_1802_00330_b200 import bnb
    meta = load_solve(case)
    spec = golden_spec(meta["system"])
    eng = bnb.engine_for(spec)
    _set_codegen(eng, 1)
    eng.set_option("graph", 0)
    eng.set_option("filter_tab", 1)
    try:
        out = eng.solve(bnb.native_config(bnb.SolverConfig(**meta["config"])))
    finally:
        eng.set_option("graph", 1)
        eng.set_option("filter_tab", 0)
    check_against_golden(case, out, meta)


@pytest.mark.parametrize("codegen", [0, 1], ids=["tables", "specialised"])
@pytest.mark.parametrize("case", solve_cases())
def test_solve_host_loop_warp_tabulated_filter(native, case, codegen):
    """Host-driven rounds with the warp-tabulated filter forced on (k_filter_wt, 5 <= n <= 16)."""
    from paper_1802_00330_b200 import bnb
    meta = load_solve(case)
    spec = golden_spec(meta["system"])
    eng = bnb.engine_for(spec)
    _set_codegen(eng, codegen)
    eng.set_option("graph", 0)
    eng.set_option("filter_wt", 1)
    try:
        out = eng.solve(bnb.native_config(bnb.SolverConfig(**meta["config"])))
    finally:
        eng.set_option("graph", 1)
        eng.set_option("filter_wt", -1)
        eng.set_option("codegen", 1)
    check_against_golden(case, out, meta)


@pytest.mark.parametrize("case", solve_cases())
def test_solve_host_loop_without_constant_j(native, case):
    """Host-driven rounds with every J entry through the HS scratch ("jconst" off)."""
    from paper_1802_00330_b200 import bnb
    meta = load_solve(case)
    spec = golden_spec(meta["system"])
    eng = bnb.engine_for(spec)
    eng.set_option("graph", 0)
    eng.set_option("hs_fused", 0)  # every HS round through eval / lin / sweep
    eng.set_option("jconst", 0)
    try:
        out = eng.solve(bnb.native_config(bnb.SolverConfig(**meta["config"])))
    finally:
        eng.set_option("graph", 1)
        eng.set_option("hs_fused", 1)
        eng.set_option("jconst", 1)
    check_against_golden(case, out, meta)


@pytest.mark.parametrize("case", solve_cases())
def test_solve_host_loop_three_kernel_hs(native, case):
    """Host-driven rounds with every HS round through eval / lin / sweep (constant J on)."""
    from paper_1802_00330_b200 import bnb
    meta = load_solve(case)
    spec = golden_spec(meta["system"])
    eng = bnb.engine_for(spec)
    eng.set_option("graph", 0)
    eng.set_option("hs_fused", 0)
    try:
        out = eng.solve(bnb.native_config(bnb.SolverConfig(**meta["config"])))
    finally:
        eng.set_option("graph", 1)
        eng.set_option("hs_fused", 1)
    check_against_golden(case, out, meta)


@pytest.mark.parametrize("lin", [2, 3], ids=["thread_per_box", "pair_per_box"])
@pytest.mark.parametrize("case", solve_cases())
def test_solve_host_loop_gauss_jordan_variants(native, case, lin):
    """Three-kernel HS with the thread-per-box (k_hs_lin_tps) and the two-threads-per-box
    (k_hs_lin_tp2) Gauss-Jordan forced at every n <= 12."""
    from paper_1802_00330_b200 import bnb
    meta = load_solve(case)
    spec = golden_spec(meta["system"])
    eng = bnb.engine_for(spec)
    eng.set_option("graph", 0)
    eng.set_option("hs_fused", 0)
    eng.set_option("lin_tpb", lin)
    try:
        out = eng.solve(bnb.native_config(bnb.SolverConfig(**meta["config"])))
    finally:
        eng.set_option("graph", 1)
        eng.set_option("hs_fused", 1)
        eng.set_option("lin_tpb", 2)
    check_against_golden(case, out, meta)


@pytest.mark.parametrize("case", solve_cases()[:12])
def test_solve_persistent_small_rounds(native, case):
    """The experimental persistent small-round kernel (grid barriers, ping-pong frontier)."""
    from paper_1802_00330_b200 import bnb
    meta = load_solve(case)
    spec = golden_spec(meta["system"])
    eng = bnb.engine_for(spec)
    eng.set_option("small_rounds", 1)
    try:
        out = eng.solve(bnb.native_config(bnb.SolverConfig(**meta["config"])))
    finally:
        eng.set_option("small_rounds", 0)
    check_against_golden(case, out, meta)


def test_solve_returns_reference_shaped_objects(native):
    from paper_1802_00330_b200 import SolverConfig, solve
    spec = golden_spec("circle_line")
    res = solve(spec, SolverConfig(target_width=1e-6))
    assert res.status == "width_reached" and res.reached_width
    assert len(res.boxes) == 2 and all(rb.certified for rb in res.boxes)
    assert [st.boxes_after_hs for st in res.stats] == [4, 8, 2, 2, 2]
    r0 = res.boxes[0].box
    assert r0[0].lo == float.fromhex(load_solve("circle_line")["lo"][0][0])


def test_config_validation_errors(native):
    from paper_1802_00330_b200 import SolverConfig, solve
    spec = golden_spec("circle_line")
    for bad in (dict(target_width=0.0), dict(max_boxes=0), dict(max_rounds=0), dict(worker_count=0),
                dict(batch_size=0), dict(hs_enable_round=-1), dict(engine="cuda")):
        with pytest.raises(ValueError):
            solve(spec, SolverConfig(**bad))


def test_init_width_below_target(native):
    from paper_1802_00330_b200 import SolverConfig, solve_arrays
    spec = golden_spec("circle_line")
    out = solve_arrays(spec, SolverConfig(target_width=10.0))
    assert out["status"] == "width_reached" and out["lo"].shape[0] == 1 and out["stats"] == []


@pytest.mark.parametrize("name,kw,rounds", [
    ("katsura6", dict(), 3),
    ("katsura6", dict(), 4),  # 117k-row frontier: exercises the device radix sort path
    ("eco8", dict(), 2),
    ("brown8", dict(target_width=1e-8), 2),
    ("broyden_banded12", dict(target_width=1e-8), 1),
    ("noon5", dict(), 4),
    ("cyclic5", dict(), 4),
    ("kinema", dict(), 3),
])
def test_round_matched_vs_oracle(native, name, kw, rounds):
    """Large configs: identical frontiers (bit patterns + flags) and round stats
    for the first rounds, checked against the multithreaded oracle."""
    from paper_1802_00330_b200 import SolverConfig, solve_arrays
    spec = golden_spec(name)
    out = solve_arrays(spec, SolverConfig(max_rounds=rounds, **kw))
    ref = oracle_sys(name).solve(spec.init_lo, spec.init_hi, max_rounds=rounds, threads=os.cpu_count(), **kw)
    assert out["status"] == ref["status"]
    for st, o in zip(out["stats"], ref["stats"]):
        assert [st["round"], st["boxes_in"], st["boxes_after_filter"], st["boxes_after_hs"]] == \
            [int(o[0]), int(o[1]), int(o[2]), int(o[3])], name
        assert bits(st["width"]) == bits(o[4])
    order = canonical_sort(ref["lo"], ref["hi"])
    assert_bits_equal(out["lo"], ref["lo"][order], f"{name} lo")
    assert_bits_equal(out["hi"], ref["hi"][order], f"{name} hi")
    assert np.array_equal(out["cert"], ref["cert"][order])
    assert np.array_equal(out["unsplit"], ref["unsplit"][order])


# ------------------------------------------------------------------ sharded protocol on the device

SHARD_CASES = ["circle_line", "broyden_tri6", "katsura3", "quirk17b", "rediff3_rounds3", "brown5", "katsura6_r3"]


@pytest.mark.parametrize("case", SHARD_CASES)
def test_sharded_protocol_single_rank_vs_golden(native, case):
    """dist.solve_sharded through the rb_shard_* / rb_round_* C-ABI on one GPU
    (partition + device export/import + dedup exercised with world = 1)."""
    from paper_1802_00330_b200 import SolverConfig
    from paper_1802_00330_b200.dist import CudaShardBackend, solve_sharded
    meta = load_solve(case)
    spec = golden_spec(meta["system"])
    res = solve_sharded(spec, SolverConfig(**meta["config"]), backend=CudaShardBackend(spec, 0), force_protocol=True)
    assert res.status == meta["status"], case
    assert [[s.round, s.boxes_in, s.boxes_after_filter, s.boxes_after_hs] for s in res.stats] == \
        [w[:4] for w in meta["stats"]], case
    lo = np.array([[iv.lo for iv in rb.box] for rb in res.boxes]).reshape(-1, spec.n)
    hi = np.array([[iv.hi for iv in rb.box] for rb in res.boxes]).reshape(-1, spec.n)
    out = {"status": res.status, "lo": lo, "hi": hi,
           "cert": np.array([rb.certified for rb in res.boxes], bool),
           "unsplit": np.array([rb.unsplittable for rb in res.boxes], bool),
           "stats": [dict(round=s.round, boxes_in=s.boxes_in, boxes_after_filter=s.boxes_after_filter,
                          boxes_after_hs=s.boxes_after_hs, width=s.width) for s in res.stats]}
    check_against_golden(case, out, meta)


def test_shard_route_export_import_roundtrip(native):
    """rb_shard_route_count / rb_shard_route / packed export+import on the device
    against the host twins (dist.thin_rows, dist.row_owner)."""
    import torch
    from paper_1802_00330_b200.dist import CudaShardBackend, row_owner, thin_rows
    spec = golden_spec("katsura6")
    rng = np.random.default_rng(3)
    lo = rng.uniform(-1, 1, (1000, spec.n)); hi = lo + rng.uniform(0, 1, lo.shape)
    thin = rng.random(1000) < 0.2  # some rows thin in one component (<= 64 ulps)
    j = rng.integers(0, spec.n, 1000)
    hi[thin, j[thin]] = np.nextafter(lo[thin, j[thin]], np.inf)
    c = (rng.random(1000) < 0.3).astype(np.uint8); u = (rng.random(1000) < 0.2).astype(np.uint8)
    for exch in (True, False):
        be = CudaShardBackend(spec, 0, device_exchange=exch)
        be.load(lo, hi, c, u, 1e-3)
        world, rank = 4, 1
        tc, other = be.route_count(world)
        assert thin_rows(lo, hi).sum() == thin.sum()
        want = np.bincount(row_owner(lo[thin], hi[thin], world), minlength=world)
        assert np.array_equal(tc, want) and other == 1000 - thin.sum()
        move = [50, 0, 0, 25]
        sc = be.route(world, rank, move)
        want_sc = tc + np.array(move)
        want_sc[rank] = tc[rank] + other - 75  # move[rank] is ignored: those rows stay
        assert np.array_equal(sc, want_sc), (sc, want_sc)
        keep = int(sc[rank])
        rows = be.export_packed(torch, keep, 1000 - keep)
        be.import_packed(torch, keep, rows)  # put them back: the shard holds the same multiset
        glo, ghi, gc, gu = be.finalize()
        key = lambda a, b: np.lexsort(tuple(b[:, i] for i in reversed(range(b.shape[1]))) +
                                      tuple(a[:, i] for i in reversed(range(a.shape[1]))))
        o1 = key(lo, hi)
        assert_bits_equal(glo, lo[o1], "lo"); assert_bits_equal(ghi, hi[o1], "hi")
        assert np.array_equal(gc, c[o1].astype(bool)) and np.array_equal(gu, u[o1].astype(bool))
        # the sent segment holds exactly the rows routed away: thin rows of other owners + 75 movers
        own = row_owner(rows[:, :spec.n].cpu().numpy(), rows[:, spec.n:2 * spec.n].cpu().numpy(), world)
        th = thin_rows(rows[:, :spec.n].cpu().numpy(), rows[:, spec.n:2 * spec.n].cpu().numpy())
        assert np.all(own[th] != rank) and (~th).sum() == 75
