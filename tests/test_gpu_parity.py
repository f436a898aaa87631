"""GPU parity: the product path (C ABI -> sm_100a kernels) against the golden
fixtures (executed reference) and the pinned oracle.

Tolerances (north_star): lists / permutation ids bit-exact; fp64 locals
relative L2 <= 1e-12 for full-rank variants and <= 1e-10 for compressed ones,
with equal ranks and equal reference-model flop counts.
"""

import os
import sys

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

FULL = ("na", "nasym", "nablk")
TOL = {v: (1e-12 if v in FULL else 1e-10) for v in O.VARIANTS}


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    return torch


def _kernel_grid(g):
    from paper_1210_7292_b200 import ChebyshevGrid, helmholtz_kernel, laplace_kernel

    k = laplace_kernel() if str(g["kernel"]) == "laplace" else helmholtz_kernel(float(g["wavenumber"]))
    return k, ChebyshevGrid(int(g["order"]))


def _lt_lw(g):
    levels = [int(l) for l in g["levels"]]
    lt = {l: sorted({tuple(int(c) for c in t) for t in g[f"t_{l}"]}) for l in levels}
    lw = dict(zip(levels, (float(w) for w in g["widths"])))
    return levels, lt, lw


def _mpoles(g, lvl, case):
    if f"mpoles_{lvl}" in g:
        return g[f"mpoles_{lvl}"]
    seed = {"sphere9": 33, "sphere_lists": 44}[case]
    n = len(g[f"cells_{lvl}"])
    rng = np.random.default_rng(seed + lvl)
    size = int(g["order"]) ** 3
    m = rng.uniform(-1, 1, (n, size))
    if str(g["kernel"]) != "laplace":
        m = m + 1j * rng.uniform(-1, 1, (n, size))
    return m


def _handler(g, variant, **kw):
    from paper_1210_7292_b200 import make_handler

    kernel, grid = _kernel_grid(g)
    levels, lt, lw = _lt_lw(g)
    if "compression" in g:
        kw.setdefault("compression", str(g["compression"]))
    h = make_handler(variant, kernel, grid, float(g["eps"]), **kw)
    h.precompute(lt, lw)
    return h, levels


CASES = [("cfg1", v) for v in O.VARIANTS] + [("helm", v) for v in O.VARIANTS] + \
    [("lapcplx", v) for v in ("na", "nablk", "iablk", "sa")] + [("sphere_lists", "nasym")] + \
    [("aca", v) for v in ("ia", "iasym", "iablk", "sa", "sarcmp")]


@pytest.mark.parametrize("case,variant", CASES)
def test_handler_matches_reference(torch_cuda, golden, case, variant):
    g = golden(case)
    h, levels = _handler(g, variant)
    for lvl in levels:
        mp = _mpoles(g, lvl, case)
        tgt, off, src, t = (g[f"{k}_{lvl}"] for k in ("tgt", "off", "src", "t"))
        batch = O.csr_to_batch(tgt, off, src, t)
        loc = np.zeros(mp.shape, dtype=np.result_type(h.kernel.dtype, mp.dtype))
        fl = h.apply_level(lvl, batch, mp, loc)
        got = loc[g[f"rows_{lvl}"]] if f"rows_{lvl}" in g else loc
        err = O.rel_l2(got, g[f"locals_{variant}_{lvl}"])
        assert err <= TOL[variant], (case, variant, lvl, err)
        assert fl == int(g[f"flops_{variant}_{lvl}"])
        assert h.flops[lvl] == int(g[f"flops_{variant}_{lvl}"])
        assert h.level_ranks(lvl) == list(g[f"ranks_{variant}_{lvl}"])
        if h.is_shared_basis:
            assert h.shared_rank(lvl) == int(g[f"shared_rank_{variant}_{lvl}"])
            rt = h.recompression_table(lvl)
            assert [(-1 if r is None else r) for _, r in rt] == list(g[f"recomp_r_{variant}_{lvl}"])
        if h.uses_blocking:
            assert h.block_stats[lvl]["columns"] == int(g[f"blk_columns_{variant}_{lvl}"])
            assert len(h.block_stats[lvl]["reps_used"]) == int(g[f"blk_reps_{variant}_{lvl}"])
    assert h.operator_count() == int(g[f"operator_count_{variant}"])
    assert h.stored_bytes() == int(g[f"stored_bytes_{variant}"])
    assert h.factorization_calls == int(g[f"factorization_calls_{variant}"])


def test_sphere9_nablk_and_sa(torch_cuda, golden):
    """l = 9 (729 nodes) on a sparse sphere tree: nablk and sa (eps 1e-8)."""
    g = golden("sphere9")
    for variant in ("nablk", "sa"):
        h, levels = _handler(g, variant, budget_bytes=4_000_000_000)
        for lvl in levels:
            mp = _mpoles(g, lvl, "sphere9")
            tgt, off, src, t = (g[f"{k}_{lvl}"] for k in ("tgt", "off", "src", "t"))
            loc = np.zeros_like(mp)
            fl = h.apply_level_csr(lvl, tgt, off, src, t, mp, loc)
            err = O.rel_l2(loc[g[f"rows_{lvl}"]], g[f"locals_{variant}_{lvl}"])
            assert err <= TOL[variant], (variant, lvl, err)
            assert fl == int(g[f"flops_{variant}_{lvl}"])
        if variant == "sa":
            assert h.shared_rank(levels[0]) == int(g[f"shared_rank_sa_{levels[0]}"])


@pytest.mark.parametrize("case", ["cfg1", "sphere_lists", "helm", "sphere9"])
def test_classifier_bit_exact(torch_cuda, golden, case):
    import ctypes

    from paper_1210_7292_b200 import _native

    lib = _native.load()
    g = golden(case)
    for lvl in g["levels"]:
        cells = np.ascontiguousarray(g[f"cells_{lvl}"], dtype=np.int32)
        n = len(cells)
        offs = np.zeros(n + 1, np.int64)
        total = ctypes.c_int64()
        _native.check(lib.cfm_classify_count(0, int(lvl), n, cells.ctypes.data, offs.ctypes.data, ctypes.byref(total)))
        src = np.zeros(total.value, np.int32)
        tv = np.zeros((total.value, 3), np.int8)
        rep = np.zeros(total.value, np.uint8)
        perm = np.zeros(total.value, np.uint8)
        _native.check(lib.cfm_classify_fill(0, int(lvl), n, cells.ctypes.data, offs.ctypes.data, src.ctypes.data,
                                            tv.ctypes.data, rep.ctypes.data, perm.ctypes.data))
        counts = np.diff(offs)
        rows = np.nonzero(counts)[0]
        assert np.array_equal(rows, g[f"tgt_{lvl}"])
        assert np.array_equal(np.concatenate([[0], np.cumsum(counts[rows])]), g[f"off_{lvl}"])
        assert np.array_equal(src, g[f"src_{lvl}"])
        assert np.array_equal(tv, g[f"t_{lvl}"])
        full_cone, _ = O.cone_of(O.full_far_field())
        exp_rep, exp_perm = [], []
        for t in tv:
            ts, fl, od = O.canonicalize(tuple(int(c) for c in t))
            exp_rep.append(full_cone.index(ts))
            exp_perm.append(O.perm_id(fl, od))
        assert np.array_equal(rep, np.asarray(exp_rep, np.uint8))
        assert np.array_equal(perm, np.asarray(exp_perm, np.uint8))


@pytest.mark.parametrize("variant", ["nablk", "na", "iablk", "sarcmp"])
def test_cells_path_equals_csr_path(torch_cuda, golden, variant):
    """Device-built lists (classifier -> plan) give the same locals as the
    reference's host batch, bitwise (same lists, same plan)."""
    torch = torch_cuda
    g = golden("cfg1")
    h, levels = _handler(g, variant)
    for lvl in levels:
        mp = g[f"mpoles_{lvl}"]
        tgt, off, src, t = (g[f"{k}_{lvl}"] for k in ("tgt", "off", "src", "t"))
        a = np.zeros_like(mp)
        fa = h.apply_level_csr(lvl, tgt, off, src, t, mp, a)
        h.plan_level_cells(lvl, g[f"cells_{lvl}"])
        b = torch.zeros(mp.shape, dtype=torch.float64, device="cuda")
        fb = h.apply_planned(lvl, torch.from_numpy(mp).cuda(), b)
        assert fa == fb
        assert np.array_equal(a, b.cpu().numpy())


def test_edge_cases(torch_cuda, golden):
    from paper_1210_7292_b200 import PrecomputeIncompleteError, make_handler

    g = golden("cfg1")
    kernel, grid = _kernel_grid(g)
    h = make_handler("nablk", kernel, grid, 1e-5)
    mp = g["mpoles_3"]
    loc = np.zeros_like(mp)
    with pytest.raises(PrecomputeIncompleteError):
        h.apply_level(3, [(0, [(100, (3, 0, 0))])], mp, loc)
    levels, lt, lw = _lt_lw(g)
    h.precompute(lt, lw)
    assert h.apply_level(3, [], mp, loc) == 0
    with pytest.raises(PrecomputeIncompleteError):
        h.apply_level(7, [(0, [(1, (2, 0, 0))])], mp, loc)
    with pytest.raises(KeyError):  # PrecomputeIncompleteError is a KeyError, as in the reference
        h.apply_level(3, [(0, [(1, (1, 0, 0))])], mp, loc)
    assert np.all(loc == 0)
    # empty far lists, a single pair, a duplicated target and duplicated pairs
    batch = [(5, []), (7, [(300, (2, 1, 0))]), (9, [(40, (3, 3, 3)), (41, (-2, 0, 0))]),
             (9, [(40, (3, 3, 3))])]
    orc, _ = _oracle(g, "nablk")
    ref = np.zeros_like(mp)
    fr = orc.apply_faithful(3, batch, mp, ref)
    fg = h.apply_level(3, batch, mp, loc)
    assert fg == fr
    assert O.rel_l2(loc, ref) <= 1e-13
    assert np.all(loc[5] == 0)


def _oracle(g, variant):
    kname = str(g["kernel"])
    prof, dt, deg = (O.laplace_profile, np.float64, -1.0) if kname == "laplace" else \
        (O.helmholtz_profile(float(g["wavenumber"])), np.complex128, None)
    levels, lt, lw = _lt_lw(g)
    return O.OracleM2L(variant, prof, dt, int(g["order"]), float(g["eps"]), deg).precompute(lt, lw), levels


def test_torch_tensors_in_place(torch_cuda, golden):
    torch = torch_cuda
    g = golden("helm")
    h, levels = _handler(g, "iablk")
    for lvl in levels:
        mp = g[f"mpoles_{lvl}"]
        tgt, off, src, t = (g[f"{k}_{lvl}"] for k in ("tgt", "off", "src", "t"))
        loc = torch.zeros(mp.shape, dtype=torch.complex128, device="cuda")
        h.apply_level_csr(lvl, tgt, off, src, t, torch.from_numpy(mp).cuda(), loc)
        torch.cuda.synchronize()
        assert O.rel_l2(loc.cpu().numpy(), g[f"locals_iablk_{lvl}"]) <= 1e-10


def _full_level(level):
    side = 1 << level
    return np.stack(np.meshgrid(*(np.arange(side),) * 3, indexing="ij"), -1).reshape(-1, 3).astype(np.int32)


@pytest.mark.parametrize("order,level,variant", [(5, 5, "nablk"), (5, 5, "iablk"), (7, 4, "nablk")])
def test_full_level_against_oracle(torch_cuda, order, level, variant):
    """Full cube levels (BASELINE configs 2/4 shapes at smaller depth), all
    targets, device-built lists, against the vectorized oracle."""
    torch = torch_cuda
    from paper_1210_7292_b200 import ChebyshevGrid, laplace_kernel, make_handler

    cells = _full_level(level)
    tgt, off, src, t = O.far_lists(cells, level)
    transfers = sorted({tuple(int(c) for c in v) for v in t})
    lw = {level: 1.0 / (1 << level)}
    eps = 1e-5
    h = make_handler(variant, laplace_kernel(), ChebyshevGrid(order), eps)
    h.precompute({level: transfers}, lw)
    st = h.plan_level_cells(level, cells)
    assert st["pairs"] == off[-1] == (6 * 2**level - 8) ** 3 - (3 * 2**level - 2) ** 3
    rng = np.random.default_rng(level)
    mp = rng.uniform(-1, 1, (len(cells), order**3))
    loc = torch.zeros(mp.shape, dtype=torch.float64, device="cuda")
    fl = h.apply_planned(level, torch.from_numpy(mp).cuda(), loc)
    orc = O.OracleM2L(variant, O.laplace_profile, np.float64, order, eps, -1.0).precompute({level: transfers}, lw)
    ref = np.zeros_like(mp)
    fr = orc.apply_fast(level, tgt, off, src, t, mp, ref)
    assert fl == fr
    assert O.rel_l2(loc.cpu().numpy(), ref) <= TOL[variant]


@pytest.mark.gpu
def test_rank1_ktail_matches_padded_dmma(torch_cuda, monkeypatch):
    """l = 5 (125 = 3 x 32 + 29 inner columns): the last k-step of every entry
    runs as a rank-1 DFMA update (default) instead of a DMMA over three zero
    columns (CFM_KTAIL=0) on the one-CTA-per-tile kernel (CFM_STEP_PERSIST=0; the
    persistent step kernel has no k-tail).  Full level 5: both agree to rounding
    and match the oracle at the full-rank tolerance."""
    torch = torch_cuda
    from paper_1210_7292_b200 import ChebyshevGrid, laplace_kernel, make_handler

    monkeypatch.setenv("CFM_STEP_PERSIST", "0")
    order, level = 5, 5
    cells = _full_level(level)
    tgt, off, src, t = O.far_lists(cells, level)
    transfers = sorted({tuple(int(c) for c in v) for v in t})
    lw = {level: 1.0 / (1 << level)}
    h = make_handler("nablk", laplace_kernel(), ChebyshevGrid(order), 1e-5)
    h.precompute({level: transfers}, lw)
    h.plan_level_cells(level, cells)
    mp = torch.from_numpy(np.random.default_rng(11).uniform(-1, 1, (len(cells), order**3))).cuda()
    out = {}
    for v in ("1", "0"):
        monkeypatch.setenv("CFM_KTAIL", v)
        loc = torch.zeros(mp.shape, dtype=torch.float64, device="cuda")
        h.apply_planned(level, mp, loc)
        out[v] = loc.cpu().numpy()
    orc = O.OracleM2L("nablk", O.laplace_profile, np.float64, order, 1e-5, -1.0).precompute({level: transfers}, lw)
    ref = np.zeros(mp.shape)
    orc.apply_fast(level, tgt, off, src, t, mp.cpu().numpy(), ref)
    assert O.rel_l2(out["1"], out["0"]) <= 1e-14
    assert O.rel_l2(out["1"], ref) <= TOL["nablk"]


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["iablk", "iasym", "ia"])
def test_two_stage_lowrank_matches_fused_and_oracle(torch_cuda, variant, monkeypatch):
    """Dense low-rank levels run as two stages (Y = V_t^H x per source and class
    transfer, then U_t Y per target).  Full level 5 at l = 5 (32,768 cells):
    both two-stage layouts (2: target-major Y + dense stage 2, the default;
    1: source-major Y + rank-segment stage 2) are taken, match the oracle
    (<= 1e-10) and the fused single-kernel path (CFM_LR_TWOSTAGE=0) to
    rounding, with equal flops."""
    torch = torch_cuda
    from paper_1210_7292_b200 import ChebyshevGrid, laplace_kernel, make_handler

    order, level, eps = 5, 5, 1e-5
    cells = _full_level(level)
    tgt, off, src, t = O.far_lists(cells, level)
    transfers = sorted({tuple(int(c) for c in v) for v in t})
    lw = {level: 1.0 / (1 << level)}
    rng = np.random.default_rng(7)
    mp = torch.from_numpy(rng.uniform(-1, 1, (len(cells), order**3))).cuda()
    out, flops = {}, {}
    for ts in ("2", "1", "0"):
        monkeypatch.setenv("CFM_LR_TWOSTAGE", ts)
        h = make_handler(variant, laplace_kernel(), ChebyshevGrid(order), eps)
        h.precompute({level: transfers}, lw)
        h.plan_level_cells(level, cells)
        assert h.plan_stats(level)["two_stage"] == (ts != "0")
        loc = torch.zeros(mp.shape, dtype=torch.float64, device="cuda")
        flops[ts] = h.apply_planned(level, mp, loc)
        loc2 = torch.zeros_like(loc)
        h.apply_planned(level, mp, loc2)  # repeated applies reuse the stage buffers
        assert torch.equal(loc, loc2)
        out[ts] = loc.cpu().numpy()
    orc = O.OracleM2L(variant, O.laplace_profile, np.float64, order, eps, -1.0).precompute({level: transfers}, lw)
    ref = np.zeros(mp.shape)
    fr = orc.apply_fast(level, tgt, off, src, t, mp.cpu().numpy(), ref)
    assert flops["2"] == flops["1"] == flops["0"] == fr
    for ts in ("2", "1"):
        assert O.rel_l2(out[ts], ref) <= 1e-10
        assert O.rel_l2(out[ts], out["0"]) <= 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("shape", ["sparse", "slab"])
def test_two_stage_target_major_missing_pairs(torch_cuda, shape, monkeypatch):
    """Target-major two-stage path on levels whose targets miss part of their
    class's transfers (a cube with 10% of the cells removed; a 32 x 32 x 12 slab):
    the Y_T columns of absent pairs stay zero, locals match the oracle
    (<= 1e-10) also when the apply is repeated on non-zero locals, and rows of
    empty targets are untouched."""
    torch = torch_cuda
    from paper_1210_7292_b200 import ChebyshevGrid, laplace_kernel, make_handler

    monkeypatch.setenv("CFM_LR_TWOSTAGE", "2")
    monkeypatch.setenv("CFM_PLAN_MODE", "target")
    order, level, eps = 5, 5, 1e-5
    cells = _full_level(level)
    rng = np.random.default_rng(23)
    if shape == "sparse":
        cells = cells[rng.random(len(cells)) >= 0.1]
    else:
        cells = cells[cells[:, 2] < 12]
    tgt, off, src, t = O.far_lists(cells, level)
    transfers = sorted({tuple(int(c) for c in v) for v in t})
    lw = {level: 1.0 / (1 << level)}
    h = make_handler("iablk", laplace_kernel(), ChebyshevGrid(order), eps)
    h.precompute({level: transfers}, lw)
    h.plan_level_cells(level, cells)
    assert h.plan_stats(level)["two_stage"]
    mp = torch.from_numpy(rng.uniform(-1, 1, (len(cells), order**3))).cuda()
    loc = torch.full(mp.shape, 0.5, dtype=torch.float64, device="cuda")
    h.apply_planned(level, mp, loc)
    h.apply_planned(level, 2.0 * mp, loc)
    orc = O.OracleM2L("iablk", O.laplace_profile, np.float64, order, eps, -1.0).precompute({level: transfers}, lw)
    ref = np.full(mp.shape, 0.5)
    orc.apply_fast(level, tgt, off, src, t, 3.0 * mp.cpu().numpy(), ref)
    assert O.rel_l2(loc.cpu().numpy() - 0.5, ref - 0.5) <= 1e-10


@pytest.mark.gpu
def test_two_stage_kstep_skip_bitwise(torch_cuda, monkeypatch):
    """Stage 2 skips the k-steps of a rank segment past the rank (their U_t
    columns and Y rows are exact zeros): bitwise equal to running all four
    k-steps of every segment (CFM_SEG_KSKIP=0), and within 1e-10 of the oracle."""
    torch = torch_cuda
    from paper_1210_7292_b200 import ChebyshevGrid, laplace_kernel, make_handler

    order, level, eps = 5, 5, 1e-5
    cells = _full_level(level)
    tgt, off, src, t = O.far_lists(cells, level)
    transfers = sorted({tuple(int(c) for c in v) for v in t})
    lw = {level: 1.0 / (1 << level)}
    monkeypatch.setenv("CFM_LR_TWOSTAGE", "1")
    h = make_handler("iablk", laplace_kernel(), ChebyshevGrid(order), eps)
    h.precompute({level: transfers}, lw)
    h.plan_level_cells(level, cells)
    assert h.plan_stats(level)["two_stage"]
    mp = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, (len(cells), order**3))).cuda()
    out = {}
    for v in ("1", "0"):
        monkeypatch.setenv("CFM_SEG_KSKIP", v)
        loc = torch.full(mp.shape, 0.25, dtype=torch.float64, device="cuda")
        h.apply_planned(level, mp, loc)
        out[v] = loc
    assert torch.equal(out["1"], out["0"])
    orc = O.OracleM2L("iablk", O.laplace_profile, np.float64, order, eps, -1.0).precompute({level: transfers}, lw)
    ref = np.full(mp.shape, 0.25)
    orc.apply_fast(level, tgt, off, src, t, mp.cpu().numpy(), ref)
    assert O.rel_l2(out["1"].cpu().numpy(), ref) <= 1e-10


@pytest.mark.gpu
def test_hybrid_plan_matches_target_tiles(torch_cuda, monkeypatch):
    """Hybrid plans (default; CFM_HYBRID=0 disables): the less-than-half-full target tiles
    of a full cube level go to a pair-mode sub-plan.  Per level (apply_planned)
    and through apply_levels, the locals match the plain target-tile plan to
    rounding and the oracle to <= 1e-12."""
    torch = torch_cuda
    from paper_1210_7292_b200 import ChebyshevGrid, full_far_field_vectors, laplace_kernel, make_handler

    order = 5
    levels = [3, 4]
    cells = {l: _full_level(l) for l in levels}
    rng = np.random.default_rng(17)
    mp = {l: torch.from_numpy(rng.uniform(-1, 1, (len(cells[l]), order**3))).cuda() for l in levels}
    out = {}
    for hyb in ("1", "0"):
        monkeypatch.setenv("CFM_HYBRID", hyb)
        h = make_handler("nablk", laplace_kernel(), ChebyshevGrid(order), 1e-5)
        h.precompute({l: full_far_field_vectors() for l in levels}, {l: 1.0 / (1 << l) for l in levels})
        for l in levels:
            h.plan_level_cells(l, cells[l])
        loc = {l: torch.zeros_like(mp[l]) for l in levels}
        h.apply_levels({l: (mp[l], loc[l]) for l in levels})
        single = torch.zeros_like(mp[4])
        h.apply_planned(4, mp[4], single)
        assert torch.equal(single, loc[4])
        out[hyb] = {l: loc[l].cpu().numpy() for l in levels}
    for l in levels:
        tgt, off, src, t = O.far_lists(cells[l], l)
        orc = O.OracleM2L("nablk", O.laplace_profile, np.float64, order, 1e-5, -1.0).precompute(
            {l: sorted({tuple(int(c) for c in v) for v in t})}, {l: 1.0 / (1 << l)})
        ref = np.zeros(mp[l].shape)
        orc.apply_fast(l, tgt, off, src, t, mp[l].cpu().numpy(), ref)
        assert O.rel_l2(out["1"][l], ref) <= 1e-12
        assert O.rel_l2(out["1"][l], out["0"][l]) <= 1e-14


@pytest.mark.gpu
def test_two_stage_skips_sparse_levels(torch_cuda, monkeypatch):
    """A sparse (sphere) level in target tiles keeps the fused low-rank kernel:
    the two-stage source GEMM would compute mostly unneeded class segments."""
    from paper_1210_7292_b200 import ChebyshevGrid, full_far_field_vectors, laplace_kernel, make_handler

    monkeypatch.setenv("CFM_PLAN_MODE", "target")
    rng = np.random.default_rng(3)
    pts = rng.normal(size=(20000, 3))
    pts /= np.linalg.norm(pts, axis=1, keepdims=True)
    level = 5
    side = 1 << level
    cells = np.unique(np.minimum(((pts + 1.0) / 2.0 * side).astype(np.int64), side - 1), axis=0).astype(np.int32)
    h = make_handler("iablk", laplace_kernel(), ChebyshevGrid(5), 1e-5)
    h.precompute({level: full_far_field_vectors()}, {level: 2.0 / side})
    st = h.plan_level_cells(level, cells)
    assert st["mode"] == "target" and not h.plan_stats(level)["two_stage"]


def test_linearity_full_size_level(torch_cuda):
    """Size-independent property at BASELINE config 2's deepest level (l=5,
    262,144 cells, 46.3 M pairs): M2L(a x + b y) == a M2L(x) + b M2L(y), and a
    sampled set of targets matches the oracle."""
    torch = torch_cuda
    from paper_1210_7292_b200 import ChebyshevGrid, laplace_kernel, make_handler

    level, order = 6, 5
    cells = _full_level(level)
    h = make_handler("nablk", laplace_kernel(), ChebyshevGrid(order), 1e-5)
    full = O.full_far_field()
    h.precompute({2: full, level: full}, {2: 0.25, level: 1.0 / 64})
    st = h.plan_level_cells(level, cells)
    assert st["pairs"] == 46_298_376
    gen = torch.Generator(device="cuda").manual_seed(1)
    x = torch.rand((len(cells), order**3), dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
    y = torch.rand((len(cells), order**3), dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
    outs = []
    for m in (x, y, 0.75 * x - 1.5 * y):
        o = torch.zeros_like(x)
        h.apply_planned(level, m, o)
        outs.append(o)
    lin = 0.75 * outs[0] - 1.5 * outs[1]
    assert (torch.linalg.norm(outs[2] - lin) / torch.linalg.norm(outs[2])).item() <= 1e-13
    # sampled targets against the oracle (first 64 rows in reference order + a random sample)
    rng = np.random.default_rng(3)
    rows = np.unique(np.concatenate([np.arange(64), rng.choice(len(cells), 192, replace=False)]))
    tgt, off, src, t = O.far_lists(cells, level, targets=rows)
    assert np.array_equal(tgt, rows)
    orc = O.OracleM2L("nablk", O.laplace_profile, np.float64, order, 1e-5, -1.0).precompute(
        {2: full, level: full}, {2: 0.25, level: 1.0 / 64})
    xm = x.cpu().numpy()
    ref = np.zeros_like(xm)
    orc.apply_fast(level, tgt, off, src, t, xm, ref)
    assert O.rel_l2(outs[0].cpu().numpy()[rows], ref[rows]) <= 1e-12


@pytest.mark.parametrize("variant", ["nablk", "iablk", "sa"])
def test_apply_levels_equals_per_level(torch_cuda, golden, variant):
    """One multi-level launch gives bitwise the per-level results and flops."""
    torch = torch_cuda
    g = golden("cfg1")
    h, levels = _handler(g, variant)
    for lvl in levels:
        h.plan_level_cells(lvl, g[f"cells_{lvl}"])
    arrays, ref = {}, {}
    fl_ref = 0
    for lvl in levels:
        mp = torch.from_numpy(g[f"mpoles_{lvl}"]).cuda()
        ref[lvl] = torch.zeros_like(mp)
        fl_ref += h.apply_planned(lvl, mp, ref[lvl])
        arrays[lvl] = (mp, torch.zeros_like(mp))
    fl = h.apply_levels(arrays)
    assert fl == fl_ref
    for lvl in levels:
        assert torch.equal(arrays[lvl][1], ref[lvl])
        assert O.rel_l2(arrays[lvl][1].cpu().numpy(), g[f"locals_{variant}_{lvl}"]) <= TOL[variant]
    # host buffers through the same call
    host = {lvl: (g[f"mpoles_{lvl}"], np.zeros_like(g[f"mpoles_{lvl}"])) for lvl in levels}
    h.apply_levels(host)
    for lvl in levels:
        assert np.array_equal(host[lvl][1], ref[lvl].cpu().numpy())


PAIR_CASES = [("cfg1", v) for v in ("na", "nablk", "iablk", "sa", "sarcmp")] + \
    [("helm", v) for v in ("nablk", "iablk", "sarcmp")] + [("lapcplx", v) for v in ("nablk", "iablk", "sa")]


@pytest.mark.parametrize("case,variant", PAIR_CASES)
def test_pair_mode_matches_reference(torch_cuda, golden, case, variant, monkeypatch):
    """Pair-mode plans (per-transfer-vector entries + ordered per-target
    reduction, used for sparse trees) give the reference locals too."""
    monkeypatch.setenv("CFM_PLAN_MODE", "pair")
    g = golden(case)
    h, levels = _handler(g, variant)
    for lvl in levels:
        mp = _mpoles(g, lvl, case)
        tgt, off, src, t = (g[f"{k}_{lvl}"] for k in ("tgt", "off", "src", "t"))
        loc = np.zeros(mp.shape, dtype=np.result_type(h.kernel.dtype, mp.dtype))
        fl = h.apply_level_csr(lvl, tgt, off, src, t, mp, loc)
        assert h.last_csr_plan_info()["mode"] == "pair"
        err = O.rel_l2(loc, g[f"locals_{variant}_{lvl}"])
        assert err <= TOL[variant], (case, variant, lvl, err)
        assert fl == int(g[f"flops_{variant}_{lvl}"])


def test_sparse_level_picks_pair_mode(torch_cuda, golden):
    g = golden("sphere9")
    h, levels = _handler(g, "nablk")
    lvl = levels[-1]
    st = h.plan_level_cells(lvl, g[f"cells_{lvl}"])
    assert st["mode"] == "pair" and st["target_fill"] < 0.6


@pytest.mark.parametrize("mode", ["target", "pair"])
def test_sharded_plans_equal_single_gpu(torch_cuda, golden, mode, monkeypatch):
    """Two Morton-range shards planned with plan_level_cells_subset, each
    reading only its own rows plus its halo, reproduce the single-plan locals
    bitwise (per-target accumulation order does not depend on the partition)."""
    torch = torch_cuda
    from paper_1210_7292_b200.distributed import partition_rows

    monkeypatch.setenv("CFM_PLAN_MODE", mode)
    g = golden("sphere_lists")
    lvl = 4
    cells = g[f"cells_{lvl}"]
    mp = torch.from_numpy(_mpoles(g, lvl, "sphere_lists")).cuda()
    h, _ = _handler(g, "nablk")
    h.plan_level_cells(lvl, cells)
    ref = torch.zeros_like(mp)
    h.apply_planned(lvl, mp, ref)
    out = torch.zeros_like(mp)
    for part in partition_rows(cells, 2):
        hs, _ = _handler(g, "nablk")
        st, srcs = hs.plan_level_cells_subset(lvl, cells, part)
        local = torch.zeros_like(mp)
        local[torch.as_tensor(srcs, device="cuda")] = mp[torch.as_tensor(srcs, device="cuda")]
        loc = torch.zeros_like(mp)
        hs.apply_planned(lvl, local, loc)
        rows = torch.as_tensor(part, device="cuda")
        out[rows] = loc[rows]
    assert torch.equal(out, ref)


@pytest.mark.parametrize("order,hybrid", [(4, "0"), (5, "0"), (5, "1"), (5, "late3")])
def test_copy_pipeline_host_buffers_bitwise(torch_cuda, order, hybrid, monkeypatch):
    """Host buffers on a large level go through the slab copy pipeline
    (multipole/locals slabs streamed while the kernel runs, gated by device
    flags; l = 4 streams both, l = 5 -- full-operator mode -- streams the
    locals, with the last slab split in halves/quarters/eighths, level 5 is
    the middle launch group, and the target-tile levels 4 and 5 download while
    level 6 still runs); the result must equal the device-resident path bitwise, including
    accumulation into non-zero host locals.  (Hybrid plans off: the
    device-resident reference then runs the same row-ordered tile plans as the
    pipelined call.  With hybrid plans on -- the bench's e2e setting -- the
    device-resident reference runs hybrid plans for levels 4 and 6, so the
    pipelined result agrees to rounding instead.)"""
    torch = torch_cuda
    from paper_1210_7292_b200 import ChebyshevGrid, laplace_kernel, make_handler

    if hybrid == "late3":
        # levels 4, 5 and 6 all host-pipelined: three late levels, each launched when its own
        # multipoles are in (smallest first), its locals slabs uploaded right behind them
        monkeypatch.setenv("CFM_PIPE_MIN_ROWS", "4096")
        hybrid = "0"
    monkeypatch.setenv("CFM_HYBRID", hybrid)
    lv = (3, 4, 5, 6)  # l = 5: level 5 runs as the middle launch group (uploaded during the first launch)
    cells = {l: _full_level(l) for l in lv}
    full = O.full_far_field()
    h = make_handler("nablk", laplace_kernel(), ChebyshevGrid(order), 1e-5)
    h.precompute({l: full for l in lv}, {l: 1.0 / (1 << l) for l in lv})
    st = {l: h.plan_level_cells(l, cells[l]) for l in lv}
    rng = np.random.default_rng(9)
    mp = {l: rng.uniform(-1, 1, (len(cells[l]), order**3)) for l in lv}
    loc = {l: rng.uniform(-1, 1, mp[l].shape) for l in lv}
    ref = {l: torch.from_numpy(loc[l].copy()).cuda() for l in lv}
    h.apply_levels({l: (torch.from_numpy(mp[l]).cuda(), ref[l]) for l in lv})
    pin = {l: torch.from_numpy(loc[l].copy()).pin_memory() for l in lv}
    for _ in range(2):  # twice: flags and counters must reset between calls
        a = {l: pin[l].numpy().copy() for l in lv}
        h.apply_levels({l: (mp[l], a[l]) for l in lv})
        for l in lv:
            r = ref[l].cpu().numpy()
            if hybrid == "0":
                assert np.array_equal(a[l], r), l
            else:
                assert O.rel_l2(a[l], r) <= 1e-14, l
    assert st[6]["pairs"] == (6 * 64 - 8) ** 3 - (3 * 64 - 2) ** 3


@pytest.mark.parametrize("case", ["cfg1", "helm", "lapcplx", "sphere9", "sphere_lists"])
def test_gpu_tree_matches_reference(torch_cuda, golden, case):
    """GPU octree (§8f rank 1): occupied cells per level equal the reference's
    build_tree output (golden), leaf particle lists equal the oracle's."""
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from geometry import cube_points, sphere_points

    from paper_1210_7292_b200.octree import build_tree_gpu

    g = golden(case)
    pts = {"cfg1": lambda: cube_points(10_000, 1), "helm": lambda: sphere_points(3_000, 5),
           "lapcplx": lambda: cube_points(2_000, 11), "sphere9": lambda: sphere_points(20_000, 3),
           "sphere_lists": lambda: sphere_points(30_000, 21)}[case]()
    center, hw = tuple(g["bbox_center"]), float(g["bbox_half"])
    tree = build_tree_gpu(pts, center, hw, int(g["depth"]))
    for lvl in g["levels"]:
        assert np.array_equal(tree.cells(int(lvl)), g[f"cells_{lvl}"].astype(np.int32))
    off, perm = tree.leaf_particles()
    depth = int(g["depth"])
    side = 1 << depth
    low = np.asarray(center) - hw
    ijk = np.minimum(((pts - low) / (2 * hw) * side).astype(np.int64), side - 1)
    key = (ijk[:, 0] * side + ijk[:, 1]) * side + ijk[:, 2]
    order = np.lexsort((np.arange(len(pts)), key))
    assert np.array_equal(perm, order)
    assert off[-1] == len(pts) and len(off) - 1 == len(np.unique(key))


def test_gpu_tree_errors(torch_cuda):
    from paper_1210_7292_b200.octree import build_tree_gpu

    with pytest.raises(ValueError):
        build_tree_gpu(np.array([[2.0, 0.5, 0.5]]), (0.5, 0.5, 0.5), 0.5, 3)
    with pytest.raises(ValueError):
        build_tree_gpu(np.array([[0.2, 0.5, 0.5]]), (0.5, 0.5, 0.5), 0.5, 1)
    t = build_tree_gpu(np.array([[1.0, 1.0, 1.0], [0.0, 0.0, 0.0]]), (0.5, 0.5, 0.5), 0.5, 2)
    assert np.array_equal(t.cells(2), [[0, 0, 0], [3, 3, 3]])


@pytest.mark.parametrize("case", ["cfg1", "sphere_lists"])
def test_device_classifier_matches_reference(torch_cuda, golden, case):
    import ctypes

    from paper_1210_7292_b200 import _native

    torch = torch_cuda
    lib = _native.load()
    g = golden(case)
    for lvl in g["levels"]:
        cells = torch.from_numpy(g[f"cells_{lvl}"].astype(np.int32)).cuda()
        n = len(cells)
        offs = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        tot = ctypes.c_int64()
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        _native.check(lib.cfm_classify_count_device(0, int(lvl), n, cells.data_ptr(), offs.data_ptr(),
                                                    ctypes.byref(tot), st))
        src = torch.empty(tot.value, dtype=torch.int32, device="cuda")
        code = torch.empty(tot.value, dtype=torch.int16, device="cuda")
        _native.check(lib.cfm_classify_fill_device(0, int(lvl), n, cells.data_ptr(), offs.data_ptr(), src.data_ptr(),
                                                   code.data_ptr(), st))
        torch.cuda.synchronize()
        o = offs.cpu().numpy()
        rows = np.nonzero(np.diff(o))[0]
        assert np.array_equal(rows, g[f"tgt_{lvl}"])
        assert np.array_equal(src.cpu().numpy(), g[f"src_{lvl}"])
        t = g[f"t_{lvl}"].astype(np.int64)
        assert np.array_equal(code.cpu().numpy(), (t[:, 0] + 3) * 49 + (t[:, 1] + 3) * 7 + (t[:, 2] + 3))


FMM_CASES = [("fmm_cube", "nablk"), ("fmm_cube", "iablk"), ("fmm_helm", "nablk"), ("fmm_helm", "iablk"),
             ("fmm_lapcplx", "nablk")]


@pytest.mark.parametrize("case,variant", FMM_CASES)
def test_gpu_fmm_pipeline_matches_reference(torch_cuda, golden, case, variant):
    """§8f ranks 1-3: GPU tree, P2M, M2M, M2L, L2L, L2P, P2P against the
    reference's FmmPlan.run potentials (and its upward-pass multipoles)."""
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from geometry import cube_points, sphere_points

    from paper_1210_7292_b200.fmm import B200FmmPlan

    g = golden(case)
    if case == "fmm_cube":
        pts = cube_points(6_000, 41)
        w = np.random.default_rng(42).uniform(-1.0, 1.0, len(pts))
    elif case == "fmm_helm":
        pts = sphere_points(4_000, 43)
        rng = np.random.default_rng(44)
        w = rng.uniform(-1, 1, len(pts)) + 1j * rng.uniform(-1, 1, len(pts))
    else:
        pts = cube_points(3_000, 45)
        rng = np.random.default_rng(46)
        w = rng.uniform(-1, 1, len(pts)) + 1j * rng.uniform(-1, 1, len(pts))
    kernel, _ = _kernel_grid(g)
    plan = B200FmmPlan(pts, tuple(g["bbox_center"]), float(g["bbox_half"]), int(g["depth"]), kernel,
                       int(g["order"]), float(g["eps"]), variant=variant)
    pot = plan.run(w)
    err = O.rel_l2(pot, g[f"potentials_{variant}"])
    assert err <= 1e-12, err
    depth = int(g["depth"])
    mp = plan._last["mpoles"]
    assert O.rel_l2(mp[depth].cpu().numpy(), g["leaf_mpoles"]) <= 1e-13
    for lvl in g["levels"]:
        assert O.rel_l2(mp[int(lvl)].cpu().numpy(), g[f"up_mpoles_{lvl}"]) <= 1e-13
    assert plan.m2l_seconds > 0


def test_default_stream_ordering(torch_cuda, golden):
    """Handler work on stream NULL is ordered after the caller's default-stream
    kernels: a producer kernel writing the multipoles right before apply must be
    seen by the M2L (large enough that a race would show)."""
    torch = torch_cuda
    from paper_1210_7292_b200 import ChebyshevGrid, laplace_kernel, make_handler

    level, order = 5, 5
    cells = _full_level(level)
    full = O.full_far_field()
    h = make_handler("nablk", laplace_kernel(), ChebyshevGrid(order), 1e-5)
    h.precompute({level: full}, {level: 1.0 / 32})
    h.plan_level_cells(level, cells)
    x = torch.zeros((len(cells), order**3), dtype=torch.float64, device="cuda")
    ref = torch.zeros_like(x)
    src = torch.rand_like(x)
    h.apply_planned(level, src, ref)
    for _ in range(3):
        x.zero_()
        big = torch.rand((4096, 4096), dtype=torch.float64, device="cuda")
        big = big @ big  # keep the default stream busy
        x.copy_(src + 0.0 * big[0, 0])
        out = torch.zeros_like(x)
        h.apply_planned(level, x, out)
        assert torch.equal(out, ref)


@pytest.mark.parametrize("variant", ["nablk", "iablk", "sa"])
@pytest.mark.parametrize("order", ["C", "F"])
def test_concurrent_apply_threads(torch_cuda, golden, variant, order):
    """FmmPlan._m2l calls apply_level from several threads with disjoint target
    chunks sharing mpoles/locals (engine.py:145-155); the result and the flop
    accounting must equal the reference's (F-order locals take the staged
    write-back path)."""
    import threading

    g = golden("cfg1")
    h, levels = _handler(g, variant)
    for lvl in levels:
        mp = _mpoles(g, lvl, "cfg1")
        tgt, off, src, t = (g[f"{k}_{lvl}"] for k in ("tgt", "off", "src", "t"))
        batch = O.csr_to_batch(tgt, off, src, t)
        loc = np.zeros(mp.shape, order=order)
        chunks = [batch[i::6] for i in range(6)]
        flops = [0] * len(chunks)
        errors = []

        def work(i):
            try:
                flops[i] = h.apply_level(lvl, chunks[i], mp, loc)
            except Exception as e:  # pragma: no cover - surfaced below
                errors.append(e)

        ths = [threading.Thread(target=work, args=(i,)) for i in range(len(chunks))]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        assert not errors, errors
        err = O.rel_l2(loc, g[f"locals_{variant}_{lvl}"])
        assert err <= TOL[variant], (variant, lvl, err)
        assert h.flops[lvl] == sum(flops)
        if variant != "sa":  # SA counts distinct sources per call, so chunking changes its total (m2l.py:373-379)
            assert sum(flops) == int(g[f"flops_{variant}_{lvl}"])


@pytest.mark.parametrize("order", [4, 5, 9])
def test_device_assembly_matches_host(torch_cuda, order):
    """cfm_assemble_operators vs assemble_for_transfer (kernels.py:167-179):
    Laplace bit-identical, Helmholtz to rounding (CUDA vs libm sin/cos)."""
    from paper_1210_7292_b200 import ChebyshevGrid, helmholtz_kernel, laplace_kernel
    from paper_1210_7292_b200.numerics import assemble_for_transfer
    from paper_1210_7292_b200.precompute import assemble_stack
    from paper_1210_7292_b200.symmetry import full_far_field_vectors

    grid = ChebyshevGrid(order)
    ts = full_far_field_vectors()
    if order == 9:
        ts = ts[::8]
    for kernel, width in ((laplace_kernel(), 0.25), (laplace_kernel(), 1.0 / 3.0), (helmholtz_kernel(8 * np.pi), 0.125),
                          (helmholtz_kernel(1.0), 0.5)):
        dev = assemble_stack(kernel, ts, width, grid, 0).cpu().numpy()
        host = np.stack([assemble_for_transfer(kernel, t, width, grid) for t in ts])
        if kernel.name == "laplace":
            assert np.array_equal(dev, host), np.abs(dev - host).max()
        else:
            assert np.abs(dev - host).max() <= 1e-15 * np.abs(host).max()


def test_device_assembly_rejects_bad_input(torch_cuda):
    from paper_1210_7292_b200 import ChebyshevGrid, laplace_kernel
    from paper_1210_7292_b200.precompute import assemble_stack

    with pytest.raises(ValueError):
        assemble_stack(laplace_kernel(), [(1, 1, 1)], 0.25, ChebyshevGrid(4), 0)
    with pytest.raises(ValueError):
        assemble_stack(laplace_kernel(), [(2, 0, 0)], -1.0, ChebyshevGrid(4), 0)


@pytest.mark.parametrize("case,variant", [("cfg1", "ia"), ("cfg1", "iablk"), ("cfg1", "sa"), ("cfg1", "sarcmp"),
                                          ("helm", "sa"), ("helm", "iasym"), ("aca", "sa")])
def test_host_precompute_path(torch_cuda, golden, case, variant):
    """precompute_on='host' (the reference's host assembly + LAPACK) gives the
    same locals, ranks and accounting as the default device precompute."""
    g = golden(case)
    h_dev, levels = _handler(g, variant)
    h_host, _ = _handler(g, variant, precompute_on="host")
    assert h_dev.precompute_on == "device" and h_host.precompute_on == "host"
    for lvl in levels:
        mp = _mpoles(g, lvl, case)
        tgt, off, src, t = (g[f"{k}_{lvl}"] for k in ("tgt", "off", "src", "t"))
        for h in (h_dev, h_host):
            loc = np.zeros(mp.shape, dtype=np.result_type(h.kernel.dtype, mp.dtype))
            h.apply_level_csr(lvl, tgt, off, src, t, mp, loc)
            assert O.rel_l2(loc, g[f"locals_{variant}_{lvl}"]) <= TOL[variant]
            assert h.level_ranks(lvl) == list(g[f"ranks_{variant}_{lvl}"])
    for attr in ("operator_count", "stored_bytes"):
        assert getattr(h_dev, attr)() == getattr(h_host, attr)()
    assert h_dev.factorization_calls == h_host.factorization_calls


@pytest.mark.parametrize("mode", ["target", "pair"])
@pytest.mark.parametrize("case", ["sphere_lists", "cube_l5"])
def test_interior_boundary_split_equals_single_gpu(torch_cuda, golden, case, mode, monkeypatch):
    """The overlapped multi-GPU step, one shard at a time on one GPU: interior
    targets (distributed.split_interior) applied while the shard's halo rows
    are still zero, boundary targets after they are filled -- two handlers,
    as bench.py uses them -- reproduce the single-plan locals bitwise (with the
    plan mode fixed: target and pair plans sum a target's pairs in different
    orders, so a subset whose fill picks the other mode agrees to ~1e-15)."""
    torch = torch_cuda
    monkeypatch.setenv("CFM_PLAN_MODE", mode)
    from paper_1210_7292_b200 import ChebyshevGrid, full_far_field_vectors, laplace_kernel, make_handler
    from paper_1210_7292_b200.distributed import owner_of_rows, partition_rows, split_interior

    if case == "sphere_lists":
        g = golden("sphere_lists")
        lvl = 4
        cells = g[f"cells_{lvl}"]
        mp = torch.from_numpy(_mpoles(g, lvl, "sphere_lists")).cuda()
        mk = lambda: _handler(g, "nablk")[0]  # noqa: E731
    else:  # l = 5: full-operator TMA path
        lvl, order = 4, 5
        side = 1 << lvl
        cells = np.stack(np.meshgrid(*(np.arange(side),) * 3, indexing="ij"), -1).reshape(-1, 3).astype(np.int32)
        mp = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, (len(cells), order**3))).cuda()

        def mk():
            h = make_handler("nablk", laplace_kernel(), ChebyshevGrid(order), 1e-5)
            h.precompute({lvl: full_far_field_vectors()}, {lvl: 1.0 / side})
            return h
    h = mk()
    h.plan_level_cells(lvl, cells)
    ref = torch.zeros_like(mp)
    h.apply_planned(lvl, mp, ref)
    out = torch.zeros_like(mp)
    parts = partition_rows(cells, 3)
    owner = owner_of_rows(parts, len(cells))
    for r, part in enumerate(parts):
        inner, bnd = split_interior(cells, lvl, part, owner)
        assert len(bnd) > 0
        local = torch.zeros_like(mp)
        rows = torch.as_tensor(part, device="cuda")
        local[rows] = mp[rows]
        loc = torch.zeros_like(mp)
        if len(inner):
            hi = mk()
            hi.plan_level_cells_subset(lvl, cells, inner)
            hi.apply_planned(lvl, local, loc)  # halo rows still zero
        hb = mk()
        _, srcs = hb.plan_level_cells_subset(lvl, cells, bnd)
        idx = torch.as_tensor(srcs, device="cuda")
        local[idx] = mp[idx]  # the exchange
        hb.apply_planned(lvl, local, loc)
        out[rows] = loc[rows]
    assert torch.equal(out, ref)


def test_applies_on_different_streams(torch_cuda):
    """Back-to-back applies from two CUDA streams share the handler's scratch
    (padded sources, pair rows): the second waits for the first."""
    torch = torch_cuda
    from paper_1210_7292_b200 import ChebyshevGrid, full_far_field_vectors, laplace_kernel, make_handler

    lvl, order = 4, 5
    side = 1 << lvl
    cells = np.stack(np.meshgrid(*(np.arange(side),) * 3, indexing="ij"), -1).reshape(-1, 3).astype(np.int32)
    h = make_handler("nablk", laplace_kernel(), ChebyshevGrid(order), 1e-5)
    h.precompute({lvl: full_far_field_vectors()}, {lvl: 1.0 / side})
    h.plan_level_cells(lvl, cells)
    rng = np.random.default_rng(9)
    mps = [torch.from_numpy(rng.uniform(-1, 1, (len(cells), order**3))).cuda() for _ in range(4)]
    ref = []
    for m in mps:
        y = torch.zeros_like(m)
        h.apply_levels({lvl: (m, y)})
        ref.append(y)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [torch.zeros_like(m) for m in mps]
    torch.cuda.synchronize()
    for i, m in enumerate(mps):
        with torch.cuda.stream(streams[i % 2]):
            h.apply_levels({lvl: (m, outs[i])})
    torch.cuda.synchronize()
    for a, b in zip(outs, ref):
        assert torch.equal(a, b)


@pytest.mark.parametrize("order", [5, 7])
def test_merged_pair_levels_bitwise(torch_cuda, order, monkeypatch):
    """Sparse (sphere) levels in pair mode on the full-operator path: the
    merged multi-level pair plan of apply_levels gives bitwise the per-level
    results (same per-pair products, same per-target summation order), and
    matches the oracle."""
    torch = torch_cuda
    from paper_1210_7292_b200 import ChebyshevGrid, full_far_field_vectors, laplace_kernel, make_handler

    monkeypatch.setenv("CFM_PLAN_MODE", "pair")
    rng = np.random.default_rng(21)
    pts = rng.normal(size=(20000, 3))
    pts /= np.linalg.norm(pts, axis=1, keepdims=True)
    depth = 5
    side = 1 << depth
    leaf = np.unique(np.minimum(((pts + 1.0) / 2.0 * side).astype(np.int64), side - 1), axis=0)
    cells = {depth: leaf}
    for lvl in range(depth - 1, 1, -1):
        cells[lvl] = np.unique(cells[lvl + 1] >> 1, axis=0)
    levels = sorted(cells)
    h = make_handler("nablk", laplace_kernel(), ChebyshevGrid(order), 1e-5)
    h.precompute({l: full_far_field_vectors() for l in levels}, {l: 2.0 / (1 << l) for l in levels})
    arrays, ref = {}, {}
    for lvl in levels:
        st = h.plan_level_cells(lvl, cells[lvl].astype(np.int32))
        assert st["mode"] == "pair"
        mp = torch.from_numpy(rng.uniform(-1, 1, (len(cells[lvl]), order**3))).cuda()
        ref[lvl] = torch.zeros_like(mp)
        h.apply_planned(lvl, mp, ref[lvl])
        arrays[lvl] = (mp, torch.zeros_like(mp))
    h.apply_levels(arrays)
    h.apply_levels(arrays)  # the cached merged plan is reused
    for lvl in levels:
        assert torch.equal(arrays[lvl][1], 2 * ref[lvl])
    lvl = levels[1]
    tgt, off, src, t = O.far_lists(cells[lvl], lvl)
    orc = O.OracleM2L("nablk", O.laplace_profile, np.float64, order, 1e-5, -1.0).precompute(
        {lvl: O.full_far_field()}, {lvl: 2.0 / (1 << lvl)})
    want = np.zeros((len(cells[lvl]), order**3))
    orc.apply_fast(lvl, tgt, off, src, t, arrays[lvl][0].cpu().numpy(), want)
    assert O.rel_l2(ref[lvl].cpu().numpy(), want) <= 1e-12


def test_full_operator_edge_cases(torch_cuda, monkeypatch):
    """Full-operator path edge cases: a level with no far pairs, a one-cell
    level, odd row counts, merged pair plan with an empty level, repeated and
    interleaved apply_levels / apply_planned calls."""
    torch = torch_cuda
    from paper_1210_7292_b200 import ChebyshevGrid, full_far_field_vectors, laplace_kernel, make_handler

    order = 5
    cells = {2: np.array([[1, 1, 1]]),                      # one cell: no far pairs
             3: np.array([[0, 0, 0], [7, 7, 7], [0, 7, 3]]),  # three scattered cells
             4: np.array([[0, 0, 0], [15, 15, 15], [3, 9, 12], [8, 1, 5], [14, 0, 7]])}
    levels = sorted(cells)
    h = make_handler("nablk", laplace_kernel(), ChebyshevGrid(order), 1e-5)
    h.precompute({l: full_far_field_vectors() for l in levels}, {l: 1.0 / (1 << l) for l in levels})
    rng = np.random.default_rng(2)
    arrays, ref = {}, {}
    for lvl in levels:
        st = h.plan_level_cells(lvl, cells[lvl].astype(np.int32))
        mp = torch.from_numpy(rng.uniform(-1, 1, (len(cells[lvl]), order**3))).cuda()
        ref[lvl] = torch.zeros_like(mp)
        h.apply_planned(lvl, mp, ref[lvl])
        arrays[lvl] = (mp, torch.zeros_like(mp))
        tgt, off, src, t = O.far_lists(cells[lvl], lvl)
        assert st["pairs"] == len(src)
        if len(src):
            orc = O.OracleM2L("nablk", O.laplace_profile, np.float64, order, 1e-5, -1.0).precompute(
                {lvl: O.full_far_field()}, {lvl: 1.0 / (1 << lvl)})
            want = np.zeros((len(cells[lvl]), order**3))
            orc.apply_fast(lvl, tgt, off, src, t, mp.cpu().numpy(), want)
            assert O.rel_l2(ref[lvl].cpu().numpy(), want) <= 1e-12
        else:
            assert not torch.any(ref[lvl])
    for _ in range(2):
        h.apply_levels(arrays)
    for lvl in levels:
        assert torch.equal(arrays[lvl][1], 2 * ref[lvl])
    # host buffers through the same path
    host = {lvl: (arrays[lvl][0].cpu().numpy(), np.zeros((len(cells[lvl]), order**3))) for lvl in levels}
    h.apply_levels(host)
    for lvl in levels:
        assert np.array_equal(host[lvl][1], ref[lvl].cpu().numpy())


def _shell_cells(level):
    side = 1 << level
    c = _full_level(level).astype(np.float64)
    r = np.linalg.norm((c + 0.5) / side - 0.5, axis=1)
    return _full_level(level)[np.abs(r - 0.4) < 1.5 / side]


@pytest.mark.parametrize("case", ["cube4", "sparse5", "shell6"])
def test_device_classifier_bit_exact(torch_cuda, case):
    """cfm_classify_count_device / cfm_classify_fill_device (the device far
    lists of B200FmmPlan and the bench's classifier line; one warp per
    occupied sibling group) against the oracle's restatement of
    build_interaction_lists: per target the same source rows in the same
    order and the same t codes, bit for bit; empty lists included."""
    import ctypes

    torch = torch_cuda
    from paper_1210_7292_b200 import _native

    if case == "cube4":
        level, cells = 4, _full_level(4)
    elif case == "sparse5":
        level = 5
        cells = _full_level(5)
        cells = cells[np.random.default_rng(3).random(len(cells)) < 0.25]
    else:
        level, cells = 6, _shell_cells(6)
    cells = np.ascontiguousarray(cells.astype(np.int32))
    n = len(cells)
    lib = _native.load()
    d = torch.from_numpy(cells).cuda()
    offs = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    tot = ctypes.c_int64()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _native.check(lib.cfm_classify_count_device(0, level, n, d.data_ptr(), offs.data_ptr(), ctypes.byref(tot), st))
    src = torch.empty(max(tot.value, 1), dtype=torch.int32, device="cuda")
    code = torch.empty(max(tot.value, 1), dtype=torch.int16, device="cuda")
    _native.check(lib.cfm_classify_fill_device(0, level, n, d.data_ptr(), offs.data_ptr(), src.data_ptr(),
                                               code.data_ptr(), st))
    torch.cuda.synchronize()
    offs, src, code = offs.cpu().numpy(), src.cpu().numpy()[: tot.value], code.cpu().numpy()[: tot.value]
    tgt, o_off, o_src, o_t = O.far_lists(cells, level)
    counts = np.zeros(n, np.int64)
    counts[tgt] = np.diff(o_off)
    assert tot.value == o_off[-1]
    assert np.array_equal(np.diff(offs), counts)
    ref_src = np.zeros(tot.value, np.int64)
    ref_code = np.zeros(tot.value, np.int64)
    for k, i in enumerate(tgt):
        a, b = offs[i], offs[i + 1]
        ref_src[a:b] = o_src[o_off[k]:o_off[k + 1]]
        tt = o_t[o_off[k]:o_off[k + 1]]
        ref_code[a:b] = (tt[:, 0] + 3) * 49 + (tt[:, 1] + 3) * 7 + (tt[:, 2] + 3)
    assert np.array_equal(src.astype(np.int64), ref_src)
    assert np.array_equal(code.astype(np.int64), ref_code)


@pytest.mark.gpu
@pytest.mark.parametrize("order,eps", [(6, 1e-5), (7, 1e-7), (4, 1e-4)])
def test_two_stage_target_major_other_orders(torch_cuda, order, eps, monkeypatch):
    """Target-major two-stage path at other expansion sizes: l = 6 (216 rows: two
    128-row result blocks per stage-2 tile, 7 K-chunks in stage 1), l = 7 with
    ranks above 32 (343 rows, three row blocks), and l = 4 (n = 64: below the
    full-operator TMA sizes, so the level must fall back to the fused kernel).
    Full level 4 (4,096 cells), iablk, vs the oracle (<= 1e-10)."""
    torch = torch_cuda
    from paper_1210_7292_b200 import ChebyshevGrid, laplace_kernel, make_handler

    monkeypatch.setenv("CFM_LR_TWOSTAGE", "2")
    level = 4
    cells = _full_level(level)
    tgt, off, src, t = O.far_lists(cells, level)
    transfers = sorted({tuple(int(c) for c in v) for v in t})
    lw = {level: 1.0 / (1 << level)}
    h = make_handler("iablk", laplace_kernel(), ChebyshevGrid(order), eps)
    h.precompute({level: transfers}, lw)
    h.plan_level_cells(level, cells)
    assert h.plan_stats(level)["two_stage"] == (order >= 5)
    mp = torch.from_numpy(np.random.default_rng(29).uniform(-1, 1, (len(cells), order**3))).cuda()
    loc = torch.full(mp.shape, -0.75, dtype=torch.float64, device="cuda")
    flops = h.apply_planned(level, mp, loc)
    orc = O.OracleM2L("iablk", O.laplace_profile, np.float64, order, eps, -1.0).precompute({level: transfers}, lw)
    ref = np.full(mp.shape, -0.75)
    fr = orc.apply_fast(level, tgt, off, src, t, mp.cpu().numpy(), ref)
    assert flops == fr
    assert O.rel_l2(loc.cpu().numpy() + 0.75, ref + 0.75) <= 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("order,shape", [(5, "cube"), (9, "shell")])
def test_persistent_step_kernel_matches_tile_kernel(torch_cuda, order, shape, monkeypatch):
    """The persistent step kernel (default) against the one-CTA-per-tile kernel
    (CFM_STEP_PERSIST=0), multi-level apply_levels and per-level apply_planned:
    l = 5 on full levels 3-4 (target tiles + hybrid pair entries), l = 9 on a
    spherical shell (pair entries, 89-row last block: the dead-m-tile path).
    Both run the same chunks in the same order per accumulator; only the
    rank-1 k-tail of the l = 5 tile kernel differs (round-off)."""
    torch = torch_cuda
    from paper_1210_7292_b200 import ChebyshevGrid, full_far_field_vectors, laplace_kernel, make_handler

    levels = (3, 4)
    cells = {}
    for l in levels:
        c = _full_level(l)
        if shape == "shell":
            r = np.linalg.norm((c + 0.5) / (1 << l) * 2 - 1, axis=1)
            c = c[(r > 0.6) & (r < 0.95)]
        cells[l] = c
    rng = np.random.default_rng(31)
    mp = {l: torch.from_numpy(rng.uniform(-1, 1, (len(cells[l]), order**3))).cuda() for l in levels}
    out, single = {}, {}
    for persist in ("1", "0"):
        monkeypatch.setenv("CFM_STEP_PERSIST", persist)
        h = make_handler("nablk", laplace_kernel(), ChebyshevGrid(order), 1e-8)
        h.precompute({l: full_far_field_vectors() for l in levels}, {l: 1.0 / (1 << l) for l in levels})
        for l in levels:
            h.plan_level_cells(l, cells[l])
        loc = {l: torch.full_like(mp[l], 0.125) for l in levels}
        h.apply_levels({l: (mp[l], loc[l]) for l in levels})
        one = torch.full_like(mp[4], 0.125)
        h.apply_planned(4, mp[4], one)
        out[persist] = {l: loc[l].cpu().numpy() for l in levels}
        single[persist] = one.cpu().numpy()
    for l in levels:
        assert O.rel_l2(out["1"][l], out["0"][l]) <= 1e-14, (l, O.rel_l2(out["1"][l], out["0"][l]))
        tgt, off, src, t = O.far_lists(cells[l], l)
        orc = O.OracleM2L("nablk", O.laplace_profile, np.float64, order, 1e-8, -1.0).precompute(
            {l: sorted({tuple(int(c) for c in v) for v in t})}, {l: 1.0 / (1 << l)})
        ref = np.full(mp[l].shape, 0.125)
        orc.apply_fast(l, tgt, off, src, t, mp[l].cpu().numpy(), ref)
        assert O.rel_l2(out["1"][l] - 0.125, ref - 0.125) <= 1e-12
    assert O.rel_l2(single["1"], single["0"]) <= 1e-14
    assert O.rel_l2(single["1"], out["1"][4]) <= 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("path", ["twopass_ft", "twopass", "fused"])
@pytest.mark.parametrize("mode", ["target", "pair"])
def test_lowrank_paths_on_sparse_levels(torch_cuda, path, mode, monkeypatch):
    """The three low-rank kernels paths on a sparse level (spherical shell at
    level 4, iablk l = 5) as target tiles and as pair entries: the fused kernel,
    the two-pass path on the permuted-gather kernels (what ranks above 64 take)
    and the two-pass path on the full-operator kernels (per-transfer factors,
    persistent step kernel; the default for complex operators), each vs the
    oracle (<= 1e-10).  Target tiles of such a level are re-ordered by row after
    they are built: the per-entry slots of the two-pass paths must follow that
    order (regression: they were built before it and dropped live columns)."""
    torch = torch_cuda
    from paper_1210_7292_b200 import ChebyshevGrid, full_far_field_vectors, laplace_kernel, make_handler

    monkeypatch.setenv("CFM_PLAN_MODE", mode)
    monkeypatch.setenv("CFM_LR_TWOSTAGE", "0")
    monkeypatch.setenv("CFM_LOWRANK_FUSED", "1" if path == "fused" else "0")
    monkeypatch.setenv("CFM_LR_TWOPASS", "1" if path == "twopass_ft" else "0")
    order, level, eps = 5, 4, 1e-5
    cells = _full_level(level)
    r = np.linalg.norm((cells + 0.5) / (1 << level) * 2 - 1, axis=1)
    cells = cells[(r > 0.55) & (r < 0.95)]
    tgt, off, src, t = O.far_lists(cells, level)
    lw = {level: 1.0 / (1 << level)}
    h = make_handler("iablk", laplace_kernel(), ChebyshevGrid(order), eps)
    h.precompute({level: full_far_field_vectors()}, lw)
    st = h.plan_level_cells(level, cells)
    assert st["mode"] == mode
    mp = torch.from_numpy(np.random.default_rng(37).uniform(-1, 1, (len(cells), order**3))).cuda()
    loc = torch.full(mp.shape, 0.5, dtype=torch.float64, device="cuda")
    h.apply_planned(level, mp, loc)
    orc = O.OracleM2L("iablk", O.laplace_profile, np.float64, order, eps, -1.0).precompute(
        {level: sorted({tuple(int(c) for c in v) for v in t})}, lw)
    ref = np.full(mp.shape, 0.5)
    orc.apply_fast(level, tgt, off, src, t, mp.cpu().numpy(), ref)
    assert O.rel_l2(loc.cpu().numpy() - 0.5, ref - 0.5) <= 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("twopass", ["1", "0"])
def test_lowrank_ranks_above_64(torch_cuda, twopass, monkeypatch):
    """ia at l = 7, eps = 1e-9: ranks above 64, which the fused kernel cannot
    hold -- the level takes the two-pass path, on the full-operator kernels
    (default) or on the permuted-gather kernels (CFM_LR_TWOPASS=0).  Full
    level 3 (target tiles) vs the oracle (<= 1e-10), ranks equal."""
    torch = torch_cuda
    from paper_1210_7292_b200 import ChebyshevGrid, laplace_kernel, make_handler

    monkeypatch.setenv("CFM_LR_TWOPASS", twopass)
    monkeypatch.setenv("CFM_LR_TWOSTAGE", "0")
    # the per-pair intermediate in ~10 chunks of tiles (default 1 GB per chunk): later chunks
    # address their slots relative to the chunk (a TMA map based below the buffer faults)
    monkeypatch.setenv("CFM_Y_CHUNK_MB", "8")
    order, level, eps = 7, 3, 1e-9
    cells = _full_level(level)
    tgt, off, src, t = O.far_lists(cells, level)
    transfers = sorted({tuple(int(c) for c in v) for v in t})
    lw = {level: 1.0 / (1 << level)}
    h = make_handler("ia", laplace_kernel(), ChebyshevGrid(order), eps)
    h.precompute({level: transfers}, lw)
    h.plan_level_cells(level, cells)
    assert max(h.level_ranks(level)) > 64
    mp = torch.from_numpy(np.random.default_rng(41).uniform(-1, 1, (len(cells), order**3))).cuda()
    loc = torch.zeros(mp.shape, dtype=torch.float64, device="cuda")
    flops = h.apply_planned(level, mp, loc)
    orc = O.OracleM2L("ia", O.laplace_profile, np.float64, order, eps, -1.0).precompute({level: transfers}, lw)
    assert orc.level_ranks(level) == h.level_ranks(level)
    ref = np.zeros(mp.shape)
    fr = orc.apply_fast(level, tgt, off, src, t, mp.cpu().numpy(), ref)
    assert flops == fr
    assert O.rel_l2(loc.cpu().numpy(), ref) <= 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("envs", [{"CFM_TS_KERNEL": "step"}, {"CFM_TS_PERSIST": "0"},
                                  {"CFM_TS_PERSIST": "0", "CFM_STEP_PERSIST": "0"}, {"CFM_TS_SKEW": "0"}])
def test_two_stage_target_major_kernel_variants(torch_cuda, envs, monkeypatch):
    """The other kernels that can run the target-major two-stage path: the
    dynamic-queue step kernel (its Y_T-scatter mode), the generic launch path
    with and without the persistent step kernel (one CTA per tile on
    tile_gemm_ws_kernel), and unskewed consumer halves.  Full level 4, iablk
    l = 5, vs the oracle (<= 1e-10)."""
    torch = torch_cuda
    from paper_1210_7292_b200 import ChebyshevGrid, laplace_kernel, make_handler

    monkeypatch.setenv("CFM_LR_TWOSTAGE", "2")
    for k, v in envs.items():
        monkeypatch.setenv(k, v)
    order, level, eps = 5, 4, 1e-5
    cells = _full_level(level)
    tgt, off, src, t = O.far_lists(cells, level)
    transfers = sorted({tuple(int(c) for c in v) for v in t})
    lw = {level: 1.0 / (1 << level)}
    h = make_handler("iablk", laplace_kernel(), ChebyshevGrid(order), eps)
    h.precompute({level: transfers}, lw)
    h.plan_level_cells(level, cells)
    assert h.plan_stats(level)["two_stage"]
    mp = torch.from_numpy(np.random.default_rng(43).uniform(-1, 1, (len(cells), order**3))).cuda()
    loc = torch.full(mp.shape, 1.5, dtype=torch.float64, device="cuda")
    h.apply_planned(level, mp, loc)
    orc = O.OracleM2L("iablk", O.laplace_profile, np.float64, order, eps, -1.0).precompute({level: transfers}, lw)
    ref = np.full(mp.shape, 1.5)
    orc.apply_fast(level, tgt, off, src, t, mp.cpu().numpy(), ref)
    assert O.rel_l2(loc.cpu().numpy() - 1.5, ref - 1.5) <= 1e-10
