"""The device planner (csrc/plan_device.cu) against the host plan builder
(plan.hpp build_plan_csr + plan.cu's row-order dispatch / slabs / hybrid split,
CFM_DEVICE_PLAN=0): identical plan statistics and bitwise identical locals,
device-resident (hybrid plans) and from host buffers (row-ordered plans with
the slab pipeline), on full and partially occupied levels."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _cube(level):
    s = 1 << level
    return np.stack(np.meshgrid(*(np.arange(s),) * 3, indexing="ij"), -1).reshape(-1, 3).astype(np.int32)


def _sparse(level, keep, seed):
    c = _cube(level)
    rng = np.random.default_rng(seed)
    return c[rng.uniform(size=len(c)) < keep]


@pytest.mark.parametrize("case", ["cube5_l5", "cube4_l7", "sparse6_l5", "shell5_l5"])
def test_device_plan_matches_host_plan(case, monkeypatch):
    import torch

    from paper_1210_7292_b200 import ChebyshevGrid, full_far_field_vectors, laplace_kernel, make_handler

    if case == "cube5_l5":
        level, order, cells = 5, 5, _cube(5)
    elif case == "cube4_l7":
        level, order, cells = 4, 7, _cube(4)
    elif case == "sparse6_l5":
        level, order, cells = 6, 5, _sparse(6, 0.6, 3)
    else:  # a spherical shell: boundary-heavy, many partial tiles
        level, order = 5, 5
        c = _cube(level).astype(np.float64) + 0.5 - 16
        r = np.linalg.norm(c, axis=1)
        cells = _cube(level)[(r > 9) & (r < 14)]
    n = order**3
    rng = np.random.default_rng(1)
    mp_h = rng.uniform(-1, 1, (len(cells), n))
    out = {}
    for dev_plan in ("1", "0"):
        monkeypatch.setenv("CFM_DEVICE_PLAN", dev_plan)
        h = make_handler("nablk", laplace_kernel(), ChebyshevGrid(order), 1e-5)
        h.precompute({level: full_far_field_vectors()}, {level: 1.0 / (1 << level)})
        st = h.plan_level_cells(level, cells)
        mp = torch.from_numpy(mp_h).cuda()
        loc = torch.zeros_like(mp)
        fl = h.apply_levels({level: (mp, loc)})
        torch.cuda.synchronize()
        pin_mp = torch.from_numpy(mp_h).pin_memory()
        pin_loc = torch.zeros(mp_h.shape, dtype=torch.float64).pin_memory()
        h.apply_levels({level: (pin_mp.numpy(), pin_loc.numpy())})
        out[dev_plan] = (dict((k, v) for k, v in st.items() if k != "counts"), st["counts"].copy(), fl,
                         loc.cpu().numpy(), pin_loc.numpy().copy())
    (st1, c1, f1, d1, p1), (st0, c0, f0, d0, p0) = out["1"], out["0"]
    assert st1 == st0
    assert np.array_equal(c1, c0) and f1 == f0
    assert np.array_equal(d1, d0), float(np.abs(d1 - d0).max())
    assert np.array_equal(p1, p0), float(np.abs(p1 - p0).max())
    tgt, off, src, t = O.far_lists(cells, level)
    orc = O.OracleM2L("nablk", O.laplace_profile, np.float64, order, 1e-5, -1.0).precompute(
        {level: O.full_far_field()}, {level: 1.0 / (1 << level)})
    ref = np.zeros_like(mp_h)
    orc.apply_fast(level, tgt, off, src, t, mp_h, ref)
    assert O.rel_l2(d1, ref) <= 1e-12


def test_device_plan_for_csr_subsets_matches_host(monkeypatch):
    """plan_level_csr with a rank-like subset of ascending target rows (the
    shard-local lists ShardedM2L plans) takes the device planner too: bitwise
    equal to the host builder."""
    import torch

    from paper_1210_7292_b200 import ChebyshevGrid, full_far_field_vectors, laplace_kernel, make_handler

    level, order = 5, 5
    cells = _cube(level)
    rows = np.nonzero(cells[:, 0] < 12)[0]  # a Morton-free slab of targets, ascending
    tgt, off, src, t = O.far_lists(cells, level, targets=rows)
    n = order**3
    mp_h = np.random.default_rng(2).uniform(-1, 1, (len(cells), n))
    out = {}
    for dev_plan in ("1", "0"):
        monkeypatch.setenv("CFM_DEVICE_PLAN", dev_plan)
        h = make_handler("nablk", laplace_kernel(), ChebyshevGrid(order), 1e-5)
        h.precompute({level: full_far_field_vectors()}, {level: 1.0 / (1 << level)})
        st = h.plan_level_csr(level, tgt, off, src, t, len(cells))
        mp = torch.from_numpy(mp_h).cuda()
        loc = torch.zeros_like(mp)
        fl = h.apply_levels({level: (mp, loc)})
        torch.cuda.synchronize()
        out[dev_plan] = ({k: v for k, v in st.items() if k != "counts"}, fl, loc.cpu().numpy())
    assert out["1"][0] == out["0"][0] and out["1"][1] == out["0"][1]
    assert np.array_equal(out["1"][2], out["0"][2])


def test_device_planner_edge_levels():
    """Levels the device planner must hand back or handle: no pairs at all, a
    sparse level that plans as pair entries (host builder), a dense level whose
    every tile is full (no hybrid leftovers); results vs the oracle."""
    import torch

    from paper_1210_7292_b200 import ChebyshevGrid, full_far_field_vectors, laplace_kernel, make_handler

    order, n = 5, 125
    cases = {
        "single_cell": (3, np.array([[1, 2, 3]], np.int32)),
        "two_far_cells": (4, np.array([[0, 0, 0], [8, 8, 8]], np.int32)),
        "sparse_pairs": (5, _sparse(5, 0.05, 7)),
        "full_cube_l4": (4, _cube(4)),
    }
    for name, (level, cells) in cases.items():
        h = make_handler("nablk", laplace_kernel(), ChebyshevGrid(order), 1e-5)
        h.precompute({level: full_far_field_vectors()}, {level: 1.0 / (1 << level)})
        st = h.plan_level_cells(level, cells)
        mp_h = np.random.default_rng(4).uniform(-1, 1, (len(cells), n))
        mp = torch.from_numpy(mp_h).cuda()
        loc = torch.zeros_like(mp)
        fl = h.apply_levels({level: (mp, loc)})
        torch.cuda.synchronize()
        tgt, off, src, t = O.far_lists(cells, level)
        ref = np.zeros_like(mp_h)
        if len(src):
            orc = O.OracleM2L("nablk", O.laplace_profile, np.float64, order, 1e-5, -1.0).precompute(
                {level: O.full_far_field()}, {level: 1.0 / (1 << level)})
            orc.apply_fast(level, tgt, off, src, t, mp_h, ref)
        assert st["pairs"] == len(src), name
        assert fl == 2 * n * n * len(src), name
        got = loc.cpu().numpy()
        assert (np.abs(got).max() == 0.0) if not len(src) else O.rel_l2(got, ref) <= 1e-12, name


def test_lowrank_host_pipeline_bitwise(monkeypatch):
    """iablk from pinned host buffers over levels 4-6 of a full cube (level 6
    two-stage, streamed: stage 1 in chunks of row-ordered source tiles that start
    on the first multipole slabs, stage 2 in chunks of row-ordered target tiles
    that wait for their locals slabs and whose rows download while later chunks
    run), non-zero initial locals: bitwise the device-resident apply, and the
    same with the slabs off (CFM_TS_SLABS=0 is read once per process, so the
    whole-array variant is covered by CFM_LR_PIPELINE=0)."""
    import torch

    from paper_1210_7292_b200 import ChebyshevGrid, full_far_field_vectors, laplace_kernel, make_handler

    order, n, levels = 5, 125, (4, 5, 6)
    h = make_handler("iablk", laplace_kernel(), ChebyshevGrid(order), 1e-5)
    h.precompute({l: full_far_field_vectors() for l in levels}, {l: 1.0 / (1 << l) for l in levels})
    rng = np.random.default_rng(9)
    mp_h = {l: rng.uniform(-1, 1, ((1 << l) ** 3, n)) for l in levels}
    for l in levels:
        h.plan_level_cells(l, _cube(l))
    assert h.plan_stats(6)["two_stage"]
    loc0 = {l: rng.uniform(-1, 1, mp_h[l].shape) for l in levels}  # locals accumulate: non-zero start
    dev = {l: (torch.from_numpy(mp_h[l]).cuda(), torch.from_numpy(loc0[l]).cuda()) for l in levels}
    fl_d = h.apply_levels(dev)
    torch.cuda.synchronize()
    out = {}
    for pipe in ("1", "0"):
        monkeypatch.setenv("CFM_LR_PIPELINE", pipe)
        arrs = {l: (torch.from_numpy(mp_h[l]).pin_memory().numpy(),
                    torch.from_numpy(loc0[l].copy()).pin_memory().numpy()) for l in levels}
        fl = h.apply_levels(arrs)
        assert fl == fl_d
        out[pipe] = {l: arrs[l][1].copy() for l in levels}
    for l in levels:
        d = dev[l][1].cpu().numpy()
        assert np.array_equal(out["1"][l], d), (l, float(np.abs(out["1"][l] - d).max()))
        assert np.array_equal(out["0"][l], d)
