"""Generate the golden fixtures under tests/golden/ by EXECUTING the reference.

Run here (not on the GPU box), from the repo root:

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

The reference package (``chebfmm``, read-only under /root/reference) ships no
tests and no golden vectors, so parity is pinned by
running its own code on seeded inputs and storing the outputs here.  Every
array below is produced by a reference call; nothing is written by hand.
The fixtures are small (a few MB) and travel with the repo; the GPU box never
reads /root/reference.

Reference call sites used (file:line under /root/reference/pkg/src/chebfmm):
  octree.full_far_field_vectors (octree.py:201), symmetry.canonicalize
  (symmetry.py:63), permutation_index_table (:86), SymmetryMap (:114),
  build_tree (octree.py:93), build_interaction_lists (:148),
  FmmPlan._level_data/_p2m/_m2m (engine.py:98-138), make_handler /
  precompute / apply_level (m2l.py:539,136,279), accounting (m2l.py:458-536),
  assemble_for_transfer (kernels.py:167).
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

try:
    import chebfmm  # noqa: F401
except ImportError:  # pragma: no cover
    sys.exit("set PYTHONPATH=/root/reference/pkg/src to generate golden fixtures")

from chebfmm.engine import FmmPlan
from chebfmm.interp import AffineMap, ChebyshevGrid
from chebfmm.kernels import assemble_for_transfer, helmholtz_kernel, laplace_kernel
from chebfmm.m2l import VARIANTS, make_handler
from chebfmm.octree import (
    build_interaction_lists,
    build_tree,
    full_far_field_vectors,
    unique_transfer_vectors,
)
from chebfmm.symmetry import (
    SymmetryMap,
    canonicalize,
    inverse_permutation_table,
    permutation_index_table,
)

OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(OUT))
from geometry import cube_points, sphere_points  # noqa: E402
AXIS_ORDERS = [(1, 2, 3), (1, 3, 2), (2, 1, 3), (2, 3, 1), (3, 1, 2), (3, 2, 1)]


def spec_id(spec) -> int:
    f = spec.axial_flips
    return (int(f[0]) | int(f[1]) << 1 | int(f[2]) << 2) * 6 + AXIS_ORDERS.index(tuple(spec.axis_order))


def symmetry_fixture() -> None:
    far = full_far_field_vectors()
    t_sym, flips, order, sid = [], [], [], []
    for t in far:
        ts, spec = canonicalize(t)
        t_sym.append(ts)
        flips.append(spec.axial_flips)
        order.append(spec.axis_order)
        sid.append(spec_id(spec))
    smap = SymmetryMap(far)
    rep_idx = [smap.assignment[tuple(t)][0] for t in far]
    # one table per spec id (all 48 ids are reachable from the 316 list)
    specs = {}
    for t in far:
        _, spec = canonicalize(t)
        specs.setdefault(spec_id(spec), spec)
    out = dict(
        far316=np.asarray(far, np.int8),
        t_sym=np.asarray(t_sym, np.int8),
        flips=np.asarray(flips, bool),
        axis_order=np.asarray(order, np.int8),
        spec_id=np.asarray(sid, np.int16),
        cone=np.asarray(smap.cone, np.int8),
        rep_idx=np.asarray(rep_idx, np.int16),
        spec_ids_present=np.asarray(sorted(specs), np.int16),
    )
    for order_l in (2, 3, 4, 5, 7, 9):
        tab = np.full((48, order_l**3), -1, np.int16)
        inv = np.full((48, order_l**3), -1, np.int16)
        for k, spec in specs.items():
            tab[k] = permutation_index_table(spec, order_l)
            inv[k] = inverse_permutation_table(spec, order_l)
        out[f"table_l{order_l}"] = tab
        out[f"inv_l{order_l}"] = inv
    # partial list: SymmetryMap on a subset (rep index is into the subset's cone)
    rng = np.random.default_rng(7)
    sub = [far[i] for i in sorted(rng.choice(len(far), 50, replace=False))]
    sub_map = SymmetryMap(sub)
    out["sub50"] = np.asarray(sub, np.int8)
    out["sub50_cone"] = np.asarray(sub_map.cone, np.int8)
    out["sub50_rep_idx"] = np.asarray([sub_map.assignment[tuple(t)][0] for t in sub], np.int16)
    np.savez_compressed(OUT / "symmetry.npz", **out)
    print("symmetry.npz", {k: v.shape for k, v in out.items()})


def _csr(batch):
    tgt = np.asarray([b[0] for b in batch], np.int32)
    counts = np.asarray([len(b[1]) for b in batch], np.int64)
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    src = np.asarray([s for b in batch for s, _ in b[1]], np.int32)
    tv = np.asarray([t for b in batch for _, t in b[1]], np.int8).reshape(-1, 3)
    return tgt, off, src, tv


def run_case(name, points, weights, bbox, depth, kernel, order, eps, variants,
             budget=2_000_000_000, store_rows=None, seeded_mpoles=None, extra=None, compression="svd",
             potentials_for=None):
    """Build tree/lists with the reference, run every variant's apply_level per
    level on identical multipoles, and store inputs + outputs + accounting."""
    t0 = time.time()
    tree = build_tree(points, bbox, depth)
    lists = build_interaction_lists(tree)
    grid = ChebyshevGrid(order)
    levels = lists.far_levels()
    lt = {lvl: unique_transfer_vectors(lists, lvl) for lvl in levels}
    lw = {lvl: tree.cell_width(lvl) for lvl in levels}
    out = dict(order=order, eps=eps, depth=depth, levels=np.asarray(levels), compression=np.asarray(compression),
               widths=np.asarray([lw[l] for l in levels]),
               kernel=np.asarray(kernel.name), bbox_center=np.asarray(bbox.center),
               bbox_half=bbox.half_width)
    if kernel.wavenumber is not None:
        out["wavenumber"] = kernel.wavenumber
    base = make_handler("nablk", kernel, grid, eps)
    plan = FmmPlan(tree, lists, grid, kernel, base, eps, 1)
    lv = plan._level_data(weights)
    if seeded_mpoles is None:
        plan._p2m(weights, lv[depth])
        plan._m2m(lv)
    for lvl in levels:
        d = lv[lvl]
        cells = np.asarray([c.ijk for c in d.cells], np.int16)
        tgt, off, src, tv = _csr(d.batch)
        out[f"cells_{lvl}"] = cells
        out[f"tgt_{lvl}"], out[f"off_{lvl}"], out[f"src_{lvl}"], out[f"t_{lvl}"] = tgt, off, src, tv
        if seeded_mpoles is not None:
            rng = np.random.default_rng(seeded_mpoles + lvl)
            m = rng.uniform(-1, 1, d.mpoles.shape)
            if np.iscomplexobj(d.mpoles):
                m = m + 1j * rng.uniform(-1, 1, d.mpoles.shape)
            d.mpoles[...] = m
        else:
            out[f"mpoles_{lvl}"] = d.mpoles.copy()
        if store_rows is not None:
            rng = np.random.default_rng(1000 + lvl)
            rows = np.sort(rng.choice(len(cells), min(store_rows, len(cells)), replace=False))
            out[f"rows_{lvl}"] = rows.astype(np.int32)
    for v in variants:
        h = make_handler(v, kernel, grid, eps, budget_bytes=budget, compression=compression)
        tp = time.time()
        h.precompute(lt, lw)
        tp = time.time() - tp
        for lvl in levels:
            d = lv[lvl]
            loc = np.zeros_like(d.locals_)
            h.apply_level(lvl, d.batch, d.mpoles, loc)
            if store_rows is not None:
                loc = loc[out[f"rows_{lvl}"]]
            out[f"locals_{v}_{lvl}"] = loc
            out[f"flops_{v}_{lvl}"] = h.flops.get(lvl, 0)
            out[f"ranks_{v}_{lvl}"] = np.asarray(h.level_ranks(lvl), np.int32)
            if h.is_shared_basis:
                out[f"shared_rank_{v}_{lvl}"] = h.shared_rank(lvl)
                rt = h.recompression_table(lvl)
                out[f"recomp_t_{v}_{lvl}"] = np.asarray([t for t, _ in rt], np.int8)
                out[f"recomp_r_{v}_{lvl}"] = np.asarray([-1 if r is None else r for _, r in rt], np.int32)
            if h.uses_blocking:
                bs = h.block_stats[lvl]
                out[f"blk_columns_{v}_{lvl}"] = bs["columns"]
                out[f"blk_products_{v}_{lvl}"] = bs["products"]
                out[f"blk_reps_{v}_{lvl}"] = len(bs["reps_used"])
                # the flush sequence itself: (representative transfer vector, columns) per flush
                out[f"blk_flush_t_{v}_{lvl}"] = np.asarray([r for r, _ in bs["flushes"]], np.int8).reshape(-1, 3)
                out[f"blk_flush_c_{v}_{lvl}"] = np.asarray([c for _, c in bs["flushes"]], np.int32)
        if potentials_for and v in potentials_for:
            # full reference pipeline (engine.py:201-222) with this handler
            plan_v = FmmPlan(tree, lists, grid, kernel, h, eps, 1)
            out[f"potentials_{v}"] = plan_v.run(weights)
            if "leaf_mpoles" not in out:
                lv2 = plan_v._level_data(weights)
                plan_v._p2m(weights, lv2[depth])
                out["leaf_mpoles"] = lv2[depth].mpoles.copy()
                plan_v._m2m(lv2)
                for lvl2 in levels:
                    out[f"up_mpoles_{lvl2}"] = lv2[lvl2].mpoles.copy()
        out[f"operator_count_{v}"] = h.operator_count()
        out[f"stored_bytes_{v}"] = h.stored_bytes()
        out[f"factorization_calls_{v}"] = h.factorization_calls
        out[f"precompute_s_{v}"] = tp
        print(f"  {name}:{v} precompute {tp:.1f}s", flush=True)
    if extra:
        extra(out, tree, lists, grid, kernel, lt, lw)
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(f"{name}.npz in {time.time() - t0:.1f}s; levels {levels}; pairs",
          {l: int(out[f'off_{l}'][-1]) for l in levels})


def main() -> None:
    only = set(sys.argv[1:])
    if only:
        if "aca" in only:
            aca_case()
        if "fmm" in only:
            fmm_cases()
        if "cfg3" in only:
            cfg3_case()
        if "cfg5" in only:
            cfg5_case()
        if "cfg1" in only:
            cfg1_case()
        if "fmmtrace" in only:
            fmmtrace_case()
        return
    symmetry_fixture()

    cfg1_case()
    _other_cases()


def cfg1_case() -> None:
    # BASELINE config 1: N=10,000 uniform cube, height 4 -> reference depth 3,
    # l=4, Laplace, charges U[-1,1]; multipoles from the reference's P2M/M2M.
    pts = cube_points(10_000, seed=1)
    w = np.random.default_rng(2).uniform(-1.0, 1.0, len(pts))

    def cfg1_extra(out, tree, lists, grid, kernel, lt, lw):
        ref = min(lt)
        cone = SymmetryMap(sorted(set().union(*lt.values()))).cone
        out["K_rep"] = np.stack([assemble_for_transfer(kernel, t, lw[ref], grid) for t in cone])
        out["K_rep_t"] = np.asarray(cone, np.int8)

    run_case("cfg1", pts, w, AffineMap((0.5, 0.5, 0.5), 0.5), 3, laplace_kernel(), 4, 1e-5,
             VARIANTS, extra=cfg1_extra)


def _other_cases() -> None:

    # Helmholtz (complex128) on a radius-1 sphere, k = 8*pi, l = 4, eps = 1e-4:
    # config 5's non-directional pipeline at fixture scale, complex charges.
    pts = sphere_points(3_000, seed=5)
    rng = np.random.default_rng(6)
    wc = rng.uniform(-1, 1, len(pts)) + 1j * rng.uniform(-1, 1, len(pts))
    run_case("helm", pts, wc, AffineMap((0.0, 0.0, 0.0), 1.0), 3, helmholtz_kernel(8 * np.pi),
             4, 1e-4, VARIANTS)

    # Laplace with complex weights: real operators x complex128 multipoles.
    pts = cube_points(2_000, seed=11)
    rng = np.random.default_rng(12)
    wc = rng.uniform(-1, 1, len(pts)) + 1j * rng.uniform(-1, 1, len(pts))
    run_case("lapcplx", pts, wc, AffineMap((0.5, 0.5, 0.5), 0.5), 3, laplace_kernel(), 3, 1e-3,
             ("na", "nablk", "iablk", "sa"))

    # Config 3 flavour: unit sphere, l = 9, nablk vs sa (eps = 1e-8), seeded
    # multipoles (M2L is linear), sampled output rows to keep the fixture small.
    pts = sphere_points(20_000, seed=3)
    w = np.random.default_rng(4).uniform(-1.0, 1.0, len(pts))
    run_case("sphere9", pts, w, AffineMap((0.0, 0.0, 0.0), 1.0), 3, laplace_kernel(), 9, 1e-8,
             ("nablk", "sa"), budget=4_000_000_000, store_rows=48, seeded_mpoles=33)

    # Classifier bit-exactness on a sparse tree (lists only, plus one variant).
    pts = sphere_points(30_000, seed=21)
    w = np.random.default_rng(22).uniform(-1.0, 1.0, len(pts))
    run_case("sphere_lists", pts, w, AffineMap((0.0, 0.0, 0.0), 1.0), 4, laplace_kernel(), 3, 1e-3,
             ("nasym",), seeded_mpoles=44, store_rows=32)

    aca_case()


def fmm_cases() -> None:
    """End-to-end potentials of the reference pipeline (P2M, M2M, M2L, L2L, L2P,
    P2P; engine.py:201-222) for the GPU FMM path."""
    pts = cube_points(6_000, seed=41)
    w = np.random.default_rng(42).uniform(-1.0, 1.0, len(pts))
    run_case("fmm_cube", pts, w, AffineMap((0.5, 0.5, 0.5), 0.5), 3, laplace_kernel(), 4, 1e-5,
             ("nablk", "iablk"), potentials_for=("nablk", "iablk"))
    pts = sphere_points(4_000, seed=43)
    rng = np.random.default_rng(44)
    wc = rng.uniform(-1, 1, len(pts)) + 1j * rng.uniform(-1, 1, len(pts))
    run_case("fmm_helm", pts, wc, AffineMap((0.0, 0.0, 0.0), 1.0), 3, helmholtz_kernel(8 * np.pi), 4, 1e-4,
             ("nablk", "iablk"), potentials_for=("nablk", "iablk"))
    pts = cube_points(3_000, seed=45)
    rng = np.random.default_rng(46)
    wc = rng.uniform(-1, 1, len(pts)) + 1j * rng.uniform(-1, 1, len(pts))
    run_case("fmm_lapcplx", pts, wc, AffineMap((0.5, 0.5, 0.5), 0.5), 3, laplace_kernel(), 5, 1e-5,
             ("nablk",), potentials_for=("nablk",))


def cfg3_case() -> None:
    """BASELINE config 3 at its full shape: 8e6 points on the unit sphere
    (bbox centre 0, half width 1), height 6 = reference depth 5 (levels 2-5,
    296,768 far pairs; the sparse levels 4-5 run the GPU's merged pair-mode
    plans), l = 9, Laplace, nablk vs sa at eps = 1e-8 (budget 4e9 since the SA
    estimate is 2.69e9 > the 2e9 default, m2l.py:171-186).  Seeded multipoles
    (M2L is linear) and 64 sampled output rows per level keep the fixture small;
    flops / ranks / shared rank are over whole levels.  The points are exactly
    bench.py's cfg3 points (sphere_points(8e6, seed=3))."""
    pts = sphere_points(8_000_000, seed=3)
    w = np.random.default_rng(4).uniform(-1.0, 1.0, len(pts))
    run_case("cfg3", pts, w, AffineMap((0.0, 0.0, 0.0), 1.0), 5, laplace_kernel(), 9, 1e-8,
             ("nablk", "sa"), budget=4_000_000_000, store_rows=64, seeded_mpoles=303)


def cfg5_case() -> None:
    """BASELINE config 5's pinnable (non-directional) part at its full shape:
    2e6 points on the radius-1 sphere, height 6 = depth 5 (leaf width 1/16 =
    lambda/4 at k = 8 pi), l = 5, Helmholtz e^{ikr}/(4 pi r) complex128,
    iablk and iasym at eps = 1e-4 (per-level ranks up to 45 at level 2: the
    realified 90-row factors exceed the fused kernel's 64 and take the
    two-pass path).  Complex seeded multipoles (re, im ~ U[-1,1]), 64 sampled
    rows per level.  Points = bench.py's cfg5 points (sphere_points(2e6, seed=5))."""
    pts = sphere_points(2_000_000, seed=5)
    rng = np.random.default_rng(6)
    wc = rng.uniform(-1, 1, len(pts)) + 1j * rng.uniform(-1, 1, len(pts))
    run_case("cfg5", pts, wc, AffineMap((0.0, 0.0, 0.0), 1.0), 5, helmholtz_kernel(8 * np.pi), 5, 1e-4,
             ("iablk", "iasym"), store_rows=64, seeded_mpoles=505)


def fmmtrace_case() -> None:
    """The reference's own caller, recorded: FmmPlan.run with threads=3 (the
    engine.py:145-155 thread pool) on a reference handler wrapped by a
    recorder that stores every apply_level call FmmPlan makes (level, chunk
    batch) plus the level arrays after the M2L phase.  The GPU test replays
    exactly that call sequence through the B200 handler."""
    import threading

    from chebfmm.engine import build_plan

    pts = cube_points(5_000, seed=51)
    w = np.random.default_rng(52).uniform(-1.0, 1.0, len(pts))
    bbox = AffineMap((0.5, 0.5, 0.5), 0.5)
    depth, order, eps, threads = 3, 5, 1e-5, 3
    tree = build_tree(pts, bbox, depth)
    lists = build_interaction_lists(tree)
    levels = lists.far_levels()
    lt = {lvl: unique_transfer_vectors(lists, lvl) for lvl in levels}
    lw = {lvl: tree.cell_width(lvl) for lvl in levels}
    out = dict(order=order, eps=eps, depth=depth, levels=np.asarray(levels), threads=threads,
               widths=np.asarray([lw[l] for l in levels]), kernel=np.asarray("laplace"))
    for variant in ("nablk", "iablk"):
        inner = make_handler(variant, laplace_kernel(), ChebyshevGrid(order), eps)
        inner.precompute(lt, lw)

        class Recorder:
            def __init__(self):
                self.calls, self.lock = [], threading.Lock()

            def __getattr__(self, name):
                return getattr(inner, name)

            def apply_level(self, level, batch, mpoles, locals_out):
                with self.lock:
                    self.calls.append((level, batch[0][0] if batch else -1, _csr(batch)))
                return inner.apply_level(level, batch, mpoles, locals_out)

        rec = Recorder()
        plan = build_plan(pts, bbox, depth, laplace_kernel(), order, eps, variant=variant, threads=threads,
                          handler=rec)
        snap = {}
        orig = plan._m2l

        def m2l(lv, orig=orig, snap=snap):
            orig(lv)
            for lvl, d in lv.items():
                snap[lvl] = (d.mpoles.copy(), d.locals_.copy())

        plan._m2l = m2l
        out[f"potentials_{variant}"] = plan.run(w)
        calls = sorted(rec.calls, key=lambda c: (c[0], c[1]))  # chunk order within a level
        for i, (lvl, _, (tgt, off, src, tv)) in enumerate(calls):
            out[f"call_{variant}_{i}_level"] = lvl
            out[f"call_{variant}_{i}_tgt"], out[f"call_{variant}_{i}_off"] = tgt, off
            out[f"call_{variant}_{i}_src"], out[f"call_{variant}_{i}_t"] = src, tv
        out[f"n_calls_{variant}"] = len(calls)
        for lvl in levels:
            out[f"mpoles_{variant}_{lvl}"], out[f"locals_{variant}_{lvl}"] = snap[lvl]
            out[f"flops_{variant}_{lvl}"] = inner.flops.get(lvl, 0)
    np.savez_compressed(OUT / "fmmtrace.npz", **out)
    print("fmmtrace.npz", {k: out[k] for k in out if k.startswith("n_calls")})


def aca_case() -> None:
    # compression="aca" (lowrank.py:65-184, m2l.py:206-214 / 241-255): cube,
    # l = 4, eps = 1e-4, multipoles from the reference's P2M/M2M.
    pts = cube_points(3_000, seed=31)
    w = np.random.default_rng(32).uniform(-1.0, 1.0, len(pts))
    run_case("aca", pts, w, AffineMap((0.5, 0.5, 0.5), 0.5), 3, laplace_kernel(), 4, 1e-4,
             ("ia", "iasym", "iablk", "sa", "sarcmp"), compression="aca")


if __name__ == "__main__":
    main()
