"""Product host-side numerics (precompute inputs) against the golden fixtures."""

import numpy as np

from oracle import oracle as O
from paper_1210_7292_b200 import (
    ChebyshevGrid,
    assemble_for_transfer,
    canonicalize,
    cheb_roots,
    full_far_field_vectors,
    helmholtz_kernel,
    laplace_kernel,
    permutation_table,
    truncated_svd,
)
from paper_1210_7292_b200.symmetry import SymmetryMap, inverse_permutation_table


def test_roots_and_nodes():
    for order in range(2, 10):
        r = cheb_roots(order)
        assert np.array_equal(r, O.cheb_roots(order))
        assert np.array_equal(r, -r[::-1])
        assert np.array_equal(ChebyshevGrid(order).nodes3d, O.nodes3d(order))


def test_symmetry_matches_reference(golden):
    g = golden("symmetry")
    far = full_far_field_vectors()
    assert np.array_equal(np.asarray(far), g["far316"])
    for i, t in enumerate(far):
        ts, spec = canonicalize(t)
        assert ts == tuple(g["t_sym"][i])
        assert spec.perm_id == g["spec_id"][i]
    assert np.array_equal(np.asarray(SymmetryMap(far).cone), g["cone"])
    for order in (2, 3, 4, 5, 7, 9):
        for pid in range(48):
            assert np.array_equal(permutation_table(pid, order), g[f"table_l{order}"][pid])
            assert np.array_equal(inverse_permutation_table(pid, order), g[f"inv_l{order}"][pid])


def test_operator_assembly_bitwise(golden):
    g = golden("cfg1")
    grid = ChebyshevGrid(4)
    w = float(g["widths"][0])
    for k, t in enumerate(g["K_rep_t"]):
        K = assemble_for_transfer(laplace_kernel(), tuple(int(c) for c in t), w, grid)
        assert np.array_equal(K, g["K_rep"][k])


def test_operator_identity_through_permutations():
    """K_t = P K_rep P^T for all 316 vectors, both kernels (<=1e-13)."""
    for kernel in (laplace_kernel(), helmholtz_kernel(1.0)):
        for order in (2, 3, 4):
            grid = ChebyshevGrid(order)
            reps = {}
            for t in full_far_field_vectors():
                ts, spec = canonicalize(t)
                if ts not in reps:
                    reps[ts] = assemble_for_transfer(kernel, ts, 0.5, grid)
                K = assemble_for_transfer(kernel, t, 0.5, grid)
                tab = permutation_table(spec.perm_id, order)
                Kp = reps[ts][np.ix_(tab, tab)]
                assert np.max(np.abs(K - Kp)) <= 1e-13 * np.max(np.abs(K))


def test_lowrank_ranks_match_reference(golden):
    g = golden("cfg1")
    grid = ChebyshevGrid(4)
    levels = [int(l) for l in g["levels"]]
    w = float(g["widths"][0])
    transfers = sorted({tuple(int(c) for c in t) for l in levels for t in g[f"t_{l}"]})
    ranks = {t: truncated_svd(assemble_for_transfer(laplace_kernel(), t, w, grid), float(g["eps"])).rank
             for t in transfers}
    assert [ranks[t] for t in transfers] == list(g["ranks_ia_2"]) or \
        [ranks[t] for t in transfers if t in set(map(tuple, g["t_2"].tolist()))] == list(g["ranks_ia_2"])


def _ops(kernel, order, width, ts):
    return np.stack([assemble_for_transfer(kernel, t, width, ChebyshevGrid(order)) for t in ts])


def test_randomized_truncated_svd_matches_lapack():
    """The device path's randomized truncated SVD (precompute.truncated_svds_device,
    run here on CPU tensors) gives the reference's ranks (lowrank.py:53-62:
    #{s_i > eps s_1}) and factors whose product matches the LAPACK truncation;
    a full-rank operator (sketch tail above the threshold) falls back to LAPACK."""
    import torch

    from paper_1210_7292_b200.precompute import truncated_svds_device

    cases = [(laplace_kernel(), 9, 1e-8, 2.0 / 4, [(3, 0, 0), (2, 2, 1), (3, 3, 3), (-2, 3, -1)]),
             (laplace_kernel(), 5, 1e-5, 1.0 / 4, [(2, 0, 0), (3, 2, 1)]),
             (helmholtz_kernel(8 * np.pi), 7, 1e-4, 2.0 / 4, [(2, 1, 0), (3, 3, 2)])]
    for kernel, order, eps, width, ts in cases:
        ops = _ops(kernel, order, width, ts)
        dev = truncated_svds_device(torch.from_numpy(ops), eps)
        for a, f in zip(ops, dev):
            ref = truncated_svd(a, eps)
            assert f.rank == ref.rank, (order, f.rank, ref.rank)
            prod = f.left @ f.right.conj().T
            ref_prod = ref.left @ ref.right.conj().T
            assert np.linalg.norm(prod - ref_prod) <= 1e-12 * np.linalg.norm(ref_prod)
    full = np.random.default_rng(0).standard_normal((2, 200, 200))
    got = truncated_svds_device(torch.from_numpy(full), 1e-6)
    for a, f in zip(full, got):
        assert f.rank == truncated_svd(a, 1e-6).rank == 200


def test_flush_log_behaves_like_the_reference_list():
    """block_stats[level]["flushes"] (m2l.py:406, :429 of the reference) is a
    list of (rep, columns) tuples; the handler's lazy log keeps references to the
    per-plan lists and must read, compare and grow like that list."""
    from paper_1210_7292_b200.m2l import _FlushLog

    per_plan = [((1, 0, 0), 256), ((1, 1, 0), 17)]
    log, ref = _FlushLog(), []
    for _ in range(3):
        log.extend(per_plan)
        ref.extend(per_plan)
    log.append(((3, 2, 1), 5))
    ref.append(((3, 2, 1), 5))
    assert log == ref and ref == log and len(log) == len(ref) == 7
    assert list(log) == ref and log[0] == ref[0] and log[-1] == ref[-1] and log[2:4] == ref[2:4]
    assert per_plan == [((1, 0, 0), 256), ((1, 1, 0), 17)]  # the shared per-plan list is never mutated
    log.extend(per_plan)
    assert len(log) == 9 and log != ref
    assert _FlushLog() == [] and not _FlushLog()
