"""Operator precompute on the GPU.

The reference builds its M2L operator cache on the host (``M2LHandler.precompute``,
m2l.py:136-273): ``assemble_for_transfer`` per transfer vector
(kernels.py:167-179), ``truncated_svd`` per operator for the IA variants
(lowrank.py:53-62), and for SA the two SVDs of the row / column
concatenations of all 316 operators (m2l.py:216-273).  At l = 9 the SA
precompute is ~60 s on the host; here:

* assembly is one sm_100a kernel (``cfm_assemble_operators``) for all
  transfer vectors, bit-identical to the host assembly for Laplace;
* the SA concatenation SVDs go through a tall-skinny QR (cuSOLVER geqrf) and
  an SVD of the small n x n triangle: for A^H = Q R, A = R^H Q^H and
  svd(R^H) = U S W^H gives the singular values S and left vectors U of A;
  for the column stack C = Q R, svd(R) = U S V^H gives S and V of C.  The
  cores C_t = diag(s) V_t^H B are U_r^H K_t B (same product, one batched GEMM);
* the per-operator truncated SVDs of the IA variants (square, independent)
  run as host LAPACK calls in parallel threads on the device-assembled
  operators: cuSOLVER's per-matrix gesvdj measured slower for them.

The truncation rule is the reference's (``eps_rank``: s_k > eps * s_1), so
ranks are the reference's; the factors agree to rounding (the parity tests
compare locals at 1e-10 and ranks exactly).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .numerics import FOUR_PI, LowRankFactors, eps_rank, grid_nodes


def device_kernel_kind(kernel):
    """(kind, wavenumber) for kernels the assembly kernel implements, else None.

    Recognised by name (the reference's ``laplace_kernel`` / ``helmholtz_kernel``,
    kernels.py:100-112) and confirmed on sample radii, so a custom profile
    under a borrowed name falls back to host assembly."""
    name = getattr(kernel, "name", None)
    r = np.array([0.37, 1.9, 11.0])
    if name == "laplace":
        kind, k = 0, 0.0
        want = 1.0 / (FOUR_PI * r)
    elif name == "helmholtz" and getattr(kernel, "wavenumber", None) is not None:
        kind, k = 1, float(kernel.wavenumber)
        want = np.exp(1j * k * r) / (FOUR_PI * r)
    else:
        return None
    try:
        got = np.asarray(kernel.profile(r))
    except Exception:
        return None
    if got.shape != want.shape or not np.allclose(got, want, rtol=1e-14, atol=0.0):
        return None
    return kind, k


def assemble_stack(kernel, vectors, width: float, grid, device: int):
    """Operators K_t for all ``vectors`` as one device tensor [T, n, n]."""
    import torch

    kk = device_kernel_kind(kernel)
    if kk is None:
        raise ValueError(f"no device assembly for kernel {getattr(kernel, 'name', kernel)!r}")
    kind, k = kk
    nodes = np.ascontiguousarray(grid_nodes(grid), dtype=np.float64)
    n = nodes.shape[0]
    tr = np.ascontiguousarray(np.asarray(vectors, dtype=np.int64).reshape(-1, 3).astype(np.int8))
    dev = torch.device("cuda", device)
    out = torch.empty((len(tr), n, n), dtype=torch.complex128 if kind else torch.float64, device=dev)
    if len(tr):
        st = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        _native.check(_native.load().cfm_assemble_operators(
            device, kind, k, n, nodes.ctypes.data, float(width), len(tr), tr.ctypes.data,
            ctypes.c_void_p(out.data_ptr()), st))
    return out


def _check_eps(eps: float) -> None:
    if not 0.0 < eps < 1.0:
        raise ValueError(f"accuracy must lie in (0, 1), got {eps}")


def _host_tsvd(a, eps):
    u, s, vh = np.linalg.svd(a, full_matrices=False)
    r = eps_rank(s, eps)
    return LowRankFactors(u[:, :r] * s[:r], vh[:r].conj().T)


def truncated_svds(stack, eps: float) -> list[LowRankFactors]:
    """``truncated_svd`` (lowrank.py:53-62) of every operator in a stack.

    The operators are square and independent, and cuSOLVER's per-matrix
    gesvdj is slower than LAPACK for them (l = 9: 55 s vs 28 s for 316
    operators, profiles/r01_precompute.json), so the SVDs run on the host,
    one operator per thread with single-threaded BLAS."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    _check_eps(eps)
    host = stack if isinstance(stack, np.ndarray) else stack.cpu().numpy()
    if not np.all(np.isfinite(host)):
        raise ValueError("matrix has non-finite entries")
    workers = max(1, min(len(host), os.cpu_count() or 1, 64))
    if workers == 1 or host.shape[-1] < 64:
        return [_host_tsvd(a, eps) for a in host]
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        threadpool_limits = None
    if threadpool_limits is not None:
        with threadpool_limits(limits=1, user_api="blas"):
            with ThreadPoolExecutor(workers) as ex:
                return list(ex.map(lambda a: _host_tsvd(a, eps), host))
    with ThreadPoolExecutor(workers) as ex:
        return list(ex.map(lambda a: _host_tsvd(a, eps), host))


def shared_basis(stack, eps: float):
    """SA shared bases (m2l.py:216-273) from a device stack [T, n, n].

    Returns (u [n, r], b [n, r], cores [T, r, r]) as host arrays, where r is
    max(eps_rank(row singular values), eps_rank(column singular values))."""
    import torch

    _check_eps(eps)
    t_count, n, _ = stack.shape
    row_h = stack.permute(0, 2, 1).reshape(t_count * n, n).conj()  # (hstack_t K_t)^H, [T n, n]
    q, r_row = torch.linalg.qr(row_h)
    del q
    u_row, s_row, _ = torch.linalg.svd(r_row.mH)  # row = R^H Q^H
    col = stack.reshape(t_count * n, n)  # vstack_t K_t
    q, r_col = torch.linalg.qr(col)
    del q
    _, s_col, vh_col = torch.linalg.svd(r_col)  # col = Q R, R = U S V^H
    r = max(eps_rank(s_row.cpu().numpy(), eps), eps_rank(s_col.cpu().numpy(), eps))
    u = u_row[:, :r].contiguous()
    b = vh_col[:r].conj().T.contiguous()
    cores = torch.matmul(torch.matmul(u.mH.unsqueeze(0), stack), b.unsqueeze(0))  # U^H K_t B
    return u.cpu().numpy(), b.cpu().numpy(), cores.cpu().numpy()
