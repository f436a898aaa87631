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
* compression="aca": the partially pivoted ACA of every operator on the
  device (one CTA each, csrc/aca.cu), the recompression on the host;
* the per-operator truncated SVDs of the IA variants (square, independent,
  numerically low rank) run on the device as a batched randomized range
  finder with one power iteration: Y = K Omega (k = 128 columns), Q = qr(Y),
  Q = qr(K (K^H Q)), B = Q^H K, B^H = Q_b R_b, svd(R_b^H) = U_2 S W_2^H, so
  K = (Q U_2) S (Q_b W_2)^H up to the part of K outside the sketch, whose
  size is s_k -- checked per operator to lie far below eps * s_1 (else that
  operator takes the host LAPACK SVD).  The small k x k SVDs run on host
  threads.  Batched cuSOLVER gesvdj on the full operators measured slower
  than host LAPACK (l = 9: 55 s vs 28 s), this path takes ~0.1-0.3 s.

The truncation rule is the reference's (``eps_rank``: s_k > eps * s_1), so
ranks are the reference's; the factors agree to rounding (the parity tests
compare locals at 1e-10 and ranks exactly).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .numerics import FOUR_PI, LowRankFactors, aca_plus_svd, eps_rank, grid_nodes, truncated_svd


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


SKETCH = 128          # randomized range: columns of the sketch
TAIL_MARGIN = 1e-4    # the sketch's smallest singular value must lie below TAIL_MARGIN * eps * s_1


def _pool_map(fn, items):
    import os
    from concurrent.futures import ThreadPoolExecutor

    workers = max(1, min(len(items), os.cpu_count() or 1, 64))
    if workers == 1:
        return [fn(a) for a in items]
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        threadpool_limits = None
    if threadpool_limits is not None:
        with threadpool_limits(limits=1, user_api="blas"):
            with ThreadPoolExecutor(workers) as ex:
                return list(ex.map(fn, items))
    with ThreadPoolExecutor(workers) as ex:  # pragma: no cover
        return list(ex.map(fn, items))


QR_STREAMS = 16


def _batched_qr(y):
    """Reduced QR of every matrix of a batch.  torch's batched CUDA QR runs the
    per-matrix cuSOLVER calls one after another (0.6 ms each at 729 x 128,
    latency-bound); issuing them round-robin on several streams overlaps them."""
    import torch

    if y.device.type != "cuda" or y.shape[0] < 2 * QR_STREAMS:
        return torch.linalg.qr(y)[0]
    q = torch.empty_like(y)
    cur = torch.cuda.current_stream(y.device)
    streams = [torch.cuda.Stream(y.device) for _ in range(QR_STREAMS)]
    for s in streams:
        s.wait_stream(cur)
    for i in range(y.shape[0]):
        with torch.cuda.stream(streams[i % QR_STREAMS]):
            q[i] = torch.linalg.qr(y[i])[0]
    for s in streams:
        cur.wait_stream(s)
    y.record_stream(cur)
    return q


def truncated_svds_device(stack, eps: float) -> list[LowRankFactors]:
    """``truncated_svd`` (lowrank.py:53-62: rank = #{s_i > eps * s_1}, left =
    U_r diag(s_r), right = V_r) of every operator of a device stack [T, n, n]
    by a batched randomized SVD (module docstring).  Operators whose sketch
    does not reach far enough below the threshold fall back to the host SVD."""
    import torch

    _check_eps(eps)
    t_count, n, _ = stack.shape
    k = min(n, SKETCH)
    dev = stack.device
    gen = torch.Generator(device=dev).manual_seed(0x5EED)
    if stack.is_complex():
        om = torch.complex(torch.randn(n, k, generator=gen, device=dev, dtype=torch.float64),
                           torch.randn(n, k, generator=gen, device=dev, dtype=torch.float64))
    else:
        om = torch.randn(n, k, generator=gen, device=dev, dtype=torch.float64)
    q = _batched_qr(torch.matmul(stack, om))
    q = _batched_qr(torch.matmul(stack.mH, q))                # one power iteration (K^H range)
    q = _batched_qr(torch.matmul(stack, q))
    b = torch.matmul(q.mH, stack)                             # [T, k, n]
    qb = _batched_qr(b.mH.contiguous())                       # B^H = Q_b R_b
    rb = torch.matmul(qb.mH, b.mH)                            # R_b = Q_b^H B^H
    rbh = rb.mH.resolve_conj().cpu().numpy()                  # [T, k, k]

    def small(a):
        return np.linalg.svd(a, full_matrices=True)

    parts = _pool_map(small, list(rbh))
    s = np.stack([x[1] for x in parts])
    rmax = max([eps_rank(si, eps) for si in s] + [1])
    # only the leading rmax singular vectors leave the device
    u2 = torch.from_numpy(np.ascontiguousarray(np.stack([x[0][:, :rmax] for x in parts]))).to(dev)
    w2 = torch.from_numpy(np.ascontiguousarray(np.stack([x[2][:rmax].conj().T for x in parts]))).to(dev)  # W_2
    u_full = torch.matmul(q, u2).cpu().numpy()                # [T, n, rmax]
    v_full = torch.matmul(qb, w2).cpu().numpy()               # [T, n, rmax]
    out: list = [None] * t_count
    redo = []
    for i in range(t_count):
        si = s[i]
        r = eps_rank(si, eps)
        tail_ok = k == n or (si[0] > 0 and si[-1] <= TAIL_MARGIN * eps * si[0] and r < k - 8)
        if not tail_ok:
            redo.append(i)
            continue
        out[i] = LowRankFactors(np.ascontiguousarray(u_full[i][:, :r] * si[:r]),
                                np.ascontiguousarray(v_full[i][:, :r]))
    if redo:
        host = stack[redo].cpu().numpy()
        for i, f in zip(redo, _pool_map(lambda a: _host_tsvd(a, eps), list(host))):
            out[i] = f
    return out


def truncated_svds(stack, eps: float) -> list[LowRankFactors]:
    """``truncated_svd`` (lowrank.py:53-62) of every operator in a stack:
    on the device (randomized, truncated_svds_device) for device stacks of
    operators larger than the sketch (n > 128, l >= 6), else host LAPACK, one
    operator per thread."""
    _check_eps(eps)
    if not isinstance(stack, np.ndarray):
        import torch

        if not bool(torch.isfinite(torch.view_as_real(stack) if stack.is_complex() else stack).all()):
            raise ValueError("matrix has non-finite entries")
        if stack.shape[-1] > SKETCH and len(stack):
            return truncated_svds_device(stack, eps)
    host = stack if isinstance(stack, np.ndarray) else stack.cpu().numpy()
    if not np.all(np.isfinite(host)):
        raise ValueError("matrix has non-finite entries")
    if host.shape[-1] < 64:
        return [_host_tsvd(a, eps) for a in host]
    return _pool_map(lambda a: _host_tsvd(a, eps), list(host))


ACA_MAX_CROSSES = 192


def aca_plus_svds_device(stack, eps: float) -> list[LowRankFactors]:
    """``aca_plus_svd`` (lowrank.py:163-184) of every operator of a device
    stack [T, n, n]: the partially pivoted ACA runs on the device, one CTA per
    operator (cfm_aca_batch, csrc/aca.cu: the reference's pivoting, updates
    and stopping rule), the QR + truncated-SVD recompression of the crosses on
    host threads.  A stagnated ACA falls back to the dense truncated SVD
    (via_fallback=True, as the reference); an operator needing more than
    ACA_MAX_CROSSES crosses reruns the host ACA."""
    import torch

    _check_eps(eps)
    t_count, n, _ = stack.shape
    if t_count == 0:
        return []
    cplx = stack.is_complex()
    kmax = min(n, ACA_MAX_CROSSES)
    dev = stack.device
    ops = stack.contiguous()
    u = torch.empty((t_count, kmax, n), dtype=stack.dtype, device=dev)
    v = torch.empty_like(u)
    ranks = np.zeros(t_count, np.int32)
    flags = np.zeros(t_count, np.int32)
    st = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    _native.check(_native.load().cfm_aca_batch(
        dev.index, n, int(cplx), t_count, ctypes.c_void_p(ops.data_ptr()), float(eps), kmax,
        ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(v.data_ptr()), ranks.ctypes.data, flags.ctypes.data, st))
    host_ops = ops.cpu().numpy()
    u_h = u.cpu().numpy()
    v_h = v.cpu().numpy()

    def finish(i):
        k, flag = int(ranks[i]), int(flags[i])
        if flag == 2:  # cross cap: the reference algorithm on the host
            a = host_ops[i]
            return aca_plus_svd(lambda r, c: a[np.asarray(r), np.asarray(c)], n, n, eps)
        if flag == 0:  # stagnation (lowrank.py:174-178)
            out = truncated_svd(host_ops[i], eps)
            out.via_fallback = True
            return out
        u_mat = np.ascontiguousarray(u_h[i, :k].T)
        v_mat = np.ascontiguousarray(v_h[i, :k].conj().T)
        if k == 0:
            return LowRankFactors(u_mat, v_mat)
        qu, ru = np.linalg.qr(u_mat)
        qv, rv = np.linalg.qr(v_mat)
        uc, s, vch = np.linalg.svd(ru @ rv.conj().T)
        r = eps_rank(s, eps)
        return LowRankFactors(qu @ (uc[:, :r] * s[:r]), qv @ vch[:r].conj().T)

    return _pool_map(finish, list(range(t_count)))


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
