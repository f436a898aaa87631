"""Host-side numerics for the M2L precompute (operator cache construction).

This is the product's own restatement of the reference's precompute-side
building blocks; it runs once per handler on the host (SURVEY.md §2 rows 4-6:
"precompute-side only") and feeds the device operator cache:

  cheb_roots            interp.py:45-70   descending, mirrored, exact 0 middle root
  ChebyshevGrid         interp.py:198-236 nodes3d[m] = (r[a1], r[a2], r[a3]), a1 fastest
  AffineMap             interp.py:164-195
  Kernel / laplace / helmholtz   kernels.py:34-112  (1/(4 pi r), e^{ikr}/(4 pi r))
  assemble_for_transfer kernels.py:142-179 source cell at the origin, target at w*t
  truncated_svd         lowrank.py:47-62  rank = #{s > eps * s_1}, sigma folded left
  aca / aca_plus_svd    lowrank.py:65-184 partially pivoted ACA + QR/SVD recompression

The arithmetic follows the reference expression by expression, so operators
are bit-identical for identical inputs and the truncation ranks agree (rank
parity is what makes compressed variants comparable at 1e-10).
The handler also accepts the reference's own ``Kernel``/``ChebyshevGrid``
objects (duck typing on ``profile``, ``dtype``, ``homogeneity_degree``,
``order``).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from functools import lru_cache
from typing import Callable

import numpy as np

FOUR_PI = 4.0 * np.pi


# ----------------------------------------------------------------- Chebyshev grid
def cheb_roots(order: int) -> np.ndarray:
    """Roots of T_order, largest first; the second half mirrors the first."""
    if order < 2:
        raise ValueError(f"interpolation order must be >= 2, got {order}")
    half = order // 2
    k = np.arange(1, half + 1)
    first = np.cos((2 * k - 1) * np.pi / (2 * order))
    roots = np.empty(order)
    roots[:half] = first
    if order % 2:
        roots[half] = 0.0
    roots[order - half:] = -first[::-1]
    return roots


@lru_cache(maxsize=None)
def component_indices(order: int) -> np.ndarray:
    """0-based (a1, a2, a3) of every flat node index, shape (3, order^3)."""
    j = np.arange(order**3)
    comp = np.stack([j % order, (j // order) % order, j // (order * order)])
    comp.setflags(write=False)
    return comp


@dataclass(frozen=True)
class AffineMap:
    """Map from the reference cube [-1,1]^3 onto an axis-aligned cell."""

    center: tuple
    half_width: float

    def __post_init__(self):
        if not self.half_width > 0:
            raise ValueError(f"half_width must be positive, got {self.half_width}")
        object.__setattr__(self, "center", tuple(float(c) for c in self.center))

    def forward(self, ref_points) -> np.ndarray:
        return np.asarray(self.center) + self.half_width * np.asarray(ref_points, dtype=float)

    @property
    def low(self) -> np.ndarray:
        return np.asarray(self.center) - self.half_width


class ChebyshevGrid:
    """Tensor Chebyshev grid; ``nodes3d[m]`` is the node of flat index m."""

    def __init__(self, order: int):
        self.order = int(order)
        roots = cheb_roots(self.order)
        roots.setflags(write=False)
        self.roots1d = roots
        self.nodes3d = roots[component_indices(self.order)].T.copy()
        self.nodes3d.setflags(write=False)

    @property
    def size(self) -> int:
        return self.order**3

    def nodes_in_cell(self, cell: AffineMap) -> np.ndarray:
        return cell.forward(self.nodes3d)

    def __repr__(self) -> str:
        return f"ChebyshevGrid(order={self.order})"


def grid_nodes(grid) -> np.ndarray:
    """Reference-cube nodes of any grid object exposing ``order``."""
    nodes = getattr(grid, "nodes3d", None)
    if nodes is not None:
        return np.asarray(nodes)
    return ChebyshevGrid(grid.order).nodes3d


# ----------------------------------------------------------------------- kernels
def _laplace_profile(r):
    return 1.0 / (FOUR_PI * r)


@dataclass(frozen=True)
class Kernel:
    """Radial kernel K(x, y) = profile(|x - y|)."""

    name: str
    profile: Callable
    dtype: np.dtype = field(default=np.dtype(np.float64))
    homogeneity_degree: float | None = None
    wavenumber: float | None = None


def laplace_kernel() -> Kernel:
    """1/(4 pi r), homogeneous of degree -1 (kernels.py:100-102)."""
    return Kernel("laplace", _laplace_profile, np.dtype(np.float64), homogeneity_degree=-1.0)


def helmholtz_kernel(wavenumber: float = 1.0) -> Kernel:
    """exp(i k r)/(4 pi r), complex, not homogeneous (kernels.py:105-112)."""
    k = float(wavenumber)

    def profile(r):
        return np.exp(1j * k * r) / (FOUR_PI * r)

    return Kernel("helmholtz", profile, np.dtype(np.complex128), wavenumber=k)


def kernel_matrix(kernel, targets: np.ndarray, sources: np.ndarray) -> np.ndarray:
    """Dense K(targets[i], sources[j]) for well-separated point sets."""
    t = np.asarray(targets, dtype=float)
    s = np.asarray(sources, dtype=float)
    r = np.sqrt(np.sum((t[:, None, :] - s[None, :, :]) ** 2, axis=-1))
    if np.any(r == 0.0):
        raise ValueError(f"{getattr(kernel, 'name', 'kernel')} kernel is singular at x == y")
    return kernel.profile(r)


def assemble_for_transfer(kernel, transfer, width: float, grid) -> np.ndarray:
    """l^3 x l^3 M2L operator for transfer vector t at cell width w.

    Rows are target nodes (cell centred at w*t), columns source nodes (cell at
    the origin); kernels.py:142-179.
    """
    t = tuple(int(c) for c in transfer)
    if t[0] * t[0] + t[1] * t[1] + t[2] * t[2] <= 3:
        raise ValueError(f"cells with transfer vector {t} are not admissible (|t| <= sqrt(3))")
    half = 0.5 * width
    nodes = grid_nodes(grid)
    x = np.asarray((width * t[0], width * t[1], width * t[2])) + half * nodes
    y = np.asarray((0.0, 0.0, 0.0)) + half * nodes
    return kernel_matrix(kernel, x, y)


def node_evaluator(kernel, x_nodes, y_nodes):
    """(i, j) -> K(x_nodes[i], y_nodes[j]) for ACA sampling (m2l.py:64-73)."""

    def evaluate(i, j):
        xi = x_nodes[np.asarray(i)]
        yj = y_nodes[np.asarray(j)]
        r = np.sqrt(np.sum((xi - yj) ** 2, axis=-1))
        return kernel.profile(r)

    return evaluate


# ---------------------------------------------------------------------- low rank
@dataclass
class LowRankFactors:
    """A ~ left @ right^H; ``right`` has orthonormal columns."""

    left: np.ndarray
    right: np.ndarray
    via_fallback: bool = False

    @property
    def rank(self) -> int:
        return self.left.shape[1]

    def reconstruct(self) -> np.ndarray:
        return self.left @ self.right.conj().T

    def apply(self, vec: np.ndarray) -> np.ndarray:
        return self.left @ (self.right.conj().T @ vec)


def eps_rank(s: np.ndarray, eps: float) -> int:
    """Smallest r with s_{r+1} <= eps * s_1 (lowrank.py:47-50, m2l.py:545-548)."""
    if s.size == 0 or s[0] == 0.0:
        return 0
    return int(np.count_nonzero(s > eps * s[0]))


def truncated_svd(matrix, eps: float) -> LowRankFactors:
    a = np.asarray(matrix)
    if not np.all(np.isfinite(a)):
        raise ValueError("matrix has non-finite entries")
    if not 0.0 < eps < 1.0:
        raise ValueError(f"accuracy must lie in (0, 1), got {eps}")
    u, s, vh = np.linalg.svd(a, full_matrices=False)
    r = eps_rank(s, eps)
    return LowRankFactors(u[:, :r] * s[:r], vh[:r].conj().T)


def aca(evaluator, n_rows: int, n_cols: int, eps: float, max_rank: int | None = None):
    """Partially pivoted adaptive cross approximation (lowrank.py:65-160).

    Returns (U, V, converged) with A ~ U V^H.  Row pivots are probed among the
    preferred row and the first few unused rows when a residual row vanishes;
    the stopping rule is |u_k| |v_k| <= eps |S_k|_F with the Frobenius norm of
    the running approximation updated incrementally.
    """
    if max_rank is None:
        max_rank = min(n_rows, n_cols)
    cols_all = np.arange(n_cols)
    rows_all = np.arange(n_rows)
    us: list[np.ndarray] = []
    vs: list[np.ndarray] = []
    used_rows: set[int] = set()
    used_cols: set[int] = set()
    frob_sq = 0.0
    pivot_row = 0
    converged = False
    for _ in range(max_rank):
        residual_row = None
        probes = [pivot_row] + [r for r in range(n_rows) if r not in used_rows][:4]
        for cand in probes:
            if cand in used_rows:
                continue
            trial = np.asarray(evaluator(cand, cols_all), dtype=None).copy()
            for u_k, v_k in zip(us, vs):
                trial -= u_k[cand] * v_k
            if np.max(np.abs(trial)) > 0.0:
                pivot_row = cand
                residual_row = trial
                break
        if residual_row is None:
            converged = bool(us)
            break
        used_rows.add(pivot_row)
        masked = residual_row.copy()
        if used_cols:
            masked[sorted(used_cols)] = 0.0
        jcol = int(np.argmax(np.abs(masked)))
        pivot = residual_row[jcol]
        if pivot == 0.0:
            converged = False
            break
        used_cols.add(jcol)
        v_new = residual_row / pivot
        u_new = np.asarray(evaluator(rows_all, jcol), dtype=None).copy()
        for u_k, v_k in zip(us, vs):
            u_new -= v_k[jcol] * u_k
        cross = sum(np.vdot(u_k, u_new) * np.vdot(v_k, v_new) for u_k, v_k in zip(us, vs))
        inc_sq = float(np.real(np.vdot(u_new, u_new)) * np.real(np.vdot(v_new, v_new)))
        frob_sq = max(frob_sq + 2.0 * float(np.real(cross)) + inc_sq, 0.0)
        us.append(u_new)
        vs.append(v_new)
        if inc_sq <= (eps**2) * frob_sq:
            converged = True
            break
        next_col = np.abs(u_new)
        next_col[sorted(used_rows)] = 0.0
        pivot_row = int(np.argmax(next_col))
    else:
        converged = True
    if not us:
        dtype = np.asarray(evaluator(0, 0)).dtype
        return np.zeros((n_rows, 0), dtype=dtype), np.zeros((n_cols, 0), dtype=dtype), converged
    return np.column_stack(us), np.column_stack([v.conj() for v in vs]), converged


def aca_plus_svd(evaluator, n_rows: int, n_cols: int, eps: float, max_rank: int | None = None) -> LowRankFactors:
    """ACA, then QR of both factors and a truncated SVD of the small core
    (lowrank.py:163-184); falls back to a dense truncated SVD on stagnation."""
    u_mat, v_mat, converged = aca(evaluator, n_rows, n_cols, eps, max_rank)
    if not converged:
        dense = np.asarray(evaluator(np.arange(n_rows)[:, None], np.arange(n_cols)[None, :]))
        out = truncated_svd(dense, eps)
        out.via_fallback = True
        return out
    if u_mat.shape[1] == 0:
        return LowRankFactors(u_mat, v_mat)
    qu, ru = np.linalg.qr(u_mat)
    qv, rv = np.linalg.qr(v_mat)
    uc, s, vch = np.linalg.svd(ru @ rv.conj().T)
    r = eps_rank(s, eps)
    return LowRankFactors(qu @ (uc[:, :r] * s[:r]), qv @ vch[:r].conj().T)


# ------------------------------------------------------------ interpolation (P2M/M2M/L2L/L2P)
def cheb_polys(x, order: int) -> np.ndarray:
    """T_k(x), k = 1..order-1, by the three-term recurrence (interp.py:88-103)."""
    x = np.asarray(x, dtype=float)
    t = np.empty(x.shape + (order - 1,))
    if order >= 2:
        t[..., 0] = x
    for k in range(1, order - 1):
        if k == 1:
            t[..., 1] = 2.0 * x * x - 1.0
        else:
            t[..., k] = 2.0 * x * t[..., k - 1] - t[..., k - 2]
    return t


def weight_matrix_1d(x, order: int) -> np.ndarray:
    """S_l(x_m, root_i) = 1/l + (2/l) sum_k T_k(x_m) T_k(root_i), shape (n, l) (interp.py:106-111)."""
    x = np.atleast_1d(np.asarray(x, dtype=float))
    return 1.0 / order + (2.0 / order) * (cheb_polys(x, order) @ cheb_polys(cheb_roots(order), order).T)


@lru_cache(maxsize=None)
def child_shift_matrix(order: int, octant: tuple) -> np.ndarray:
    """Moment transfer child octant -> parent, (parent nodes x child nodes) (engine.py:41-63)."""
    roots = cheb_roots(order)
    axes = [weight_matrix_1d((0.5 if octant[i] else -0.5) + 0.5 * roots, order) for i in range(3)]
    mat = np.kron(axes[2], np.kron(axes[1], axes[0])).T.copy()
    mat.setflags(write=False)
    return mat


def octant_code(ijk) -> np.ndarray:
    """Octant of a cell inside its parent, 4*cx + 2*cy + cz (lexicographic child order)."""
    ijk = np.asarray(ijk, dtype=np.int64).reshape(-1, 3) & 1
    return ijk[:, 0] * 4 + ijk[:, 1] * 2 + ijk[:, 2]


def octant_of_code(code: int) -> tuple:
    return ((code >> 2) & 1, (code >> 1) & 1, code & 1)
