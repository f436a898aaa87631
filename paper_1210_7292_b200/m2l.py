"""B200 M2L handler: a drop-in for the reference's ``M2LHandler``.

Reference interface mirrored (m2l.py, /root/reference/pkg/src/chebfmm):

  M2LHandler(variant, kernel, grid, epsilon, compression="svd",
             block_size=128, budget_bytes=2e9)                 :93-130
  precompute(level_transfers, level_widths) -> self            :136-169
  apply_level(level, batch, mpoles, locals_out) -> int flops   :279-305
  apply_to_target(level, target_row, far_list, mpoles, locals_out) :307-310
  operator_count / stored_bytes / level_ranks / shared_rank /
  recompression_table / flop_report / reset_counters           :458-536
  flops, block_stats, factorization_calls attributes           :127-129
  BudgetExceededError(RuntimeError), PrecomputeIncompleteError(KeyError) :56-61

so ``build_plan(..., handler=B200M2LHandler(...))`` (engine.py:252) or
``FmmPlan(tree, lists, grid, kernel, handler, ...)`` (bench.py:305) run the
reference FMM with its M2L phase on the GPU.

Precompute (operator assembly, truncated SVD / ACA, shared bases) runs on the
host exactly as the reference defines it, then the operator cache is uploaded
once.  ``apply_level`` converts the Python batch to CSR and calls the C ABI;
``apply_level_csr`` / ``plan_level_cells`` + ``apply_planned`` skip the Python
lists entirely (device-built interaction lists).  Expansion arrays may be
numpy (host; copied in and out) or CUDA tensors (used in place).  There is no
CPU fallback.
"""

from __future__ import annotations

import collections.abc
import ctypes
import threading
import time

import numpy as np

from . import _native
from .numerics import (
    AffineMap,
    LowRankFactors,
    aca_plus_svd,
    assemble_for_transfer,
    eps_rank,
    grid_nodes,
    node_evaluator,
    truncated_svd,
)
from .precompute import aca_plus_svds_device, assemble_stack, device_kernel_kind, shared_basis, truncated_svds
from .symmetry import SymmetryMap

__all__ = [
    "VARIANTS",
    "DEFAULT_BUDGET_BYTES",
    "BudgetExceededError",
    "PrecomputeIncompleteError",
    "B200M2LHandler",
    "M2LHandler",
    "make_handler",
]

VARIANTS = ("na", "nasym", "nablk", "sa", "sarcmp", "ia", "iasym", "iablk")
DEFAULT_BUDGET_BYTES = 2_000_000_000


def _reference_exceptions():
    """If the reference package is importable, subclass its exception types so
    callers catching ``chebfmm.m2l.BudgetExceededError`` keep working."""
    try:  # pragma: no cover - depends on the user's environment
        from chebfmm import m2l as ref  # type: ignore

        return ref.BudgetExceededError, ref.PrecomputeIncompleteError
    except Exception:
        return RuntimeError, KeyError


_BUDGET_BASE, _PRECOMPUTE_BASE = _reference_exceptions()


class BudgetExceededError(_BUDGET_BASE):
    """Estimated precompute memory exceeds the budget (m2l.py:56-57)."""


class PrecomputeIncompleteError(_PRECOMPUTE_BASE):
    """Apply met a level or transfer vector with no precomputed operator (m2l.py:60-61)."""


def _as_t(t) -> tuple[int, int, int]:
    return (int(t[0]), int(t[1]), int(t[2]))


def _tarray(ts) -> np.ndarray:
    return np.ascontiguousarray(np.asarray([_as_t(t) for t in ts], dtype=np.int8).reshape(-1, 3))


class _Group:
    """One precompute unit: transfer list at a width (m2l.py:76-87)."""

    def __init__(self, transfers, width: float):
        self.transfers = sorted(_as_t(t) for t in transfers)
        self.width = float(width)
        self.symmetry = SymmetryMap(self.transfers)


def _batch_to_csr(batch):
    """Reference batch [(tgt, [(src, t), ...]), ...] (engine.py:113-119) -> CSR
    numpy arrays (targets, offsets, sources, int8 t[P, 3]).

    Walked in C (libcfm_batch.so, several threads, ~10 ns per pair instead of
    ~380 ns for the Python loop); objects outside the fast shapes (numpy
    scalars, big ints, other sequence types) take the Python conversion."""
    lib = _native.load_batch()
    n = len(batch)
    off = np.empty(n + 1, np.int64)
    n_pairs = ctypes.c_int64()
    if lib.cfm_batch_count(batch, None, ctypes.byref(n_pairs), off.ctypes.data) == 0:
        P = n_pairs.value
        tgt = np.empty(n, np.int64)
        src = np.empty(P, np.int64)
        t = np.empty((P, 3), np.int8)
        if lib.cfm_batch_fill(batch, off.ctypes.data, tgt.ctypes.data, src.ctypes.data, t.ctypes.data, 0) == 0:
            return tgt, off, src, t
    return _batch_to_csr_py(batch)


def _batch_to_csr_py(batch):
    """Python conversion of any batch the C walker declines."""
    n = len(batch)
    tgt = np.empty(n, np.int64)
    counts = np.empty(n, np.int64)
    srcs: list[int] = []
    ts: list[tuple] = []
    for i, (row, far) in enumerate(batch):
        tgt[i] = row
        counts[i] = len(far)
        for s, t in far:
            srcs.append(s)
            ts.append(t)
    off = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=off[1:])
    src = np.asarray(srcs, dtype=np.int64) if srcs else np.zeros(0, np.int64)
    t = np.asarray(ts, dtype=np.int64).reshape(-1, 3) if ts else np.zeros((0, 3), np.int64)
    if t.size and (t.min() < -128 or t.max() > 127):
        t = np.clip(t, -128, 127)  # far outside [-3,3]: reported as missing operator by the native side
    return tgt, off, src, np.ascontiguousarray(t.astype(np.int8))


class _FlushLog(collections.abc.Sequence):
    """``block_stats[level]["flushes"]``: the reference's list of one ``(rep,
    columns)`` tuple per GEMM flush (m2l.py:406, :429), grown by every apply.
    A planned level flushes the same ~pairs / block_size tuples at every step
    (181 k at BASELINE config 2's level 6), so ``extend`` keeps a reference to
    the per-plan list instead of copying it (1.3 ms of the timed step and
    unbounded growth otherwise); reading materialises the concatenation.
    Compares equal to the plain list the reference builds."""

    __slots__ = ("_chunks", "_flat")

    def __init__(self, items=()):
        self._chunks = [list(items)] if items else []
        self._flat = None

    def extend(self, items):
        self._chunks.append(items if isinstance(items, list) else list(items))
        self._flat = None

    def append(self, item):
        self.extend([item])

    def _list(self):
        if self._flat is None:
            self._flat = [x for c in self._chunks for x in c]
            self._chunks = [self._flat]
        return self._flat

    def __len__(self):
        return sum(len(c) for c in self._chunks)

    def __iter__(self):
        return iter(self._list())

    def __getitem__(self, i):
        return self._list()[i]

    def __eq__(self, other):
        if isinstance(other, _FlushLog):
            other = other._list()
        return self._list() == other

    def __ne__(self, other):
        return not self == other

    __hash__ = None

    def __repr__(self):
        return repr(self._list())


class B200M2LHandler:
    """Precompute/apply/account interface of all eight variants, on a B200."""

    def __init__(self, variant: str, kernel, grid, epsilon: float, compression: str = "svd",
                 block_size: int = 128, budget_bytes: int = DEFAULT_BUDGET_BYTES, device: int | None = None,
                 precompute_on: str = "device"):
        if variant not in VARIANTS:
            raise ValueError(f"unknown M2L variant {variant!r}; expected one of {VARIANTS}")
        if compression not in ("svd", "aca"):
            raise ValueError(f"unknown compression {compression!r}; expected svd or aca")
        self.variant = variant
        self.kernel = kernel
        self.grid = grid
        self.epsilon = float(epsilon)
        self.compression = compression
        self.block_size = int(block_size)  # accepted for API parity; the GPU tiles are 64 columns
        self.budget_bytes = int(budget_bytes)
        if precompute_on not in ("device", "host"):
            raise ValueError(f"precompute_on must be 'device' or 'host', got {precompute_on!r}")
        # device assembly / SVDs (precompute.py) for the kernels the assembly kernel implements
        self.precompute_on = precompute_on if device_kernel_kind(kernel) is not None else "host"
        self.precompute_seconds = 0.0

        self.uses_symmetry = variant in ("nasym", "nablk", "iasym", "iablk")
        self.uses_blocking = variant in ("nablk", "iablk")
        self.is_dense = variant in ("na", "nasym", "nablk")
        self.is_shared_basis = variant in ("sa", "sarcmp")

        self._groups: dict[object, _Group] = {}
        self._level_group: dict[int, object] = {}
        self._level_scale: dict[int, float] = {}
        # host-side metadata of the operator cache (shapes/ranks; data lives on the GPU)
        self._dense: dict[object, dict] = {}
        self._lowrank: dict[object, dict] = {}
        self._sa: dict[object, dict] = {}
        self._group_key_id: dict[object, int] = {}

        self.factorization_calls = 0
        self.flops: dict[int, int] = {}
        self.block_stats: dict[int, dict] = {}
        self._precomputed = False
        self._lock = threading.RLock()  # FmmPlan may call apply_level from several threads (engine.py:145-155)

        self._lib = _native.load()
        self._op_complex = np.issubdtype(np.dtype(kernel.dtype), np.complexfloating)
        self._device = self._pick_device(device)
        self._order = int(grid.order)
        self._size = self._order**3
        h = ctypes.c_void_p()
        _native.check(self._lib.cfm_handler_create(self._device, _native.VARIANT_IDS[variant], self._order,
                                                   int(self._op_complex), ctypes.byref(h)))
        self._h = h
        self._planned: dict[int, dict] = {}
        self._rep_code_tab: dict[object, np.ndarray] = {}
        self._flush_cache: dict[tuple, tuple] = {}  # (native plan id, block_size) -> block statistics of one apply
        self.last_plan_cache_hit = False  # the last apply_level(_csr) reused a cached plan of the same batch
        self._acct: dict[int, tuple] = {}  # level -> (plan stats, group key, flops, block summary)

    @staticmethod
    def _pick_device(device):
        if device is not None:
            return int(device)
        try:
            import torch

            if torch.cuda.is_available():
                return int(torch.cuda.current_device())
        except Exception:  # pragma: no cover
            pass
        return 0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.cfm_handler_destroy(h)
            except Exception:  # pragma: no cover
                pass
            self._h = None

    def _check(self, rc):
        _native.check(rc, PrecomputeIncompleteError, BudgetExceededError)

    # ------------------------------------------------------------------
    # precompute (m2l.py:136-273)
    # ------------------------------------------------------------------
    def precompute(self, level_transfers, level_widths) -> "B200M2LHandler":
        t0 = time.perf_counter()
        try:
            return self._precompute(level_transfers, level_widths)
        finally:
            self.precompute_seconds = time.perf_counter() - t0

    def _operators(self, vectors, width: float):
        """Operators for ``vectors`` at ``width``: a device tensor [T, n, n]
        (device precompute) or a host array (assemble_for_transfer)."""
        if self.precompute_on == "device":
            return assemble_stack(self.kernel, vectors, width, self.grid, self._device)
        dt = np.complex128 if self._op_complex else np.float64
        if not vectors:
            return np.zeros((0, self._size, self._size), dt)
        return np.stack([assemble_for_transfer(self.kernel, t, width, self.grid) for t in vectors]).astype(dt)

    @staticmethod
    def _host(a):
        return a if isinstance(a, np.ndarray) else a.cpu().numpy()

    def _precompute(self, level_transfers, level_widths) -> "B200M2LHandler":
        levels = sorted(lvl for lvl, ts in level_transfers.items() if ts)
        if not levels:
            self._precomputed = True
            return self
        degree = getattr(self.kernel, "homogeneity_degree", None)
        if degree is not None:
            union = set()
            for lvl in levels:
                union.update(_as_t(t) for t in level_transfers[lvl])
            ref_level = levels[0]
            ref_width = level_widths[ref_level]
            group = _Group(sorted(union), ref_width)
            self._groups["ref"] = group
            for lvl in levels:
                self._level_group[lvl] = "ref"
                self._level_scale[lvl] = (level_widths[lvl] / ref_width) ** degree
            self._check_budget([group])
            self._build_group("ref", group)
        else:
            groups = []
            for lvl in levels:
                group = _Group(level_transfers[lvl], level_widths[lvl])
                self._groups[lvl] = group
                self._level_group[lvl] = lvl
                self._level_scale[lvl] = 1.0
                groups.append(group)
            self._check_budget(groups)
            for lvl in levels:
                self._build_group(lvl, self._groups[lvl])
        for lvl in levels:
            key = self._group_key_id[self._level_group[lvl]]
            self._check(self._lib.cfm_set_level(self._h, int(lvl), key, float(self._level_scale[lvl])))
        self._planned.clear()
        self._acct.clear()
        self._precomputed = True
        return self

    def _check_budget(self, groups) -> None:
        size = self._size
        itemsize = np.dtype(self.kernel.dtype).itemsize
        estimate = 0
        for g in groups:
            n_ops = len(g.symmetry.cone) if self.uses_symmetry else len(g.transfers)
            if self.is_shared_basis:
                estimate += 2 * len(g.transfers) * size * size * itemsize
            else:
                estimate += n_ops * size * size * itemsize
        if estimate > self.budget_bytes:
            raise BudgetExceededError(
                f"variant {self.variant}: estimated precompute memory {estimate} B exceeds budget "
                f"{self.budget_bytes} B"
            )

    def _key_id(self, key) -> int:
        if key not in self._group_key_id:
            self._group_key_id[key] = len(self._group_key_id)
        return self._group_key_id[key]

    def _build_group(self, key, group: _Group) -> None:
        kid = self._key_id(key)
        tr = _tarray(group.transfers)
        dt = np.complex128 if self._op_complex else np.float64
        if self.is_dense:
            vectors = group.symmetry.cone if self.uses_symmetry else group.transfers
            ops = np.ascontiguousarray(self._host(self._operators(list(vectors), group.width)), dtype=dt)
            self._dense[key] = {"vectors": list(vectors), "nbytes": [ops[0].nbytes] * len(vectors)}
            self._check(self._lib.cfm_set_dense_group(self._h, kid, len(tr), tr.ctypes.data, len(vectors),
                                                      _tarray(vectors).ctypes.data, ops.ctypes.data))
        elif self.is_shared_basis:
            self._build_shared_basis(key, kid, group)
        else:
            vectors = group.symmetry.cone if self.uses_symmetry else group.transfers
            if self.compression == "svd" and self.precompute_on == "device":
                facs = truncated_svds(self._operators(list(vectors), group.width), self.epsilon)
                self.factorization_calls += len(facs)
            elif self.compression == "aca" and self.precompute_on == "device":
                facs = aca_plus_svds_device(self._operators(list(vectors), group.width), self.epsilon)
                self.factorization_calls += len(facs)
            else:
                facs = [self._factorize(t, group.width) for t in vectors]
            ranks = np.asarray([f.rank for f in facs], np.int32)
            left = np.concatenate([np.ascontiguousarray(f.left, dtype=dt).ravel() for f in facs]) if facs else np.zeros(0, dt)
            right = np.concatenate([np.ascontiguousarray(f.right, dtype=dt).ravel() for f in facs]) if facs else np.zeros(0, dt)
            left = np.ascontiguousarray(left)
            right = np.ascontiguousarray(right)
            self._lowrank[key] = {
                "vectors": list(vectors),
                "ranks": {t: f.rank for t, f in zip(vectors, facs)},
                "nbytes": {t: f.left.nbytes + f.right.nbytes for t, f in zip(vectors, facs)},
                "fallback": {t: f.via_fallback for t, f in zip(vectors, facs)},
            }
            vt = _tarray(vectors)
            self._check(self._lib.cfm_set_lowrank_group(self._h, kid, len(tr), tr.ctypes.data, len(vectors),
                                                        vt.ctypes.data, ranks.ctypes.data, left.ctypes.data,
                                                        right.ctypes.data))

    def _factorize(self, t, width: float) -> LowRankFactors:
        self.factorization_calls += 1
        if self.compression == "svd":
            return truncated_svd(assemble_for_transfer(self.kernel, t, width, self.grid), self.epsilon)
        size = self._size
        half = 0.5 * width
        nodes = grid_nodes(self.grid)
        x_nodes = AffineMap((width * t[0], width * t[1], width * t[2]), half).forward(nodes)
        y_nodes = AffineMap((0.0, 0.0, 0.0), half).forward(nodes)
        return aca_plus_svd(node_evaluator(self.kernel, x_nodes, y_nodes), size, size, self.epsilon)

    def _build_shared_basis(self, key, kid: int, group: _Group) -> None:
        """U, B from SVDs of the row/column concatenations; C_t = diag(s) V_t^H B
        (m2l.py:216-273)."""
        size = self._size
        transfers = group.transfers
        stack = self._operators(list(transfers), group.width)
        cores = {}
        if self.compression == "svd" and self.precompute_on == "device":
            u, b, core_stack = shared_basis(stack, self.epsilon)
            self.factorization_calls += 2
            for k, t in enumerate(transfers):
                cores[t] = ("dense", core_stack[k])
            self._finish_shared_basis(key, kid, transfers, u, b, cores)
            return
        stack = self._host(stack)
        row = np.hstack(list(stack))
        col = np.vstack(list(stack))
        del stack
        if self.compression == "svd":
            u_row, s_row, vh_row = np.linalg.svd(row, full_matrices=False)
            _, s_col, vh_col = np.linalg.svd(col, full_matrices=False)
            r = max(eps_rank(s_row, self.epsilon), eps_rank(s_col, self.epsilon))
            self.factorization_calls += 2
            u = u_row[:, :r]
            sigma = s_row[:r]
            vh = vh_row[:r]
            b = vh_col[:r].conj().T
        else:
            row_fac = aca_plus_svd(lambda i, j: row[np.asarray(i), np.asarray(j)], size, row.shape[1], self.epsilon)
            col_fac = aca_plus_svd(lambda i, j: col[np.asarray(i), np.asarray(j)], col.shape[0], size, self.epsilon)
            self.factorization_calls += 2
            sigma = np.linalg.norm(row_fac.left, axis=0)
            u = row_fac.left / sigma
            vh = row_fac.right.conj().T
            b = col_fac.right
        for k, t in enumerate(transfers):
            cores[t] = ("dense", (sigma[:, None] * vh[:, k * size:(k + 1) * size]) @ b)
        self._finish_shared_basis(key, kid, transfers, u, b, cores)

    def _finish_shared_basis(self, key, kid: int, transfers, u, b, cores) -> None:
        r_u, r_b = u.shape[1], b.shape[1]
        if self.variant == "sarcmp" and cores:
            keys = list(cores)
            facs = truncated_svds(np.stack([cores[t][1] for t in keys]), self.epsilon)
            self.factorization_calls += len(keys)
            for t, fac in zip(keys, facs):
                if fac.rank * (r_u + r_b) < r_u * r_b:
                    cores[t] = ("factored", fac)
        dt = np.complex128 if self._op_complex else np.float64
        core_rank = np.asarray([-1 if cores[t][0] == "dense" else cores[t][1].rank for t in transfers], np.int32)
        parts = []
        for t in transfers:
            kind, c = cores[t]
            if kind == "dense":
                parts.append(np.ascontiguousarray(c, dtype=dt).ravel())
            else:
                parts.append(np.ascontiguousarray(c.left, dtype=dt).ravel())
                parts.append(np.ascontiguousarray(c.right, dtype=dt).ravel())
        core_data = np.ascontiguousarray(np.concatenate(parts) if parts else np.zeros(0, dt))
        u_c = np.ascontiguousarray(u, dtype=dt)
        b_c = np.ascontiguousarray(b, dtype=dt)
        tr = _tarray(transfers)
        self._check(self._lib.cfm_set_shared_group(self._h, kid, int(r_u), int(r_b), u_c.ctypes.data,
                                                   b_c.ctypes.data, len(transfers), tr.ctypes.data,
                                                   core_rank.ctypes.data, core_data.ctypes.data))
        self._sa[key] = {
            "u_nbytes": u_c.nbytes,
            "b_nbytes": b_c.nbytes,
            "rank": max(r_u, r_b),
            "r_u": r_u,
            "r_b": r_b,
            "cores": {t: (kind, (c.nbytes if kind == "dense" else c.left.nbytes + c.right.nbytes),
                          (None if kind == "dense" else c.rank)) for t, (kind, c) in cores.items()},
        }

    # ------------------------------------------------------------------
    # apply (m2l.py:279-310)
    # ------------------------------------------------------------------
    def _level_key(self, level: int):
        if not self._precomputed:
            raise PrecomputeIncompleteError("handler has not been precomputed")
        key = self._level_group.get(level)
        if key is None:
            raise PrecomputeIncompleteError(f"no operators precomputed for level {level}")
        return key

    def _result_dtype(self, mpoles):
        return np.result_type(np.dtype(self.kernel.dtype), mpoles.dtype)

    def _prepare(self, mpoles, locals_out):
        """Validate expansion arrays; returns (x, y, writeback, data_complex, n_rows)."""
        is_np = isinstance(mpoles, np.ndarray)
        if is_np != isinstance(locals_out, np.ndarray):
            raise TypeError("mpoles and locals_out must both be numpy arrays or both CUDA tensors")
        if is_np:
            rdt = self._result_dtype(mpoles)
            if mpoles.ndim != 2 or mpoles.shape[1] != self._size:
                raise ValueError(f"mpoles must have shape (rows, {self._size})")
            if locals_out.shape != mpoles.shape:
                raise ValueError("locals_out must have the shape of mpoles")
            if not np.can_cast(rdt, locals_out.dtype, casting="same_kind"):
                raise TypeError(f"cannot accumulate {rdt} contributions into {locals_out.dtype} locals")
            work_dt = np.complex128 if np.issubdtype(locals_out.dtype, np.complexfloating) or np.issubdtype(rdt, np.complexfloating) else np.float64
            x = np.ascontiguousarray(mpoles, dtype=work_dt)
            if locals_out.dtype == work_dt and locals_out.flags.c_contiguous:
                y, wb = locals_out, None
            else:
                y, wb = np.ascontiguousarray(locals_out, dtype=work_dt), locals_out
            return x, y, wb, int(work_dt == np.complex128), mpoles.shape[0]
        import torch  # CUDA tensors

        if not (mpoles.is_cuda and locals_out.is_cuda):
            raise TypeError("torch expansion tensors must live on the GPU")
        if mpoles.dim() != 2 or mpoles.shape[1] != self._size or locals_out.shape != mpoles.shape:
            raise ValueError(f"expansion tensors must have shape (rows, {self._size})")
        if mpoles.dtype not in (torch.float64, torch.complex128) or locals_out.dtype != (
            torch.complex128 if (self._op_complex or mpoles.dtype == torch.complex128) else torch.float64
        ):
            raise TypeError("expansion tensors must be float64/complex128 matching the result type")
        if mpoles.dtype == torch.float64 and locals_out.dtype == torch.complex128:
            mpoles = mpoles.to(torch.complex128)
        x = mpoles.contiguous()
        if not locals_out.is_contiguous():
            raise ValueError("locals_out tensor must be contiguous")
        return x, locals_out, None, int(locals_out.dtype == torch.complex128), mpoles.shape[0]

    @staticmethod
    def _stream_of(x):
        if isinstance(x, np.ndarray):
            return None
        import torch

        return ctypes.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)

    def apply_level(self, level: int, batch, mpoles, locals_out) -> int:
        """Apply the level's M2L interactions for a batch of target cells.

        ``batch`` is [(target_row, [(source_row, transfer), ...]), ...]; the
        contributions are accumulated into ``locals_out`` and the counted flops
        are returned and added to ``self.flops[level]`` (m2l.py:279-305).
        """
        if not self._precomputed:
            raise PrecomputeIncompleteError("handler has not been precomputed")
        if not batch:
            return 0
        self._level_key(level)
        tgt, off, src, t = _batch_to_csr(batch)
        return self.apply_level_csr(level, tgt, off, src, t, mpoles, locals_out)

    def apply_to_target(self, level: int, target_row: int, far_list, mpoles, locals_out) -> int:
        return self.apply_level(level, [(target_row, far_list)], mpoles, locals_out)

    def apply_level_csr(self, level: int, tgt, offsets, src, t, mpoles, locals_out) -> int:
        """Fast path: the batch as CSR arrays (targets, offsets, sources, t[P,3])."""
        key = self._level_key(level)
        tgt = np.ascontiguousarray(tgt, dtype=np.int64)
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        src = np.ascontiguousarray(src, dtype=np.int64)
        t = np.ascontiguousarray(t, dtype=np.int8).reshape(-1, 3)
        if off.shape != (len(tgt) + 1,) or (len(tgt) and (off[0] != 0 or off[-1] != len(src) or len(t) != len(src))):
            raise ValueError("inconsistent CSR batch")
        if off[-1] == 0:
            self._record(level, key, np.zeros(343, np.int64), 0, planned=False)
            return 0
        n_targets_nonempty = int(np.count_nonzero(np.diff(off)))
        n_sources = int(np.unique(src).size) if self.is_shared_basis else 0
        counts = np.zeros(343, np.int64)
        # one critical section from the staging copy to the accounting: concurrent
        # callers with disjoint target rows of shared arrays stay correct
        with self._lock:
            x, y, wb, data_complex, n_rows = self._prepare(mpoles, locals_out)
            self._check(self._lib.cfm_apply_level_csr(
                self._h, int(level), len(tgt), tgt.ctypes.data, off.ctypes.data, src.ctypes.data, t.ctypes.data,
                data_complex, _native.ptr(x), int(n_rows), _native.ptr(y), self._stream_of(x), counts.ctypes.data))
            if wb is not None:
                wb[...] = y
            info = self.last_csr_plan_info()
            self.last_plan_cache_hit = info["cache_hit"]
            flops = self._count_flops(key, counts, n_targets_nonempty, n_sources)
            summary = None
            if self.uses_blocking:
                # the flush sequence is a function of the batch, like the plan:
                # computed once per plan and reused while the plan is cached
                ck = (info["plan_id"], self.block_size)
                summary = self._flush_cache.get(ck)
                if summary is None:
                    summary = self._flush_summary(key, t)
                    if len(self._flush_cache) >= 64:
                        self._flush_cache.pop(next(iter(self._flush_cache)))
                    self._flush_cache[ck] = summary
            self._record(level, key, counts, flops, summary=summary)
        return flops

    def last_csr_plan_info(self) -> dict:
        """Plan of the last apply_level / apply_level_csr call (batch plans are
        cached apart from the level plans of plan_level_*)."""
        hit, mode, ts, pid = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_uint64()
        self._check(self._lib.cfm_last_csr_plan_info(self._h, ctypes.byref(hit), ctypes.byref(mode),
                                                     ctypes.byref(ts), ctypes.byref(pid)))
        return {"cache_hit": bool(hit.value), "mode": {0: "target", 1: "pair"}.get(mode.value),
                "two_stage": bool(ts.value), "plan_id": int(pid.value)}

    def _rep_of_code(self, key) -> np.ndarray:
        """t-code -> representative index of a group (symmetry.assignment)."""
        tab = self._rep_code_tab.get(key)
        if tab is None:
            tab = np.full(343, -1, np.int16)
            for t, (rep_idx, _) in self._groups[key].symmetry.assignment.items():
                tab[(t[0] + 3) * 49 + (t[1] + 3) * 7 + (t[2] + 3)] = rep_idx
            self._rep_code_tab[key] = tab
        return tab

    def _flush_summary(self, key, t):
        """block_stats of one blocked apply of a batch exactly as the reference
        counts them (m2l.py:397-452): the flush sequence of its pairs in batch
        order for buffers of ``block_size`` columns (computed in C)."""
        cone = self._groups[key].symmetry.cone
        P = len(t)
        cap = P // max(self.block_size, 1) + len(cone) + 1
        reps = np.empty(cap, np.int32)
        cols = np.empty(cap, np.int32)
        k = _native.load_batch().cfm_flush_sequence(P, t.ctypes.data, self._rep_of_code(key).ctypes.data, len(cone),
                                                    self.block_size, reps.ctypes.data, cols.ctypes.data, cap)
        if k < 0:
            raise PrecomputeIncompleteError(f"variant {self.variant}: a transfer vector has no operator")
        flushes = [(cone[r], c) for r, c in zip(reps[:k].tolist(), cols[:k].tolist())]
        return P, int(k), flushes, {cone[r] for r in np.unique(reps[:k]).tolist()}

    # -------- device-built lists: classify on the GPU, plan once, apply many
    def plan_level_cells(self, level: int, cells_ijk, complex_data: bool | None = None) -> dict:
        """Classify the far lists of a level on the GPU from its sorted occupied
        cells (int32 [n, 3], row order) and cache the apply plan."""
        self._level_key(level)
        cells = np.ascontiguousarray(cells_ijk, dtype=np.int32).reshape(-1, 3)
        if complex_data is None:
            complex_data = self._op_complex
        counts = np.zeros(343, np.int64)
        with self._lock:
            self._check(self._lib.cfm_plan_level_cells(self._h, int(level), len(cells), cells.ctypes.data,
                                                       int(bool(complex_data)), None, counts.ctypes.data))
        stats = self.plan_stats(level)
        stats["counts"] = counts
        stats["n_rows"] = len(cells)
        stats["complex"] = bool(complex_data)
        self._planned[level] = stats
        return stats

    def plan_level_cells_subset(self, level: int, cells_ijk, target_rows, complex_data: bool | None = None):
        """Plan only ``target_rows`` of a level (a multi-GPU rank's range).
        Returns (stats, source_rows) where source_rows are the rows the planned
        targets read (owned rows plus the halo to receive)."""
        self._level_key(level)
        cells = np.ascontiguousarray(cells_ijk, dtype=np.int32).reshape(-1, 3)
        rows = np.ascontiguousarray(target_rows, dtype=np.int64)
        if complex_data is None:
            complex_data = self._op_complex
        counts = np.zeros(343, np.int64)
        nsrc = ctypes.c_int64()
        srcs = np.zeros(len(cells), np.int64)
        with self._lock:
            self._check(self._lib.cfm_plan_level_cells_subset(
                self._h, int(level), len(cells), cells.ctypes.data, len(rows), rows.ctypes.data,
                int(bool(complex_data)), None, counts.ctypes.data, ctypes.byref(nsrc), srcs.ctypes.data))
        stats = self.plan_stats(level)
        stats["counts"] = counts
        stats["n_rows"] = len(cells)
        stats["complex"] = bool(complex_data)
        self._planned[level] = stats
        return stats, srcs[: nsrc.value].copy()

    def plan_level_csr(self, level: int, tgt, offsets, src, t, n_rows: int, complex_data: bool | None = None) -> dict:
        """Cache the apply plan of a level from CSR lists (targets, offsets,
        sources, int8 t[P, 3]) over level arrays of ``n_rows`` rows; rows may
        be any local numbering (a multi-GPU rank's owned + halo rows).  Then
        :meth:`apply_planned` / :meth:`apply_levels` run it."""
        self._level_key(level)
        tgt = np.ascontiguousarray(tgt, dtype=np.int64)
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        src = np.ascontiguousarray(src, dtype=np.int64)
        t = np.ascontiguousarray(t, dtype=np.int8).reshape(-1, 3)
        if off.shape != (len(tgt) + 1,) or (len(tgt) and (off[0] != 0 or off[-1] != len(src) or len(t) != len(src))):
            raise ValueError("inconsistent CSR batch")
        if complex_data is None:
            complex_data = self._op_complex
        counts = np.zeros(343, np.int64)
        with self._lock:
            self._check(self._lib.cfm_plan_level_csr(self._h, int(level), len(tgt), tgt.ctypes.data, off.ctypes.data,
                                                     src.ctypes.data, t.ctypes.data, int(bool(complex_data)),
                                                     int(n_rows), counts.ctypes.data))
        stats = self.plan_stats(level)
        stats["counts"] = counts
        stats["n_rows"] = int(n_rows)
        stats["complex"] = bool(complex_data)
        self._planned[level] = stats
        return stats

    def plan_stats(self, level: int) -> dict:
        vals = [ctypes.c_int64() for _ in range(6)]
        self._check(self._lib.cfm_plan_stats(self._h, int(level), *[ctypes.byref(v) for v in vals]))
        names = ("tiles", "entries", "pairs", "slots", "targets", "sources")
        out = {k: int(v.value) for k, v in zip(names, vals)}
        mode, fill = ctypes.c_int(), ctypes.c_double()
        self._check(self._lib.cfm_plan_info(self._h, int(level), ctypes.byref(mode), ctypes.byref(fill)))
        out["mode"] = "pair" if mode.value == 1 else "target"
        out["target_fill"] = fill.value
        ts = ctypes.c_int()
        self._check(self._lib.cfm_plan_two_stage(self._h, int(level), ctypes.byref(ts)))
        out["two_stage"] = bool(ts.value)
        return out

    def apply_planned(self, level: int, mpoles, locals_out) -> int:
        """Apply a level planned with :meth:`plan_level_cells` (same flops/accounting)."""
        key = self._level_key(level)
        st = self._planned.get(level)
        if st is None:
            raise PrecomputeIncompleteError(f"level {level} has no device plan; call plan_level_cells first")
        with self._lock:
            x, y, wb, data_complex, n_rows = self._prepare(mpoles, locals_out)
            if bool(data_complex) != (st["complex"] or self._op_complex):
                raise ValueError("expansion dtype differs from the one the level was planned for")
            self._check(self._lib.cfm_apply_planned(self._h, int(level), _native.ptr(x), int(n_rows), _native.ptr(y),
                                                    self._stream_of(x)))
            if wb is not None:
                wb[...] = y
            flops, summary = self._planned_acct(level, key, st)
            self._record(level, key, st["counts"], flops, summary=summary)
        return flops

    def _planned_acct(self, level, key, st):
        """Flops and block statistics of one apply of a planned level: fixed by the
        plan, so computed once per plan (a per-call Python pass over the 316
        transfer vectors of every level cost ~1.4 ms per step)."""
        cached = self._acct.get(level)
        if cached is None or cached[0] is not st or cached[1] != key:
            flops = self._count_flops(key, st["counts"], st["targets"], st["sources"])
            cached = self._acct[level] = (st, key, flops, self._record_summary(level, key, st["counts"]))
        return cached[2], cached[3]

    def apply_levels(self, arrays) -> int:
        """Apply several planned levels of one M2L step together.

        ``arrays`` maps level -> (mpoles, locals_out).  Dense variants run all
        levels in a single kernel launch; returns the total counted flops and
        records per-level accounting exactly as per-level calls would."""
        with self._lock:
            return self._apply_levels_locked(arrays)

    def _apply_levels_locked(self, arrays) -> int:
        levels = sorted(arrays)
        prepared = []
        for lvl in levels:
            self._level_key(lvl)
            st = self._planned.get(lvl)
            if st is None:
                raise PrecomputeIncompleteError(f"level {lvl} has no device plan; call plan_level_cells first")
            x, y, wb, data_complex, n_rows = self._prepare(*arrays[lvl])
            if bool(data_complex) != (st["complex"] or self._op_complex):
                raise ValueError("expansion dtype differs from the one the level was planned for")
            prepared.append((lvl, x, y, wb, n_rows, st))
        if not prepared:
            return 0
        n = len(prepared)
        lv = (ctypes.c_int * n)(*[p[0] for p in prepared])
        xs = (ctypes.c_void_p * n)(*[_native.ptr(p[1]) for p in prepared])
        ys = (ctypes.c_void_p * n)(*[_native.ptr(p[2]) for p in prepared])
        rows = (ctypes.c_int64 * n)(*[int(p[4]) for p in prepared])
        self._check(self._lib.cfm_apply_levels(self._h, n, lv, xs, rows, ys, self._stream_of(prepared[0][1])))
        total = 0
        for lvl, x, y, wb, n_rows, st in prepared:
            if wb is not None:
                wb[...] = y
            key = self._level_group[lvl]
            flops, summary = self._planned_acct(lvl, key, st)
            self._record(lvl, key, st["counts"], flops, summary=summary)
            total += flops
        return total

    def last_apply_stats(self) -> tuple[float, int]:
        ms = ctypes.c_double()
        n = ctypes.c_int64()
        self._check(self._lib.cfm_last_apply_stats(self._h, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    # -------- accounting model (m2l.py:21-26, :333,336,358,361,379-394,423,426)
    def _op_cost(self, key, t) -> int:
        size = self._size
        if self.is_dense:
            return 2 * size * size
        group = self._groups[key]
        if self.is_shared_basis:
            sa = self._sa[key]
            kind, _, r_t = sa["cores"][t]
            return 2 * sa["r_u"] * sa["r_b"] if kind == "dense" else 2 * r_t * (sa["r_u"] + sa["r_b"])
        lr = self._lowrank[key]
        rep = group.symmetry.lookup(t)[0] if self.uses_symmetry else t
        return 4 * size * lr["ranks"][rep]

    def _count_flops(self, key, counts, n_targets, n_sources) -> int:
        group = self._groups[key]
        total = 0
        for code in np.nonzero(counts)[0]:
            c = int(code)
            t = (c // 49 - 3, (c // 7) % 7 - 3, c % 7 - 3)
            if t not in group.symmetry.assignment:
                raise PrecomputeIncompleteError(f"variant {self.variant}: no operator for transfer vector {t}")
            total += int(counts[c]) * self._op_cost(key, t)
        if self.is_shared_basis:
            sa = self._sa[key]
            total += 2 * self._size * sa["r_b"] * int(n_sources) + 2 * self._size * sa["r_u"] * int(n_targets)
        return int(total)

    def _record_summary(self, level, key, counts, planned: bool = True):
        """Per-call block statistics of a counts vector: (columns, products, [(rep, columns)] flushes)."""
        if not self.uses_blocking:
            return None
        group = self._groups[key]
        per_rep: dict = {}
        for code in np.nonzero(counts)[0]:
            c = int(code)
            t = (c // 49 - 3, (c // 7) % 7 - 3, c % 7 - 3)
            rep = group.symmetry.lookup(t)[0]
            per_rep[rep] = per_rep.get(rep, 0) + int(counts[c])
        # products = the reference's flush count for these columns (each
        # representative flushes every block_size columns plus once for the
        # remainder, m2l.py:412-451), whatever the pair order; planned levels
        # have no reference batch order, so their flush list holds the same
        # multiset of (rep, columns) grouped by representative
        bs = max(self.block_size, 1)
        flushes = []
        for rep in sorted(per_rep, key=lambda r: group.symmetry.cone.index(r)):
            full, rem = divmod(per_rep[rep], bs)
            flushes.extend([(rep, bs)] * full)
            if rem:
                flushes.append((rep, rem))
        return int(counts.sum()), len(flushes), flushes, set(per_rep)

    def _record(self, level, key, counts, flops, planned: bool = True, summary=None) -> None:
        self.flops[level] = self.flops.get(level, 0) + flops
        if self.uses_blocking:
            if summary is None:
                summary = self._record_summary(level, key, counts, planned)
            pairs, products, flushes, reps = summary
            st = self.block_stats.setdefault(
                level, {"columns": 0, "products": 0, "reps_used": set(), "flushes": _FlushLog()})
            st["columns"] += pairs
            st["products"] += products
            st["reps_used"].update(reps)
            st["flushes"].extend(flushes)

    # ------------------------------------------------------------------
    # accounting (m2l.py:458-536)
    # ------------------------------------------------------------------
    def operator_count(self) -> int:
        count = 0
        for d in self._dense.values():
            count += len(d["vectors"])
        for d in self._lowrank.values():
            count += len(d["vectors"])
        for sa in self._sa.values():
            count += len(sa["cores"])
        return count

    def stored_bytes(self) -> int:
        total = 0
        for d in self._dense.values():
            total += sum(d["nbytes"])
        for d in self._lowrank.values():
            total += sum(d["nbytes"].values())
        for sa in self._sa.values():
            total += sa["u_nbytes"] + sa["b_nbytes"] + sum(nb for _, nb, _ in sa["cores"].values())
        return total

    def level_ranks(self, level: int) -> list[int]:
        key = self._level_group.get(level)
        if key is None:
            return []
        group = self._groups[key]
        if self.is_dense:
            return [self._size for _ in group.transfers]
        if self.is_shared_basis:
            sa = self._sa[key]
            return [sa["rank"] if sa["cores"][t][0] == "dense" else sa["cores"][t][2] for t in group.transfers]
        lr = self._lowrank[key]
        if self.uses_symmetry:
            return [lr["ranks"][group.symmetry.lookup(t)[0]] for t in group.transfers]
        return [lr["ranks"][t] for t in group.transfers]

    def shared_rank(self, level: int):
        key = self._level_group.get(level)
        if key is None or not self.is_shared_basis:
            return None
        return self._sa[key]["rank"]

    def recompression_table(self, level: int):
        key = self._level_group.get(level)
        if key is None or key not in self._sa:
            return []
        sa = self._sa[key]
        return [(t, sa["cores"][t][2] if sa["cores"][t][0] == "factored" else None) for t in self._groups[key].transfers]

    def flop_report(self) -> list[dict]:
        if not self.flops:
            raise RuntimeError("flop report requires at least one apply")
        stored = self.stored_bytes()
        return [{"level": lvl, "variant": self.variant, "flops": n, "bytes": stored}
                for lvl, n in sorted(self.flops.items())]

    def reset_counters(self) -> None:
        self.flops = {}
        self.block_stats = {}


M2LHandler = B200M2LHandler


def make_handler(variant: str, kernel, grid, epsilon: float, **kwargs) -> B200M2LHandler:
    """Construct an (unprecomputed) handler for a variant tag (m2l.py:539-542)."""
    return B200M2LHandler(variant, kernel, grid, epsilon, **kwargs)
