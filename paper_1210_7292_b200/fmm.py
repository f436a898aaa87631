"""Whole FMM evaluation on the GPU around the B200 M2L.

Mirrors the reference's ``FmmPlan.run`` (engine.py:201-222):

  tree + lists   octree.py:93-178   GPU octree build + device interaction lists
  P2M            engine.py:122-127  leaf multipoles from particle weights
  M2M            engine.py:129-138  child -> parent (8 octant operators, tile kernel)
  M2L            engine.py:140-157  B200M2LHandler.apply_levels (one launch, all levels)
  L2L            engine.py:159-168  parent -> child (transposed octant operators)
  L2P            engine.py:170-175  locals -> particle potentials
  P2P            engine.py:177-199  near field (27 neighbour leaves, coincident skipped)

Everything stays on the device between stages; ``run`` returns the
potentials in the original particle order, and ``m2l_seconds`` is the device
time of the M2L phase (the reference's timer, engine.py:212-214).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .m2l import make_handler
from .numerics import ChebyshevGrid, child_shift_matrix, octant_of_code
from .octree import build_tree_gpu


class B200FmmPlan:
    """Precomputed state for repeated fast summations over fixed particles."""

    def __init__(self, points, center, half_width: float, depth: int, kernel, order: int, epsilon: float,
                 variant: str = "iablk", compression: str = "svd", block_size: int = 128,
                 budget_bytes: int = 2_000_000_000, device: int = 0):
        import torch

        self.torch = torch
        self.device = torch.device("cuda", device)
        self.kernel = kernel
        self.order = int(order)
        self.depth = int(depth)
        self.epsilon = float(epsilon)
        self.n_points = len(points)
        self.tree = build_tree_gpu(points, center, half_width, depth, device=device)
        self.cells = {lvl: self.tree.cells(lvl) for lvl in range(0, depth + 1)}
        self.widths = {lvl: 2.0 * half_width / (1 << lvl) for lvl in range(0, depth + 1)}
        self.handler = make_handler(variant, kernel, ChebyshevGrid(order), epsilon, compression=compression,
                                    block_size=block_size, budget_bytes=budget_bytes, device=device)
        # transfer vectors per level from the device classifier (unique_transfer_vectors, octree.py:195-198)
        lib = _native.load()
        self._lib = lib
        level_transfers = {}
        for lvl in range(2, depth + 1):
            c = torch.from_numpy(self.cells[lvl]).to(self.device)
            n = len(c)
            offs = torch.empty(n + 1, dtype=torch.int64, device=self.device)
            tot = ctypes.c_int64()
            st = ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
            _native.check(lib.cfm_classify_count_device(device, lvl, n, c.data_ptr(), offs.data_ptr(),
                                                        ctypes.byref(tot), st))
            src = torch.empty(max(tot.value, 1), dtype=torch.int32, device=self.device)
            code = torch.empty(max(tot.value, 1), dtype=torch.int16, device=self.device)
            _native.check(lib.cfm_classify_fill_device(device, lvl, n, c.data_ptr(), offs.data_ptr(), src.data_ptr(),
                                                       code.data_ptr(), st))
            codes = torch.unique(code[: tot.value]).cpu().numpy().astype(np.int64)
            level_transfers[lvl] = [(int(k) // 49 - 3, (int(k) // 7) % 7 - 3, int(k) % 7 - 3) for k in codes]
        self.handler.precompute(level_transfers, {l: self.widths[l] for l in level_transfers})
        self.m2l_levels = [l for l, ts in level_transfers.items() if ts]
        self._complex_ops = np.issubdtype(np.dtype(kernel.dtype), np.complexfloating)
        self._planned_complex = None
        mats = np.ascontiguousarray(np.stack([child_shift_matrix(self.order, octant_of_code(c)) for c in range(8)]))
        h = ctypes.c_void_p()
        _native.check(lib.cfm_fmm_create(self.tree._t, self.order, mats.ctypes.data, ctypes.byref(h)))
        self._f = h
        self.m2l_seconds = 0.0

    def __del__(self):
        f = getattr(self, "_f", None)
        if f is not None and f.value:
            try:
                self._lib.cfm_fmm_destroy(f)
            except Exception:  # pragma: no cover
                pass
            self._f = None

    def _plan(self, complex_data: bool):
        if self._planned_complex == complex_data:
            return
        for lvl in self.m2l_levels:
            self.handler.plan_level_cells(lvl, self.cells[lvl], complex_data=complex_data)
        self._planned_complex = complex_data

    def run(self, weights):
        """Potentials at every particle for the given source weights (engine.py:201-222)."""
        torch = self.torch
        w = np.asarray(weights)
        if w.shape != (self.n_points,):
            raise ValueError(f"weights must have shape ({self.n_points},), got {w.shape}")
        rdt = np.result_type(np.dtype(self.kernel.dtype), w.dtype)
        cplx = np.issubdtype(rdt, np.complexfloating)
        tdt = torch.complex128 if cplx else torch.float64
        self._plan(cplx)
        dc = 2 if cplx else 1
        n = self.order**3
        dev = self.device
        wd = torch.from_numpy(np.ascontiguousarray(w.astype(rdt))).to(dev)
        levels = list(range(2, self.depth + 1))
        mp = {l: torch.zeros((len(self.cells[l]), n), dtype=tdt, device=dev) for l in levels}
        loc = {l: torch.zeros_like(mp[l]) for l in levels}
        st = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        lib = self._lib
        out = torch.zeros(self.n_points, dtype=tdt, device=dev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
        ev[0].record()
        _native.check(lib.cfm_fmm_p2m(self._f, wd.data_ptr(), int(cplx), mp[self.depth].data_ptr(), st))
        ev[1].record()
        for lvl in range(self.depth, 2, -1):
            _native.check(lib.cfm_fmm_m2m(self._f, lvl, mp[lvl].data_ptr(), mp[lvl - 1].data_ptr(), int(cplx), st))
        ev[2].record()
        if self.m2l_levels:
            self.handler.apply_levels({l: (mp[l], loc[l]) for l in self.m2l_levels})
        ev[3].record()
        for lvl in range(2, self.depth):
            _native.check(lib.cfm_fmm_l2l(self._f, lvl, loc[lvl].data_ptr(), loc[lvl + 1].data_ptr(), int(cplx), st))
        ev[4].record()
        _native.check(lib.cfm_fmm_l2p(self._f, loc[self.depth].data_ptr(), int(cplx), out.data_ptr(), st))
        ev[5].record()
        kind = 0 if getattr(self.kernel, "wavenumber", None) is None else 1
        k = float(getattr(self.kernel, "wavenumber", 0.0) or 0.0)
        _native.check(lib.cfm_fmm_p2p(self._f, kind, k, wd.data_ptr(), int(cplx), out.data_ptr(), int(cplx), st))
        ev[6].record()
        torch.cuda.synchronize(dev)
        names = ("p2m", "m2m", "m2l", "l2l", "l2p", "p2p")
        self.stage_ms = {nm: ev[i].elapsed_time(ev[i + 1]) for i, nm in enumerate(names)}
        self.m2l_seconds = self.stage_ms["m2l"] * 1e-3
        self._last = {"mpoles": mp, "locals": loc}
        return out.cpu().numpy()
