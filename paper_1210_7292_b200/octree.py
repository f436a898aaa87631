"""Octree construction on the GPU.

Restates the reference's ``build_tree`` (octree.py:93-127) on the device:
leaf index of every particle with the same fp64 operation order
(``min(trunc((p - low) / width * 2^depth), 2^depth - 1)``), occupied cells per
level in the reference's row order (lexicographic ijk), and the leaf particle
lists (ascending particle indices inside a leaf).  Feeds
``B200M2LHandler.plan_level_cells`` without any host-side tree.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native


class GpuTree:
    """Uniform octree built on a CUDA device."""

    def __init__(self, points, center, half_width: float, depth: int, device: int = 0):
        pts = np.ascontiguousarray(points, dtype=np.float64)
        if pts.ndim != 2 or pts.shape[1] != 3:
            raise ValueError("particles must have shape (n, 3)")
        self._lib = _native.load()
        self.depth = int(depth)
        self.n_points = len(pts)
        c = np.ascontiguousarray(center, dtype=np.float64).reshape(3)
        h = ctypes.c_void_p()
        _native.check(self._lib.cfm_tree_build(int(device), pts.ctypes.data, len(pts), c.ctypes.data,
                                               float(half_width), int(depth), ctypes.byref(h)))
        self._t = h

    def __del__(self):
        t = getattr(self, "_t", None)
        if t is not None and t.value:
            try:
                self._lib.cfm_tree_destroy(t)
            except Exception:  # pragma: no cover
                pass
            self._t = None

    def n_cells(self, level: int) -> int:
        n = ctypes.c_int64()
        _native.check(self._lib.cfm_tree_level_size(self._t, int(level), ctypes.byref(n)))
        return n.value

    def cells(self, level: int) -> np.ndarray:
        """Occupied cells of a level, int32 [n, 3], reference row order."""
        out = np.zeros((self.n_cells(level), 3), dtype=np.int32)
        if len(out):
            _native.check(self._lib.cfm_tree_level_cells(self._t, int(level), out.ctypes.data))
        return out

    def leaf_particles(self):
        """(offsets [n_leaves + 1], particle indices [n]) of the leaves, in row order."""
        nl = self.n_cells(self.depth)
        off = np.zeros(nl + 1, dtype=np.int64)
        perm = np.zeros(self.n_points, dtype=np.int64)
        _native.check(self._lib.cfm_tree_leaf_particles(self._t, off.ctypes.data, perm.ctypes.data))
        return off, perm


def build_tree_gpu(points, center, half_width: float, depth: int, device: int = 0) -> GpuTree:
    return GpuTree(points, center, half_width, depth, device)
