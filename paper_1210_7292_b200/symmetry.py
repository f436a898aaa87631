"""Cone representatives and reflection permutations (host side).

Product restatement of the reference's symmetry module (symmetry.py:44-149),
used by the handler's precompute to decide which operators to build (one per
cone representative for the symmetric variants) and by tests.  The device
applies the same permutations from index tables built in C++
(csrc/symmetry.hpp); both follow:

  canonicalize(t): flips = (t_i < 0); axis_order = stable sort of the axes by
    (-|t_i|, i), 1-based; t_sym = |t|[axis_order]          (symmetry.py:63-75)
  table[j] = m(reorder(flip(components(j))))                (symmetry.py:86-102)
  K_t[i, j] = K_rep[table[i], table[j]]                      (symmetry.py:10-12)
"""

from __future__ import annotations

from functools import lru_cache
from typing import NamedTuple

import numpy as np

from .numerics import component_indices

AXIS_ORDERS = ((1, 2, 3), (1, 3, 2), (2, 1, 3), (2, 3, 1), (3, 1, 2), (3, 2, 1))


class PermutationSpec(NamedTuple):
    axial_flips: tuple
    axis_order: tuple

    @property
    def is_identity(self) -> bool:
        return not any(self.axial_flips) and tuple(self.axis_order) == (1, 2, 3)

    @property
    def perm_id(self) -> int:
        f = self.axial_flips
        return (int(f[0]) | int(f[1]) << 1 | int(f[2]) << 2) * 6 + AXIS_ORDERS.index(tuple(self.axis_order))


def spec_from_id(perm_id: int) -> PermutationSpec:
    flips = perm_id // 6
    return PermutationSpec(tuple(bool(flips >> a & 1) for a in range(3)), AXIS_ORDERS[perm_id % 6])


def canonicalize(t) -> tuple[tuple[int, int, int], PermutationSpec]:
    t = tuple(int(c) for c in t)
    a = [abs(c) for c in t]
    order = tuple(i + 1 for i in sorted(range(3), key=lambda i: (-a[i], i)))
    return tuple(a[i - 1] for i in order), PermutationSpec(tuple(c < 0 for c in t), order)


@lru_cache(maxsize=None)
def permutation_table(perm_id: int, order: int) -> np.ndarray:
    spec = spec_from_id(perm_id)
    comp = component_indices(order).copy()
    for axis in range(3):
        if spec.axial_flips[axis]:
            comp[axis] = order - 1 - comp[axis]
    comp = comp[[i - 1 for i in spec.axis_order]]
    table = comp[0] + comp[1] * order + comp[2] * order * order
    table.setflags(write=False)
    return table


@lru_cache(maxsize=None)
def inverse_permutation_table(perm_id: int, order: int) -> np.ndarray:
    table = permutation_table(perm_id, order)
    inv = np.empty_like(table)
    inv[table] = np.arange(table.size)
    inv.setflags(write=False)
    return inv


def is_far(t) -> bool:
    return t[0] * t[0] + t[1] * t[1] + t[2] * t[2] > 3


def full_far_field_vectors() -> list[tuple[int, int, int]]:
    """The 316 admissible far-field transfer vectors, lexicographic."""
    r = range(-3, 4)
    return [(a, b, c) for a in r for b in r for c in r if is_far((a, b, c))]


def tcode(t) -> int:
    return (int(t[0]) + 3) * 49 + (int(t[1]) + 3) * 7 + (int(t[2]) + 3)


class SymmetryMap:
    """Sorted cone of a transfer list and the total assignment t -> (rep idx, spec)."""

    def __init__(self, vectors):
        assignment = {}
        reps = set()
        for t in vectors:
            t = tuple(int(c) for c in t)
            rep, spec = canonicalize(t)
            reps.add(rep)
            assignment[t] = (rep, spec)
        self.cone = sorted(reps)
        index = {rep: i for i, rep in enumerate(self.cone)}
        self.assignment = {t: (index[rep], spec) for t, (rep, spec) in assignment.items()}

    def __len__(self) -> int:
        return len(self.cone)

    def lookup(self, t):
        idx, spec = self.assignment[tuple(t)]
        return self.cone[idx], spec
