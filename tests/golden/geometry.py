"""Seeded synthetic inputs shared by the golden generator, the tests and bench.py.

BASELINE.json's configs are generator-defined (no public dataset): uniform
points in the unit cube (bbox centre (0.5,0.5,0.5), half width 0.5) or uniform
on a radius-R sphere (Gaussian triples normalised; bbox centre 0, half width R),
charges U[-1,1] from the next seed.
"""

import numpy as np


def cube_points(n, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(0.0, 1.0, (n, 3))


def sphere_points(n, seed, radius=1.0):
    rng = np.random.default_rng(seed)
    p = rng.standard_normal((n, 3))
    return radius * p / np.linalg.norm(p, axis=1, keepdims=True)
