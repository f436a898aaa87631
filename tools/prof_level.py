"""Minimal driver for ncu: plan one full-cube level and apply it a few times.

    python tools/prof_level.py --level 6 --order 5 --variant nablk --reps 3
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--level", type=int, default=6)
    ap.add_argument("--order", type=int, default=5)
    ap.add_argument("--variant", default="nablk")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--eps", type=float, default=1e-5)
    a = ap.parse_args()
    import torch

    from paper_1210_7292_b200 import ChebyshevGrid, full_far_field_vectors, laplace_kernel, make_handler

    side = 1 << a.level
    cells = np.stack(np.meshgrid(*(np.arange(side),) * 3, indexing="ij"), -1).reshape(-1, 3).astype(np.int32)
    full = full_far_field_vectors()
    h = make_handler(a.variant, laplace_kernel(), ChebyshevGrid(a.order), a.eps)
    h.precompute({2: full, a.level: full}, {2: 0.25, a.level: 1.0 / side})
    st = h.plan_level_cells(a.level, cells)
    n = a.order**3
    mp = torch.rand((len(cells), n), dtype=torch.float64, device="cuda")
    loc = torch.zeros_like(mp)
    for _ in range(a.reps):
        t0 = time.perf_counter()
        h.apply_planned(a.level, mp, loc)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        ms, launches = h.last_apply_stats()
        flops = st["pairs"] * (2 * n * n if a.variant in ("na", "nasym", "nablk") else 0)
        print(f"level {a.level} l={a.order} {a.variant}: {st} device {ms:.3f} ms wall {dt*1e3:.1f} ms "
              f"launches {launches} {flops / (ms * 1e-3) / 1e12:.2f} TF/s")


if __name__ == "__main__":
    main()
