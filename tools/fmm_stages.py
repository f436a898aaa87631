"""Per-stage device times of the whole GPU FMM (B200FmmPlan.run) on a bench config."""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--variant", default=None)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    from paper_1210_7292_b200 import helmholtz_kernel, laplace_kernel
    from paper_1210_7292_b200.fmm import B200FmmPlan

    n, depth, order, geom, variant, eps = bench.CONFIGS[a.config]
    pts, center, half = bench.bench_points(a.config)
    kernel = helmholtz_kernel(bench.HELMHOLTZ[a.config]) if a.config in bench.HELMHOLTZ else laplace_kernel()
    t0 = time.perf_counter()
    plan = B200FmmPlan(pts, center, half, depth, kernel, order, eps, variant=a.variant or variant)
    setup = time.perf_counter() - t0
    rng = np.random.default_rng(1)
    w = rng.uniform(-1, 1, len(pts))
    for _ in range(a.reps):
        t0 = time.perf_counter()
        plan.run(w)
        wall = time.perf_counter() - t0
        print({k: round(v, 3) for k, v in plan.stage_ms.items()}, "total_device_ms",
              round(sum(plan.stage_ms.values()), 3), "wall_s", round(wall, 3), "setup_s", round(setup, 2))


if __name__ == "__main__":
    main()
