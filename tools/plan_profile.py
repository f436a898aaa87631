"""Plan-time breakdown (CFM_TRACE=1 prints the native stages) for a config's levels."""
import os
import sys
import time

os.environ.setdefault("CFM_TRACE", "1")
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1210_7292_b200 import ChebyshevGrid, full_far_field_vectors, make_handler  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
cells, widths, _ = bench.gpu_level_cells(cfg, 0)
n, depth, order, geom, variant, eps = bench.CONFIGS[cfg]
h = make_handler(variant, bench._kernel_of(cfg), ChebyshevGrid(order), eps, device=0)
h.precompute({l: full_far_field_vectors() for l in cells}, widths)
for l in sorted(cells):
    t0 = time.perf_counter()
    st = h.plan_level_cells(l, cells[l].astype("int32"))
    print(f"level {l}: {st['pairs']} pairs, plan {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
