"""Reference-call-path probe (config 2): apply_level with the Python batch and
pageable arrays, broken into batch->CSR, first call (plans built) and cached
calls."""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_1210_7292_b200 import ChebyshevGrid, full_far_field_vectors, laplace_kernel, make_handler  # noqa: E402
from paper_1210_7292_b200.m2l import _batch_to_csr  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cells, widths, _ = bench.gpu_level_cells(cfg, 0)
levels = sorted(cells)
n, depth, order, geom, variant, eps = bench.CONFIGS[cfg]
h = make_handler(variant, laplace_kernel(), ChebyshevGrid(order), eps, device=0)
h.precompute({l: full_far_field_vectors() for l in levels}, widths)
t0 = time.perf_counter()
batches = bench.reference_batches(cells, 0)
out = {"batch_build_s": time.perf_counter() - t0}
for l in levels:
    t0 = time.perf_counter()
    _batch_to_csr(batches[l])
    out[f"csr_ms_L{l}"] = (time.perf_counter() - t0) * 1e3
# one steady-state call per level, broken down (plans cached by the first call)
mp = {l: np.random.default_rng(l).uniform(-1, 1, (len(cells[l]), order**3)) for l in levels}
loc = {l: np.zeros_like(mp[l]) for l in levels}
for l in levels:
    h.apply_level(l, batches[l], mp[l], loc[l])
for l in levels:
    t0 = time.perf_counter()
    h.apply_level(l, batches[l], mp[l], loc[l])
    out[f"call_ms_L{l}"] = (time.perf_counter() - t0) * 1e3
    out[f"kernel_ms_L{l}"] = h.last_apply_stats()[0]
del batches
out["e2e"] = bench.reference_api_e2e(h, cells, levels, order**3, np.float64, 3, 0)
print(json.dumps(out, indent=1))
