"""One bench step (all levels, one launch) for ncu: plans BASELINE config 2 and
applies it `--reps` times with device-resident expansions."""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--variant", default=None)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--gpu-tree", action="store_true", help="level cells from the GPU octree (large configs)")
    ap.add_argument("--signed", action="store_true", help="multipoles U[-1,1] (as bench.py) instead of U[0,1]")
    ap.add_argument("--host", action="store_true", help="pinned host numpy buffers (the e2e path)")
    ap.add_argument("--flush", action="store_true", help="write 256 MB (> L2) and synchronize before each step")
    ap.add_argument("--order", type=int, default=None, help="expansion order override (same tree)")
    ap.add_argument("--levels", default=None, help="comma list: apply only these levels (all are planned)")
    a = ap.parse_args()
    import torch

    from paper_1210_7292_b200 import ChebyshevGrid, full_far_field_vectors, laplace_kernel, make_handler

    n, depth, order, geom, variant, eps = bench.CONFIGS[a.config]
    variant = a.variant or variant
    order = a.order or order
    if a.gpu_tree:
        cells, widths, _ = bench.gpu_level_cells(a.config, 0)
    else:
        cells, widths = bench.cached_level_cells(a.config)
    levels = sorted(cells)
    full = full_far_field_vectors()
    h = make_handler(variant, laplace_kernel(), ChebyshevGrid(order), eps,
                     budget_bytes=4_000_000_000 if variant in ("sa", "sarcmp") else 2_000_000_000)
    h.precompute({l: full for l in levels}, widths)
    for l in levels:
        h.plan_level_cells(l, cells[l].astype("int32"))
    mp = {l: torch.rand((len(cells[l]), order**3), dtype=torch.float64, device="cuda") for l in levels}
    if a.signed:
        mp = {l: v * 2 - 1 for l, v in mp.items()}
    loc = {l: torch.zeros_like(mp[l]) for l in levels}
    if a.host:
        hm = {l: torch.empty(mp[l].shape, dtype=mp[l].dtype, pin_memory=True) for l in levels}
        hl = {l: torch.zeros(mp[l].shape, dtype=mp[l].dtype, pin_memory=True) for l in levels}
        for l in levels:
            hm[l].copy_(mp[l].cpu())
        mp = {l: hm[l].numpy() for l in levels}
        loc = {l: hl[l].numpy() for l in levels}
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda") if a.flush else None
    if a.levels:
        levels = [int(x) for x in a.levels.split(",")]
    for i in range(a.reps):
        if flush is not None:
            flush.fill_(float(i))
            torch.cuda.synchronize()
        t0 = time.perf_counter()
        h.apply_levels({l: (mp[l], loc[l]) for l in levels})
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        print("step device ms %.3f launches %d" % h.last_apply_stats(), "host call ms %.3f" % ((t1 - t0) * 1e3))


if __name__ == "__main__":
    main()
