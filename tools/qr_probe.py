"""Timing of the batched linear algebra the device IA precompute uses (l = 9:
316 operators of 729 x 729, sketch 128)."""
import json
import time

import torch


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return round(best * 1e3, 2)


dev = torch.device("cuda")
T, n, k = 316, 729, 128
a = torch.randn(T, n, n, dtype=torch.float64, device=dev)
y = torch.randn(T, n, k, dtype=torch.float64, device=dev)
r = torch.randn(T, k, k, dtype=torch.float64, device=dev)
out = {
    "matmul_K_Omega_ms": t(lambda: torch.matmul(a, y)),
    "qr_reduced_ms": t(lambda: torch.linalg.qr(y)),
    "geqrf_ms": t(lambda: torch.geqrf(y)),
    "svd_kxk_batched_ms": t(lambda: torch.linalg.svd(r)),
    "svd_kxk_gesvdj_ms": t(lambda: torch.linalg.svd(r, driver="gesvdj")),
    "svd_kxk_gesvda_ms": t(lambda: torch.linalg.svd(r, driver="gesvda")),
    "qr_tall_one_ms": t(lambda: torch.linalg.qr(y[0])),
}
print(json.dumps(out, indent=1))
