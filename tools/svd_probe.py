"""Probe cuSOLVER (via torch.linalg) SVD/QR timings for GPU precompute sizing."""
import time, torch
dev = torch.device("cuda")
def t(f, rep=2):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(rep): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / rep
for b, n in ((16, 125), (316, 125), (16, 343), (16, 729), (64, 729)):
    a = torch.randn(b, n, n, dtype=torch.float64, device=dev)
    for drv in (None, "gesvd", "gesvdj", "gesvda"):
        try:
            print(b, n, drv, "%.4f s" % t(lambda: torch.linalg.svd(a, full_matrices=False, driver=drv)), flush=True)
        except Exception as e:
            print(b, n, drv, "ERR", str(e)[:80], flush=True)
    print(b, n, "eigh", "%.4f s" % t(lambda: torch.linalg.eigh(a @ a.mT)), flush=True)
for n, N in ((125, 316 * 125), (729, 316 * 729)):
    a = torch.randn(N, n, dtype=torch.float64, device=dev)
    print("qr", N, n, "%.4f s" % t(lambda: torch.linalg.qr(a)), flush=True)
    print("svd tall", N, n, "%.4f s" % t(lambda: torch.linalg.svd(a, full_matrices=False), 1), flush=True)
    c = torch.randn(2, 316, n, n, dtype=torch.complex128, device=dev)
    print("c128 svd", n, "%.4f s" % t(lambda: torch.linalg.svd(c[0, :16], full_matrices=False), 1), flush=True)
