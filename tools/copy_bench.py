"""Host<->device copy rates on the box: pinned, pageable (driver staging) and
cudaHostRegister of a pageable numpy array (cost of registering included).
Informs how the handler moves the reference's pageable level arrays
(engine.py:104-108 allocates them with np.zeros)."""

import json
import time

import numpy as np
import torch


def t_ms(fn, reps=5):
    best = 1e30
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) * 1e3)
    return best


def main():
    out = {}
    cudart = torch.cuda.cudart()
    for mb in (64, 262, 1024):
        n = mb * (1 << 20) // 8
        a = np.random.default_rng(0).uniform(size=n)
        d = torch.empty(n, dtype=torch.float64, device="cuda")
        pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
        pin.copy_(torch.from_numpy(a))
        ta = torch.from_numpy(a)
        r = {}
        r["h2d_pinned_ms"] = t_ms(lambda: d.copy_(pin, non_blocking=True))
        r["h2d_pageable_ms"] = t_ms(lambda: d.copy_(ta))
        r["d2h_pinned_ms"] = t_ms(lambda: pin.copy_(d, non_blocking=True))
        r["d2h_pageable_ms"] = t_ms(lambda: ta.copy_(d))

        def reg():
            rc = cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
            assert int(rc) == 0, rc
            d.copy_(ta, non_blocking=True)
            torch.cuda.synchronize()
            cudart.cudaHostUnregister(a.ctypes.data)

        r["h2d_register_copy_unregister_ms"] = t_ms(reg)

        def reg_only():
            cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
            cudart.cudaHostUnregister(a.ctypes.data)

        r["register_unregister_ms"] = t_ms(reg_only)
        t0 = time.perf_counter()
        for _ in range(3):
            pin.numpy()[:] = a
        r["host_memcpy_1thread_ms"] = (time.perf_counter() - t0) / 3 * 1e3
        for k in list(r):
            r[k.replace("_ms", "_GBps")] = mb * 1.048576e-3 / (r[k] * 1e-3) if r[k] > 0 else None
        out[f"{mb}MB"] = r
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
