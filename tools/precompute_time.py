"""Time M2LHandler.precompute on the device vs the host path."""
import json, sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_1210_7292_b200 import ChebyshevGrid, helmholtz_kernel, laplace_kernel, make_handler
from paper_1210_7292_b200.symmetry import full_far_field_vectors

ts = full_far_field_vectors()
cases = [("cfg2 nablk l5", "nablk", laplace_kernel(), 5, 1e-5, [2, 3, 4, 5, 6], 1.0),
         ("cfg2 iablk l5", "iablk", laplace_kernel(), 5, 1e-5, [2, 3, 4, 5, 6], 1.0),
         ("cfg3 sa l9 eps1e-8", "sa", laplace_kernel(), 9, 1e-8, [2, 3, 4, 5], 2.0),
         ("cfg3 sarcmp l9 eps1e-8", "sarcmp", laplace_kernel(), 9, 1e-8, [2, 3, 4, 5], 2.0),
         ("cfg3 ia l9 eps1e-8", "ia", laplace_kernel(), 9, 1e-8, [2, 3, 4, 5], 2.0),
         ("cfg4 nablk l7", "nablk", laplace_kernel(), 7, 1e-5, [2, 3, 4, 5, 6, 7], 1.0),
         ("cfg5 helm iablk l5", "iablk", helmholtz_kernel(8 * np.pi), 5, 1e-4, [2, 3, 4, 5], 2.0)]
only = sys.argv[1:] or None
res = {}
for name, var, ker, order, eps, levels, side in cases:
    lt = {l: ts for l in levels}
    lw = {l: side / (1 << l) for l in levels}
    row = {}
    for where in ("device", "host"):
        if where == "host" and var in ("sa", "sarcmp", "ia") and "--host-sa" not in sys.argv:
            continue
        h = make_handler(var, ker, ChebyshevGrid(order), eps, precompute_on=where, budget_bytes=8_000_000_000)
        if where == "device":  # warm the CUDA context / cuSOLVER handles once
            make_handler(var, ker, ChebyshevGrid(order), eps, budget_bytes=8_000_000_000).precompute(
                {levels[-1]: ts[:4]}, {levels[-1]: lw[levels[-1]]})
        h.precompute(lt, lw)
        row[where] = round(h.precompute_seconds, 3)
        row["ranks_" + where] = (h.shared_rank(levels[0]) if h.is_shared_basis else
                                 (None if h.is_dense else sum(h.level_ranks(levels[0]))))
    res[name] = row
    print(name, row, flush=True)
json.dump(res, open("gpurun_out/precompute_time.json", "w"), indent=1)
