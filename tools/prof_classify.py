"""Device classifier of BASELINE config 2's deepest level (262,144 cells,
46.3 M far pairs) for ncu: count pass once, then REPS fill passes."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
from paper_1210_7292_b200 import _native  # noqa: E402


def main(reps=3, level=6):
    lib = _native.load()
    side = 1 << level
    cells = np.stack(np.meshgrid(*(np.arange(side),) * 3, indexing="ij"), -1).reshape(-1, 3).astype(np.int32)
    d = torch.from_numpy(cells).cuda()
    n = len(cells)
    offs = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    tot = ctypes.c_int64()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _native.check(lib.cfm_classify_count_device(0, level, n, d.data_ptr(), offs.data_ptr(), ctypes.byref(tot), st))
    src = torch.empty(tot.value, dtype=torch.int32, device="cuda")
    code = torch.empty(tot.value, dtype=torch.int16, device="cuda")
    for _ in range(reps):
        _native.check(lib.cfm_classify_fill_device(0, level, n, d.data_ptr(), offs.data_ptr(), src.data_ptr(),
                                                   code.data_ptr(), st))
    torch.cuda.synchronize()
    print("pairs", tot.value)


if __name__ == "__main__":
    main()
