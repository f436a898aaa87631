"""cProfile of one device precompute (default: l = 9 ia, eps 1e-8, levels 2-5)."""
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
from paper_1210_7292_b200 import ChebyshevGrid, laplace_kernel, make_handler  # noqa: E402
from paper_1210_7292_b200.symmetry import full_far_field_vectors  # noqa: E402

var = sys.argv[1] if len(sys.argv) > 1 else "ia"
ts = full_far_field_vectors()
lt = {l: ts for l in (2, 3, 4, 5)}
lw = {l: 2.0 / (1 << l) for l in lt}
make_handler(var, laplace_kernel(), ChebyshevGrid(9), 1e-8, budget_bytes=8_000_000_000).precompute(
    {5: ts[:4]}, {5: lw[5]})  # warm-up: CUDA context, cuSOLVER, streams
h = make_handler(var, laplace_kernel(), ChebyshevGrid(9), 1e-8, budget_bytes=8_000_000_000)
pr = cProfile.Profile()
pr.enable()
h.precompute(lt, lw)
pr.disable()
print("precompute_s", h.precompute_seconds)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
