// Segmented, ordered reduction of per-pair results into target rows (pair mode).
//
// In pair mode each tile entry holds 64 (target, source) pairs that share one
// transfer vector (one operator and one permutation), so sparse trees fill the
// DMMA tiles; the per-pair results F[pair] are then summed per target in a
// fixed order and added once, scaled, exactly the reference's
// `locals[target] += scale * acc` (m2l.py:337, :363, :393).  No atomics.
#pragma once
#include <cuda_runtime.h>

namespace cfm {

__global__ void k_pair_reduce(const double* __restrict__ F, long long f_ld, const long long* __restrict__ tgt,
                              const long long* __restrict__ off, const int* __restrict__ frow, long long n_tgt,
                              double* __restrict__ y, long long y_ld, int len, double scale, int accumulate) {
  const long long t = blockIdx.x;
  if (t >= n_tgt) return;
  const long long q0 = off[t], q1 = off[t + 1];
  double* dst = y + tgt[t] * y_ld;
  for (int i = threadIdx.x; i < len; i += blockDim.x) {
    double s = 0.0;
    for (long long q = q0; q < q1; ++q) s += F[(long long)frow[q] * f_ld + i];
    if (accumulate)
      dst[i] += scale * s;
    else
      dst[i] = scale * s;
  }
}

}  // namespace cfm
