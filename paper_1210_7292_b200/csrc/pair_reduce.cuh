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

// Several independent reductions (the pair-mode levels of one M2L step) in
// one launch: blocks [start[s], start[s+1]) reduce segment s.  Segments write
// disjoint target rows (different levels, or a level's leftover targets).
struct ReduceSeg {
  const double* F;
  long long f_ld;
  const long long* tgt;
  const long long* off;
  const int* frow;
  long long n_tgt;
  double* y;
  long long y_ld;
  int len;
  double scale;
};
constexpr int kMaxReduceSegs = 16;
struct MultiReduce {
  int n;
  long long start[kMaxReduceSegs + 1];
  ReduceSeg seg[kMaxReduceSegs];
};

__global__ void k_pair_reduce_multi(const __grid_constant__ MultiReduce m) {
  const long long b = blockIdx.x;
  int sg = 0;
  while (sg + 1 < m.n && b >= m.start[sg + 1]) ++sg;
  const ReduceSeg& r = m.seg[sg];
  const long long t = b - m.start[sg];
  if (t >= r.n_tgt) return;
  const long long q0 = r.off[t], q1 = r.off[t + 1];
  double* dst = r.y + r.tgt[t] * r.y_ld;
  for (int i = threadIdx.x; i < r.len; i += blockDim.x) {
    double acc = 0.0;
    for (long long q = q0; q < q1; ++q) acc += r.F[(long long)r.frow[q] * r.f_ld + i];
    dst[i] += r.scale * acc;
  }
}

}  // namespace cfm
