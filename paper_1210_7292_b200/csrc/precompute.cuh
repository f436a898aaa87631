// Operator assembly on the GPU.
//
// K_t[i, j] = profile(|x_i - y_j|) with target nodes x = w t + (w/2) node_i and
// source nodes y = (w/2) node_j (assemble_for_transfer, kernels.py:167-179,
// Kernel.matrix kernels.py:75-93).  The arithmetic is written with explicit
// round-to-nearest intrinsics in the reference's evaluation order (no FMA
// contraction), so the Laplace operators are bit-identical to the host
// assembly: x = (w t) + (h node), d = x - y, r = sqrt((d0^2 + d1^2) + d2^2),
// K = 1 / (4 pi r).  Helmholtz: (cos kr, sin kr) / (4 pi r) (libm vs CUDA
// sin/cos differ by an ulp, so those are equal to ~1e-16, not bitwise).
//
// Layout: out[t][i][j] row-major (targets x sources), real or interleaved
// complex; one thread per entry, the node table staged in shared memory.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace cfm {

constexpr double kFourPi = 12.566370614359172;  // 4 * pi rounded to double (== 4.0 * np.pi)

__global__ void k_assemble(int kernel, double wavenumber, int n, const double* __restrict__ nodes, double width,
                           const int8_t* __restrict__ transfers, double* __restrict__ out) {
  extern __shared__ double s_nodes[];  // n x 3 scaled by half width
  const double half = 0.5 * width;
  for (int k = threadIdx.x; k < 3 * n; k += blockDim.x) s_nodes[k] = __dmul_rn(half, nodes[k]);
  __syncthreads();
  const int t = blockIdx.y;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)n * n) return;
  const int i = int(e / n), j = int(e % n);
  const double c0 = __dmul_rn(width, double(transfers[3 * t])), c1 = __dmul_rn(width, double(transfers[3 * t + 1])),
               c2 = __dmul_rn(width, double(transfers[3 * t + 2]));
  const double d0 = __dsub_rn(__dadd_rn(c0, s_nodes[3 * i]), __dadd_rn(0.0, s_nodes[3 * j]));
  const double d1 = __dsub_rn(__dadd_rn(c1, s_nodes[3 * i + 1]), __dadd_rn(0.0, s_nodes[3 * j + 1]));
  const double d2 = __dsub_rn(__dadd_rn(c2, s_nodes[3 * i + 2]), __dadd_rn(0.0, s_nodes[3 * j + 2]));
  const double ss = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
  const double r = __dsqrt_rn(ss);
  const double den = __dmul_rn(kFourPi, r);
  const long long o = (long long)t * n * n + e;
  if (kernel == 0) {
    out[o] = __ddiv_rn(1.0, den);
  } else {
    double sn, cs;
    sincos(__dmul_rn(wavenumber, r), &sn, &cs);
    out[2 * o] = __ddiv_rn(cs, den);
    out[2 * o + 1] = __ddiv_rn(sn, den);
  }
}

}  // namespace cfm
