// GPU octree construction: the reference's build_tree
// (octree.py:93-127) restated for the device.
//
//   ref  = (p - low) / width                  (fp64, same operation order)
//   ijk  = min(trunc(ref * 2^depth), 2^depth - 1)
//   leaf = occupied ijk, sorted lexicographically (i major)   -> row order
//   leaf_particles[leaf] = ascending particle indices in the leaf
//   level L-1 cells = sorted unique parents of level L cells
//
// Keys are the lexicographic keys (i * S + j) * S + k, so sorting keys sorts
// cells in the reference's row order; a stable radix sort of (key, index)
// keeps particle indices ascending inside each leaf.  The fp64 arithmetic uses
// explicit round-to-nearest intrinsics (no FMA contraction), so the integer
// cell indices are bitwise those of numpy.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cfm {

__global__ void k_leaf_keys(const double* __restrict__ pts, long long n, double lx, double ly, double lz, double width,
                            int depth, unsigned long long* __restrict__ keys, long long* __restrict__ idx,
                            int* __restrict__ bad) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long side = 1ll << depth;
  const double low[3] = {lx, ly, lz};
  long long c[3];
  for (int a = 0; a < 3; ++a) {
    const double r = __ddiv_rn(__dsub_rn(pts[3 * i + a], low[a]), width);
    if (!(r >= 0.0 && r <= 1.0)) atomicExch(bad, 1);  // outside the box (or NaN)
    long long v = (long long)__dmul_rn(r, double(side));
    c[a] = v < side - 1 ? v : side - 1;
    if (c[a] < 0) c[a] = 0;
  }
  keys[i] = (unsigned long long)((c[0] * side + c[1]) * side + c[2]);
  idx[i] = i;
}

// parent keys of sorted unique level-L keys (side S) at level L-1 (side S/2)
__global__ void k_parent_keys(const unsigned long long* __restrict__ keys, long long n, long long side,
                              unsigned long long* __restrict__ out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k = keys[i];
  const long long z = k % side, y = (k / side) % side, x = k / (side * side);
  const long long ps = side >> 1;
  out[i] = (unsigned long long)(((x >> 1) * ps + (y >> 1)) * ps + (z >> 1));
}

__global__ void k_keys_to_ijk(const unsigned long long* __restrict__ keys, long long n, long long side,
                              int* __restrict__ ijk) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k = keys[i];
  ijk[3 * i] = int(k / (side * side));
  ijk[3 * i + 1] = int((k / side) % side);
  ijk[3 * i + 2] = int(k % side);
}

}  // namespace cfm
