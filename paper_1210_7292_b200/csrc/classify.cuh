// GPU interaction-list classifier.
//
// Restates build_interaction_lists' far part (octree.py:148-178): for every
// occupied target cell at level L >= 2, the candidates are the 8 children of
// each of the 27 neighbours of its parent; a candidate is kept iff it is
// occupied and t . t > 3 with t = ijk_target - ijk_source (octree.py:50-65).
// The reference filters neighbours through the occupied parent set first;
// a child can only be occupied if its parent is, so testing the child alone
// is equivalent.  The reference sorts each list by source ijk (octree.py:176);
// enumerating candidates with source x, then y, then z ascending produces that
// order directly, so no sort is needed.
//
// Each kept pair is classified on the fly (symmetry.py:63-75): the cone
// representative index (into the 16 sorted representatives) and the perm id.
//
// Occupancy lookup: a dense S^3 int32 grid of row indices (S = 2^L), built by
// one scatter kernel; L <= 9 keeps it at <= 512 MB of the 180 GB HBM.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "symmetry.hpp"

namespace cfm {

__constant__ int8_t c_cone_index[kNumCodes];  // t_sym code -> index in sorted cone, -1 otherwise

__global__ void k_grid_scatter(const int* __restrict__ ijk, long long n, int S, int* __restrict__ grid) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int x = ijk[3 * i], y = ijk[3 * i + 1], z = ijk[3 * i + 2];
  grid[((long long)x * S + y) * S + z] = int(i);
}

template <bool FILL>
__global__ void k_classify(const int* __restrict__ ijk, long long n, int S, const int* __restrict__ grid,
                           int* __restrict__ counts, const long long* __restrict__ off,
                           int* __restrict__ src_out, int16_t* __restrict__ code_out,
                           int8_t* __restrict__ t_out, uint8_t* __restrict__ rep_out,
                           uint8_t* __restrict__ perm_out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int x = ijk[3 * i], y = ijk[3 * i + 1], z = ijk[3 * i + 2];
  const int bx = 2 * ((x >> 1) - 1), by = 2 * ((y >> 1) - 1), bz = 2 * ((z >> 1) - 1);
  long long w = FILL ? off[i] : 0;
  int cnt = 0;
  for (int sx = bx; sx < bx + 6; ++sx) {
    if (sx < 0 || sx >= S) continue;
    const int t0 = x - sx;
    for (int sy = by; sy < by + 6; ++sy) {
      if (sy < 0 || sy >= S) continue;
      const int t1 = y - sy;
      const long long rowbase = ((long long)sx * S + sy) * S;
      for (int sz = bz; sz < bz + 6; ++sz) {
        if (sz < 0 || sz >= S) continue;
        const int t2 = z - sz;
        if (!is_far(t0, t1, t2)) continue;
        const int r = grid[rowbase + sz];
        if (r < 0) continue;
        if (FILL) {
          src_out[w] = r;
          const int c = tcode(t0, t1, t2);
          if (code_out) code_out[w] = int16_t(c);
          if (t_out) {
            t_out[3 * w] = int8_t(t0);
            t_out[3 * w + 1] = int8_t(t1);
            t_out[3 * w + 2] = int8_t(t2);
          }
          if (rep_out || perm_out) {
            int ts[3], pid;
            canonicalize(t0, t1, t2, ts, pid);
            if (rep_out) rep_out[w] = uint8_t(c_cone_index[tcode(ts[0], ts[1], ts[2])]);
            if (perm_out) perm_out[w] = uint8_t(pid);
          }
          ++w;
        } else {
          ++cnt;
        }
      }
    }
  }
  if (!FILL) counts[i] = cnt;
}

// Warp per target: lane l handles candidates l, l+32, ... (216 in source-ijk
// order); kept pairs are compacted in candidate order with ballot/popc, so
// the output order is the reference's.  Counts (FILL=false) or writes (FILL).
//
// t = ijk_target - ijk_source depends only on the target's parity class
// ((x&1, y&1, z&1): x - bx = (x&1) + 2) and the candidate index, so the far
// test and the t-code come from a per-CTA shared table (8 classes x 216) and
// the occupancy-grid offset of a candidate from a second one; the CTAs are
// persistent (grid-stride over targets) so the tables are built once per CTA.
// Interior targets (whole 6^3 candidate box inside the level) skip the bounds
// tests.  The 8 children of a parent share the candidate box: the first
// occupied sibling's warp reads the box's occupancy once (7 loads per lane)
// and emits the lists of every occupied sibling; the other siblings' warps
// stop after one 8-lane lookup.  Output positions come from each target's own
// offset, so the lists are the same as per-target enumeration.
constexpr int kCandPad = 224;  // 7 x 32 lanes >= 216 candidates

template <bool FILL>
__global__ void __launch_bounds__(256) k_classify_warp(const int* __restrict__ ijk, long long n, int S,
                                                       const int* __restrict__ grid, int* __restrict__ counts,
                                                       const long long* __restrict__ off, int* __restrict__ src_out,
                                                       int16_t* __restrict__ code_out) {
  __shared__ int16_t s_code[8 * kCandPad];  // -1: near (or padding)
  __shared__ int s_goff[kCandPad];          // (dx * S + dy) * S + dz
  __shared__ int s_dxyz[kCandPad];          // dx | dy << 8 | dz << 16
  for (int i = threadIdx.x; i < 8 * kCandPad; i += blockDim.x) {
    const int p = i / kCandPad, c = i % kCandPad;
    int16_t v = -1;
    if (c < 216) {
      const int t0 = ((p >> 2) & 1) + 2 - c / 36, t1 = ((p >> 1) & 1) + 2 - (c / 6) % 6, t2 = (p & 1) + 2 - c % 6;
      if (is_far(t0, t1, t2)) v = int16_t(tcode(t0, t1, t2));
    }
    s_code[i] = v;
  }
  for (int c = threadIdx.x; c < kCandPad; c += blockDim.x) {
    const int dx = c < 216 ? c / 36 : 0, dy = c < 216 ? (c / 6) % 6 : 0, dz = c < 216 ? c % 6 : 0;
    s_goff[c] = (dx * S + dy) * S + dz;
    s_dxyz[c] = dx | dy << 8 | dz << 16;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long w = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); w < n; w += nw) {
    const int x = __ldg(ijk + 3 * w), y = __ldg(ijk + 3 * w + 1), z = __ldg(ijk + 3 * w + 2);
    // the 8 siblings share the parent's 6^3 candidate box: the occupied
    // sibling with the lowest child index (x&1, y&1, z&1) handles all of them
    // and reads the candidates' occupancy once
    const int px = x >> 1, py = y >> 1, pz = z >> 1;
    int sib = -1;
    if (lane < 8) {
      const int cx = 2 * px + (lane >> 2), cy = 2 * py + ((lane >> 1) & 1), cz = 2 * pz + (lane & 1);
      if (cx < S && cy < S && cz < S) sib = __ldg(grid + ((long long)cx * S + cy) * S + cz);
    }
    const unsigned occ = __ballot_sync(0xffffffffu, sib >= 0) & 0xffu;
    const int me = (x & 1) << 2 | (y & 1) << 1 | (z & 1);
    if (occ & ((1u << me) - 1u)) continue;
    const int bx = 2 * (px - 1), by = 2 * (py - 1), bz = 2 * (pz - 1);
    const bool interior = bx >= 0 && by >= 0 && bz >= 0 && bx + 6 <= S && by + 6 <= S && bz + 6 <= S;
    const long long pbase = ((long long)bx * S + by) * S + bz;
    int rows[7];
#pragma unroll
    for (int r = 0; r < 7; ++r) {
      const int c = r * 32 + lane;
      rows[r] = -1;
      if (c < 216) {
        bool ok = true;
        if (!interior) {
          const int d = s_dxyz[c];
          const int sx = bx + (d & 255), sy = by + ((d >> 8) & 255), sz = bz + (d >> 16);
          ok = sx >= 0 && sx < S && sy >= 0 && sy < S && sz >= 0 && sz < S;
        }
        if (ok) rows[r] = __ldg(grid + pbase + s_goff[c]);
      }
    }
    for (unsigned m = occ; m; m &= m - 1u) {
      const int l = __ffs(m) - 1;
      const int trow = __shfl_sync(0xffffffffu, sib, l);
      const int16_t* codes = s_code + l * kCandPad;
      long long base = FILL ? __ldg(off + trow) : 0;
      int total = 0;
#pragma unroll
      for (int r = 0; r < 7; ++r) {
        const int cd = codes[r * 32 + lane];
        const bool keep = cd >= 0 && rows[r] >= 0;
        const unsigned bm = __ballot_sync(0xffffffffu, keep);
        if (FILL && keep) {
          const long long pos = base + __popc(bm & ((1u << lane) - 1u));
          src_out[pos] = rows[r];
          code_out[pos] = int16_t(cd);
        }
        base += __popc(bm);
        total += __popc(bm);
      }
      if (!FILL && lane == 0) counts[trow] = total;
    }
  }
}

// Persistent grid for k_classify_warp: one wave of resident CTAs (by the
// occupancy calculator; the fill kernel's 44 registers allow 5 x 256 threads/SM).
template <bool FILL>
inline unsigned classify_warp_blocks(long long n_cells, int device) {
  int sms = 148, per_sm = 4;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_classify_warp<FILL>, 256, 0);
  const long long need = (n_cells + 7) / 8, cap = (long long)sms * (per_sm > 0 ? per_sm : 1);
  return unsigned(need < cap ? need : cap);
}

}  // namespace cfm
