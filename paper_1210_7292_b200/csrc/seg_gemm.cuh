// Stage 2 of the two-stage low-rank M2L (ia / iasym / iablk on dense levels):
//     locals[i, c] += scale * sum_e sum_a U_{t_e}[i, 16 j_e + a] * Y_e[c, a]
// over the entries e = (transfer t, rank segment j) of a target tile, i.e. the
// reference's `acc += left[table] @ Y` (m2l.py:425, lowrank.py:43-44) with the
// rank-r intermediate Y produced by stage 1 in this kernel's reading order.
//
// Every entry is a 16-wide K slice: A = U_t[:, 16 j : 16 j + 16] (one 2-D TMA
// box of 20 x 128 from the per-transfer factor stack), B = the 64 sources'
// rank rows of Y (stage 1's packed output, one row per source): 16 TMA
// tile::gather4 copies of 4 rows x 20 columns from the entry's column
// (op_col); the rows past the rank are zero in U_t and in Y.  Two entries share one pipeline stage
// (two A and two B sub-tiles at a 20-double pitch), so the consumer warps run
// 8 k-steps (128 DMMA per warp) between barrier operations instead of 4.
// Warp specialisation as in tile_gemm_ws_kernel: one producer warp issues the
// copies (a gather per lane), 8 consumer warps run mma.sync.m8n8k4.f64 with the next stage's first
// fragments loaded before the current stage's last k-step; accumulators stay
// in registers and every target column is written once, in order, no atomics.
#pragma once
#include "tile_gemm_ws.cuh"

namespace cfm {

constexpr int kSegStages = 3;
constexpr int kSegPitch = 20;  // 16 + 4: conflict-free fragment loads

constexpr int seg_pair_smem_bytes() {
  return kSegStages * 2 * (128 + 64) * kSegPitch * 8 + 2 * kSegStages * 8 + 4 * 64;
}

__global__ void __launch_bounds__(12 * 32, 1) seg_pair_gemm_kernel(const __grid_constant__ TileParams p) {
  constexpr int BM = 128, BN = 64, WM = 4, WN = 2, STAGES = kSegStages, LD = kSegPitch;
  constexpr int NC = WM * WN * 32;
  constexpr int WTM = BM / WM, WTN = BN / WN, MT = WTM / 8, NTL = WTN / 8;
  constexpr int SUB_A = BM * LD, SUB_B = BN * LD;  // doubles per sub-tile
  constexpr unsigned STAGE_TX = unsigned(2 * (SUB_A + SUB_B) * 8);

  extern __shared__ __align__(128) double smem_seg[];
  double* As = smem_seg;                       // [STAGES][2][BM][LD]
  double* Bs = As + STAGES * 2 * SUB_A;        // [STAGES][2][BN][LD]
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + STAGES * 2 * SUB_B);
  uint64_t* empty = full + STAGES;
  int* s_col = reinterpret_cast<int*>(empty + STAGES);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tile = p.tile_base + int(blockIdx.x);
  const int e_begin = p.tile_off[tile], e_end = p.tile_off[tile + 1];
  const int n_pairs = (e_end - e_begin + 1) / 2;
  for (int c = tid; c < BN; c += blockDim.x) s_col[c] = p.tile_col[(long long)tile * BN + c];
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NC / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (tid >= NC) {
    // ---- producer warp: per stage two entries, each A = one 2-D box (lane 0 /
    // lane 16) and B = 16 tile::gather4 copies of 4 source rows x 20 columns
    // at the entry's column, one per lane (lane l: entry l / 16, rows 4 (l % 16)
    // .. +3).  Each lane's source rows and the entry's column/operator of the
    // next stage are loaded before waiting for its slot, so the index loads'
    // latency hides under the wait.  The odd last entry (no partner) reads
    // row -1 everywhere (zeros, skipped by the consumers' k-step mask).
    if (warp != NC / 32) return;
    const int hl = lane >> 4, jl = lane & 15;
    auto fetch = [&](int q, int4& rows, int& col, int& op) {
      const int e = e_begin + 2 * q + hl;
      const bool live = q < n_pairs && e < e_end;
      rows = live ? __ldg(reinterpret_cast<const int4*>(p.entry_src + (long long)e * BN) + jl) : make_int4(-1, -1, -1, -1);
      op = __ldg(p.entry_code + (live ? e : e_begin));
      col = live ? __ldg(p.op_col + op) : 0;
    };
    int4 rows_n;
    int col_n, op_n;
    fetch(0, rows_n, col_n, op_n);
    for (int q = 0; q < n_pairs; ++q) {
      const int s = q % STAGES;
      const int4 rows = rows_n;
      const int col = col_n, op = op_n;
      if (q + 1 < n_pairs) fetch(q + 1, rows_n, col_n, op_n);
      if (lane == 0) {
        if (q >= STAGES) mbar_wait_backoff(empty + s, ((q / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(full + s, STAGE_TX);
      }
      __syncwarp();
      if (jl == 0)
        tma_load_2d(As + (s * 2 + hl) * SUB_A, &p.tmap_a, (op & 1) * p.ft_colseg, (op >> 1) * p.ft_rows, full + s);
      tma_gather4(Bs + (s * 2 + hl) * SUB_B + 4 * jl * LD, &p.tmap_b, col, rows, full + s);
    }
    return;
  }

  // ---- consumers
  const int g = lane >> 2, tg = lane & 3;
  const int wm = warp % WM, wn = warp / WM;
  double acc[MT][NTL][2];
#pragma unroll
  for (int mi = 0; mi < MT; ++mi)
#pragma unroll
    for (int nj = 0; nj < NTL; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;
  const int aoff = (wm * WTM + g) * LD + tg, boff = (wn * WTN + g) * LD + tg;
  double a0[MT], b0[NTL], a1[MT], b1[NTL];
  // k-step kk (0..31) of stage s: sub-tile kk / 16, column kk % 16
  auto load = [&](double* a, double* b, int s, int kk) {
    const double* as = As + (s * 2 + (kk >> 4)) * SUB_A + aoff + (kk & 15);
    const double* bs = Bs + (s * 2 + (kk >> 4)) * SUB_B + boff + (kk & 15);
#pragma unroll
    for (int mi = 0; mi < MT; ++mi) a[mi] = as[mi * 8 * LD];
#pragma unroll
    for (int nj = 0; nj < NTL; ++nj) b[nj] = bs[nj * 8 * LD];
  };
  auto mma = [&](const double* a, const double* b) {
#pragma unroll
    for (int mi = 0; mi < MT; ++mi)
#pragma unroll
      for (int nj = 0; nj < NTL; ++nj) dmma884(acc[mi][nj][0], acc[mi][nj][1], a[mi], b[nj]);
  };
  // live k-steps of a stage (bit 4h + j: k-step j of its entry h): a rank
  // segment narrower than 16 leaves exact zeros in its last k-steps, and the
  // odd last entry pairs with an all-zero sub-tile -- those DMMAs are skipped
  auto stage_mask = [&](int q) -> unsigned {
    unsigned m = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = e_begin + 2 * q + h;
      if (e < e_end) {
        const int ks = p.seg_ksteps ? __ldg(p.seg_ksteps + __ldg(p.entry_code + e)) : 4;
        m |= ((1u << ks) - 1u) << (4 * h);
      }
    }
    return m;
  };
  if (n_pairs > 0) {
    mbar_wait(full, 0);
    load(a0, b0, 0, 0);
    unsigned msk = stage_mask(0);
    for (int q = 0; q < n_pairs; ++q) {
      const int s = q % STAGES;
      const unsigned msk_next = q + 1 < n_pairs ? stage_mask(q + 1) : 0u;
#pragma unroll
      for (int kk = 0; kk < 32; kk += 8) {
        load(a1, b1, s, kk + 4);
        if ((msk >> (kk >> 2)) & 1u) mma(a0, b0);
        if (kk + 8 < 32) {
          load(a0, b0, s, kk + 8);
        } else if (q + 1 < n_pairs) {
          const int s1 = (q + 1) % STAGES;
          mbar_wait(full + s1, ((q + 1) / STAGES) & 1);
          load(a0, b0, s1, 0);
        }
        if ((msk >> ((kk + 4) >> 2)) & 1u) mma(a1, b1);
      }
      msk = msk_next;
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
    }
  }
  if (e_begin == e_end && p.accumulate) return;
  // ---- epilogue: ordered, atomic-free write of this tile's target columns
#pragma unroll
  for (int mi = 0; mi < MT; ++mi) {
    const int row = wm * WTM + mi * 8 + g;
    if (row >= p.nr) continue;
#pragma unroll
    for (int nj = 0; nj < NTL; ++nj)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int v = s_col[wn * WTN + nj * 8 + 2 * tg + h];
        if (v < 0) continue;
        double* dst = p.y + (long long)v * p.y_ld + row;
        const double val = p.scale * acc[mi][nj][h];
        if (p.accumulate)
          *dst += val;
        else
          *dst = val;
      }
  }
}

}  // namespace cfm
