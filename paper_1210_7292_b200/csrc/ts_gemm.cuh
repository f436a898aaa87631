// Persistent GEMM kernel of the target-major two-stage low-rank path (sm_100a).
//
// Both stages of the path are plain dense GEMMs over uniform tiles:
//   stage 1  Y_T <- V_c (128-row blocks of the class stack) x X[64 sources]^T,
//            every 128-row block (= one plan entry, K = n) scattered to the
//            pair targets' Y_T rows when it ends;
//   stage 2  locals[64 targets] += scale * U_c (n x R_c) x Y_T[targets]^T,
//            K = R_c in 128-column blocks (one plan entry each), one ordered
//            read-modify-write of the targets' rows when the tile ends.
// tile_gemm_ws_kernel runs them with one CTA per tile; a tile is only ~76
// K-chunks (160 us), so the per-CTA launch, table loads, first-TMA latency and
// the epilogue drain (~11 us, measured from the two kernels' efficiencies)
// cost 6-7%.  Here one CTA per SM walks its tiles (static round-robin; the
// tiles are uniform) and the operand ring never drains: the producer lane runs
// ahead into the next tile while the consumers finish the current one, no
// shared-memory tables, no CTA-wide barrier after the start.  The two consumer
// halves (wn = 0 / 1) start `skew` chunks apart, so the two consumer warps of an SM
// sub-partition reach their epilogues at different times and one of them
// keeps the FP64 tensor pipe busy.
//
// Operands as in the full-operator mode of tile_gemm_ws_kernel: A = one 2-D
// TMA box (KC + 4 columns x 128 rows, landing with the conflict-free 36-double
// pitch) of the operator stack, B = 16 TMA tile::gather4 copies of the 64
// source rows (row -1 = empty slot, out of bounds, arrives as zeros); 8
// consumer warps (4 x 2, 32 x 32 warp tiles) run LDS -> DMMA.8x8x4 on a
// 4-stage ring with full/empty mbarriers.
#pragma once
#include "tile_gemm_ws.cuh"

namespace cfm {

struct TsGemmParams {
  int n_work;             // tiles x row blocks of this launch
  int nrb;                // row blocks (of 128 result rows) per tile
  int tile_base;          // first tile of this launch in the plan
  const int* tile_col;    // [tiles * 64] stage 1: source rows, stage 2: target rows (-1: empty column)
  const int* tile_off;    // [tiles + 1] entry range per tile (every tile has >= 1 entry)
  const int* entry_code;  // [E] operator block id (code_op null) or transfer code
  const int* code_op;     // optional transfer code -> operator block id
  const int* entry_src;   // [E * 64] rows of tmap_b (-1: empty)
  int nk;                 // inner length of an entry
  int nr;                 // result rows (stage 1: 128 per entry; stage 2: n)
  int a_rows;             // rows per operator block in the A stack
  int skew;               // chunks the odd consumer half starts behind the even one (0: off)
  // stage 1 output: row i of entry code c, source column v -> y[nbr[v * nslots + (info >> 8)] + (info & 255)],
  // info = rowinfo[c * 128 + i] (-1: padding row; nbr -1: the source has no such pair)
  double* y;
  const int* rowinfo;
  const int* nbr;
  int nslots;
  // stage 2 output: loc[v * loc_ld + row] += scale * acc
  double* loc;
  long long loc_ld;
  double scale;
  CUtensorMap tmap_a, tmap_b;
};

constexpr int kTsStages = 4;
constexpr int kTsKC = 32;
constexpr int kTsThreads = 9 * 32;  // 8 consumer warps + the producer warp
constexpr int ts_gemm_smem_bytes() { return kTsStages * (128 + 64) * (kTsKC + 4) * 8 + 2 * kTsStages * 8; }

template <int STAGE>
__global__ void __launch_bounds__(kTsThreads, 1) ts_gemm_kernel(const __grid_constant__ TsGemmParams p) {
  constexpr int BM = 128, BN = 64, KC = kTsKC, ST = kTsStages, LD = KC + 4;
  constexpr int WM = 4, NC = 8 * 32;
  constexpr int MT = 4, NTL = 4;  // 32 x 32 warp tiles
  extern __shared__ __align__(128) double smem_ts[];
  double* As = smem_ts;
  double* Bs = As + ST * BM * LD;
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + ST * BN * LD);
  uint64_t* empty = full + ST;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NC / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int nch = (p.nk + KC - 1) / KC;

  if (warp == NC / 32) {
    // ===================== producer: one lane, TMA only =====================
    if (lane != 0) return;
    constexpr unsigned STAGE_TX = unsigned((BM + BN) * LD * 8);
    int q = 0;
    for (int w = blockIdx.x; w < p.n_work; w += gridDim.x) {
      const int tile = p.tile_base + w / p.nrb;
      const int r0 = (w % p.nrb) * BM;
      const int e0 = __ldg(p.tile_off + tile), e1 = __ldg(p.tile_off + tile + 1);
      for (int e = e0; e < e1; ++e) {
        int4 rows[BN / 4];
        const int4* srow = reinterpret_cast<const int4*>(p.entry_src + (long long)e * BN);
#pragma unroll
        for (int j = 0; j < BN / 4; ++j) rows[j] = __ldg(srow + j);
        int op = __ldg(p.entry_code + e);
        if (p.code_op) op = __ldg(p.code_op + op);
        const int arow = op * p.a_rows + r0;
        for (int kc = 0; kc < nch; ++kc, ++q) {
          const int s = q % ST;
          if (q >= ST) mbar_wait_backoff(empty + s, ((q / ST) & 1) ^ 1);
          mbar_arrive_expect_tx(full + s, STAGE_TX);
          tma_load_2d(As + s * BM * LD, &p.tmap_a, kc * KC, arow, full + s);
          double* bs = Bs + s * BN * LD;
#pragma unroll
          for (int j = 0; j < BN / 4; ++j) tma_gather4(bs + 4 * j * LD, &p.tmap_b, kc * KC, rows[j], full + s);
        }
      }
    }
    return;
  }

  // ============================ consumer warps ============================
  const int g = lane >> 2, tg = lane & 3;
  const int wm = warp % WM, wn = warp / WM;
  const int aoff = (wm * 32 + g) * LD + tg, boff = (wn * 32 + g) * LD + tg;
  double acc[MT][NTL][2];
#pragma unroll
  for (int mi = 0; mi < MT; ++mi)
#pragma unroll
    for (int nj = 0; nj < NTL; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;
  double a0[MT], b0[NTL], a1[MT], b1[NTL];
  auto load = [&](double* a, double* b, int s, int kk) {
    const double* as = As + s * BM * LD + aoff;
    const double* bs = Bs + s * BN * LD + boff;
#pragma unroll
    for (int mi = 0; mi < MT; ++mi) a[mi] = as[mi * 8 * LD + kk];
#pragma unroll
    for (int nj = 0; nj < NTL; ++nj) b[nj] = bs[nj * 8 * LD + kk];
  };
  auto mma = [&](const double* a, const double* b) {
#pragma unroll
    for (int mi = 0; mi < MT; ++mi)
#pragma unroll
      for (int nj = 0; nj < NTL; ++nj) dmma884(acc[mi][nj][0], acc[mi][nj][1], a[mi], b[nj]);
  };
  if (int(blockIdx.x) >= p.n_work) return;
  const bool skewed = p.skew > 0 && p.skew < ST;
  if (skewed && wn == 1) asm volatile("bar.sync 2, %0;\n" ::"n"(NC) : "memory");
  int q = 0;
  mbar_wait(full, 0);
  load(a0, b0, 0, 0);
  for (int w = blockIdx.x; w < p.n_work; w += gridDim.x) {
    const int tile = p.tile_base + w / p.nrb;
    const int r0 = (w % p.nrb) * BM;
    const int e0 = __ldg(p.tile_off + tile);
    const int total = (__ldg(p.tile_off + tile + 1) - e0) * nch;
    const bool more_work = w + int(gridDim.x) < p.n_work;
    for (int c = 0; c < total; ++c, ++q) {
      const int s = q % ST;
      if (skewed && wn == 0 && q == p.skew) asm volatile("bar.arrive 2, %0;\n" ::"n"(NC) : "memory");
#pragma unroll
      for (int kk = 0; kk < KC; kk += 8) {
        load(a1, b1, s, kk + 4);
        mma(a0, b0);
        if (kk + 8 < KC) {
          load(a0, b0, s, kk + 8);
        } else if (c + 1 < total || more_work) {
          // the next chunk (of this tile or the CTA's next one): wait for it and
          // load its first fragments before this chunk's last k-step
          const int s1 = (q + 1) % ST;
          mbar_wait(full + s1, ((q + 1) / ST) & 1);
          load(a0, b0, s1, 0);
        }
        mma(a1, b1);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
      if (STAGE == 1 && (c + 1) % nch == 0) {
        // the entry's 128 rows of every source: each (slot, a) row goes to the
        // Y_T row of the pair's target (the 8 lanes of a tg mostly share a slot:
        // one broadcast load, a run of up to 64 B stored)
        const int* ri = p.rowinfo + (long long)__ldg(p.entry_code + e0 + c / nch) * BM + wm * 32 + g;
        int info[MT];
#pragma unroll
        for (int mi = 0; mi < MT; ++mi) info[mi] = __ldg(ri + mi * 8);
#pragma unroll
        for (int nj = 0; nj < NTL; ++nj)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int v = __ldg(p.tile_col + (long long)tile * BN + wn * 32 + nj * 8 + 2 * tg + h);
            const int* nb = p.nbr + (long long)v * p.nslots;
            int dst[MT];
#pragma unroll
            for (int mi = 0; mi < MT; ++mi) dst[mi] = (v >= 0 && info[mi] >= 0) ? __ldg(nb + (info[mi] >> 8)) : -1;
#pragma unroll
            for (int mi = 0; mi < MT; ++mi) {
              if (dst[mi] >= 0) p.y[(long long)dst[mi] + (info[mi] & 255)] = acc[mi][nj][h];
              acc[mi][nj][h] = 0.0;
            }
          }
      }
    }
    if (STAGE == 2) {
      // ordered, atomic-free accumulate: a target column belongs to one tile
#pragma unroll
      for (int nj = 0; nj < NTL; ++nj)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int v = __ldg(p.tile_col + (long long)tile * BN + wn * 32 + nj * 8 + 2 * tg + h);
          double* dst = p.loc + (long long)v * p.loc_ld + r0 + wm * 32 + g;
          double old[MT];
#pragma unroll
          for (int mi = 0; mi < MT; ++mi) old[mi] = (v >= 0 && r0 + wm * 32 + mi * 8 + g < p.nr) ? dst[mi * 8] : 0.0;
#pragma unroll
          for (int mi = 0; mi < MT; ++mi) {
            if (v >= 0 && r0 + wm * 32 + mi * 8 + g < p.nr) dst[mi * 8] = old[mi] + p.scale * acc[mi][nj][h];
            acc[mi][nj][h] = 0.0;
          }
        }
    }
  }
  // an odd-half warp of a CTA whose even half never reached `skew` chunks cannot
  // exist: the host launches the skewed kernel only when every CTA has > skew chunks
}

}  // namespace cfm
