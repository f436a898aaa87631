// Persistent full-operator tile kernel (sm_100a): one CTA per SM walks a work
// queue of (tile, row block) items from several tile lists (the levels of an
// M2L step, the stages of the two-stage low-rank path).
//
// Same math and operand staging as the full-operator mode of
// tile_gemm_ws_kernel -- per entry acc[128 x 64] += A_op[r0.., k] X[src_c, k],
// A = one 2-D TMA box (KC + 4 columns x 128 rows, landing with the
// conflict-free 36-double pitch) of the operator stack, B = 16 TMA
// tile::gather4 copies of the entry's 64 source rows (row -1 = empty slot, out
// of bounds, arrives as zeros), 8 consumer warps (4 x 2, 32 x 32 warp tiles)
// running LDS -> DMMA.8x8x4 on a 4-stage ring with full/empty mbarriers --
// but the ring never drains between tiles.  With one CTA per tile the launch
// of the CTA, its table loads, the first TMA round trip and the epilogue
// drain cost ~11 us per tile (6-7% of a 76-chunk low-rank tile, ~1% of a
// 756-chunk nablk tile) and leave the FP64 tensor pipe idle; here
//   * the producer lane takes the next work item from a global counter
//     (atomicAdd: long tiles first, short ones fill the tail, CTAs that start
//     late simply take fewer) and streams its chunks right behind the
//     previous item's, reading the plan from global memory;
//   * it posts the item in a small shared-memory ring just before arming the
//     item's first stage, so the consumers learn it when that stage's full
//     barrier completes; a final item -1 on an empty stage ends the CTA;
//   * the consumers run one flat chunk stream: the next chunk's barrier is
//     waited for and its first fragments loaded before the current chunk's
//     last k-step, also across tiles; no shared-memory tables, no CTA-wide
//     barrier after the start;
//   * the two consumer halves (wn = 0 / 1) start `skew` chunks apart (measured
//     neutral here: inside the 4-stage ring the halves drift apart on their own;
//     worth 8% on the one-CTA-per-tile stage-1 kernel of the two-stage path).
// Output modes per segment: 0 = target tiles (registers accumulate over the
// tile's entries, one ordered read-modify-write of the targets' rows at the
// end; a target column belongs to one tile: no atomics), 1 = pair entries
// (each entry's 64 columns written to their own rows, reduced per target by
// k_pair_reduce afterwards), 2 = stage 1 of the target-major two-stage low-rank
// path (each entry's 128 rows scattered to the pair targets' Y_T rows).  Target
// tiles keep the host<->device copy pipeline of tile_gemm_ws_kernel (per-tile
// slab needs, per-slab completion counters).
#pragma once
#include "tile_gemm_ws.cuh"

namespace cfm {

struct StepSeg {
  int start;              // first work item of the segment in the launch
  int tile_base;          // plan tile of that item
  int mode;               // 0 target tiles, 1 pair entries, 2 Y_T scatter
  int src_row0;           // subtracted from every source row id (tmap_b starts at that row)
  const int* tile_col;    // [tiles * 64] output columns (mode 2: the tile's source rows)
  const int* tile_off;    // [tiles + 1] entry range per tile (every tile has >= 1 entry)
  const int* entry_code;  // [E] transfer code (StepParams::code_op maps it) or operator id
  const int* entry_src;   // [E * 64] rows of tmap_b (-1: empty)
  double* y;              // mode 0: locals; 1: per-pair rows; 2: Y_T
  long long y_ld;
  double scale;
  // mode 2: row i of entry code c, source v -> y[nbr[v * nslots + (info >> 8)] + (info & 255)],
  // info = rowinfo[c * 128 + i] (-1: padding row; nbr -1: the source has no such pair)
  const int* rowinfo;
  const int* nbr;
  int nslots;
  int code_is_op;
  // copy pipeline (mode 0; null: off)
  const unsigned* pipe_mp;
  const unsigned* pipe_loc;
  unsigned* pipe_done;
  const int* pipe_need_mp;
  const int* pipe_need_loc;
  const int* pipe_lo;
  const int* pipe_hi;
  CUtensorMap tmap_a;  // operator stack of the segment
  CUtensorMap tmap_b;  // its source rows
};

constexpr int kStepMaxSegs = 16;
struct StepParams {
  int n_seg;
  int n_work;       // (tile, row block) items of the launch
  int nrb;          // row blocks of 128 result rows per tile
  int nk;           // inner length of an entry
  int nr;           // result rows
  int a_rows;       // rows per operator in the A stack
  int skew;         // chunks the odd consumer half starts behind the even one (0: off)
  const int* code_op;   // transfer code -> operator (segments with code_is_op == 0)
  unsigned* queue;      // work counter, zero at launch
  StepSeg seg[kStepMaxSegs];
};

constexpr int kStepStages = 4;
constexpr int kStepKC = 32;
constexpr int kStepThreads = 9 * 32;  // 8 consumer warps + the producer warp
constexpr int kStepRing = 8;          // posted work items
constexpr int step_gemm_smem_bytes() {
  return kStepStages * (128 + 64) * (kStepKC + 4) * 8 + 2 * kStepStages * 8 + kStepRing * 4;
}

// SCATTER: compile output mode 2 (two-stage launches); MPART: the last row block has dead m-tiles
// (128 - nr % 128 >= 8: l = 9), skipped per warp on a separate path, so the full row blocks keep the
// flat unrolled stream of the l = 5 launches.
template <bool SCATTER, bool MPART>
__global__ void __launch_bounds__(kStepThreads, 1) step_gemm_kernel(const __grid_constant__ StepParams p) {
  constexpr int BM = 128, BN = 64, KC = kStepKC, ST = kStepStages, LD = KC + 4;
  constexpr int WM = 4, NC = 8 * 32;
  constexpr int MT = 4, NTL = 4;  // 32 x 32 warp tiles
  extern __shared__ __align__(128) double smem_step[];
  double* As = smem_step;
  double* Bs = As + ST * BM * LD;
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + ST * BN * LD);
  uint64_t* empty = full + ST;
  volatile int* s_work = reinterpret_cast<volatile int*>(empty + ST);
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
  auto seg_of = [&](int w) {
    int si = 0;
    while (si + 1 < p.n_seg && w >= p.seg[si + 1].start) ++si;
    return si;
  };

  if (warp == NC / 32) {
    // ===================== producer: one lane, TMA only =====================
    if (lane != 0) return;
    constexpr unsigned STAGE_TX = unsigned((BM + BN) * LD * 8);
    int q = 0, wc = 0;
    for (;; ++wc) {
      const int w = int(atomicAdd(p.queue, 1u));
      if (w >= p.n_work) break;
      const StepSeg& sg = p.seg[seg_of(w)];
      const int tile = sg.tile_base + (w - sg.start) / p.nrb;
      const int r0 = ((w - sg.start) % p.nrb) * BM;
      const int e0 = __ldg(sg.tile_off + tile), e1 = __ldg(sg.tile_off + tile + 1);
      if (e0 == e1) {
        // a tile without entries (its slab counters still move): posted on an empty stage
        const int s = q % ST;
        if (q >= ST) mbar_wait_backoff(empty + s, ((q / ST) & 1) ^ 1);
        s_work[wc % kStepRing] = w;
        mbar_arrive(full + s);
        ++q;
        continue;
      }
      if (sg.pipe_mp) wait_flag_geq(sg.pipe_mp, unsigned(__ldg(sg.pipe_need_mp + tile)));
      for (int e = e0; e < e1; ++e) {
        int4 rows[BN / 4];
        const int4* srow = reinterpret_cast<const int4*>(sg.entry_src + (long long)e * BN);
#pragma unroll
        for (int j = 0; j < BN / 4; ++j) rows[j] = __ldg(srow + j);
        if (sg.src_row0) {
#pragma unroll
          for (int j = 0; j < BN / 4; ++j) {
            rows[j].x -= rows[j].x >= 0 ? sg.src_row0 : 0;
            rows[j].y -= rows[j].y >= 0 ? sg.src_row0 : 0;
            rows[j].z -= rows[j].z >= 0 ? sg.src_row0 : 0;
            rows[j].w -= rows[j].w >= 0 ? sg.src_row0 : 0;
          }
        }
        int op = __ldg(sg.entry_code + e);
        if (!sg.code_is_op) op = __ldg(p.code_op + op);
        const int arow = op * p.a_rows + r0;
        for (int kc = 0; kc < nch; ++kc, ++q) {
          const int s = q % ST;
          if (q >= ST) mbar_wait_backoff(empty + s, ((q / ST) & 1) ^ 1);
          if (e == e0 && kc == 0) s_work[wc % kStepRing] = w;  // published by the arrive below (release)
          mbar_arrive_expect_tx(full + s, STAGE_TX);
          tma_load_2d(As + s * BM * LD, &sg.tmap_a, kc * KC, arow, full + s);
          double* bs = Bs + s * BN * LD;
#pragma unroll
          for (int j = 0; j < BN / 4; ++j) tma_gather4(bs + 4 * j * LD, &sg.tmap_b, kc * KC, rows[j], full + s);
        }
      }
    }
    // end marker on an empty stage
    const int s = q % ST;
    if (q >= ST) mbar_wait_backoff(empty + s, ((q / ST) & 1) ^ 1);
    s_work[wc % kStepRing] = -1;
    mbar_arrive(full + s);
    return;
  }

  // ============================ consumer warps ============================
  // Interleaved warp tiles: warp (wm, wn) owns the m-tiles (mi * 4 + wm) * 8, so in a
  // partial last row block (l = 7: 87 of 128 rows) every SM sub-partition keeps
  // about the same number of live m-tiles; the dead ones are skipped.
  const int g = lane >> 2, tg = lane & 3;
  const int wm = warp % WM, wn = warp / WM;
  const int aoff = (wm * 8 + g) * LD + tg, boff = (wn * 32 + g) * LD + tg;
  constexpr int MSTEP = WM * 8;  // rows between a warp's m-tiles
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
    for (int mi = 0; mi < MT; ++mi) a[mi] = as[mi * MSTEP * LD + kk];
#pragma unroll
    for (int nj = 0; nj < NTL; ++nj) b[nj] = bs[nj * 8 * LD + kk];
  };
  auto mma = [&](const double* a, const double* b) {
#pragma unroll
    for (int mi = 0; mi < MT; ++mi)
#pragma unroll
      for (int nj = 0; nj < NTL; ++nj) dmma884(acc[mi][nj][0], acc[mi][nj][1], a[mi], b[nj]);
  };
  int q = 0, wc = 0;
  mbar_wait(full, 0);
  int w = s_work[0];
  if (w < 0) return;  // no work for this CTA (both halves see the same marker)
  const bool skewed = p.skew > 0 && p.skew < ST && p.skew < nch;
  if (skewed && wn == 1) asm volatile("bar.sync 2, %0;\n" ::"n"(NC) : "memory");
  bool arrived = false;
  load(a0, b0, 0, 0);
  while (w >= 0) {
    const StepSeg& sg = p.seg[seg_of(w)];
    const int tile = sg.tile_base + (w - sg.start) / p.nrb;
    const int r0 = ((w - sg.start) % p.nrb) * BM;
    const int e0 = __ldg(sg.tile_off + tile);
    const int total = (__ldg(sg.tile_off + tile + 1) - e0) * nch;
    const int mode = sg.mode;
    if (total == 0) {
      // empty tile: consume its empty stage, pick up the next chunk
      const int s = q % ST, s1 = (q + 1) % ST;
      mbar_wait(full + s1, ((q + 1) / ST) & 1);
      load(a0, b0, s1, 0);
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
      ++q;
    }
    int ml = MT;  // live m-tiles of this warp in this row block
    if (MPART) {
      ml = 0;
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
        if (r0 + (mi * WM + wm) * 8 < p.nr) ml = mi + 1;
    }
    if (MPART && ml < MT && total > 0) {
      // a partial row block: the same chunk stream over this warp's ML live m-tiles
      auto run_partial = [&](auto mlc) {
        constexpr int ML = decltype(mlc)::value;
        auto loadp = [&](double* a, double* b, int s, int kk) {
          const double* as = As + s * BM * LD + aoff;
          const double* bs = Bs + s * BN * LD + boff;
#pragma unroll
          for (int mi = 0; mi < ML; ++mi) a[mi] = as[mi * MSTEP * LD + kk];
#pragma unroll
          for (int nj = 0; nj < NTL; ++nj) b[nj] = bs[nj * 8 * LD + kk];
        };
        auto mmap = [&](const double* a, const double* b) {
#pragma unroll
          for (int mi = 0; mi < ML; ++mi)
#pragma unroll
            for (int nj = 0; nj < NTL; ++nj) dmma884(acc[mi][nj][0], acc[mi][nj][1], a[mi], b[nj]);
        };
        for (int c = 0; c < total; ++c, ++q) {
          const int s = q % ST;
          if (skewed && wn == 0 && !arrived && q >= p.skew) {
            asm volatile("bar.arrive 2, %0;\n" ::"n"(NC) : "memory");
            arrived = true;
          }
          const bool last_of_entry = (c + 1) % nch == 0;
#pragma unroll
          for (int kk = 0; kk < KC; kk += 8) {
            loadp(a1, b1, s, kk + 4);
            mmap(a0, b0);
            if (kk + 8 < KC) {
              loadp(a0, b0, s, kk + 8);
            } else {
              const int s1 = (q + 1) % ST;
              mbar_wait(full + s1, ((q + 1) / ST) & 1);
              load(a0, b0, s1, 0);  // (maybe another item's chunk: all m-tiles)
            }
            mmap(a1, b1);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(empty + s);
          if (mode == 1 && last_of_entry) {
            const int e = e0 + c / nch;
#pragma unroll
            for (int nj = 0; nj < NTL; ++nj)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const long long v = (long long)e * BN + wn * 32 + nj * 8 + 2 * tg + h;
                const bool live = __ldg(sg.entry_src + v) >= 0;
                double* dst = sg.y + v * sg.y_ld + r0 + wm * 8 + g;
#pragma unroll
                for (int mi = 0; mi < MT; ++mi) {
                  if (live && r0 + (mi * WM + wm) * 8 + g < p.nr) dst[mi * MSTEP] = sg.scale * acc[mi][nj][h];
                  acc[mi][nj][h] = 0.0;
                }
              }
          }
        }
      };
      if (ml == 3) run_partial(std::integral_constant<int, 3>{});
      else run_partial(std::integral_constant<int, 2>{});  // (rows past the operator are never stored)
    } else
    for (int c = 0; c < total; ++c, ++q) {
      const int s = q % ST;
      if (skewed && wn == 0 && !arrived && q >= p.skew) {
        asm volatile("bar.arrive 2, %0;\n" ::"n"(NC) : "memory");
        arrived = true;
      }
      const bool last_of_entry = (c + 1) % nch == 0;
      // the next chunk always exists (this tile's, the next item's first, or the
      // end marker's empty stage): it is waited for and its first fragments
      // loaded before this chunk's last k-step
#pragma unroll
      for (int kk = 0; kk < KC; kk += 8) {
        load(a1, b1, s, kk + 4);
        mma(a0, b0);
        if (kk + 8 < KC) {
          load(a0, b0, s, kk + 8);
        } else {
          const int s1 = (q + 1) % ST;
          mbar_wait(full + s1, ((q + 1) / ST) & 1);
          load(a0, b0, s1, 0);
        }
        mma(a1, b1);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
      if (mode != 0 && last_of_entry) {
        const int e = e0 + c / nch;
        if (mode == 1) {
          // pair entries: the entry's 64 columns are 64 (target, source) pairs,
          // written to rows e * 64 + c of the per-pair buffer
#pragma unroll
          for (int nj = 0; nj < NTL; ++nj)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const long long v = (long long)e * BN + wn * 32 + nj * 8 + 2 * tg + h;
              const bool live = __ldg(sg.entry_src + v) >= 0;
              double* dst = sg.y + v * sg.y_ld + r0 + wm * 8 + g;
#pragma unroll
              for (int mi = 0; mi < MT; ++mi) {
                if (live && r0 + (mi * WM + wm) * 8 + g < p.nr) dst[mi * MSTEP] = sg.scale * acc[mi][nj][h];
                acc[mi][nj][h] = 0.0;
              }
            }
        } else if (SCATTER) {
          // Y_T scatter: each (slot, a) row of every source goes to the Y_T row
          // of the pair's target (the 8 lanes of a tg mostly share a slot: one
          // broadcast load, a run of up to 64 B stored)
          const int* ri = sg.rowinfo + (long long)__ldg(sg.entry_code + e) * BM + wm * 8 + g;
          int info[MT];
#pragma unroll
          for (int mi = 0; mi < MT; ++mi) info[mi] = __ldg(ri + mi * MSTEP);
#pragma unroll
          for (int nj = 0; nj < NTL; ++nj)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int v = __ldg(sg.tile_col + (long long)tile * BN + wn * 32 + nj * 8 + 2 * tg + h);
              const int* nb = sg.nbr + (long long)v * sg.nslots;
              int dst[MT];
#pragma unroll
              for (int mi = 0; mi < MT; ++mi) dst[mi] = (v >= 0 && info[mi] >= 0) ? __ldg(nb + (info[mi] >> 8)) : -1;
#pragma unroll
              for (int mi = 0; mi < MT; ++mi) {
                if (dst[mi] >= 0) sg.y[(long long)dst[mi] + (info[mi] & 255)] = acc[mi][nj][h];
                acc[mi][nj][h] = 0.0;
              }
            }
        }
      }
    }
    if (mode == 0) {
      // ordered, atomic-free accumulate: a target column belongs to one tile
      if (sg.pipe_loc && total) wait_flag_geq(sg.pipe_loc, sg.pipe_need_loc ? unsigned(__ldg(sg.pipe_need_loc + tile)) : 1u);
      if (total)
#pragma unroll
      for (int nj = 0; nj < NTL; ++nj)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int v = __ldg(sg.tile_col + (long long)tile * BN + wn * 32 + nj * 8 + 2 * tg + h);
          double* dst = sg.y + (long long)v * sg.y_ld + r0 + wm * 8 + g;
          double old[MT];
#pragma unroll
          for (int mi = 0; mi < MT; ++mi) old[mi] = (v >= 0 && r0 + (mi * WM + wm) * 8 + g < p.nr) ? dst[mi * MSTEP] : 0.0;
#pragma unroll
          for (int mi = 0; mi < MT; ++mi) {
            if (v >= 0 && r0 + (mi * WM + wm) * 8 + g < p.nr) dst[mi * MSTEP] = old[mi] + sg.scale * acc[mi][nj][h];
            acc[mi][nj][h] = 0.0;
          }
        }
      if (sg.pipe_done) {
        // every consumer's rows are visible device-wide before the slab counters move
        __threadfence();
        asm volatile("bar.sync 1, %0;\n" ::"n"(NC) : "memory");
        if (tid == 0)
          for (int k = __ldg(sg.pipe_lo + tile); k <= __ldg(sg.pipe_hi + tile); ++k) atomicAdd(sg.pipe_done + k, 1u);
      }
    }
    ++wc;
    w = s_work[wc % kStepRing];  // posted before the stage this warp already waited for
  }
  if (skewed && wn == 0 && !arrived) asm volatile("bar.arrive 2, %0;\n" ::"n"(NC) : "memory");  // (only empty tiles)
}

}  // namespace cfm
