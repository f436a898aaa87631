// Fused low-rank M2L tile kernel (ia / iasym / iablk), warp-specialized.
//
// Reference: LowRankFactors.apply (lowrank.py:43-44) inside the symmetric
// apply (m2l.py:353-362) and its blocked flush (m2l.py:425):
//     out = left @ (right^H @ w[inv]);  acc += out[table]
// Per tile entry (one transfer vector, 64 columns) the CTA computes
//     phase 1:  Y[a, c]  = sum_k rightH[a, k] * X[src_c, inv[k]]      (a < rank)
//     phase 2:  acc[i, c] += sum_a left[table[i], a] * Y[a, c]
// with Y kept in shared memory (double-buffered, one named barrier per entry),
// so per-pair intermediates never touch HBM.  Producer warps stream phase-1
// chunks (rightH rows + gathered permuted sources) and phase-2 chunks (the
// row-gathered left factor) through one cp.async/mbarrier ring; consumer
// warps run mma.sync.m8n8k4.f64 (DMMA) for both phases.
#pragma once
#include <type_traits>

#include "tile_gemm_ws.cuh"

namespace cfm {

struct LowRankParams {
  // plan (same layout as TileParams)
  int n_tiles;
  int tile_base;
  const int* tile_col;
  const int* tile_off;
  const int* entry_code;
  const int* entry_src;
  const int* code_op;
  const int* code_rperm;  // row table id for phase 2 (-1 identity)
  const int* code_cperm;  // inverse table id for phase 1 (-1 identity)
  // factors: rightH op o = vh + o * vh_stride (RP rows x vh_ld), left op o = u + o * u_stride (nr rows x u_ld)
  const double* vh;
  long long vh_stride;
  int vh_ld;
  const double* u;
  long long u_stride;
  int u_ld;
  const int* rank;  // per op (realified)
  int n_ops;        // <= 344
  int nr, nk;
  const short* rowtab;
  const short* invtab;
  const double* x;
  long long x_ld;
  int x_dc;
  double* y;
  long long y_ld;
  int y_dc;
  double scale;
  int accumulate;
  int pair_out;
  int tabs_smem;  // host decided the 48 permutation tables fit in shared memory
};

template <int RP, int KC, int STAGES>
constexpr int lr_smem_bytes() {
  // ring: A region (128 rows, both phases) + B region (64 cols, phase 1); Y double buffer; barriers
  return STAGES * (128 + 64) * (KC + 4) * 8 + 4 * 64 * (RP + 4) * 8 + 2 * STAGES * 8 + 4 * 344;
}

// VB: sources are contiguous zero-padded rows and the factors are the
// per-transfer permuted ones (no permutation in the copies): B is staged with
// 16-B cp.async pieces instead of 8-B element gathers.
template <int RP, int KC, int STAGES, bool VB = false>
__global__ void __launch_bounds__(12 * 32, 1) lowrank_ws_kernel(const __grid_constant__ LowRankParams p) {
  constexpr int BM = 128, BN = 64, WM = 4, WN = 2;
  constexpr int NC = 8 * 32, NP = 4 * 32;
  constexpr int WTM = BM / WM, WTN = BN / WN;  // phase-2 warp tile 32 x 32
  constexpr int MT = WTM / 8, NTL = WTN / 8;
  constexpr int MT1 = RP / 8;                  // phase-1 m-tiles (each warp: all RP rows x 8 columns)
  constexpr int LDA = KC + 4, LDB = KC + 4, LDY = RP + 4;
  constexpr int A1_PIECES = RP * (KC / 2), A2_PIECES = BM * (KC / 2);
  constexpr int B_PER_T = VB ? BN * KC / 2 / NP : BN * KC / NP;  // 16-B pieces (VB) or 8-B elements per thread
  constexpr int B_TPC = VB ? KC / 2 : KC;                          // threads per column
  static_assert(A1_PIECES % NP == 0 && A2_PIECES % NP == 0 && (BN * KC) % NP == 0, "mapping");
  static_assert(NP % KC == 0, "B mapping");
  static_assert(RP % 8 == 0 && RP <= 64, "rank pad");

  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = As + STAGES * BM * LDA;
  double* Ys = Bs + STAGES * BN * LDB;  // [2 buffers][2 k-groups][BN][LDY] partial Y
  uint64_t* full = reinterpret_cast<uint64_t*>(Ys + 4 * BN * LDY);
  uint64_t* empty = full + STAGES;
  int* s_rank = reinterpret_cast<int*>(empty + STAGES);
  int* s_col = s_rank + 344;
  int* s_op = s_col + 64;
  int* s_rp = s_op + 344;
  int* s_cp = s_rp + 344;
  int* s_ecode = s_cp + 344;
  short* s_rowtab = reinterpret_cast<short*>(s_ecode + kMaxTileEntries);
  const bool tabs_in_smem = p.tabs_smem != 0;
  short* s_invtab = s_rowtab + 48 * p.nr + 8;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int tile = p.tile_base + int(blockIdx.x);
  const int r0 = blockIdx.y * BM;
  const int e_begin = p.tile_off[tile], e_end = p.tile_off[tile + 1];

  for (int c = tid; c < BN; c += NC + NP) s_col[c] = p.tile_col[(long long)tile * BN + c];
  for (int c = tid; c < 343; c += NC + NP) {
    s_op[c] = p.code_op[c];
    s_rp[c] = p.code_rperm[c];
    s_cp[c] = p.code_cperm[c];
  }
  for (int c = tid; c < p.n_ops; c += NC + NP) s_rank[c] = min(p.rank[c], RP);
  const int n_cached = min(e_end - e_begin, kMaxTileEntries);
  for (int i = tid; i < n_cached; i += NC + NP) s_ecode[i] = p.entry_code[e_begin + i];
  if (tabs_in_smem) {
    for (int i = tid; i < 48 * p.nr; i += NC + NP) s_rowtab[i] = p.rowtab[i];
    for (int i = tid; i < 48 * p.nk; i += NC + NP) s_invtab[i] = p.invtab[i];
  }
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, NP);
      mbar_init(empty + s, NC / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const short* rowtab = tabs_in_smem ? s_rowtab : p.rowtab;
  const short* invtab = tabs_in_smem ? s_invtab : p.invtab;
  auto code_of = [&](int e) -> int {
    const int i = e - e_begin;
    return i < kMaxTileEntries ? s_ecode[i] : __ldg(p.entry_code + e);
  };
  struct LInfo {
    int op, rperm, cperm, rank, n1, n2;
  };
  auto decode = [&](int e) -> LInfo {
    LInfo d;
    const int code = code_of(e);
    d.op = s_op[code];
    d.rperm = s_rp[code];
    d.cperm = s_cp[code];
    d.rank = d.op >= 0 ? s_rank[d.op] : 0;
    d.n1 = d.rank > 0 ? (p.nk + KC - 1) / KC : 0;
    d.n2 = d.rank > 0 ? (d.rank + KC - 1) / KC : 0;
    return d;
  };
  auto next_live = [&](int e, LInfo& d) -> int {
    while (e < e_end) {
      d = decode(e);
      if (d.n1) break;
      ++e;
    }
    return e;
  };

  if (tid >= NC) {
    // ======================= producer warps =======================
    const int pt = tid - NC;
    LInfo d;
    int e = next_live(e_begin, d);
    int q = 0;
    // source columns of the next entry are fetched one entry ahead
    int nsrc[B_PER_T];
    auto fetch_src = [&](int ee) {
#pragma unroll
      for (int u = 0; u < B_PER_T; ++u)
        nsrc[u] = ee < e_end ? __ldg(p.entry_src + (long long)ee * BN + pt / B_TPC + u * (NP / B_TPC)) : -1;
    };
    fetch_src(e);
    while (e < e_end) {
      const double* vbase = p.vh + (long long)d.op * p.vh_stride;
      const double* ubase = p.u + (long long)d.op * p.u_stride;
      const double* bcol[B_PER_T];
#pragma unroll
      for (int u = 0; u < B_PER_T; ++u) {
        const int v = nsrc[u];
        bcol[u] = (v >= 0) ? p.x + (long long)(v / p.x_dc) * p.x_ld + (v % p.x_dc) : nullptr;
      }
      LInfo dn;
      const int en = next_live(e + 1, dn);
      fetch_src(en);
      // phase 1 chunks: rightH rows (a < rank) and gathered sources
      for (int kc = 0; kc < d.n1; ++kc, ++q) {
        const int s = q % STAGES;
        if (q >= STAGES) mbar_wait_backoff(empty + s, ((q / STAGES) & 1) ^ 1);
        const int k0 = kc * KC;
        double* as = As + s * BM * LDA;
        double* bs = Bs + s * BN * LDB;
#pragma unroll
        for (int u = 0; u < A1_PIECES / NP; ++u) {
          const int id = pt + u * NP;
          const int a = id / (KC / 2), kp = id % (KC / 2);
          const bool ok = a < d.rank;
          cp_async16(as + a * LDA + 2 * kp, ok ? (const void*)(vbase + (long long)a * p.vh_ld + k0 + 2 * kp)
                                               : (const void*)p.vh, ok);
        }
        if (VB) {
          const int kp = pt % B_TPC;
          const bool kvalid = k0 + 2 * kp < p.nk;  // (the pair past n reads a zero pad element)
#pragma unroll
          for (int u = 0; u < B_PER_T; ++u) {
            const int c = pt / B_TPC + u * (NP / B_TPC);
            const bool ok = kvalid && bcol[u] != nullptr;
            cp_async16(bs + c * LDB + 2 * kp, ok ? (const void*)(bcol[u] + k0 + 2 * kp) : (const void*)p.vh, ok);
          }
        } else {
          const int kk = pt % KC;
          const int k = k0 + kk;
          const bool kvalid = k < p.nk;
          int j = k;
          if (kvalid && d.cperm >= 0) j = invtab[d.cperm * p.nk + k];
#pragma unroll
          for (int u = 0; u < B_PER_T; ++u) {
            const int c = pt / KC + u * (NP / KC);
            const bool ok = kvalid && bcol[u] != nullptr;
            cp_async8(bs + c * LDB + kk, ok ? (const void*)(bcol[u] + (long long)p.x_dc * j) : (const void*)p.vh, ok);
          }
        }
        mbar_cp_async_arrive(full + s);
      }
      // phase 2 chunks: left rows gathered by the row table, columns a < rank
      int orow[A2_PIECES / NP];
#pragma unroll
      for (int u = 0; u < A2_PIECES / NP; ++u) {
        const int id = pt + u * NP;
        const int i = id / (KC / 2);
        const int gr = r0 + i;
        orow[u] = gr < p.nr ? (d.rperm >= 0 ? rowtab[d.rperm * p.nr + gr] : gr) : -1;
      }
      for (int kc = 0; kc < d.n2; ++kc, ++q) {
        const int s = q % STAGES;
        if (q >= STAGES) mbar_wait_backoff(empty + s, ((q / STAGES) & 1) ^ 1);
        const int k0 = kc * KC;
        double* as = As + s * BM * LDA;
#pragma unroll
        for (int u = 0; u < A2_PIECES / NP; ++u) {
          const int id = pt + u * NP;
          const int i = id / (KC / 2), kp = id % (KC / 2);
          const bool ok = orow[u] >= 0;
          cp_async16(as + i * LDA + 2 * kp,
                     ok ? (const void*)(ubase + (long long)orow[u] * p.u_ld + k0 + 2 * kp) : (const void*)p.u, ok);
        }
        mbar_cp_async_arrive(full + s);
      }
      e = en;
      d = dn;
    }
    cp_async_wait<0>();
    return;
  }

  // ======================= consumer warps =======================
  const int g = lane >> 2, tg = lane & 3;
  const int wm = warp % WM, wn = warp / WM;
  double acc[MT][NTL][2];
#pragma unroll
  for (int mi = 0; mi < MT; ++mi)
#pragma unroll
    for (int nj = 0; nj < NTL; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;

  LInfo d;
  int e = next_live(e_begin, d);
  int q = 0;
  // phase-1 layout: warp = (k-group kg in {0,1}) x (column group cg of 16 columns);
  // kg takes every other k-step, partial sums land in Yp[kg] and are added in a
  // fixed order when phase 2 reads them (deterministic, no atomics)
  const int kg = warp >> 2, cg = warp & 3;
  int ybuf = 0;
  while (e < e_end) {
    double* yp0 = Ys + ybuf * 2 * BN * LDY;
    double* yp1 = yp0 + BN * LDY;
    // ---- phase 1: Y (rank x 64), specialized on the live m-tiles (no predicated MMAs)
    double yacc[MT1][2][2];
#pragma unroll
    for (int mi = 0; mi < MT1; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) yacc[mi][nj][0] = yacc[mi][nj][1] = 0.0;
    const int mlive = (d.rank + 7) / 8;
    auto phase1 = [&](auto live_c) {
      constexpr int ML = decltype(live_c)::value;
      for (int kc = 0; kc < d.n1; ++kc, ++q) {
        const int s = q % STAGES;
        mbar_wait(full + s, (q / STAGES) & 1);
        const double* as = As + s * BM * LDA + g * LDA + tg;
        const double* bs = Bs + s * BN * LDB + (cg * 16 + g) * LDB + tg;
        const int kmax = min(KC, p.nk - kc * KC);
#pragma unroll
        for (int kk = kg * 4; kk < KC; kk += 8) {
          if (kk < kmax) {
            const double b0 = bs[kk], b1 = bs[8 * LDB + kk];
            double a[ML];
#pragma unroll
            for (int mi = 0; mi < ML; ++mi) a[mi] = as[mi * 8 * LDA + kk];
#pragma unroll
            for (int mi = 0; mi < ML; ++mi) {
              dmma884(yacc[mi][0][0], yacc[mi][0][1], a[mi], b0);
              dmma884(yacc[mi][1][0], yacc[mi][1][1], a[mi], b1);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
      }
    };
    if (mlive <= 1) phase1(std::integral_constant<int, 1>{});
    else if (mlive == 2) phase1(std::integral_constant<int, 2>{});
    else if (mlive == 3 || MT1 < 4) phase1(std::integral_constant<int, (MT1 < 3 ? MT1 : 3)>{});
    else if (mlive <= 4 || MT1 <= 4) phase1(std::integral_constant<int, (MT1 < 4 ? MT1 : 4)>{});
    else phase1(std::integral_constant<int, MT1>{});
    // partial Y -> smem as the phase-2 B operand layout: Yp[kg][col][a]
    double* yp = kg ? yp1 : yp0;
#pragma unroll
    for (int mi = 0; mi < MT1; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj)
#pragma unroll
        for (int h = 0; h < 2; ++h) yp[(cg * 16 + nj * 8 + 2 * tg + h) * LDY + mi * 8 + g] = yacc[mi][nj][h];
    // one barrier per entry: Yp[ybuf] complete; also every warp has finished the
    // previous entry's phase 2, so Yp[ybuf ^ 1] may be overwritten next entry
    asm volatile("bar.sync 1, %0;\n" ::"n"(NC) : "memory");
    // ---- phase 2: acc += left[table] (128 x rank) * (Yp0 + Yp1) (rank x 64)
    for (int kc = 0; kc < d.n2; ++kc, ++q) {
      const int s = q % STAGES;
      mbar_wait(full + s, (q / STAGES) & 1);
      const double* as = As + s * BM * LDA + (wm * WTM + g) * LDA + tg;
      const int yoff = (wn * WTN + g) * LDY + kc * KC + tg;
      const int kmax = min(KC, d.rank - kc * KC);
#pragma unroll 2
      for (int kk = 0; kk < kmax; kk += 4) {
        double a[MT], b[NTL];
#pragma unroll
        for (int mi = 0; mi < MT; ++mi) a[mi] = as[mi * 8 * LDA + kk];
#pragma unroll
        for (int nj = 0; nj < NTL; ++nj) b[nj] = yp0[yoff + nj * 8 * LDY + kk] + yp1[yoff + nj * 8 * LDY + kk];
#pragma unroll
        for (int mi = 0; mi < MT; ++mi)
#pragma unroll
          for (int nj = 0; nj < NTL; ++nj) dmma884(acc[mi][nj][0], acc[mi][nj][1], a[mi], b[nj]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
    }
    ybuf ^= 1;
    if (p.pair_out) {
#pragma unroll
      for (int mi = 0; mi < MT; ++mi) {
        const int row = r0 + wm * WTM + mi * 8 + g;
#pragma unroll
        for (int nj = 0; nj < NTL; ++nj) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = wn * WTN + nj * 8 + 2 * tg + h;
            if (row < p.nr && __ldg(p.entry_src + (long long)e * BN + c) >= 0) {
              const long long v = (long long)e * BN + c;
              double* dst = p.y + (v / p.y_dc) * p.y_ld + (v % p.y_dc) + (long long)p.y_dc * row;
              const double val = p.scale * acc[mi][nj][h];
              if (p.accumulate)
                *dst += val;
              else
                *dst = val;
            }
            acc[mi][nj][h] = 0.0;
          }
        }
      }
    }
    e = next_live(e + 1, d);
  }
  if (p.pair_out) return;
  if (e_begin == e_end && p.accumulate) return;
#pragma unroll
  for (int mi = 0; mi < MT; ++mi) {
    const int row = r0 + wm * WTM + mi * 8 + g;
    if (row >= p.nr) continue;
#pragma unroll
    for (int nj = 0; nj < NTL; ++nj) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = wn * WTN + nj * 8 + 2 * tg + h;
        const int v = s_col[c];
        if (v < 0) continue;
        double* dst = p.y + (long long)(v / p.y_dc) * p.y_ld + (v % p.y_dc) + (long long)p.y_dc * row;
        const double val = p.scale * acc[mi][nj][h];
        if (p.accumulate)
          *dst += val;
        else
          *dst = val;
      }
    }
  }
}

}  // namespace cfm
