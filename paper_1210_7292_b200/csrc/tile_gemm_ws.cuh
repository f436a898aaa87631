// Warp-specialized variant of tile_gemm_kernel (same math, same plan).
//
// 4 producer warps walk the tile's (entry, K-chunk) stream and issue the
// cp.async gathers (operator rows by the row table, source columns by the
// inverse table); each producer thread signals the stage's "full" mbarrier
// with cp.async.mbarrier.arrive.noinc when its copies land.  8 consumer warps
// wait on "full", run the LDS -> DMMA.8x8x4 loop on the stage and release it
// on the "empty" mbarrier.  There is no CTA-wide barrier in the main loop, so
// the consumer warps keep the FP64 tensor pipe fed while the producers run
// STAGES-1 chunks ahead.
#pragma once
#include <type_traits>

#include "tile_gemm.cuh"

namespace cfm {

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_cp_async_arrive(uint64_t* bar) {
  unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(a), "r"(bytes)
               : "memory");
}
// TMA bulk copy global -> shared, completion counted on an mbarrier (bytes).
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, uint64_t* bar) {
  unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(d),
               "l"(gmem), "r"(bytes), "r"(b)
               : "memory");
}

// 2-D TMA tile copy global -> shared (box from the tensor map), bytes on an mbarrier.
__device__ __forceinline__ void tma_load_2d(void* smem, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(d), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(b)
      : "memory");
}

// L2 eviction-priority policies for TMA copies (createpolicy): operator tiles
// are re-read by every tile of a level and should stay L2-resident; source rows
// stream through.
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_2d_hint(void* smem, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                                 uint64_t pol) {
  unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(d),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(b), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_gather4_hint(void* smem, const CUtensorMap* map, int c0, int4 r, uint64_t* bar,
                                                 uint64_t pol) {
  unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;\n" ::"r"(d),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(b), "l"(pol)
      : "memory");
}

// 2-D TMA tile::gather4: rows r.x..r.w of the map, columns [c0, c0 + box), landing
// back to back in shared memory (4 x box doubles), bytes on an mbarrier.
__device__ __forceinline__ void tma_gather4(void* smem, const CUtensorMap* map, int c0, int4 r, uint64_t* bar) {
  unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(d),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(b)
      : "memory");
}

__device__ __forceinline__ bool mbar_try(uint64_t* bar, unsigned parity) {
  unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  unsigned ok;
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
  return ok != 0;
}
// Producer-side wait with exponential nanosleep backoff: a spinning producer
// warp would steal issue slots from the DMMA consumer warps of its SMSP.
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, unsigned parity) {
  unsigned ns = 32;
  while (!mbar_try(bar, parity)) {
    __nanosleep(ns);
    ns = ns < 512 ? ns * 2 : 512;
  }
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

template <int BM, int BN, int KC, int STAGES>
constexpr int ws_ring_bytes() {
  return STAGES * (BM + BN) * (KC + 4) * 8 + 2 * STAGES * 8;
}

// Several independent tile lists (e.g. all octree levels of one M2L step) in
// one launch: tiles [start[s], start[s+1]) of the launch belong to segment s.
// CTA b works on tile b / nrb, row block b % nrb: the row blocks of a tile run
// side by side and share its source columns in L2.
constexpr int kMaxSegments = 16;  // (config 4: 6 levels + 4 short-tile lists + 4 hybrid pair lists + the merged pair plan = 15)
struct MultiTileParams {
  int n_seg;
  int nrb;  // row blocks per tile
  int start[kMaxSegments + 1];
  TileParams seg[kMaxSegments];
};

// FTM: 0 = permuted-gather staging, 1 = full-operator TMA staging, 2 = full-operator
// TMA staging with interleaved warp tiles that skip rows past the operator and
// empty trailing columns of pair entries (used when a launch has either)
template <int BM, int BN, int WM, int WN, int KC, int STAGES, bool SKIP_ROWS, bool BULK_A = false, int FTM = 0>
__global__ void __launch_bounds__((WM * WN + 4) * 32, 1) tile_gemm_ws_kernel(const __grid_constant__ MultiTileParams mp) {
  constexpr bool FT = FTM != 0;
  constexpr bool IL = FTM == 2;
  int sidx = 0;
  const int ltile = int(blockIdx.x) / mp.nrb;
  while (sidx + 1 < mp.n_seg && ltile >= mp.start[sidx + 1]) ++sidx;
  const TileParams& p = mp.seg[sidx];
  constexpr int NC = WM * WN * 32;  // consumer threads
  constexpr int NP = 4 * 32;        // producer threads
  constexpr int WTM = BM / WM, WTN = BN / WN;
  constexpr int MT = WTM / 8, NTL = WTN / 8;
  constexpr int LDA = KC + 4, LDB = KC + 4;
  constexpr int A_PIECES = BM * (KC / 2);
  constexpr int A_PER_T = A_PIECES / NP;
  constexpr int B_ELEMS = BN * KC;
  constexpr int B_PER_T = B_ELEMS / NP;
  static_assert(A_PIECES % NP == 0 && B_ELEMS % NP == 0, "tile/thread mismatch");
  static_assert(NP % KC == 0, "B mapping needs NP multiple of KC");
  static_assert(BN <= 64, "s_col sized for 64 columns");
  static_assert(!BULK_A || BM == NP, "bulk A path: one operator row per producer thread");
  static_assert(!FT || (BN % 32 == 0 && !BULK_A), "full-operator path: whole B columns per lane");

  extern __shared__ __align__(128) double smem_ws[];  // TMA tile destinations need 128-B alignment
  double* As = smem_ws;
  double* Bs = As + STAGES * BM * LDA;
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + STAGES * BN * LDB);
  uint64_t* empty = full + STAGES;
  int* s_col = reinterpret_cast<int*>(empty + STAGES);
  int* s_op = s_col + 64;
  int* s_rp = s_op + 344;
  int* s_cp = s_rp + 344;
  int* s_ecode = s_cp + 344;
  short* s_rowtab = reinterpret_cast<short*>(s_ecode + kMaxTileEntries);
  unsigned char* s_encols = reinterpret_cast<unsigned char*>(s_rowtab);  // full-operator mode (no perm tables)
  const bool tabs_in_smem = tile_perm_tabs_fit(p.nr, p.nk);
  short* s_invtab = s_rowtab + 48 * p.nr + 8;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int tile = p.tile_base + ltile - mp.start[sidx];
  const int r0 = (int(blockIdx.x) % mp.nrb) * BM;
  const int e_begin = p.tile_off[tile], e_end = p.tile_off[tile + 1];

  for (int c = tid; c < BN; c += NC + NP) s_col[c] = p.tile_col[(long long)tile * BN + c];
  if (!p.code_is_op) {
    for (int c = tid; c < 343; c += NC + NP) {
      s_op[c] = p.code_op[c];
      s_rp[c] = p.code_rperm[c];
      s_cp[c] = p.code_cperm[c];
    }
  }
  const int n_cached = min(e_end - e_begin, kMaxTileEntries);
  for (int i = tid; i < n_cached; i += NC + NP) s_ecode[i] = p.entry_code[e_begin + i];
  if (IL && p.entry_ncols)
    for (int i = tid; i < n_cached; i += NC + NP) s_encols[i] = p.entry_ncols[e_begin + i];
  if (tabs_in_smem) {
    if (p.rowtab)
      for (int i = tid; i < 48 * p.nr; i += NC + NP) s_rowtab[i] = p.rowtab[i];
    if (p.invtab)
      for (int i = tid; i < 48 * p.nk; i += NC + NP) s_invtab[i] = p.invtab[i];
  }
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, FT ? 1 : (BULK_A ? NP + 1 : NP));
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
  auto next_live = [&](int e, EntryInfo& d) -> int {
    while (e < e_end) {
      d = decode_code<KC>(p, code_of(e), s_op, s_rp, s_cp, r0);
      if (d.nchunks) break;
      ++e;
    }
    return e;
  };

  if (FT && tid >= NC) {
    // ============ producer, full-operator mode: one warp, TMA only ============
    // per chunk: one 2-D tile copy of the operator block (BM rows x KC+4
    // columns, landing with the LDA pitch) and BN/4 tile::gather4 copies of
    // the source rows (4 rows x KC+4 columns each, landing with the LDB pitch;
    // empty slots carry row -1, out of bounds, and arrive as zeros).  Lane 0
    // issues everything; the entry's source rows are read once per entry.
    if (tid >= NC + 32) return;
    if (p.pipe_mp && e_begin < e_end) wait_flag_geq(p.pipe_mp, unsigned(p.pipe_need_mp[tile]));
    if (lane != 0) return;
    static_assert(BN % 4 == 0 && LDA == LDB, "gather4 rows land with the A pitch");
    constexpr unsigned STAGE_TX = unsigned((BM * LDA + BN * LDB) * 8);
    const uint64_t pol_a = l2_policy_evict_last();
    const uint64_t pol_b = (p.l2_hints & 4) ? l2_policy_evict_last() : l2_policy_evict_first();
    EntryInfo d;
    d.nchunks = 0;
    int e = next_live(e_begin, d);
    int q = 0;
    while (e < e_end) {
      int4 rows[BN / 4];
      const int4* srow = reinterpret_cast<const int4*>(p.entry_src + (long long)e * BN);
      if (!p.b_block) {
#pragma unroll
        for (int j = 0; j < BN / 4; ++j) rows[j] = __ldg(srow + j);
        if (p.x_row0) {
#pragma unroll
          for (int j = 0; j < BN / 4; ++j) {
            rows[j].x -= rows[j].x >= 0 ? p.x_row0 : 0;
            rows[j].y -= rows[j].y >= 0 ? p.x_row0 : 0;
            rows[j].z -= rows[j].z >= 0 ? p.x_row0 : 0;
            rows[j].w -= rows[j].w >= 0 ? p.x_row0 : 0;
          }
        }
      }
      const int arow = (d.op >> p.ft_opshift) * p.ft_rows + r0;
      const int acol = (d.op & ((1 << p.ft_opshift) - 1)) * p.ft_colseg;
      for (int kc = 0; kc < d.nchunks; ++kc, ++q) {
        const int s = q % STAGES;
        if (q >= STAGES) mbar_wait_backoff(empty + s, ((q / STAGES) & 1) ^ 1);
        const int k0 = kc * KC;
        double* bs = Bs + s * BN * LDB;
        if (CFM_DEBUG(p) & (4 | 32 | 64)) {
          // timing experiments only (stale stage data): debug 4 no copies,
          // 32 no source gathers, 64 no operator tile
          if (CFM_DEBUG(p) & 4) {
            mbar_arrive(full + s);
          } else if (CFM_DEBUG(p) & 32) {
            mbar_arrive_expect_tx(full + s, unsigned(BM * LDA * 8));
            tma_load_2d(As + s * BM * LDA, &p.tmap_a, acol + k0, arow, full + s);
          } else {
            mbar_arrive_expect_tx(full + s, unsigned(BN * LDB * 8));
#pragma unroll
            for (int j = 0; j < BN / 4; ++j) tma_gather4(bs + 4 * j * LDB, &p.tmap_b, k0, rows[j], full + s);
          }
          continue;
        }
        mbar_arrive_expect_tx(full + s, STAGE_TX);
        // l2_hints bit 0: operator tiles evict_last; bit 1: sources evict_first;
        // bit 2: sources evict_last (experiments; 0 = no policy)
        if (p.l2_hints & 1)
          tma_load_2d_hint(As + s * BM * LDA, &p.tmap_a, acol + k0, arow, full + s, pol_a);
        else
          tma_load_2d(As + s * BM * LDA, &p.tmap_a, acol + k0, arow, full + s);
        if (p.l2_hints & 6) {
          if (p.b_block) {
            tma_load_2d_hint(bs, &p.tmap_b, k0, e * BN, full + s, pol_b);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 4; ++j) tma_gather4_hint(bs + 4 * j * LDB, &p.tmap_b, k0, rows[j], full + s, pol_b);
          }
        } else {
          if (p.b_block) {
            tma_load_2d(bs, &p.tmap_b, k0, e * BN, full + s);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 4; ++j) tma_gather4(bs + 4 * j * LDB, &p.tmap_b, k0, rows[j], full + s);
          }
        }
      }
      e = next_live(e + 1, d);
    }
    return;
  }
  if (tid >= NC) {
    // ======================= producer warps =======================
    const int pt = tid - NC;
    if (p.pipe_mp && e_begin < e_end) wait_flag_geq(p.pipe_mp, unsigned(p.pipe_need_mp[tile]));
    EntryInfo d;
    d.nchunks = 0;
    int e = next_live(e_begin, d);
    int q = 0;
    int nxt_src[B_PER_T];
    int nxt_e = -1;
    auto prefetch_src = [&](int ee) {
      nxt_e = ee;
      if (ee < e_end) {
#pragma unroll
        for (int u = 0; u < B_PER_T; ++u)
          nxt_src[u] = __ldg(p.entry_src + (long long)ee * BN + pt / KC + u * (NP / KC));
      }
    };
    const double* a_row[A_PER_T];
    bool a_ok[A_PER_T];
    const double* a_rowb[BM / NP > 0 ? BM / NP : 1];
    const double* b_col[B_PER_T];
    while (e < e_end) {
      // per-entry pointers
      const double* opbase = p.ops + (long long)d.op * p.op_stride;
#pragma unroll
      for (int u = 0; u < A_PER_T; ++u) {
        const int id = pt + u * NP;
        const int i = id / (KC / 2), kp = id % (KC / 2);
        const int gr = r0 + i;
        a_ok[u] = gr < d.rows;
        int orow = gr;
        if (a_ok[u] && d.rperm >= 0) orow = rowtab[d.rperm * p.nr + gr];
        a_row[u] = opbase + (long long)(a_ok[u] ? orow : 0) * p.op_ld + 2 * kp;
      }
      if (BULK_A) {
#pragma unroll
        for (int u = 0; u < BM / NP; ++u) {
          const int gr = r0 + pt + u * NP;
          const bool ok = gr < d.rows;
          int orow = gr;
          if (ok && d.rperm >= 0) orow = rowtab[d.rperm * p.nr + gr];
          a_rowb[u] = ok ? opbase + (long long)orow * p.op_ld : p.zero_row;
        }
      }
      if (nxt_e != e) prefetch_src(e);
#pragma unroll
      for (int u = 0; u < B_PER_T; ++u) {
        const int v = nxt_src[u];
        b_col[u] = (v >= 0) ? p.x + (long long)(v / p.x_dc) * p.x_ld + (v % p.x_dc) : nullptr;
      }
      prefetch_src(e + 1);
      for (int kc = 0; kc < d.nchunks; ++kc, ++q) {
        const int s = q % STAGES;
        if (q >= STAGES) {
          if (CFM_DEBUG(p) & 2)
            mbar_wait(empty + s, ((q / STAGES) & 1) ^ 1);
          else
            mbar_wait_backoff(empty + s, ((q / STAGES) & 1) ^ 1);
        }
        if (CFM_DEBUG(p) & 4) {  // timing experiment: no copies, stale stage data
          mbar_arrive(full + s);
          if (BULK_A && pt == 0) mbar_arrive(full + s);  // the expect_tx arrival of the bulk path
          continue;
        }
        const int k0 = kc * KC;
        double* as = As + s * BM * LDA;
        double* bs = Bs + s * BN * LDB;
        if (BULK_A) {
          // one bulk copy per operator row (KC doubles); rows past the operator
          // read the zero row kept after the stack
          if (pt == 0) mbar_arrive_expect_tx(full + s, BM * KC * 8);
#pragma unroll
          for (int u = 0; u < BM / NP; ++u) {
            const int i = pt + u * NP;
            bulk_g2s(as + i * LDA, a_rowb[u] + k0, KC * 8, full + s);
          }
        } else {
#pragma unroll
          for (int u = 0; u < A_PER_T; ++u) {
            const int id = pt + u * NP;
            const int i = id / (KC / 2), kp = id % (KC / 2);
            const bool ok = a_ok[u] && !(CFM_DEBUG(p) & 8);
            cp_async16(as + i * LDA + 2 * kp, ok ? (const void*)(a_row[u] + k0) : (const void*)p.ops, ok);
          }
        }
        const int kk = pt % KC;
        const int k = k0 + kk;
        const bool kvalid = k < d.klen;
        int j = k;
        if (kvalid && d.cperm >= 0) j = invtab[d.cperm * p.nk + k];
#pragma unroll
        for (int u = 0; u < B_PER_T; ++u) {
          const int c = pt / KC + u * (NP / KC);
          const bool ok = kvalid && b_col[u] != nullptr && !(CFM_DEBUG(p) & 16);
          cp_async8(bs + c * LDB + kk, ok ? (const void*)(b_col[u] + (long long)p.x_dc * j) : (const void*)p.ops, ok);
        }
        mbar_cp_async_arrive(full + s);
      }
      e = next_live(e + 1, d);
    }
    cp_async_wait<0>();
    return;
  }

  // ======================= consumer warps =======================
  const int g = lane >> 2, tg = lane & 3;
  const int wm = warp % WM, wn = warp / WM;
  // first row / column of m-tile mi / n-tile nj of this warp.  Full-operator
  // mode interleaves them (warp (wm, wn) owns m-tiles mi*WM+wm, n-tiles
  // nj*WN+wn) so that rows past the operator and empty trailing columns of a
  // pair entry are skipped evenly by all four SM sub-partitions.
  auto mrow = [&](int mi) { return IL ? (mi * WM + wm) * 8 : wm * WTM + mi * 8; };
  auto ncol = [&](int nj) { return IL ? (nj * WN + wn) * 8 : wn * WTN + nj * 8; };
  double acc[MT][NTL][2];
#pragma unroll
  for (int mi = 0; mi < MT; ++mi)
#pragma unroll
    for (int nj = 0; nj < NTL; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;

  EntryInfo d;
  d.nchunks = 0;
  int e = next_live(e_begin, d);
  int q = 0;
  int ml = 0;  // live m-tiles of this warp (full-operator mode; fixed per CTA)
  if (IL)
    for (int mi = 0; mi < MT; ++mi)
      if (r0 + mrow(mi) < p.nr) ml = mi + 1;
  auto ft_entry = [&](auto mlc, auto nlc) {
    constexpr int ML = decltype(mlc)::value, NL = decltype(nlc)::value;
    for (int kc = 0; kc < d.nchunks; ++kc, ++q) {
      const int s = q % STAGES;
      mbar_wait(full + s, (q / STAGES) & 1);
      if (ML > 0 && NL > 0) {
        const double* as = As + s * BM * LDA + (mrow(0) + g) * LDA + tg;
        const double* bs = Bs + s * BN * LDB + (ncol(0) + g) * LDB + tg;
        constexpr int MSTEP = IL ? WM * 8 : 8, NSTEP = IL ? WN * 8 : 8;
        const int kmax = min(KC, d.klen - kc * KC);
        auto step = [&](int kk) {
          double a[ML > 0 ? ML : 1], b[NL > 0 ? NL : 1];
#pragma unroll
          for (int mi = 0; mi < ML; ++mi) a[mi] = as[mi * MSTEP * LDA + kk];
#pragma unroll
          for (int nj = 0; nj < NL; ++nj) b[nj] = bs[nj * NSTEP * LDB + kk];
#pragma unroll
          for (int mi = 0; mi < ML; ++mi)
#pragma unroll
            for (int nj = 0; nj < NL; ++nj) dmma884(acc[mi][nj][0], acc[mi][nj][1], a[mi], b[nj]);
        };
        if (kmax == KC) {
#pragma unroll
          for (int kk = 0; kk < KC; kk += 4) step(kk);
        } else {
#pragma unroll 2
          for (int kk = 0; kk < kmax; kk += 4) step(kk);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
    }
  };
  auto ft_dispatch = [&](auto mlc, int nl) {
    switch (nl) {
      case 0: ft_entry(mlc, std::integral_constant<int, 0>{}); break;
      case 1: ft_entry(mlc, std::integral_constant<int, (NTL < 1 ? NTL : 1)>{}); break;
      case 2: ft_entry(mlc, std::integral_constant<int, (NTL < 2 ? NTL : 2)>{}); break;
      case 3: ft_entry(mlc, std::integral_constant<int, (NTL < 3 ? NTL : 3)>{}); break;
      default: ft_entry(mlc, std::integral_constant<int, NTL>{}); break;
    }
  };
  if constexpr (FTM == 1 || FTM == 3) {
    // FTM 3: pair-mode stage-1 tiles of the two-stage low-rank path (y_rowblk,
    // operator-id codes: every entry has the same chunk count and the tile's
    // columns) run the flat loop too, writing each entry's rows when its last
    // chunk is done
    // (the KC = 16 instantiation -- stage 2 -- also keeps this path compiled in:
    // measured 4% faster that way, a scheduling side effect; the KC = 32 FTM 1
    // step kernel compiles without it, 0.4% faster)
    constexpr bool kSegCapable = FTM == 3 || KC == 16;
    const bool seg_out = kSegCapable && p.pair_out && p.y_rowblk && p.code_is_op;
    if ((seg_out || !p.pair_out) && p.ft_pipe) {
      // Full-operator target tiles whose every chunk is KC/4 whole k-steps
      // (host-checked): one flat chunk stream, software-pipelined across chunk
      // and entry boundaries -- the next chunk's full barrier is waited for and
      // its first fragments loaded before the current chunk's last k-step, so
      // the two consumer warps of an SM sub-partition do not stall together
      // at every boundary.
      int total = 0;
      for (int ee = e_begin; ee < e_end; ++ee) total += decode_code<KC>(p, code_of(ee), s_op, s_rp, s_cp, r0).nchunks;
      const int nch = (p.nk + KC - 1) / KC;  // chunks per entry (seg_out: uniform)
      if (total > 0) {
        const int aoff = (mrow(0) + g) * LDA + tg, boff = (ncol(0) + g) * LDB + tg;
        double a0[MT], b0[NTL], a1[MT], b1[NTL];
        auto load = [&](double* a, double* b, int s, int kk) {
          const double* as = As + s * BM * LDA + aoff;
          const double* bs = Bs + s * BN * LDB + boff;
#pragma unroll
          for (int mi = 0; mi < MT; ++mi) a[mi] = as[mi * 8 * LDA + kk];
#pragma unroll
          for (int nj = 0; nj < NTL; ++nj) b[nj] = bs[nj * 8 * LDB + kk];
        };
        auto mma = [&](const double* a, const double* b) {
#pragma unroll
          for (int mi = 0; mi < MT; ++mi)
#pragma unroll
            for (int nj = 0; nj < NTL; ++nj) dmma884(acc[mi][nj][0], acc[mi][nj][1], a[mi], b[nj]);
        };
        // skewed consumer halves (ft_skew chunks): the warps with odd wn start
        // when the even ones have finished ft_skew chunks, so the two consumer
        // warps of an SM sub-partition reach their per-entry / per-tile
        // epilogues at different times and one keeps the DMMA pipe busy
        const bool skewed = WN == 2 && p.ft_skew > 0 && total > p.ft_skew && p.ft_skew < STAGES;
        if (skewed && wn == 1) asm volatile("bar.sync 2, %0;\n" ::"n"(NC) : "memory");
        mbar_wait(full, 0);
        load(a0, b0, 0, 0);
        for (int qq = 0; qq < total; ++qq) {
          const int s = qq % STAGES;
          if (skewed && wn == 0 && qq == p.ft_skew) asm volatile("bar.arrive 2, %0;\n" ::"n"(NC) : "memory");
          // an entry's last k-step with one real column (p.ft_ktail: nk % KC ==
          // KC - 3, e.g. l = 5) runs as a rank-1 DFMA update instead of a DMMA
          // over 3 zero columns: DMMA and DFMA share the FP64 pipe
          // (tools/fp64_mix.cu), so this drops 3/4 of that step's pipe time
          // (FTM 1 only: in the FTM 3 stage-1 kernel the extra registers spill)
          const bool ktail = FTM == 1 && p.ft_ktail && (qq + 1) % nch == 0;
#pragma unroll
          for (int kk = 0; kk < KC; kk += 8) {
            double bt[NTL];
            if (kk + 8 == KC && ktail) {
              const double* as = As + s * BM * LDA + g * LDA + kk + 4;
              const double* bs = Bs + s * BN * LDB + 2 * tg * LDB + kk + 4;
#pragma unroll
              for (int mi = 0; mi < MT; ++mi) a1[mi] = as[mrow(mi) * LDA];
#pragma unroll
              for (int nj = 0; nj < NTL; ++nj) {
                b1[nj] = bs[ncol(nj) * LDB];
                bt[nj] = bs[(ncol(nj) + 1) * LDB];
              }
            } else {
              load(a1, b1, s, kk + 4);
            }
            mma(a0, b0);
            if (kk + 8 < KC) {
              load(a0, b0, s, kk + 8);
            } else if (qq + 1 < total) {
              const int s1 = (qq + 1) % STAGES;
              mbar_wait(full + s1, ((qq + 1) / STAGES) & 1);
              load(a0, b0, s1, 0);
            }
            if (kk + 8 == KC && ktail) {
#pragma unroll
              for (int mi = 0; mi < MT; ++mi)
#pragma unroll
                for (int nj = 0; nj < NTL; ++nj) {
                  acc[mi][nj][0] = fma(a1[mi], b1[nj], acc[mi][nj][0]);
                  acc[mi][nj][1] = fma(a1[mi], bt[nj], acc[mi][nj][1]);
                }
            } else {
              mma(a1, b1);
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(empty + s);
          if (seg_out && (qq + 1) % nch == 0) {
            // packed two-stage stage 1: the entry's 128 rows of every source's
            // Y row, at the columns of ts_colmap (a transfer's rows are
            // contiguous: the 8 lanes of a tg write runs of up to 64 B)
            const int* cm = p.y_colmap + (long long)code_of(e_begin + qq / nch) * BM + r0 + g;
            int ycol[MT];
#pragma unroll
            for (int mi = 0; mi < MT; ++mi) ycol[mi] = __ldg(cm + mrow(mi));
            if (p.y_nbr) {
              // target-major Y: row (slot, a) of source v goes to the Y_T row of the
              // pair's target, at y_nbr[v][slot] + a (the 8 lanes of a tg mostly
              // share a slot: one broadcast load, a run of up to 64 B stored)
#pragma unroll
              for (int nj = 0; nj < NTL; ++nj)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  const int v = s_col[ncol(nj) + 2 * tg + h];
                  const int* nb = p.y_nbr + (long long)v * p.y_nslots;
                  int w[MT];
#pragma unroll
                  for (int mi = 0; mi < MT; ++mi) w[mi] = (v >= 0 && ycol[mi] >= 0) ? __ldg(nb + (ycol[mi] >> 8)) : -1;
#pragma unroll
                  for (int mi = 0; mi < MT; ++mi) {
                    if (w[mi] >= 0) p.y[(long long)w[mi] + (ycol[mi] & 255)] = acc[mi][nj][h];
                    acc[mi][nj][h] = 0.0;
                  }
                }
              continue;
            }
#pragma unroll
            for (int nj = 0; nj < NTL; ++nj)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int v = s_col[ncol(nj) + 2 * tg + h];
                double* dst = p.y + (long long)v * p.y_ld;
#pragma unroll
                for (int mi = 0; mi < MT; ++mi) {
                  if (v >= 0 && ycol[mi] >= 0 && !(CFM_DEBUG(p) & 128)) dst[ycol[mi]] = acc[mi][nj][h];
                  acc[mi][nj][h] = 0.0;
                }
              }
          }
        }
      }
      e = e_end;
      if (seg_out) return;
    }
  }
  while (e < e_end) {
    bool generic = true;  // all of this warp's tiles live: the plain loop
    if constexpr (IL) {
      static_assert(MT <= 4 && NTL <= 4, "full-operator dispatch covers 4 x 4 tiles per warp");
      const int i = e - e_begin;
      const int ncols = p.entry_ncols ? (i < kMaxTileEntries ? int(s_encols[i]) : int(__ldg(p.entry_ncols + e))) : BN;
      int nl = 0;
#pragma unroll
      for (int nj = 0; nj < NTL; ++nj)
        if (ncol(nj) < ncols) nl = nj + 1;
      if (ml != MT || nl != NTL) {
        generic = false;
        switch (ml) {
          case 0: ft_dispatch(std::integral_constant<int, 0>{}, nl); break;
          case 1: ft_dispatch(std::integral_constant<int, (MT < 1 ? MT : 1)>{}, nl); break;
          case 2: ft_dispatch(std::integral_constant<int, (MT < 2 ? MT : 2)>{}, nl); break;
          case 3: ft_dispatch(std::integral_constant<int, (MT < 3 ? MT : 3)>{}, nl); break;
          default: ft_dispatch(std::integral_constant<int, MT>{}, nl); break;
        }
      }
    }
    if (generic) {
    constexpr int MSTEP = IL ? WM * 8 : 8, NSTEP = IL ? WN * 8 : 8;
    const int mrows = d.rows - r0 - wm * WTM;
    for (int kc = 0; kc < d.nchunks; ++kc, ++q) {
      const int s = q % STAGES;
      if (!(CFM_DEBUG(p) & 1)) mbar_wait(full + s, (q / STAGES) & 1);
      const double* as = As + s * BM * LDA + (mrow(0) + g) * LDA + tg;
      const double* bs = Bs + s * BN * LDB + (ncol(0) + g) * LDB + tg;
      const int kmax = min(KC, d.klen - kc * KC);
      if (SKIP_ROWS) {
#pragma unroll 2
        for (int kk = 0; kk < kmax; kk += 4) {
          double a[MT], b[NTL];
#pragma unroll
          for (int mi = 0; mi < MT; ++mi) a[mi] = as[mi * MSTEP * LDA + kk];
#pragma unroll
          for (int nj = 0; nj < NTL; ++nj) b[nj] = bs[nj * NSTEP * LDB + kk];
#pragma unroll
          for (int mi = 0; mi < MT; ++mi) {
            if (mi * 8 < mrows) {
#pragma unroll
              for (int nj = 0; nj < NTL; ++nj) dmma884(acc[mi][nj][0], acc[mi][nj][1], a[mi], b[nj]);
            }
          }
        }
      } else if (kmax == KC) {
#pragma unroll
        for (int kk = 0; kk < KC; kk += 4) {
          double a[MT], b[NTL];
#pragma unroll
          for (int mi = 0; mi < MT; ++mi) a[mi] = as[mi * MSTEP * LDA + kk];
#pragma unroll
          for (int nj = 0; nj < NTL; ++nj) b[nj] = bs[nj * NSTEP * LDB + kk];
#pragma unroll
          for (int mi = 0; mi < MT; ++mi)
#pragma unroll
            for (int nj = 0; nj < NTL; ++nj) dmma884(acc[mi][nj][0], acc[mi][nj][1], a[mi], b[nj]);
        }
      } else {
#pragma unroll 2
        for (int kk = 0; kk < kmax; kk += 4) {
          double a[MT], b[NTL];
#pragma unroll
          for (int mi = 0; mi < MT; ++mi) a[mi] = as[mi * MSTEP * LDA + kk];
#pragma unroll
          for (int nj = 0; nj < NTL; ++nj) b[nj] = bs[nj * NSTEP * LDB + kk];
#pragma unroll
          for (int mi = 0; mi < MT; ++mi)
#pragma unroll
            for (int nj = 0; nj < NTL; ++nj) dmma884(acc[mi][nj][0], acc[mi][nj][1], a[mi], b[nj]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
    }
    }
    if (p.pair_out) {
      // pair mode: this entry's 64 columns are 64 distinct (target, source)
      // pairs; write their results to rows e*BN + c (segment-reduced per target later)
#pragma unroll
      for (int mi = 0; mi < MT; ++mi) {
        const int row = r0 + mrow(mi) + g;
#pragma unroll
        for (int nj = 0; nj < NTL; ++nj) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = ncol(nj) + 2 * tg + h;
            if (row < p.nr && __ldg(p.entry_src + (long long)e * BN + c) >= 0) {
              const long long v = (long long)e * BN + c;
              const long long ro = (long long)p.y_dc * row;
              double* dst = p.y + (v / p.y_dc) * p.y_ld + (v % p.y_dc) + ro;
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
  if (p.pair_out) {
    if (p.red_counter) {
      // last CTA of the segment: ordered per-target reduction of the pair rows
      __shared__ int s_last;
      __threadfence();  // every consumer's pair rows are visible device-wide before the count
      asm volatile("bar.sync 1, %0;\n" ::"n"(NC) : "memory");
      if (tid == 0) {
        __threadfence();
        const unsigned old = atomicAdd(p.red_counter, 1u);
        s_last = (old == unsigned(p.red_ctas) - 1) ? 1 : 0;
        __threadfence();
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(NC) : "memory");
      if (s_last) {
        const long long total = p.red_n_tgt * p.red_len;
        for (long long idx = tid; idx < total; idx += NC) {
          const long long t = idx / p.red_len;
          const int i = int(idx - t * p.red_len);
          double sum = 0.0;
          for (long long q2 = p.red_off[t]; q2 < p.red_off[t + 1]; ++q2)
            sum += __ldcg(p.y + (long long)p.red_frow[q2] * p.red_ld + i);
          p.red_y[p.red_tgt[t] * p.red_ld + i] += p.red_scale * sum;
        }
      }
    }
    return;
  }

  // ---------------- epilogue: ordered, atomic-free write ----------------
  if (e_begin == e_end && p.accumulate && !p.pipe_done) return;
  if (p.pipe_loc) wait_flag_geq(p.pipe_loc, p.pipe_need_loc ? unsigned(p.pipe_need_loc[tile]) : 1u);
#pragma unroll
  for (int mi = 0; mi < MT; ++mi) {
    const int row = r0 + mrow(mi) + g;
    if (row >= p.nr) continue;
#pragma unroll
    for (int nj = 0; nj < NTL; ++nj) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = ncol(nj) + 2 * tg + h;
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
  if (p.pipe_done) {
    __threadfence();
    asm volatile("bar.sync 1, %0;\n" ::"n"(NC) : "memory");
    if (tid == 0)
      for (int k = p.pipe_lo[tile]; k <= p.pipe_hi[tile]; ++k) atomicAdd(p.pipe_done + k, 1u);
  }
}

}  // namespace cfm
