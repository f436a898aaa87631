// Fused gather-permute -> FP64 DMMA -> ordered accumulate tile kernel (sm_100a).
//
// One CTA owns a (row block r0..r0+BM) x (tile of BN output columns) block of
// the result and walks the tile's entries.  An entry is one (transfer vector,
// occurrence) with one source column per output column; all columns of an
// entry share an operator and a permutation, so the entry is one small GEMM:
//
//   acc[i, c] += sum_k  Op[ rowtab[i] , k ] * X[ src_c , invtab[k] ]
//
// which is the reference's symmetric apply (m2l.py:353-362, blocked form
// :437-444 + :422 + :430-431):  u = w[inv]; out = K_rep @ u; acc += out[table]
// with acc[i] += out[table[i]] = sum_k K_rep[table[i], k] * w[inv[k]].
// The accumulator stays in registers across all entries of the tile, so the
// inverse-permute scatter of the reference becomes a row gather of the
// operator (rowtab) and the result is written once per tile, ordered per
// target column with no atomics (each output column belongs to one tile).
//
// Staging: the operator rows (contiguous 16-B cp.async) and the gathered,
// permuted source columns (8-B cp.async, zero-filled for empty slots) are
// streamed through a STAGES-deep shared-memory ring in K-chunks of KC; the
// MMA is mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4): tcgen05 has no f64 kind, and
// DMMA runs at the chip's FP64 peak (37.1 TF/s measured, profiles/).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

// Timing-experiment bits of TileParams::debug (they give wrong results) exist
// only in builds with -DCFM_EXPERIMENTS; release builds fold them to 0.
#ifdef CFM_EXPERIMENTS
#define CFM_DEBUG(p) ((p).debug)
#else
#define CFM_DEBUG(p) 0
#endif

namespace cfm {

struct TileParams {
  // plan
  int n_tiles;
  int tile_base;          // tile index of blockIdx.x == 0
  const int* tile_col;    // [n_tiles * BN]  virtual output id or -1
  const int* tile_off;    // [n_tiles + 1]   entry range per tile
  const int* entry_code;  // [E]             code -> (op, row perm, col perm)
  const int* entry_src;   // [E * BN]        virtual source id or -1
  const int* code_op;     // [n_codes]
  const int* code_rperm;  // [n_codes] row perm id (-1 identity)
  const int* code_cperm;  // [n_codes] col perm id (-1 identity)
  // operators: op o = ops + o * op_stride, row-major, leading dim op_ld,
  // columns zero-padded up to a multiple of KC.
  const double* ops;
  long long op_stride;
  int op_ld;
  int nr;                  // output rows
  int nk;                  // inner length
  const int* op_rows;      // optional per-op row count
  const int* op_klen;      // optional per-op inner length
  const short* rowtab;     // rowtab[p * nr + i]
  const short* invtab;     // invtab[p * nk + k]
  // data: virtual id v -> base (v / dc) * ld + (v % dc), element stride dc
  const double* x;
  long long x_ld;
  int x_dc;
  double* y;
  long long y_ld;
  int y_dc;
  double scale;
  int accumulate;
  int pair_out;  // 1: write each entry's result to y rows (e * BN + c) when the entry ends
  int debug;     // timing experiments only (bit 0: consumers skip the full-barrier wait);
                 // read through CFM_DEBUG(), which is 0 unless built with -DCFM_EXPERIMENTS
  const double* zero_row;  // >= op_ld zeros (rows past an operator, bulk-copy path)
  // pair mode, small segments: the last CTA of the segment reduces the per-pair
  // rows into the targets itself (ordered, no extra launch)
  unsigned int* red_counter;  // null: reduction launched separately
  int red_ctas;               // CTAs in the segment (tiles x row blocks)
  const long long* red_tgt;
  const long long* red_off;
  const int* red_frow;
  long long red_n_tgt;
  double* red_y;
  long long red_ld;
  int red_len;
  double red_scale;
  // host<->device copy pipeline (target mode): per-tile slab needs and
  // per-slab completion counters; null when the level is not pipelined
  const unsigned* pipe_mp;   // # multipole slabs resident
  const unsigned* pipe_loc;  // # locals slabs resident
  unsigned* pipe_done;       // per slab: CTAs done writing its rows
  const int* pipe_need_mp;
  const int* pipe_need_loc;
  const int* pipe_lo;
  const int* pipe_hi;
  // full-operator TMA mode (real dense groups, 65 < nr, nk <= 512): ops is a
  // stack of the fully permuted operators K_t (ft_rows rows each, one per
  // transfer vector, code_* map t -> its K_t with identity permutations), read
  // by one 2-D TMA tile copy per chunk through tmap_a; the sources are
  // contiguous zero-padded rows (x_ld = op_ld), one bulk copy per column
  int ft;
  int ft_rows;
  const unsigned char* entry_ncols;  // pair plans: filled columns per entry (null: all BN)
  long long n_entries;               // host-side hint: entries of the plan (kernel choice)
  long long x_rows;                  // full-operator mode: rows of the padded source array x
  int x_row0;                        // full-operator mode: subtracted from every source row id (tmap_b starts at that row)
  int ft_pipe;                       // full-operator target tiles: flat pipelined consumer loop
  int ft_skew;                       // flat loop: chunks the odd-wn consumer warps start behind the even ones (0: off)
  int ft_ktail;                      // flat loop: an entry's last k-step has one real column (DFMA rank-1)
  // two-stage low-rank mode (full-operator kernels):
  int code_is_op;   // entry codes are operator ids (no code tables, identity permutations)
  int ft_opshift;   // operator id o -> A block row (o >> ft_opshift) * ft_rows, column (o & mask) * ft_colseg
  int ft_colseg;
  int y_rowblk;     // pair-mode stage-1 output (0: off): row i of entry code c lands at
                    // y[source * y_ld + y_colmap[c * 128 + i]] (skipped where -1)
  const int* y_colmap;
  const int* y_nbr;   // target-major stage 1 (null: off): y_colmap[c * 128 + i] = (slot << 8 | a), and row i of a
  int y_nslots;       // source lands at y[y_nbr[source * y_nslots + slot] + a] (skipped where either is -1)
  int b_block;      // B of entry e = rows [e * BN, e * BN + BN) of tmap_b (one 2-D box; no gathers)
  const int* op_col;  // seg_pair_gemm_kernel: B of entry e gathered from its sources' rows of
                      // tmap_b at column op_col[entry_code[e]]
  const int* seg_ksteps;  // seg_pair_gemm_kernel: live k-steps (0..4) per entry code (null: all 4)
  int l2_hints;     // TMA copies with L2 policies: operators evict_last, sources evict_first
  int no_step;      // host-side: keep this list off the persistent step kernel (entries whose code has no
                    // operator in this launch are skipped by tile_gemm_ws_kernel only)
  CUtensorMap tmap_a;
  // full-operator mode: 2-D map over the padded sources (x_ld x x_rows), box
  // (KC + 4) x 1, read by tile::gather4 copies (4 source rows per instruction)
  CUtensorMap tmap_b;
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Wait until a copy-stream flag reaches v (written by cuStreamWriteValue32).
// Traps after ~4 s instead of hanging the device if a flag never arrives.
__device__ __forceinline__ void wait_flag_geq(const unsigned* f, unsigned v) {
  unsigned ns = 64;
  const long long t0 = clock64();
  while (ld_acquire_u32(f) < v) {
    __nanosleep(ns);
    ns = ns < 2048 ? ns * 2 : 2048;
    if (clock64() - t0 > (1ll << 33)) __trap();
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

constexpr int kMaxTileEntries = 1024;  // entry codes cached in smem per tile

// Shared-memory footprint: operand ring + per-CTA lookup tables
// (code -> op/perm, the tile's entry codes, and the 48 permutation tables
// when they fit).
template <int BM, int BN, int KC, int STAGES>
constexpr int tile_ring_bytes() {
  return STAGES * (BM + BN) * (KC + 4) * 8;
}
__host__ __device__ constexpr int tile_table_bytes(int nr, int nk, bool perm_tabs) {
  return 4 * 64 /*s_col*/ + 3 * 4 * 344 + 4 * kMaxTileEntries + (perm_tabs ? 48 * 2 * (nr + nk + 8) : 0);
}
__host__ __device__ inline bool tile_perm_tabs_fit(int nr, int nk) { return 48 * 2 * (nr + nk) <= 48 * 1024; }

// Per-entry decode shared by producer and consumer (all lookups in smem).
struct EntryInfo {
  int op, rperm, cperm, rows, klen, nchunks;
};

template <int KC>
__device__ __forceinline__ EntryInfo decode_code(const TileParams& p, int code, const int* s_op, const int* s_rp,
                                                 const int* s_cp, int r0) {
  EntryInfo d;
  if (p.code_is_op) {
    d.op = code;
    d.rperm = d.cperm = -1;
    d.rows = p.nr;
    d.klen = p.nk;
    d.nchunks = (d.rows > r0) ? (d.klen + KC - 1) / KC : 0;
    return d;
  }
  d.op = s_op[code];
  d.rperm = s_rp[code];
  d.cperm = s_cp[code];
  if (d.op < 0) {  // code handled by another launch (shared-basis dense vs factored cores)
    d.rows = 0;
    d.klen = 0;
    d.nchunks = 0;
    return d;
  }
  d.rows = p.op_rows ? __ldg(p.op_rows + d.op) : p.nr;
  d.klen = p.op_klen ? __ldg(p.op_klen + d.op) : p.nk;
  d.nchunks = (d.rows > r0) ? (d.klen + KC - 1) / KC : 0;
  return d;
}

template <int BM, int BN, int WM, int WN, int KC, int STAGES, bool SKIP_ROWS>
__global__ void __launch_bounds__(WM* WN * 32, 1) tile_gemm_kernel(const TileParams p) {
  constexpr int NT = WM * WN * 32;
  constexpr int WTM = BM / WM, WTN = BN / WN;
  constexpr int MT = WTM / 8, NTL = WTN / 8;
  constexpr int LDA = KC + 4, LDB = KC + 4;
  constexpr int A_PIECES = BM * (KC / 2);  // 16-B pieces per chunk
  constexpr int A_PER_T = A_PIECES / NT;
  constexpr int B_ELEMS = BN * KC;
  constexpr int B_PER_T = B_ELEMS / NT;
  static_assert(A_PIECES % NT == 0 && B_ELEMS % NT == 0, "tile/thread mismatch");
  static_assert(NT % KC == 0, "B mapping needs NT multiple of KC");
  static_assert(MT >= 1 && NTL >= 1, "warp tile too small");
  static_assert(BN <= 64, "s_col sized for 64 columns");

  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = As + STAGES * BM * LDA;
  int* s_col = reinterpret_cast<int*>(Bs + STAGES * BN * LDB);
  int* s_op = s_col + 64;
  int* s_rp = s_op + 344;
  int* s_cp = s_rp + 344;
  int* s_ecode = s_cp + 344;
  short* s_rowtab = reinterpret_cast<short*>(s_ecode + kMaxTileEntries);
  const bool tabs_in_smem = tile_perm_tabs_fit(p.nr, p.nk);
  short* s_invtab = s_rowtab + 48 * p.nr + 8;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tg = lane & 3;
  const int wm = warp % WM, wn = warp / WM;
  const int tile = p.tile_base + blockIdx.x;
  const int r0 = blockIdx.y * BM;
  const int e_begin = p.tile_off[tile], e_end = p.tile_off[tile + 1];

  // ---------------- per-CTA tables in shared memory ----------------
  for (int c = tid; c < BN; c += NT) s_col[c] = p.tile_col[(long long)tile * BN + c];
  for (int c = tid; c < 343; c += NT) {
    s_op[c] = p.code_op[c];
    s_rp[c] = p.code_rperm[c];
    s_cp[c] = p.code_cperm[c];
  }
  const int n_cached = min(e_end - e_begin, kMaxTileEntries);
  for (int i = tid; i < n_cached; i += NT) s_ecode[i] = p.entry_code[e_begin + i];
  if (tabs_in_smem) {
    if (p.rowtab)
      for (int i = tid; i < 48 * p.nr; i += NT) s_rowtab[i] = p.rowtab[i];
    if (p.invtab)
      for (int i = tid; i < 48 * p.nk; i += NT) s_invtab[i] = p.invtab[i];
  }
  __syncthreads();
  const short* rowtab = tabs_in_smem ? s_rowtab : p.rowtab;
  const short* invtab = tabs_in_smem ? s_invtab : p.invtab;
  auto code_of = [&](int e) -> int {
    const int i = e - e_begin;
    return i < kMaxTileEntries ? s_ecode[i] : __ldg(p.entry_code + e);
  };

  // ---------------- producer state ----------------
  int pe = e_begin, pk = 0;  // entry / chunk to issue next
  EntryInfo pinfo;
  pinfo.nchunks = 0;
  while (pe < e_end) {
    pinfo = decode_code<KC>(p, code_of(pe), s_op, s_rp, s_cp, r0);
    if (pinfo.nchunks) break;
    ++pe;
  }
  // B source indices: current entry (registers) and the prefetched next entry
  int nxt_src[B_PER_T];
  int nxt_e = -1;
  auto prefetch_src = [&](int e) {
    nxt_e = e;
    if (e < e_end) {
#pragma unroll
      for (int u = 0; u < B_PER_T; ++u) nxt_src[u] = __ldg(p.entry_src + (long long)e * BN + tid / KC + u * (NT / KC));
    }
  };
  const double* a_row[A_PER_T];
  bool a_ok[A_PER_T];
  const double* b_col[B_PER_T];
  int pe_loaded = -1;

  auto load_entry_ptrs = [&](int e, const EntryInfo& d) {
    const double* opbase = p.ops + (long long)d.op * p.op_stride;
#pragma unroll
    for (int u = 0; u < A_PER_T; ++u) {
      const int id = tid + u * NT;
      const int i = id / (KC / 2), kp = id % (KC / 2);
      const int gr = r0 + i;
      a_ok[u] = gr < d.rows;
      int orow = gr;
      if (a_ok[u] && d.rperm >= 0) orow = rowtab[d.rperm * p.nr + gr];
      a_row[u] = opbase + (long long)(a_ok[u] ? orow : 0) * p.op_ld + 2 * kp;
    }
    if (nxt_e != e) prefetch_src(e);
#pragma unroll
    for (int u = 0; u < B_PER_T; ++u) {
      const int v = nxt_src[u];
      b_col[u] = (v >= 0) ? p.x + (long long)(v / p.x_dc) * p.x_ld + (v % p.x_dc) : nullptr;
    }
    prefetch_src(e + 1);  // latency hidden behind this entry's chunks
  };

  auto issue = [&](int stage) {
    if (pe >= e_end) {
      cp_async_commit();
      return;
    }
    if (pe_loaded != pe) {
      load_entry_ptrs(pe, pinfo);
      pe_loaded = pe;
    }
    const int k0 = pk * KC;
    double* as = As + stage * BM * LDA;
    double* bs = Bs + stage * BN * LDB;
#pragma unroll
    for (int u = 0; u < A_PER_T; ++u) {
      const int id = tid + u * NT;
      const int i = id / (KC / 2), kp = id % (KC / 2);
      cp_async16(as + i * LDA + 2 * kp, a_ok[u] ? (const void*)(a_row[u] + k0) : (const void*)p.ops, a_ok[u]);
    }
    const int kk = tid % KC;
    const int k = k0 + kk;
    const bool kvalid = k < pinfo.klen;
    int j = k;
    if (kvalid && pinfo.cperm >= 0) j = invtab[pinfo.cperm * p.nk + k];
#pragma unroll
    for (int u = 0; u < B_PER_T; ++u) {
      const int c = tid / KC + u * (NT / KC);
      const bool ok = kvalid && b_col[u] != nullptr;
      cp_async8(bs + c * LDB + kk, ok ? (const void*)(b_col[u] + (long long)p.x_dc * j) : (const void*)p.ops, ok);
    }
    cp_async_commit();
    // advance producer
    if (++pk >= pinfo.nchunks) {
      pk = 0;
      ++pe;
      while (pe < e_end) {
        pinfo = decode_code<KC>(p, code_of(pe), s_op, s_rp, s_cp, r0);
        if (pinfo.nchunks) break;
        ++pe;
      }
    }
  };

  double acc[MT][NTL][2];
#pragma unroll
  for (int mi = 0; mi < MT; ++mi)
#pragma unroll
    for (int nj = 0; nj < NTL; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;

  // ---------------- consumer state ----------------
  int ce = e_begin, ck = 0;
  EntryInfo cinfo;
  cinfo.nchunks = 0;
  while (ce < e_end) {
    cinfo = decode_code<KC>(p, code_of(ce), s_op, s_rp, s_cp, r0);
    if (cinfo.nchunks) break;
    ++ce;
  }

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) issue(s);

  int q = 0;
  while (ce < e_end) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    issue((q + STAGES - 1) % STAGES);
    const int stage = q % STAGES;
    const double* as = As + stage * BM * LDA + (wm * WTM + g) * LDA + tg;
    const double* bs = Bs + stage * BN * LDB + (wn * WTN + g) * LDB + tg;
    const int kmax = min(KC, cinfo.klen - ck * KC);
    if (SKIP_ROWS) {
      const int mrows = cinfo.rows - r0 - wm * WTM;  // live rows of this warp tile
#pragma unroll 2
      for (int kk = 0; kk < kmax; kk += 4) {
        double a[MT], b[NTL];
#pragma unroll
        for (int mi = 0; mi < MT; ++mi) a[mi] = as[mi * 8 * LDA + kk];
#pragma unroll
        for (int nj = 0; nj < NTL; ++nj) b[nj] = bs[nj * 8 * LDB + kk];
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
        for (int mi = 0; mi < MT; ++mi) a[mi] = as[mi * 8 * LDA + kk];
#pragma unroll
        for (int nj = 0; nj < NTL; ++nj) b[nj] = bs[nj * 8 * LDB + kk];
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
        for (int mi = 0; mi < MT; ++mi) a[mi] = as[mi * 8 * LDA + kk];
#pragma unroll
        for (int nj = 0; nj < NTL; ++nj) b[nj] = bs[nj * 8 * LDB + kk];
#pragma unroll
        for (int mi = 0; mi < MT; ++mi)
#pragma unroll
          for (int nj = 0; nj < NTL; ++nj) dmma884(acc[mi][nj][0], acc[mi][nj][1], a[mi], b[nj]);
      }
    }
    ++q;
    if (++ck >= cinfo.nchunks) {
      ck = 0;
      ++ce;
      while (ce < e_end) {
        cinfo = decode_code<KC>(p, code_of(ce), s_op, s_rp, s_cp, r0);
        if (cinfo.nchunks) break;
        ++ce;
      }
    }
  }
  cp_async_wait<0>();

  // ---------------- epilogue: ordered, atomic-free write ----------------
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
