// C-ABI implementation (include/chebm2l.h): operator cache on the device,
// plan cache per level, and the per-variant launch sequences.
//
// Variant -> device work (reference apply paths in m2l.py):
//   na            _apply_plain  :320-338  one tile_gemm over the |T| dense operators
//   nasym, nablk  _apply_sym    :340-364  one tile_gemm over the 16 representatives
//                 _apply_blocked:397-452  with row-gather (table) + column-gather (inv)
//   ia            _apply_plain  (low-rank)      pass 1: Y = right^H P^T w   (per pair)
//   iasym, iablk  _apply_sym/_blocked (low-rank) pass 2: acc += left[table] Y (per tile)
//   sa, sarcmp    _apply_shared :366-395  W~ = B^H M[src] (per source), Z = sum C_t W~
//                                         (dense or factored cores), locals += s U Z
// The reference's own accumulation model is kept: a target's contributions are
// summed into an accumulator and added once, scaled, into locals (m2l.py:337,
// :363, :393); the blocked variant's per-column adds (:430-431) differ from that
// only by floating-point reassociation.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>
#include <chrono>

#include "../../include/chebm2l.h"
#include "classify.cuh"
#include "plan.hpp"
#include "symmetry.hpp"
#include "tile_gemm.cuh"
#include "seg_gemm.cuh"
#include "tile_gemm_ws.cuh"
#include "pair_reduce.cuh"
#include "lowrank_ws.cuh"
#include "tree.cuh"
#include "fmm.cuh"
#include "precompute.cuh"

#include <cub/cub.cuh>

namespace cfm {

static thread_local std::string g_last_error;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CUDA_CHECK(x)                                                                       \
  do {                                                                                      \
    cudaError_t _e = (x);                                                                   \
    if (_e != cudaSuccess)                                                                  \
      throw Error(CFM_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(_e));          \
  } while (0)

// ---------------------------------------------------------------- device buffers
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; bytes = o.bytes; o.p = nullptr; o.bytes = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  void alloc(size_t b) {
    if (b <= bytes && p) return;
    release();
    if (b == 0) return;
    CUDA_CHECK(cudaMalloc(&p, b));
    bytes = b;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

template <class T>
static void upload(DevBuf& d, const std::vector<T>& h) {
  d.alloc(std::max<size_t>(h.size() * sizeof(T), 16));
  if (!h.empty()) CUDA_CHECK(cudaMemcpy(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
}

static int round_up(int x, int m) { return (x + m - 1) / m * m; }

constexpr int kKC = 32;
constexpr int kPass1Run = 16;  // entries per CTA in low-rank pass 1 (per-entry outputs)

// ------------------------------------------------------------------ code maps
struct CodeMap {
  std::array<int, kNumCodes> op;
  std::array<int, kNumCodes> rperm;
  std::array<int, kNumCodes> cperm;
  DevBuf d_op, d_rperm, d_cperm;
  CodeMap() { op.fill(-1); rperm.fill(-1); cperm.fill(-1); }
  void push() {
    upload(d_op, std::vector<int>(op.begin(), op.end()));
    upload(d_rperm, std::vector<int>(rperm.begin(), rperm.end()));
    upload(d_cperm, std::vector<int>(cperm.begin(), cperm.end()));
  }
};

// A stack of real operators laid out for tile_gemm: rows x ld (ld = cols
// rounded up to KC, zero padded).
struct OpStack {
  DevBuf d;
  int n_ops = 0, rows = 0, cols = 0, ld = 0;
  long long stride = 0;
  DevBuf d_rows, d_klen;  // optional per-op row / inner counts
  bool has_rows = false, has_klen = false;
  size_t host_bytes = 0;
};

static void realify_into(const double* src, int m, int k, bool cplx, double* dst, int ld, bool conj_t = false) {
  // src: m x k (complex interleaved if cplx) row-major; dst: (m f) x (k f) with leading dim ld.
  // conj_t: use conj(src)^T instead (src is k x m then).
  if (!cplx) {
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < k; ++j) dst[(size_t)i * ld + j] = conj_t ? src[(size_t)j * m + i] : src[(size_t)i * k + j];
    return;
  }
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < k; ++j) {
      double re, im;
      if (conj_t) {
        re = src[2 * ((size_t)j * m + i)];
        im = -src[2 * ((size_t)j * m + i) + 1];
      } else {
        re = src[2 * ((size_t)i * k + j)];
        im = src[2 * ((size_t)i * k + j) + 1];
      }
      dst[(size_t)(2 * i) * ld + 2 * j] = re;
      dst[(size_t)(2 * i) * ld + 2 * j + 1] = -im;
      dst[(size_t)(2 * i + 1) * ld + 2 * j] = im;
      dst[(size_t)(2 * i + 1) * ld + 2 * j + 1] = re;
    }
}

// ------------------------------------------------------------------ groups
enum GroupKind { kDense = 0, kLowRank = 1, kShared = 2 };

struct Group {
  GroupKind kind = kDense;
  int n_ops = 0;
  CodeMap main;       // dense / pass-2 (left) / SA dense cores
  CodeMap pass1;      // low-rank pass 1 (right^H) / SA factored cores pass 1
  CodeMap sa_fac2;    // SA factored cores pass 2
  CodeMap single;     // code 0 -> op 0 (SA transforms)
  OpStack dense;      // dense ops / SA dense cores
  OpStack left, right_h;  // low-rank factors (also SA factored cores)
  OpStack sa_bh, sa_u;    // SA bases
  int r_u = 0, r_b = 0;
  bool any_dense_core = false, any_fac_core = false;
  std::array<int, kNumCodes> valid{};  // transfer vectors of the group
  // full-operator TMA mode (dense, real): one fully permuted K_t per transfer
  bool has_full = false;
  OpStack full;
  int full_rows = 0;
  CodeMap fullmap;
  CUtensorMap full_tmap;
  // low-rank counterpart: per-transfer permuted factors (U_t rows and V_t^H
  // columns permuted once), read with contiguous copies from padded sources
  bool has_lrfull = false;
  OpStack lrf_left, lrf_right_h;
  // two-stage low-rank mode (real, dense levels): stage 1 Y = V_t^H x per
  // (source, transfer) for the whole transfer set of the source's class, as a
  // dense GEMM against a per-class stack of V_t^H rows; stage 2 sums U_t Y per
  // target tile.  Classes: per axis the transfer components lie in [-3, 2]
  // (bit 0) or [-2, 3] (bit 1), which holds for every source of an octree
  // level (octree.py:157-175).  Ranks are cut in 16-wide segments (<= 2).
  bool has_ts = false;
  int ts_nb = 0;                 // 128-row blocks per class stack
  std::vector<int> ts_rank;      // per transfer index
  std::vector<int> ts_slot;      // [8][n_transfers][2] segment slot in the class stack, -1 if absent
  int ts_ntr = 0;
  OpStack ts_v;                  // 8 * ts_nb blocks of 128 rows x n
  CUtensorMap ts_vmap, ts_umap;  // box 36 x 128 over ts_v; box 20 x 128 over lrf_left
  DevBuf ts_ksteps;              // per stage-2 entry code 2k + j: k-steps holding rank columns (ceil(w / 4))
};

struct HybridPlan;
struct LevelPlan {
  HostPlan hp;
  int dc = 1;
  int mode = 0;  // 0: target tiles (accumulator per target column); 1: pair entries + ordered reduction
  double target_fill = 1.0;
  PairReduce red;
  DevBuf r_tgt, r_off, r_frow;
  // copy pipeline (target mode, large levels): rows split into n_slabs ranges
  int n_slabs = 1;
  std::vector<int64_t> slab_row0;        // n_slabs + 1 row boundaries
  std::vector<unsigned> slab_expected;   // CTAs (tiles x row blocks) writing each slab
  DevBuf p_need_mp, p_need_loc, p_lo, p_hi;
  DevBuf tile_col, tile_off, entry_code, entry_src;
  DevBuf entry_ncols;     // pair mode: filled columns per entry (uint8)
  DevBuf slot_ids, iota;  // low-rank: per-entry slots
  DevBuf runs;            // low-rank pass 1: tiles = runs of kPass1Run consecutive entries
  int64_t n_runs = 0;
  std::vector<int64_t> run_start;  // per target tile: first run
  // shared basis
  std::vector<int64_t> sources, targets;
  HostPlan src_plan, tgt_plan;
  DevBuf s_tile_col, s_tile_off, s_entry_code, s_entry_src;
  DevBuf t_tile_col, t_tile_off, t_entry_code, t_entry_src;
  int64_t n_rows = 0;
  uint64_t gen = 0;  // unique per built plan (merged plans remember what they were built from)
  // two-stage low-rank plans (Group::has_ts): stage 1 over source tiles, stage 2 over target tiles
  bool ts = false;
  HostPlan ts1, ts2;
  DevBuf ts1_col, ts1_off, ts1_code, ts1_src, ts2_col, ts2_off, ts2_code, ts2_src;
  int64_t ts_segs = 0;  // stage-2 B rows (entries x 64): the stage-1 output in stage-2 order, 20 doubles each (4 zero)
  DevBuf ts_y, ts_map;  // ts_map: stage-1 segment -> its row in ts_y (-1: no pair needs it)
  // hybrid (dense full-operator target tiles): the tiles that are less than
  // half full -- the partial last tile of each boundary class of targets --
  // go to a pair-mode sub-plan; device-resident applies run the remaining
  // tiles + the sub-plan, host-pipelined applies the full tile plan
  std::shared_ptr<HybridPlan> hyb;
};

struct HybridPlan {
  HostPlan main;  // the kept target tiles, longest first
  int64_t n_long = 0;  // leading tiles with the most entries (the rest run at the end of a launch)
  DevBuf tile_col, tile_off, entry_code, entry_src;
  LevelPlan aux;  // pair-mode plan of the leftover targets
};

// Pair-mode levels of one homogeneous full-operator group merged into one
// plan: pairs with the same transfer vector from different levels share 64-
// column entries (their operators differ only by the level scale, which the
// per-level reductions apply), so small sparse levels stop streaming a whole
// operator per nearly empty entry.  Per pair the product is computed exactly
// as in the level's own plan and every target sums its pairs in the same
// order, so results are bitwise those of the per-level plans.
struct MergedPairPlan {
  std::vector<int> levels;
  std::vector<uint64_t> gens;
  std::vector<int64_t> row_off;  // source row offset of each level in the padded buffer
  HostPlan hp;
  DevBuf tile_col, tile_off, entry_code, entry_src, entry_ncols;
  std::vector<PairReduce> red;  // per level: frows into the merged per-pair rows
  std::vector<DevBuf> r_tgt, r_off, r_frow;
};

}  // namespace cfm

using namespace cfm;

struct AuxStream {
  cudaStream_t s = nullptr;
  cudaEvent_t done = nullptr;
};
struct CsrPlanEntry {  // one cached plan of cfm_apply_level_csr and the exact batch it was built from
  int level = 0, dc_flag = 0;
  int64_t n_rows = 0;
  std::vector<int64_t> tgt, off, src;
  std::vector<int8_t> t;
  LevelPlan plan;
  size_t host_bytes() const { return (tgt.size() + off.size() + src.size()) * 8 + t.size(); }
};

struct LevelScratch {  // per-level scratch of concurrently applied levels
  DevBuf fbuf, xpad, ybuf;
  std::vector<int64_t> xpad_sig;
};

struct cfm_handler {
  int device = 0, variant = 0, order = 0, op_complex = 0;
  int n = 0, f = 1;
  bool sym = false, lowrank = false, shared = false;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  DevBuf rowtab, invtab;  // [48][n f] int16
  DevBuf zeros;           // zero row for bulk copies past an operator
  std::map<int, Group> groups;
  std::map<int, std::pair<int, double>> levels;
  std::map<int, LevelPlan> plans;
  std::list<CsrPlanEntry> csr_cache;  // plans of ad-hoc CSR batches (cfm_apply_level_csr), most recent first
  size_t csr_cache_bytes = 0;
  DevBuf x_stage, y_stage, ybuf, wt, z, fbuf, fzbuf, counters, pipe_flags;
  DevBuf xpad;                     // zero-padded source rows of full-operator levels
  long long wt_ld_zeroed = -1;     // SA: leading dimension the W~ padding was zeroed for
  std::unique_ptr<MergedPairPlan> merged;
  std::vector<int64_t> xpad_sig;   // layout the padding columns were zeroed for
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr, s_late = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr, ev_prev = nullptr, ev_x = nullptr;
  cudaEvent_t ev_late0 = nullptr, ev_late1 = nullptr;
  cudaStream_t s_mid = nullptr;  // middle launch group (e2e): its sources cross PCIe during the first launch
  cudaEvent_t ev_mid = nullptr, ev_mid1 = nullptr;
  cudaStream_t s_pad = nullptr;  // pads pipelined full-operator slabs beside the running grid
  cudaEvent_t ev_slab[16] = {}, ev_pad_done = nullptr;
  cudaEvent_t ev_last = nullptr;  // end of the previous apply's work
  cudaEvent_t ev_fork = nullptr;
  std::vector<AuxStream> aux;
  std::vector<LevelScratch> lvl_scratch;
  cudaStream_t last_stream = nullptr;
  bool have_last = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double last_ms = 0.0;
  int64_t last_launches = 0;
  bool last_csr_hit = false;  // the last cfm_apply_level_csr reused a cached plan
  int last_csr_mode = -1, last_csr_two_stage = 0;  // and that plan's mode / two-stage flag
};

namespace cfm {

// ------------------------------------------------------------------ launching
// Kernel selection (CFM_TILE_KERNEL): "ws32" warp-specialized KC=32 x 3 stages
// with TMA bulk copies of the operator rows (default, CFM_BULK_A=1), "ws16"
// KC=16 x 5 stages, "sync" the lockstep kernel, "ws16w"
// like ws16 with 16 consumer warps (32x16 warp tiles) on 128-row blocks.
// Default by inner length (measured, profiles/r01_summary.md): KC=32 with bulk
// operator rows up to nk = 512 (l <= 7), KC=16 with cp.async rows above (l = 9).
static int tile_kernel_kind(int nk = 0) {
  static int forced = [] {
    const char* v = getenv("CFM_TILE_KERNEL");
    if (!v) return -1;
    if (!strcmp(v, "ws32")) return 0;
    if (!strcmp(v, "ws16")) return 1;
    if (!strcmp(v, "sync")) return 2;
    if (!strcmp(v, "ws16w")) return 3;
    return -1;
  }();
  if (forced >= 0) return forced;
  return nk > 512 ? 1 : 0;
}

static bool use_bulk_a(int kc) {
  static int v = [] {
    const char* e = getenv("CFM_BULK_A");
    return e ? atoi(e) : -1;
  }();
  if (v >= 0) return v != 0;
  return kc >= 32;  // 256-B row chunks: bulk copies win; 128-B: cp.async wins
}

// cuTensorMapEncodeTiled, resolved at run time like the stream memory ops.
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiled resolve_encode_tiled() {
  static PFN_encodeTiled fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<PFN_encodeTiled>(nullptr);
    }
    return reinterpret_cast<PFN_encodeTiled>(f);
  }();
  return fn;
}

// Full-operator mode: the 2-D map over a segment's padded source rows
// (x_ld doubles x x_rows rows) read by tile::gather4 copies, box (KC + 4) x 1
// so each gathered row lands with the stage's LDB pitch; columns past x_ld and
// rows < 0 (empty plan slots) are out of bounds and arrive as zeros.
static void encode_source_map(TileParams& q, int kc) {
  const cuuint64_t dims[2] = {cuuint64_t(q.x_ld), cuuint64_t(std::max<long long>(q.x_rows, 1))};
  const cuuint64_t strides[1] = {cuuint64_t(q.x_ld) * sizeof(double)};
  const cuuint32_t box[2] = {cuuint32_t(kc + 4), q.b_block ? cuuint32_t(kBN) : 1u};  // b_block: one entry's rows
  const cuuint32_t estr[2] = {1u, 1u};
  const CUresult r = resolve_encode_tiled()(&q.tmap_b, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(q.x),
                                            dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(CFM_ERR_CUDA, "cuTensorMapEncodeTiled failed for the source rows");
}

static bool ft_pipe_enabled() {
  static const int v = [] {
    const char* e = getenv("CFM_FT_PIPE");
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}

// CFM_LATE_STREAM=0: later launch groups on the caller's stream, after the first
static bool use_late_stream() {
  static const bool v = [] {
    const char* e = getenv("CFM_LATE_STREAM");
    return !e || atoi(e) != 0;
  }();
  return v;
}

// CFM_MID_GROUP=0: with host buffers next to a pipelined level, the largest
// other target-tile level stays in the first launch (its upload then delays
// the first launch; with the middle group it crosses PCIe during that launch)
static bool mid_group_enabled() {
  static const bool v = [] {
    const char* e = getenv("CFM_MID_GROUP");
    return !e || atoi(e) != 0;
  }();
  return v;
}

// CFM_EARLY_TGT_D2H=0: first-group target-tile levels download after the whole call
static bool early_tgt_d2h() {
  static const bool v = [] {
    const char* e = getenv("CFM_EARLY_TGT_D2H");
    return !e || atoi(e) != 0;
  }();
  return v;
}

// CFM_KTAIL=0: the last k-step of l = 5 operators as a DMMA over zero padding (A/B)
// (read at every launch, so a test can compare both in one process)
static bool ktail_enabled() {
  const char* e = getenv("CFM_KTAIL");
  return !e || atoi(e) != 0;
}

template <int BM, int BN, int WM, int WN, int KC, int STAGES, bool SKIP>
static void launch_ws_multi(const MultiTileParams& mp_in, dim3 grid_tiles, cudaStream_t s) {
  // grid_tiles = (tiles, row blocks) -> one CTA per (tile, row block), row blocks fastest
  MultiTileParams mp = mp_in;
  mp.nrb = int(grid_tiles.y);
  const dim3 grid(unsigned(grid_tiles.x) * grid_tiles.y, 1);
  if ((long long)grid_tiles.x * grid_tiles.y >= (1ll << 31)) throw Error(CFM_ERR_VALUE, "too many tiles for one launch");
  const TileParams& q = mp.seg[0];
  const bool tabs = tile_perm_tabs_fit(q.nr, q.nk);
  const int smem = ws_ring_bytes<BM, BN, KC, STAGES>() + tile_table_bytes(q.nr, q.nk, tabs);
  if constexpr (BM == 128 && KC == 32 && !SKIP) {
    if (q.ft) {
      // tile skipping pays when a warp has no rows in the last row block or a
      // segment is a pair plan; otherwise the plain full-operator kernel
      static const int skip_env = [] {
        const char* e = getenv("CFM_FT_SKIP");
        return e ? atoi(e) : -1;
      }();
      // (measured: the skipping kernel is ~1% slower when nothing is skipped)
      long long pair_e = 0, all_e = 0;
      for (int i = 0; i < mp.n_seg; ++i) {
        all_e += mp.seg[i].n_entries;
        if (mp.seg[i].entry_ncols) pair_e += mp.seg[i].n_entries;
      }
      bool skip = int(mp.nrb) * BM - q.nr >= 32 || 4 * pair_e >= all_e;
      if (skip_env >= 0) skip = skip_env != 0;
      const int smem_ft = ws_ring_bytes<BM, BN, KC, 4>() + tile_table_bytes(q.nr, q.nk, false) + kMaxTileEntries;
      // the flat pipelined consumer loop runs whole KC-chunks: only when the last
      // chunk of an operator has KC/4 k-steps anyway (l = 5: 125 = 3 x 32 + 29)
      static const int hints_env = [] {
        const char* e = getenv("CFM_L2_HINTS");
        return e ? atoi(e) : 0;  // measured: no gain (the operator stack stays L2-resident anyway)
      }();
      for (int i = 0; i < mp.n_seg; ++i) {
        encode_source_map(mp.seg[i], KC);
        mp.seg[i].l2_hints = hints_env;
        const int rem = mp.seg[i].nk % KC;
        mp.seg[i].ft_pipe = ft_pipe_enabled() && (rem == 0 || rem > KC - 4) && !mp.seg[i].op_klen;
        mp.seg[i].ft_ktail = mp.seg[i].ft_pipe && rem == KC - 3 && !mp.seg[i].op_rows && ktail_enabled();
      }
      auto kf = q.y_map ? tile_gemm_ws_kernel<BM, BN, WM, WN, KC, 4, SKIP, false, 3>
                : skip    ? tile_gemm_ws_kernel<BM, BN, WM, WN, KC, 4, SKIP, false, 2>
                          : tile_gemm_ws_kernel<BM, BN, WM, WN, KC, 4, SKIP, false, 1>;
      CUDA_CHECK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_ft));
      kf<<<grid, (WM * WN + 4) * 32, smem_ft, s>>>(mp);
      return;
    }
  }
  if constexpr (BM == 128) {
    if (use_bulk_a(KC) && q.zero_row && q.op_ld <= 8192) {
      auto kb = tile_gemm_ws_kernel<BM, BN, WM, WN, KC, STAGES, SKIP, true>;
      CUDA_CHECK(cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      kb<<<grid, (WM * WN + 4) * 32, smem, s>>>(mp);
      return;
    }
  }
  auto kern = tile_gemm_ws_kernel<BM, BN, WM, WN, KC, STAGES, SKIP>;
  CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<grid, (WM * WN + 4) * 32, smem, s>>>(mp);
}

template <int BM, int BN, int WM, int WN, int KC, int STAGES, bool SKIP>
static void launch_ws(const TileParams& q, dim3 grid, cudaStream_t s) {
  MultiTileParams mp{};
  mp.n_seg = 1;
  mp.start[0] = 0;
  mp.start[1] = int(grid.x);
  mp.seg[0] = q;
  launch_ws_multi<BM, BN, WM, WN, KC, STAGES, SKIP>(mp, grid, s);
}

template <int BM, int BN, int WM, int WN, bool SKIP>
static void launch_sync(const TileParams& q, dim3 grid, cudaStream_t s) {
  constexpr int STAGES = 3;
  const bool tabs = tile_perm_tabs_fit(q.nr, q.nk);
  const int smem = tile_ring_bytes<BM, BN, kKC, STAGES>() + tile_table_bytes(q.nr, q.nk, tabs);
  auto kern = tile_gemm_kernel<BM, BN, WM, WN, kKC, STAGES, SKIP>;
  CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<grid, WM * WN * 32, smem, s>>>(q);
}

template <int BM, int BN, int WM, int WN>
static void launch_cfg(const TileParams& p, int n_tiles, int tile_base, cudaStream_t s) {
  TileParams q = p;
  q.tile_base = tile_base;
  dim3 grid(n_tiles, (p.nr + BM - 1) / BM);
  const int kind = p.ft ? 0 : ((p.pair_out && tile_kernel_kind(p.nk) == 2) ? 1 : tile_kernel_kind(p.nk));
  if (p.op_rows) {
    if (kind == 2) launch_sync<BM, BN, WM, WN, true>(q, grid, s);
    else if (kind == 1) launch_ws<BM, BN, WM, WN, 16, 5, true>(q, grid, s);
    else launch_ws<BM, BN, WM, WN, 32, 3, true>(q, grid, s);
  } else {
    if (kind == 2) launch_sync<BM, BN, WM, WN, false>(q, grid, s);
    else if (kind == 1) launch_ws<BM, BN, WM, WN, 16, 5, false>(q, grid, s);
    else launch_ws<BM, BN, WM, WN, 32, 3, false>(q, grid, s);
  }
  CUDA_CHECK(cudaGetLastError());
}

// ---- fused low-rank kernel (phase 1 + phase 2 in one CTA)
// Driver stream-memory ops resolved at run time (no link-time libcuda
// dependency, so the library still loads on machines without a driver).
typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static PFN_writeValue32 p_writeValue32 = nullptr;
static PFN_waitValue32 p_waitValue32 = nullptr;
static bool resolve_stream_mem_ops() {
  static int ok = [] {
    cudaDriverEntryPointQueryResult q1, q2;
    void* f1 = nullptr;
    void* f2 = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f1, cudaEnableDefault, &q1) != cudaSuccess ||
        cudaGetDriverEntryPoint("cuStreamWaitValue32", &f2, cudaEnableDefault, &q2) != cudaSuccess ||
        q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess || !f1 || !f2) {
      cudaGetLastError();
      return 0;
    }
    p_writeValue32 = reinterpret_cast<PFN_writeValue32>(f1);
    p_waitValue32 = reinterpret_cast<PFN_waitValue32>(f2);
    return 1;
  }();
  return ok != 0;
}

static bool use_copy_pipeline() {
  static int v = [] {
    const char* e = getenv("CFM_COPY_PIPELINE");
    return e ? atoi(e) : 1;
  }();
  return v != 0 && resolve_stream_mem_ops();
}

static bool use_concurrent_levels() {
  static int v = [] {
    const char* e = getenv("CFM_CONCURRENT_LEVELS");
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}

static bool use_fused_lowrank() {
  static int v = [] {
    const char* e = getenv("CFM_LOWRANK_FUSED");
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}


// Full-operator TMA mode (CFM_FULL_OPS=0 disables): real dense groups with
// 64 < n <= 1024 (l = 5..10); always the 128-row KC=32 kernel.
static bool use_full_ops(const cfm_handler* h) {
  static int v = [] {
    const char* e = getenv("CFM_FULL_OPS");
    return e ? atoi(e) : 1;
  }();
  const int nf = h->n * h->f;
  return v != 0 && !h->op_complex && nf > 64 && nf <= 1024 && resolve_encode_tiled() != nullptr;
}

template <int RP, int STAGES, bool VB, int KC = 16>
static bool launch_lowrank_cfg(LowRankParams lp_, int64_t first, int64_t count, cudaStream_t s) {
  const int fixed = lr_smem_bytes<RP, KC, STAGES>() + 4 * 64 + 3 * 4 * 344 + 4 * kMaxTileEntries;
  if (lp_.n_ops > 344 || fixed > 227 * 1024) return false;
  const int tabs = 48 * 2 * (lp_.nr + lp_.nk + 8);
  lp_.tabs_smem = (fixed + tabs <= 227 * 1024) ? 1 : 0;
  const int smem = fixed + (lp_.tabs_smem ? tabs : 0);
  auto kern = lowrank_ws_kernel<RP, KC, STAGES, VB>;
  CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int64_t max_grid = 1 << 30;
  for (int64_t base = first; base < first + count; base += max_grid) {
    const int nt = int(std::min<int64_t>(max_grid, first + count - base));
    LowRankParams q = lp_;
    q.tile_base = int(base);
    dim3 grid(nt, (lp_.nr + 127) / 128);
    kern<<<grid, 12 * 32, smem, s>>>(q);
    CUDA_CHECK(cudaGetLastError());
  }
  return true;
}

static bool launch_lowrank_fused(const LowRankParams& lp_, int rmax, int64_t first, int64_t count, cudaStream_t s,
                                 bool vb = false) {
  if (!use_fused_lowrank()) return false;
  static const int kc_env = [] {
    const char* e = getenv("CFM_LR_KC");
    return e ? atoi(e) : 16;
  }();
  if (vb) {
    if (kc_env == 32) {
      if (rmax <= 16) return launch_lowrank_cfg<16, 3, true, 32>(lp_, first, count, s);
      if (rmax <= 32) return launch_lowrank_cfg<32, 2, true, 32>(lp_, first, count, s);
    }
    if (rmax <= 16) return launch_lowrank_cfg<16, 5, true>(lp_, first, count, s);
    if (rmax <= 32) return launch_lowrank_cfg<32, 4, true>(lp_, first, count, s);
    if (rmax <= 64) return launch_lowrank_cfg<64, 2, true>(lp_, first, count, s);
    return false;
  }
  if (rmax <= 16) return launch_lowrank_cfg<16, 5, false>(lp_, first, count, s);
  if (rmax <= 32) return launch_lowrank_cfg<32, 4, false>(lp_, first, count, s);
  if (rmax <= 64) return launch_lowrank_cfg<64, 2, false>(lp_, first, count, s);
  return false;
}

// One launch over several tile lists sharing operator shapes (all levels of a
// homogeneous dense group).  Segments are launched in the given order.
static int64_t launch_multi(const std::vector<TileParams>& segs, const std::vector<int64_t>& counts, cudaStream_t s) {
  MultiTileParams mp{};
  int64_t total = 0;
  mp.n_seg = 0;
  for (size_t i = 0; i < segs.size(); ++i) {
    if (counts[i] == 0) continue;
    if (mp.n_seg == kMaxSegments) throw Error(CFM_ERR_VALUE, "too many levels in one launch");
    mp.start[mp.n_seg] = int(total);
    mp.seg[mp.n_seg] = segs[i];  // (tile_base: first tile of the segment in its plan)
    total += counts[i];
    ++mp.n_seg;
  }
  if (mp.n_seg == 0) return 0;
  if (total >= (int64_t(1) << 31)) throw Error(CFM_ERR_VALUE, "too many tiles for one launch");
  mp.start[mp.n_seg] = int(total);
  const TileParams& q = mp.seg[0];
  const int kind = q.ft ? 0 : tile_kernel_kind(q.nk);
  if (q.nr <= 32) {
    dim3 grid(unsigned(total), (q.nr + 31) / 32);
    if (kind == 0) launch_ws_multi<32, kBN, 1, 8, 32, 3, false>(mp, grid, s);
    else launch_ws_multi<32, kBN, 1, 8, 16, 5, false>(mp, grid, s);
  } else if (q.nr <= 64) {
    dim3 grid(unsigned(total), (q.nr + 63) / 64);
    if (kind == 0) launch_ws_multi<64, kBN, 2, 4, 32, 3, false>(mp, grid, s);
    else launch_ws_multi<64, kBN, 2, 4, 16, 5, false>(mp, grid, s);
  } else {
    dim3 grid(unsigned(total), (q.nr + 127) / 128);
    if (kind == 0) launch_ws_multi<128, kBN, 4, 2, 32, 3, false>(mp, grid, s);
    else if (kind == 3) launch_ws_multi<128, kBN, 4, 4, 16, 5, false>(mp, grid, s);
    else launch_ws_multi<128, kBN, 4, 2, 16, 5, false>(mp, grid, s);
  }
  CUDA_CHECK(cudaGetLastError());
  return 1;
}

// Launch tiles [first, first + count) of the plan in p.
static int64_t launch_range(const TileParams& p, int64_t first, int64_t count, cudaStream_t s) {
  int64_t launches = 0;
  const int64_t max_grid = 1 << 30;
  for (int64_t base = first; base < first + count; base += max_grid) {
    const int nt = int(std::min<int64_t>(max_grid, first + count - base));
    if (nt <= 0) break;
    if (p.nr <= 32)
      launch_cfg<32, kBN, 1, 8>(p, nt, int(base), s);
    else if (p.nr <= 64)
      launch_cfg<64, kBN, 2, 4>(p, nt, int(base), s);
    else
      launch_cfg<128, kBN, 4, 2>(p, nt, int(base), s);
    ++launches;
  }
  return launches;
}

static int64_t launch_tiles(const TileParams& p, int64_t n_tiles, cudaStream_t s) {
  return launch_range(p, 0, n_tiles, s);
}

// Two-stage low-rank stage 2 on seg_pair_gemm_kernel (two 16-wide rank
// segments per pipeline stage); CFM_SEG_PAIR=0 runs the KC = 16 full-operator
// kernel instead.
static int64_t launch_seg_pair(TileParams q, int64_t n_tiles, cudaStream_t s) {
  if (n_tiles <= 0) return 0;
  if (n_tiles >= (int64_t(1) << 31)) throw Error(CFM_ERR_VALUE, "too many tiles for one launch");
  q.tile_base = 0;
  encode_source_map(q, 16);
  const int smem = seg_pair_smem_bytes();
  CUDA_CHECK(cudaFuncSetAttribute(seg_pair_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  seg_pair_gemm_kernel<<<unsigned(n_tiles), 12 * 32, smem, s>>>(q);
  CUDA_CHECK(cudaGetLastError());
  return 1;
}

// Full-operator kernel with 16-wide K chunks (two-stage low-rank stage 2: one
// chunk per rank segment), one segment, pipelined consumer loop.
static int64_t launch_ft16(TileParams q, int64_t n_tiles, cudaStream_t s) {
  constexpr int KC = 16, STAGES = 6;
  if (n_tiles <= 0) return 0;
  if (n_tiles >= (int64_t(1) << 31)) throw Error(CFM_ERR_VALUE, "too many tiles for one launch");
  MultiTileParams mp{};
  mp.n_seg = 1;
  mp.nrb = 1;
  mp.start[0] = 0;
  mp.start[1] = int(n_tiles);
  q.tile_base = 0;
  encode_source_map(q, KC);
  q.ft_pipe = ft_pipe_enabled() && q.nk % KC == 0;
  q.l2_hints = getenv("CFM_L2_HINTS") ? atoi(getenv("CFM_L2_HINTS")) : 0;
  mp.seg[0] = q;
  auto kf = tile_gemm_ws_kernel<128, kBN, 4, 2, KC, STAGES, false, false, 1>;
  const int smem = ws_ring_bytes<128, kBN, KC, STAGES>() + tile_table_bytes(q.nr, q.nk, false) + kMaxTileEntries;
  CUDA_CHECK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kf<<<unsigned(n_tiles), (4 * 2 + 4) * 32, smem, s>>>(mp);
  CUDA_CHECK(cudaGetLastError());
  return 1;
}

static void fill_ops(TileParams& p, const OpStack& s, const CodeMap& m) {
  p.ops = s.d.as<double>();
  p.op_stride = s.stride;
  p.op_ld = s.ld;
  p.nr = s.rows;
  p.nk = s.cols;
  p.op_rows = s.has_rows ? s.d_rows.as<int>() : nullptr;
  p.op_klen = s.has_klen ? s.d_klen.as<int>() : nullptr;
  p.code_op = m.d_op.as<int>();
  p.code_rperm = m.d_rperm.as<int>();
  p.code_cperm = m.d_cperm.as<int>();
}

static void fill_plan(TileParams& p, const DevBuf& col, const DevBuf& toff, const DevBuf& code, const DevBuf& src,
                      int64_t n_tiles) {
  p.n_tiles = int(n_tiles);
  p.tile_col = col.as<int>();
  p.tile_off = toff.as<int>();
  p.entry_code = code.as<int>();
  p.entry_src = src.as<int>();
}

static void push_plan(const HostPlan& hp, DevBuf& col, DevBuf& toff, DevBuf& code, DevBuf& src) {
  upload(col, hp.tile_col);
  upload(toff, hp.tile_off);
  upload(code, hp.entry_code);
  upload(src, hp.entry_src);
}

static bool is_device_ptr(const void* ptr) {
  if (!ptr) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// ------------------------------------------------------------------ handler ops
static void build_tables(cfm_handler* h) {
  const int nf = h->n * h->f;
  std::vector<int16_t> row(size_t(kNumPerms) * nf), inv(size_t(kNumPerms) * nf);
  for (int pid = 0; pid < kNumPerms; ++pid) {
    auto tab = permutation_table(pid, h->order);
    auto itab = inverse_table(tab);
    for (int i = 0; i < h->n; ++i)
      for (int q = 0; q < h->f; ++q) {
        row[size_t(pid) * nf + i * h->f + q] = int16_t(tab[i] * h->f + q);
        inv[size_t(pid) * nf + i * h->f + q] = int16_t(itab[i] * h->f + q);
      }
  }
  upload(h->rowtab, row);
  upload(h->invtab, inv);
}

// Map every transfer of the group to (op index, perm) following the variant:
// symmetric variants go through canonicalize (symmetry.py:63-75, lookup :142-144),
// plain ones index the operator of t itself.
static void map_transfers(cfm_handler* h, Group& g, int n_transfers, const int8_t* transfers, int n_ops,
                          const int8_t* op_t, bool rows_permuted, bool cols_permuted, CodeMap& m) {
  std::array<int, kNumCodes> op_of_code;
  op_of_code.fill(-1);
  for (int i = 0; i < n_ops; ++i) {
    const int t0 = op_t[3 * i], t1 = op_t[3 * i + 1], t2 = op_t[3 * i + 2];
    if (t0 < -3 || t0 > 3 || t1 < -3 || t1 > 3 || t2 < -3 || t2 > 3)
      throw Error(CFM_ERR_VALUE, "operator transfer vector outside [-3,3]^3");
    op_of_code[tcode(t0, t1, t2)] = i;
  }
  for (int k = 0; k < n_transfers; ++k) {
    const int t0 = transfers[3 * k], t1 = transfers[3 * k + 1], t2 = transfers[3 * k + 2];
    if (t0 < -3 || t0 > 3 || t1 < -3 || t1 > 3 || t2 < -3 || t2 > 3)
      throw Error(CFM_ERR_VALUE, "transfer vector outside [-3,3]^3");
    const int c = tcode(t0, t1, t2);
    g.valid[c] = 1;
    if (h->sym) {
      int ts[3], pid;
      canonicalize(t0, t1, t2, ts, pid);
      const int o = op_of_code[tcode(ts[0], ts[1], ts[2])];
      if (o < 0) throw Error(CFM_ERR_PRECOMPUTE, "no representative operator for a transfer vector");
      m.op[c] = o;
      m.rperm[c] = rows_permuted ? pid : -1;
      m.cperm[c] = cols_permuted ? pid : -1;
    } else {
      const int o = op_of_code[c];
      if (o < 0) throw Error(CFM_ERR_PRECOMPUTE, "no operator for a transfer vector");
      m.op[c] = o;
    }
  }
}

static void make_stack(OpStack& s, int n_ops, int rows, int cols);
static void put_stack(OpStack& s, int i, const std::vector<double>& hostblock);

// Full-operator stack for the TMA tile kernel: K_t[i][j] = Op[tab_r[i]][tab_c[j]]
// for every transfer of the group (the same products the permuted apply forms,
// acc[i] += sum_k Op[rowtab[i]][k] x[invtab[k]] with j = invtab[k]), rows padded
// to a multiple of 8, columns to the KC multiple; plus the 2-D tensor map.
static void build_full_ops(cfm_handler* h, Group& g, int n_transfers, const int8_t* transfers, const double* ops) {
  const int n = h->n;
  const int rows = round_up(n, 8);
  OpStack& fs = g.full;
  make_stack(fs, n_transfers, rows, n);
  g.full_rows = rows;
  std::vector<double> blockv(fs.stride);
  std::vector<int> ident(n);
  std::iota(ident.begin(), ident.end(), 0);
  for (int k = 0; k < n_transfers; ++k) {
    const int c = tcode(transfers[3 * k], transfers[3 * k + 1], transfers[3 * k + 2]);
    const int o = g.main.op[c], rp = g.main.rperm[c], cp = g.main.cperm[c];
    const std::vector<int> tr = rp >= 0 ? permutation_table(rp, h->order) : ident;
    const std::vector<int> tc = cp >= 0 ? permutation_table(cp, h->order) : ident;
    std::fill(blockv.begin(), blockv.end(), 0.0);
    const double* src = ops + size_t(o) * n * n;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) blockv[size_t(i) * fs.ld + j] = src[size_t(tr[i]) * n + tc[j]];
    put_stack(fs, k, blockv);
    g.fullmap.op[c] = k;
  }
  g.fullmap.push();
  const cuuint64_t dims[2] = {cuuint64_t(fs.ld), cuuint64_t(n_transfers) * rows};
  const cuuint64_t strides[1] = {cuuint64_t(fs.ld) * sizeof(double)};
  const cuuint32_t box[2] = {cuuint32_t(kKC + 4), 128u};
  const cuuint32_t estr[2] = {1u, 1u};
  const CUresult r = resolve_encode_tiled()(&g.full_tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, fs.d.p, dims, strides,
                                            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(CFM_ERR_CUDA, "cuTensorMapEncodeTiled failed for the operator stack");
  g.has_full = true;
}

static void make_stack(OpStack& s, int n_ops, int rows, int cols) {
  s.n_ops = n_ops;
  s.rows = rows;
  s.cols = cols;
  s.ld = round_up(std::max(cols, 1), kKC);
  s.stride = (long long)rows * s.ld;
  s.d.alloc(std::max<size_t>(size_t(n_ops) * s.stride * sizeof(double), 16));
  CUDA_CHECK(cudaMemset(s.d.p, 0, s.d.bytes));
}

static void put_stack(OpStack& s, int i, const std::vector<double>& hostblock) {
  CUDA_CHECK(cudaMemcpy(s.d.as<double>() + (size_t)i * s.stride, hostblock.data(),
                        hostblock.size() * sizeof(double), cudaMemcpyHostToDevice));
}

static void set_per_op(OpStack& s, const std::vector<int>& rows, const std::vector<int>& klen) {
  if (!rows.empty()) {
    upload(s.d_rows, rows);
    s.has_rows = true;
  }
  if (!klen.empty()) {
    upload(s.d_klen, klen);
    s.has_klen = true;
  }
}

// Low-rank factor stacks: pass 1 op = right^H (r f x n f), pass 2 op = left (n f x r f).
static void build_lowrank_stacks(cfm_handler* h, OpStack& left, OpStack& right_h, int n_ops, const int* ranks,
                                 const double* L, const double* R, int rows_left, int rows_right) {
  // rows_left: rows of left (n or r_u); rows_right: rows of right (n or r_b)
  const int f = h->f;
  const bool cplx = h->op_complex;
  int rmax = 0;
  for (int i = 0; i < n_ops; ++i) rmax = std::max(rmax, ranks[i]);
  make_stack(left, n_ops, rows_left * f, std::max(rmax * f, 1));
  make_stack(right_h, n_ops, std::max(rmax * f, 1), rows_right * f);
  std::vector<int> rrows(n_ops), rk(n_ops);
  size_t offL = 0, offR = 0;
  const int sc = cplx ? 2 : 1;
  for (int i = 0; i < n_ops; ++i) {
    const int r = ranks[i];
    rrows[i] = r * f;
    rk[i] = r * f;
    std::vector<double> bl((size_t)left.stride, 0.0), br((size_t)right_h.stride, 0.0);
    if (r > 0) {
      realify_into(L + offL, rows_left, r, cplx, bl.data(), left.ld);
      realify_into(R + offR, r, rows_right, cplx, br.data(), right_h.ld, /*conj_t=*/true);
    }
    put_stack(left, i, bl);
    put_stack(right_h, i, br);
    offL += (size_t)rows_left * r * sc;
    offR += (size_t)rows_right * r * sc;
    left.host_bytes += (size_t)rows_left * r * sc * 8;
    right_h.host_bytes += (size_t)rows_right * r * sc * 8;
  }
  set_per_op(left, {}, rk);       // pass 2: inner length = rank
  set_per_op(right_h, rrows, {});  // pass 1: rows = rank
}

static bool use_two_stage() {  // read at every precompute (tests switch it)
  const char* e = getenv("CFM_LR_TWOSTAGE");
  return !e || atoi(e) != 0;
}

// Two-stage low-rank operators (see Group::has_ts): per class the V_t^H rows
// of its transfers in 16-row segments, and the tensor maps of both stages.
static void build_two_stage(cfm_handler* h, Group& g, int n_transfers, const int8_t* transfers,
                            const std::vector<int>& rk, const std::vector<double>& all_v) {
  g.has_ts = false;
  if (!use_two_stage()) return;
  const int n = h->n;
  int rmax = 0;
  for (int r : rk) rmax = std::max(rmax, r);
  if (rmax == 0 || rmax > 32 || g.lrf_left.ld != 32) return;
  g.ts_ntr = n_transfers;
  g.ts_rank = rk;
  g.ts_slot.assign(size_t(8) * n_transfers * 2, -1);
  int max_slots = 0;
  for (int cls = 0; cls < 8; ++cls) {
    int ns = 0;
    for (int k = 0; k < n_transfers; ++k) {
      bool in = rk[k] > 0;
      for (int a = 0; a < 3 && in; ++a) {
        const int t = transfers[3 * k + a], bit = (cls >> a) & 1;
        in = t >= (bit ? -2 : -3) && t <= (bit ? 3 : 2);
      }
      if (!in) continue;
      for (int j = 0; j * 16 < rk[k]; ++j) g.ts_slot[(size_t(cls) * n_transfers + k) * 2 + j] = ns++;
    }
    max_slots = std::max(max_slots, ns);
  }
  const int nb = (max_slots * 16 + 127) / 128;
  g.ts_nb = nb;
  make_stack(g.ts_v, 8 * nb, 128, n);
  const int vld = g.lrf_right_h.ld;
  const size_t vstride = size_t(g.lrf_right_h.stride);
  std::vector<double> blk(size_t(g.ts_v.stride));
  for (int cls = 0; cls < 8; ++cls)
    for (int b = 0; b < nb; ++b) {
      std::fill(blk.begin(), blk.end(), 0.0);
      for (int k = 0; k < n_transfers; ++k)
        for (int j = 0; j < 2; ++j) {
          const int sl = g.ts_slot[(size_t(cls) * n_transfers + k) * 2 + j];
          if (sl < 0 || sl / 8 != b) continue;
          for (int a = 0; a < 16 && 16 * j + a < rk[k]; ++a)
            std::copy_n(all_v.begin() + size_t(k) * vstride + size_t(16 * j + a) * vld, n,
                        blk.begin() + size_t((sl % 8) * 16 + a) * g.ts_v.ld);
        }
      put_stack(g.ts_v, cls * nb + b, blk);
    }
  auto encode = [](CUtensorMap* m, const OpStack& st, long long rows, unsigned box0) {
    const cuuint64_t dims[2] = {cuuint64_t(st.ld), cuuint64_t(rows)};
    const cuuint64_t strides[1] = {cuuint64_t(st.ld) * sizeof(double)};
    const cuuint32_t box[2] = {box0, 128u};
    const cuuint32_t estr[2] = {1u, 1u};
    const CUresult r = resolve_encode_tiled()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, st.d.p, dims, strides, box, estr,
                                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(CFM_ERR_CUDA, "cuTensorMapEncodeTiled failed for a two-stage stack");
  };
  encode(&g.ts_vmap, g.ts_v, (long long)8 * nb * 128, kKC + 4);
  encode(&g.ts_umap, g.lrf_left, (long long)n_transfers * n, 16 + 4);
  // stage 2 skips the k-steps of a 16-wide rank segment past the rank: their
  // U_t columns and Y rows are exact zeros, so the sums are unchanged
  std::vector<int> ks(size_t(2) * n_transfers, 0);
  for (int k = 0; k < n_transfers; ++k)
    for (int j = 0; j < 2; ++j) {
      const int w = std::min(16, std::max(0, rk[k] - 16 * j));
      ks[size_t(2) * k + j] = (w + 3) / 4;
    }
  upload(g.ts_ksteps, ks);
  g.has_ts = true;
}

// Per-transfer low-rank factors for real operators: U_t[i][a] = left_o[tab_r[i]][a],
// V_t^H[a][j] = right_o[tab_c[j]][a] (the products the permuted apply forms:
// Y[a] = sum_k right^H[a][k] x[inv[k]] = sum_j right^H[a][tab[j]] x[j]).
static void build_lowrank_full(cfm_handler* h, Group& g, int n_transfers, const int8_t* transfers, int n_ops,
                               const int* ranks, const double* L, const double* R) {
  const int n = h->n;
  int rmax = 0;
  for (int i = 0; i < n_ops; ++i) rmax = std::max(rmax, ranks[i]);
  std::vector<size_t> off(n_ops + 1, 0);
  for (int i = 0; i < n_ops; ++i) off[i + 1] = off[i] + size_t(n) * ranks[i];
  make_stack(g.lrf_left, n_transfers, n, std::max(rmax, 1));
  make_stack(g.lrf_right_h, n_transfers, std::max(rmax, 1), n);
  std::vector<int> ident(n), rk(n_transfers);
  std::iota(ident.begin(), ident.end(), 0);
  std::vector<double> bl(g.lrf_left.stride), br(g.lrf_right_h.stride);
  std::vector<double> all_v(size_t(n_transfers) * g.lrf_right_h.stride);
  for (int k = 0; k < n_transfers; ++k) {
    const int c = tcode(transfers[3 * k], transfers[3 * k + 1], transfers[3 * k + 2]);
    const int o = g.main.op[c];
    const std::vector<int> tr = g.main.rperm[c] >= 0 ? permutation_table(g.main.rperm[c], h->order) : ident;
    const std::vector<int> tc = g.pass1.cperm[c] >= 0 ? permutation_table(g.pass1.cperm[c], h->order) : ident;
    const int r = ranks[o];
    rk[k] = r;
    std::fill(bl.begin(), bl.end(), 0.0);
    std::fill(br.begin(), br.end(), 0.0);
    const double* Lo = L + off[o];
    const double* Ro = R + off[o];
    for (int i = 0; i < n; ++i)
      for (int a = 0; a < r; ++a) bl[size_t(i) * g.lrf_left.ld + a] = Lo[size_t(tr[i]) * r + a];
    for (int a = 0; a < r; ++a)
      for (int j = 0; j < n; ++j) br[size_t(a) * g.lrf_right_h.ld + j] = Ro[size_t(tc[j]) * r + a];
    put_stack(g.lrf_left, k, bl);
    put_stack(g.lrf_right_h, k, br);
    std::copy(br.begin(), br.end(), all_v.begin() + size_t(k) * br.size());
    g.fullmap.op[c] = k;
  }
  g.fullmap.push();
  set_per_op(g.lrf_left, {}, rk);
  set_per_op(g.lrf_right_h, rk, {});
  g.has_lrfull = true;
  build_two_stage(h, g, n_transfers, transfers, rk, all_v);
}

// ------------------------------------------------------------------ planning
static std::vector<int16_t> codes_from_t(int64_t P, const int8_t* t) {
  std::vector<int16_t> codes(P);
  for (int64_t q = 0; q < P; ++q) {
    const int t0 = t[3 * q], t1 = t[3 * q + 1], t2 = t[3 * q + 2];
    if (t0 < -3 || t0 > 3 || t1 < -3 || t1 > 3 || t2 < -3 || t2 > 3) {
      throw Error(CFM_ERR_PRECOMPUTE, "no operator for transfer vector (" + std::to_string(t0) + ", " +
                                          std::to_string(t1) + ", " + std::to_string(t2) + ")");
    }
    codes[q] = int16_t(tcode(t0, t1, t2));
  }
  return codes;
}

static Group& group_for_level(cfm_handler* h, int level) {
  auto it = h->levels.find(level);
  if (it == h->levels.end())
    throw Error(CFM_ERR_PRECOMPUTE, "no operators precomputed for level " + std::to_string(level));
  auto git = h->groups.find(it->second.first);
  if (git == h->groups.end()) throw Error(CFM_ERR_PRECOMPUTE, "level group has no operators");
  return git->second;
}

// Two-stage low-rank plans from a level's target-tile plan (Group::has_ts).
// Stage 1: source tiles (64 sources of one class) x ts_nb entries (one per
// 128-row block of the class stack), pair-mode output rows v = e * 64 + c
// written as 8 segments of 16 at a 20-double pitch.  Stage 2: the target tiles
// with every entry (t, 64 sources) split into its rank segments j, operator id
// 2 k + j (k = transfer index), source ids = stage-1 segment rows.  Taken only
// when stage 1 computes at most ~1.7x the segments the pairs need and the
// stage-1 output fits CFM_LR_TWOSTAGE_GB (default 24 GB).
static void build_two_stage_plan(const Group& g, LevelPlan& lp) {
  const HostPlan& hp = lp.hp;
  const int64_t n_rows = lp.n_rows;
  const int ntr = g.ts_ntr, nb = g.ts_nb;
  std::vector<int8_t> mn(size_t(n_rows) * 3, 127), mx(size_t(n_rows) * 3, -128);
  std::vector<char> used(n_rows, 0);
  int64_t need_segs = 0;
  const int64_t E = hp.n_entries();
  for (int64_t e = 0; e < E; ++e) {
    const int c = hp.entry_code[e];
    const int k = g.fullmap.op[c];
    if (k < 0 || k >= ntr || g.ts_rank[k] <= 0) return;
    int t[3];
    tcode_decode(c, t[0], t[1], t[2]);
    const int nseg = (g.ts_rank[k] + 15) / 16;
    for (int col = 0; col < kBN; ++col) {
      const int v = hp.entry_src[size_t(e) * kBN + col];
      if (v < 0) continue;
      used[v] = 1;
      need_segs += nseg;
      for (int a = 0; a < 3; ++a) {
        mn[size_t(v) * 3 + a] = std::min<int8_t>(mn[size_t(v) * 3 + a], int8_t(t[a]));
        mx[size_t(v) * 3 + a] = std::max<int8_t>(mx[size_t(v) * 3 + a], int8_t(t[a]));
      }
    }
  }
  std::vector<int8_t> cls(n_rows, -1);
  std::vector<std::vector<int64_t>> by_cls(8);
  for (int64_t v = 0; v < n_rows; ++v) {
    if (!used[v]) continue;
    int b = 0;
    for (int a = 0; a < 3; ++a) {
      if (mx[size_t(v) * 3 + a] <= 2) continue;        // fits [-3, 2]
      if (mn[size_t(v) * 3 + a] >= -2) b |= 1 << a;     // fits [-2, 3]
      else return;                                      // not an octree far list
    }
    cls[v] = int8_t(b);
    by_cls[b].push_back(v);
  }
  // stage 1 plan
  HostPlan p1;
  std::vector<int> tile1(n_rows, -1), col1(n_rows, -1);
  for (int b = 0; b < 8; ++b)
    for (size_t i = 0; i < by_cls[b].size(); i += kBN) {
      const int64_t t = p1.n_tiles++;
      p1.tile_off.push_back(int(p1.entry_code.size()));
      std::vector<int> cols(kBN, -1);
      for (int c = 0; c < kBN && i + c < by_cls[b].size(); ++c) {
        const int64_t v = by_cls[b][i + c];
        cols[c] = int(v);
        tile1[v] = int(t);
        col1[v] = c;
      }
      p1.tile_col.insert(p1.tile_col.end(), cols.begin(), cols.end());
      for (int blk = 0; blk < nb; ++blk) {
        p1.entry_code.push_back(b * nb + blk);
        p1.entry_src.insert(p1.entry_src.end(), cols.begin(), cols.end());
      }
    }
  p1.tile_off.push_back(int(p1.entry_code.size()));
  const int64_t segs1 = p1.n_entries() * kBN * 8;
  static const double budget_gb = [] {
    const char* e = getenv("CFM_LR_TWOSTAGE_GB");
    return e ? atof(e) : 24.0;
  }();
  if (segs1 >= (int64_t(1) << 31) || double(need_segs) * 1.2 * 20 * 8 > budget_gb * 1e9) return;
  if (double(p1.n_tiles) * kBN * nb * 8 > 1.7 * double(need_segs)) return;  // sparse level: fused kernel
  // stage 2 plan; its B rows (entry e2, column c) = the stage-1 segment of that pair
  std::vector<int> ymap(size_t(segs1), -1);
  HostPlan p2;
  p2.n_tiles = hp.n_tiles;
  p2.tile_col = hp.tile_col;
  p2.tile_off.reserve(hp.n_tiles + 1);
  for (int64_t t = 0; t < hp.n_tiles; ++t) {
    p2.tile_off.push_back(int(p2.entry_code.size()));
    for (int e = hp.tile_off[t]; e < hp.tile_off[t + 1]; ++e) {
      const int c = hp.entry_code[e];
      const int k = g.fullmap.op[c];
      for (int j = 0; j * 16 < g.ts_rank[k]; ++j) {
        p2.entry_code.push_back(2 * k + j);
        for (int col = 0; col < kBN; ++col) {
          const int v = hp.entry_src[size_t(e) * kBN + col];
          int id = -1;
          if (v >= 0) {
            const int sl = g.ts_slot[(size_t(cls[v]) * ntr + k) * 2 + j];
            if (sl < 0) return;
            id = int(((int64_t(tile1[v]) * nb + sl / 8) * kBN + col1[v]) * 8 + sl % 8);
            const int64_t row2 = int64_t(p2.entry_code.size() - 1) * kBN + col;
            if (row2 >= (int64_t(1) << 31)) return;
            ymap[size_t(id)] = int(row2);
          }
          p2.entry_src.push_back(id);
        }
      }
    }
  }
  p2.tile_off.push_back(int(p2.entry_code.size()));
  lp.ts1 = std::move(p1);
  lp.ts2 = std::move(p2);
  push_plan(lp.ts1, lp.ts1_col, lp.ts1_off, lp.ts1_code, lp.ts1_src);
  push_plan(lp.ts2, lp.ts2_col, lp.ts2_off, lp.ts2_code, lp.ts2_src);
  upload(lp.ts_map, ymap);
  lp.ts_segs = lp.ts2.n_entries() * kBN;
  lp.ts = true;
}

static bool full_mode(const Group& g, const LevelPlan& lp) { return g.kind == kDense && g.has_full && lp.dc == 1; }

// Hybrid plans (CFM_HYBRID=0 disables): measured at config 2 the step kernel
// drops 50.56 -> 50.28 ms; with all reductions of a step in one launch the
// step goes 50.60 -> 50.41 ms.  Read at every plan build; a forced
// CFM_PLAN_MODE disables it.
static bool use_hybrid() {
  const char* e = getenv("CFM_HYBRID");
  return (!e || atoi(e) != 0) && !getenv("CFM_PLAN_MODE");
}

// Upload a pair-mode plan's device arrays (entries, reduction, filled columns).
static void push_pair_plan(LevelPlan& lp) {
  push_plan(lp.hp, lp.tile_col, lp.tile_off, lp.entry_code, lp.entry_src);
  upload(lp.r_tgt, lp.red.tgt);
  upload(lp.r_off, lp.red.off);
  upload(lp.r_frow, lp.red.frow);
  const int64_t E = lp.hp.n_entries();
  std::vector<unsigned char> nc(std::max<int64_t>(E, 1), 0);
  for (int64_t e = 0; e < E; ++e)
    for (int c = kBN - 1; c >= 0; --c)
      if (lp.hp.entry_src[size_t(e) * kBN + c] >= 0) {
        nc[e] = static_cast<unsigned char>(c + 1);
        break;
      }
  upload(lp.entry_ncols, nc);
}

// Hybrid split of a dense full-operator target-tile plan (LevelPlan::hyb).
static void build_hybrid_plan(cfm_handler* h, LevelPlan& lp, int64_t n_targets, const int64_t* tgt,
                              const int64_t* off, const int64_t* src, const int16_t* codes,
                              const std::array<int, kNumCodes>& key) {
  const HostPlan& hp = lp.hp;
  std::vector<char> leftover_tile(hp.n_tiles, 0);
  std::vector<char> leftover_row(lp.n_rows, 0);
  int64_t n_left = 0;
  for (int64_t t = 0; t < hp.n_tiles; ++t) {
    int64_t valid = 0;
    const int64_t slots = int64_t(hp.tile_off[t + 1] - hp.tile_off[t]) * kBN;
    for (int e = hp.tile_off[t]; e < hp.tile_off[t + 1]; ++e)
      for (int c = 0; c < kBN; ++c) valid += hp.entry_src[size_t(e) * kBN + c] >= 0;
    if (slots == 0 || 2 * valid >= slots) continue;
    leftover_tile[t] = 1;
    ++n_left;
    for (int c = 0; c < kBN; ++c) {
      const int v = hp.tile_col[size_t(t) * kBN + c];
      if (v >= 0) leftover_row[v] = 1;
    }
  }
  if (n_left == 0 || n_left == hp.n_tiles) return;
  auto hy = std::make_shared<HybridPlan>();
  HostPlan& mn = hy->main;
  mn.bn = hp.bn;
  mn.dc = hp.dc;
  // kept tiles longest first (row order kept among equally long tiles): the
  // shorter boundary-class tiles run last and fill the launch's tail (this
  // plan only serves device-resident applies, which need no row order)
  std::vector<int64_t> kept;
  for (int64_t t = 0; t < hp.n_tiles; ++t)
    if (!leftover_tile[t]) kept.push_back(t);
  std::stable_sort(kept.begin(), kept.end(), [&](int64_t a, int64_t b) {
    return hp.tile_off[a + 1] - hp.tile_off[a] > hp.tile_off[b + 1] - hp.tile_off[b];
  });
  const int max_e = kept.empty() ? 0 : hp.tile_off[kept[0] + 1] - hp.tile_off[kept[0]];
  for (int64_t t : kept) hy->n_long += (hp.tile_off[t + 1] - hp.tile_off[t]) * 10 >= max_e * 9;
  for (int64_t t : kept) {
    mn.tile_col.insert(mn.tile_col.end(), hp.tile_col.begin() + t * kBN, hp.tile_col.begin() + (t + 1) * kBN);
    mn.tile_off.push_back(int(mn.entry_code.size()));
    for (int e = hp.tile_off[t]; e < hp.tile_off[t + 1]; ++e) {
      mn.entry_code.push_back(hp.entry_code[e]);
      mn.entry_src.insert(mn.entry_src.end(), hp.entry_src.begin() + size_t(e) * kBN,
                          hp.entry_src.begin() + size_t(e + 1) * kBN);
    }
    ++mn.n_tiles;
  }
  mn.tile_off.push_back(int(mn.entry_code.size()));
  // leftover targets' far lists (CSR order kept) -> pair entries
  std::vector<int64_t> t2, o2{0}, s2;
  std::vector<int16_t> c2;
  for (int64_t i = 0; i < n_targets; ++i) {
    if (off[i + 1] <= off[i] || !leftover_row[tgt[i]]) continue;
    t2.push_back(tgt[i]);
    for (int64_t q = off[i]; q < off[i + 1]; ++q) {
      s2.push_back(src[q]);
      c2.push_back(codes[q]);
    }
    o2.push_back(int64_t(s2.size()));
  }
  LevelPlan& ax = hy->aux;
  const int nkp = round_up(h->n * h->f, kKC);
  const int64_t e_est = int64_t(s2.size()) / kBN + 1;
  int ept = std::max(1, std::min(16, int(2.5e7 / (2.0 * 128 * kBN * nkp))));
  ept = std::min<int>(ept, int(std::max<int64_t>(1, e_est / (2 * 148))));
  ax.hp = build_plan_pairs(int64_t(t2.size()), t2.data(), o2.data(), s2.data(), c2.data(), 1, key, lp.n_rows, ept,
                           ax.red);
  ax.mode = 1;
  ax.dc = 1;
  ax.n_rows = lp.n_rows;
  push_pair_plan(ax);
  static uint64_t hyb_gen = uint64_t(1) << 62;
  ax.gen = ++hyb_gen;
  push_plan(mn, hy->tile_col, hy->tile_off, hy->entry_code, hy->entry_src);
  lp.hyb = std::move(hy);
}

static LevelPlan build_level_plan(cfm_handler* h, int level, int64_t n_targets, const int64_t* tgt,
                                  const int64_t* off, const int64_t* src, const int16_t* codes, int data_complex,
                                  int64_t n_rows) {
  Group& g = group_for_level(h, level);
  const int dc = (data_complex && !h->op_complex) ? 2 : 1;
  if (h->op_complex && !data_complex)
    throw Error(CFM_ERR_VALUE, "complex operators need complex128 expansions (engine.py:99)");
  std::array<int, kNumCodes> key;
  for (int c = 0; c < kNumCodes; ++c) key[c] = g.valid[c] ? std::max(g.main.op[c], 0) + 1 : -1;
  if (g.kind == kShared)
    for (int c = 0; c < kNumCodes; ++c) key[c] = g.valid[c] ? c : -1;
  LevelPlan lp;
  try {
    lp.hp = build_plan_csr(n_targets, tgt, off, src, codes, dc, key, n_rows);
    const double slots = double(lp.hp.n_entries()) * kBN;
    lp.target_fill = slots > 0 ? double(lp.hp.n_pairs) * dc / slots : 1.0;
    const char* m = getenv("CFM_PLAN_MODE");
    const bool force_pair = m && !strcmp(m, "pair");
    const bool force_target = m && !strcmp(m, "target");
    if (force_pair || (!force_target && lp.target_fill < 0.6)) {
      // dense: ~25 MFLOP of row-block work per CTA (l = 9: 2 entries, l = 5: 11) so
      // sparse levels still give many waves of CTAs and a short tail
      const int nkp = round_up(h->n * h->f, kKC);
      static const int ept_env = [] {
        const char* e = getenv("CFM_PAIR_EPT");
        return e ? atoi(e) : 0;
      }();
      // ... and at least ~2 CTAs per SM where the level has the entries for it
      // (a small level in few long CTAs is latency-bound)
      const int64_t e_est = lp.hp.n_pairs * dc / kBN + 1;
      const int ept_occ = int(std::max<int64_t>(1, e_est / (2 * 148)));
      int ept = g.kind == kDense ? std::max(1, std::min(16, int(2.5e7 / (2.0 * 128 * kBN * nkp)))) : 16;
      ept = std::min(ept, ept_occ);
      if (ept_env > 0) ept = ept_env;
      lp.hp = build_plan_pairs(n_targets, tgt, off, src, codes, dc, key, n_rows, ept, lp.red);
      lp.mode = 1;
      upload(lp.r_tgt, lp.red.tgt);
      upload(lp.r_off, lp.red.off);
      upload(lp.r_frow, lp.red.frow);
    }
  } catch (const PlanError& e) {
    throw Error(e.code == 2 ? CFM_ERR_PRECOMPUTE : CFM_ERR_VALUE, e.what());
  }
  lp.dc = dc;
  lp.n_rows = n_rows;
  push_plan(lp.hp, lp.tile_col, lp.tile_off, lp.entry_code, lp.entry_src);
  const int64_t E = lp.hp.n_entries();
  if (lp.mode == 1) {
    // filled columns per pair entry (slots are filled from column 0): the
    // full-operator kernel skips the empty trailing 8-column tiles
    std::vector<unsigned char> nc(std::max<int64_t>(E, 1), 0);
    for (int64_t e = 0; e < E; ++e)
      for (int c = kBN - 1; c >= 0; --c)
        if (lp.hp.entry_src[size_t(e) * kBN + c] >= 0) {
          nc[e] = static_cast<unsigned char>(c + 1);
          break;
        }
    upload(lp.entry_ncols, nc);
  }
  if (g.kind == kLowRank || (g.kind == kShared && g.any_fac_core)) {
    std::vector<int> slots(size_t(E) * kBN), iota(E + 1);
    for (int64_t e = 0; e < E; ++e)
      for (int c = 0; c < kBN; ++c)
        slots[size_t(e) * kBN + c] = lp.hp.entry_src[size_t(e) * kBN + c] >= 0 ? int(e * kBN + c) : -1;
    std::iota(iota.begin(), iota.end(), 0);
    upload(lp.slot_ids, slots);
    upload(lp.iota, iota);
    // runs of <= kPass1Run entries that never cross a tile boundary, so a tile
    // range [t0, t1) maps to the run range [run_start[t0], run_start[t1])
    std::vector<int> runs;
    lp.run_start.assign(lp.hp.n_tiles + 1, 0);
    for (int64_t t = 0; t < lp.hp.n_tiles; ++t) {
      lp.run_start[t] = int64_t(runs.size());
      for (int e = lp.hp.tile_off[t]; e < lp.hp.tile_off[t + 1]; e += kPass1Run) runs.push_back(e);
    }
    lp.run_start[lp.hp.n_tiles] = int64_t(runs.size());
    runs.push_back(int(E));
    lp.n_runs = int64_t(runs.size()) - 1;
    upload(lp.runs, runs);
  }
  // distinct targets / sources (SA transforms and accounting)
  {
    std::vector<char> seen_t(n_rows, 0), seen_s(n_rows, 0);
    for (int64_t i = 0; i < n_targets; ++i)
      if (off[i + 1] > off[i]) {
        seen_t[tgt[i]] = 1;
        for (int64_t q = off[i]; q < off[i + 1]; ++q) seen_s[src[q]] = 1;
      }
    for (int64_t r = 0; r < n_rows; ++r) {
      if (seen_t[r]) lp.targets.push_back(r);
      if (seen_s[r]) lp.sources.push_back(r);
    }
  }
  if (g.kind == kShared) {
    lp.src_plan = build_identity_plan(lp.sources, dc);
    lp.tgt_plan = build_identity_plan(lp.targets, dc);
    push_plan(lp.src_plan, lp.s_tile_col, lp.s_tile_off, lp.s_entry_code, lp.s_entry_src);
    push_plan(lp.tgt_plan, lp.t_tile_col, lp.t_tile_off, lp.t_entry_code, lp.t_entry_src);
  }
  if (lp.mode == 0 && lp.hp.n_tiles > 0) {
    // dispatch order ~ row order (tiles stay class-pure; a target's entry order
    // is unchanged, so results are bitwise identical), which lets the host
    // copies of multipoles/locals run in row slabs alongside the kernel
    HostPlan& hp = lp.hp;
    const int64_t nt = hp.n_tiles;
    std::vector<int64_t> tmin(nt, INT64_MAX);
    for (int64_t t = 0; t < nt; ++t)
      for (int c = 0; c < kBN; ++c) {
        const int v = hp.tile_col[size_t(t) * kBN + c];
        if (v >= 0) tmin[t] = std::min<int64_t>(tmin[t], v / dc);
      }
    std::vector<int64_t> ord(nt);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return tmin[a] < tmin[b]; });
    HostPlan np_;
    np_.bn = hp.bn; np_.dc = hp.dc; np_.n_tiles = nt; np_.n_pairs = hp.n_pairs; np_.code_count = hp.code_count;
    np_.tile_col.resize(hp.tile_col.size());
    np_.tile_off.resize(nt + 1);
    np_.entry_code.reserve(hp.entry_code.size());
    np_.entry_src.reserve(hp.entry_src.size());
    for (int64_t k = 0; k < nt; ++k) {
      const int64_t t = ord[k];
      std::copy(hp.tile_col.begin() + t * kBN, hp.tile_col.begin() + (t + 1) * kBN, np_.tile_col.begin() + k * kBN);
      np_.tile_off[k] = int(np_.entry_code.size());
      for (int e = hp.tile_off[t]; e < hp.tile_off[t + 1]; ++e) {
        np_.entry_code.push_back(hp.entry_code[e]);
        np_.entry_src.insert(np_.entry_src.end(), hp.entry_src.begin() + size_t(e) * kBN,
                             hp.entry_src.begin() + size_t(e + 1) * kBN);
      }
    }
    np_.tile_off[nt] = int(np_.entry_code.size());
    lp.hp = std::move(np_);
    push_plan(lp.hp, lp.tile_col, lp.tile_off, lp.entry_code, lp.entry_src);
    // slabs of ~32K rows (at most 16); CFM_SLAB_ROWS / CFM_MAX_SLABS for experiments
    static const int64_t slab_rows = [] {
      const char* e = getenv("CFM_SLAB_ROWS");
      return e ? std::max<int64_t>(1024, atoll(e)) : int64_t(32768);
    }();
    static const int64_t max_slabs = [] {
      const char* e = getenv("CFM_MAX_SLABS");
      return e ? std::max<int64_t>(2, atoll(e)) : int64_t(16);
    }();
    static const int64_t min_rows = [] {  // levels with fewer rows are not host-pipelined
      const char* e = getenv("CFM_PIPE_MIN_ROWS");
      return e ? atoll(e) : int64_t(0);
    }();
    int S = int(std::min<int64_t>(max_slabs, std::max<int64_t>(1, n_rows / slab_rows)));
    if (min_rows > 0) S = n_rows >= min_rows ? std::max(S, 2) : 1;
    // the last slab's download cannot start before the kernel's last wave
    // ends: split it into halves, quarters, eighths (CFM_SLAB_TAIL=0: uniform)
    static const int slab_tail = [] {
      const char* e = getenv("CFM_SLAB_TAIL");
      return e ? std::max(0, atoi(e)) : 3;
    }();
    lp.slab_row0.clear();
    for (int k = 0; k < S; ++k) lp.slab_row0.push_back(n_rows * k / S);
    if (S >= 2) {
      const int64_t a = n_rows * (S - 1) / S, len = n_rows - a;
      int64_t r = a;
      for (int d = 1; d <= slab_tail && S + d <= 16 && (len >> d) >= 1024; ++d) {
        r += len >> d;
        lp.slab_row0.push_back(r);
      }
    }
    lp.slab_row0.push_back(n_rows);
    const int S_all = int(lp.slab_row0.size()) - 1;
    lp.n_slabs = S_all;
    auto slab_of = [&](int64_t row) {
      const auto it = std::upper_bound(lp.slab_row0.begin(), lp.slab_row0.end(), row);
      return int(std::min<int64_t>(S_all - 1, std::max<int64_t>(0, (it - lp.slab_row0.begin()) - 1)));
    };
    std::vector<int> need_mp(nt, 0), need_loc(nt, 0), lo(nt, 0), hi(nt, -1);
    lp.slab_expected.assign(S_all, 0);
    const int nrb = (group_for_level(h, level).dense.rows + 127) / 128;
    for (int64_t t = 0; t < nt; ++t) {
      int l = S_all, hh = -1, m = 0;
      for (int c = 0; c < kBN; ++c) {
        const int v = lp.hp.tile_col[size_t(t) * kBN + c];
        if (v < 0) continue;
        const int k = slab_of(v / dc);
        l = std::min(l, k);
        hh = std::max(hh, k);
      }
      for (int e = lp.hp.tile_off[t]; e < lp.hp.tile_off[t + 1]; ++e)
        for (int c = 0; c < kBN; ++c) {
          const int v = lp.hp.entry_src[size_t(e) * kBN + c];
          if (v >= 0) m = std::max(m, slab_of(v / dc) + 1);
        }
      if (hh < 0) { l = 0; hh = -1; }
      need_mp[t] = m;
      need_loc[t] = hh + 1;
      lo[t] = l;
      hi[t] = hh;
      for (int k = l; k <= hh; ++k) lp.slab_expected[k] += unsigned(nrb);
    }
    upload(lp.p_need_mp, need_mp);
    upload(lp.p_need_loc, need_loc);
    upload(lp.p_lo, lo);
    upload(lp.p_hi, hi);
  }
  if (g.kind == kLowRank && g.has_ts && lp.mode == 0 && dc == 1 && lp.hp.n_tiles > 0) build_two_stage_plan(g, lp);
  if (use_hybrid() && full_mode(g, lp) && lp.mode == 0 && lp.hp.n_tiles > 0) {
    try {
      build_hybrid_plan(h, lp, n_targets, tgt, off, src, codes, key);
    } catch (const PlanError& e) {
      throw Error(e.code == 2 ? CFM_ERR_PRECOMPUTE : CFM_ERR_VALUE, e.what());
    }
  }
  static std::atomic<uint64_t> plan_gen{0};
  lp.gen = ++plan_gen;
  return lp;
}

// The level's cached plan (plan_level_* / plan_level_csr; apply_planned and
// apply_levels run it).  Ad-hoc batches of cfm_apply_level_csr never land here
// (they use the CSR plan cache below), so a cached plan is only replaced by an
// explicit re-plan of its level.
static LevelPlan& make_plan(cfm_handler* h, int level, int64_t n_targets, const int64_t* tgt, const int64_t* off,
                            const int64_t* src, const int16_t* codes, int data_complex, int64_t n_rows) {
  LevelPlan lp = build_level_plan(h, level, n_targets, tgt, off, src, codes, data_complex, n_rows);
  h->plans[level] = std::move(lp);
  return h->plans[level];
}

// Plans of the reference call path (apply_level with a batch, engine.py:140-157):
// FmmPlan rebuilds the same batches on every run (engine.py:98-120), so a plan is
// cached under its exact CSR content (targets, offsets, sources, transfer vectors,
// row count, data kind) and reused when the same batch comes back.  Keys are
// compared in full (memcmp), never by hash alone.
static constexpr size_t kCsrCacheMaxEntries = 64;
static constexpr size_t kCsrCacheMaxBytes = size_t(8) << 30;

static LevelPlan& csr_plan(cfm_handler* h, int level, int64_t n_targets, const int64_t* tgt, const int64_t* off,
                           const int64_t* src, const int8_t* t, int data_complex, int64_t n_rows, bool* hit_out) {
  const int64_t P = n_targets ? off[n_targets] : 0;
  for (auto it = h->csr_cache.begin(); it != h->csr_cache.end(); ++it) {
    CsrPlanEntry& e = *it;
    if (e.level != level || e.dc_flag != data_complex || e.n_rows != n_rows || int64_t(e.tgt.size()) != n_targets ||
        int64_t(e.src.size()) != P)
      continue;
    if (n_targets && std::memcmp(e.tgt.data(), tgt, size_t(n_targets) * 8)) continue;
    if (std::memcmp(e.off.data(), off, size_t(n_targets + 1) * 8)) continue;
    if (P && std::memcmp(e.src.data(), src, size_t(P) * 8)) continue;
    if (P && std::memcmp(e.t.data(), t, size_t(P) * 3)) continue;
    h->csr_cache.splice(h->csr_cache.begin(), h->csr_cache, it);  // most recently used first
    if (hit_out) *hit_out = true;
    return h->csr_cache.front().plan;
  }
  if (hit_out) *hit_out = false;
  auto codes = codes_from_t(P, t);
  CsrPlanEntry e;
  e.plan = build_level_plan(h, level, n_targets, tgt, off, src, codes.data(), data_complex, n_rows);
  e.level = level;
  e.dc_flag = data_complex;
  e.n_rows = n_rows;
  e.tgt.assign(tgt, tgt + n_targets);
  e.off.assign(off, off + n_targets + 1);
  e.src.assign(src, src + P);
  e.t.assign(t, t + 3 * P);
  const size_t bytes = e.host_bytes();
  h->csr_cache.push_front(std::move(e));
  h->csr_cache_bytes += bytes;
  while (h->csr_cache.size() > 1 &&
         (h->csr_cache.size() > kCsrCacheMaxEntries || h->csr_cache_bytes > kCsrCacheMaxBytes)) {
    h->csr_cache_bytes -= h->csr_cache.back().host_bytes();
    h->csr_cache.pop_back();
  }
  return h->csr_cache.front().plan;
}

// ------------------------------------------------------------------ apply
static void ensure(DevBuf& b, size_t bytes) { b.alloc(std::max<size_t>(bytes, 16)); }

static int64_t launch_reduce(const LevelPlan& lp, const double* F, long long f_ld, double* y, long long y_ld, int len,
                             double scale, cudaStream_t s) {
  const int64_t nt = int64_t(lp.red.tgt.size());
  if (nt == 0) return 0;
  k_pair_reduce<<<unsigned(nt), 128, 0, s>>>(F, f_ld, lp.r_tgt.as<long long>(), lp.r_off.as<long long>(),
                                             lp.r_frow.as<int>(), nt, y, y_ld, len, scale, 1);
  CUDA_CHECK(cudaGetLastError());
  return 1;
}

// ---- full-operator mode: sources as zero-padded rows (ld = group full.ld)

// Reserve h->xpad for levels of (rows, ld) and return each level's offset (in
// doubles); the padding columns are zeroed whenever the layout changes (rows
// are only ever written in their first n columns afterwards).
static std::vector<size_t> xpad_layout(cfm_handler* h, const std::vector<std::pair<int64_t, int>>& lay, cudaStream_t s) {
  std::vector<size_t> off(lay.size());
  std::vector<int64_t> sig;
  size_t total = 0;
  for (size_t i = 0; i < lay.size(); ++i) {
    off[i] = total;
    total += size_t(lay[i].first) * size_t(lay[i].second);
    sig.push_back(lay[i].first);
    sig.push_back(lay[i].second);
  }
  const size_t bytes = std::max<size_t>(total * sizeof(double), 16);
  const bool grow = !h->xpad.p || bytes > h->xpad.bytes;
  ensure(h->xpad, bytes);
  if (grow || sig != h->xpad_sig) {
    CUDA_CHECK(cudaMemsetAsync(h->xpad.p, 0, bytes, s));
    h->xpad_sig = sig;
  }
  return off;
}

// Zero-padded copy of rows: dst[r][k] = k < n ? src[r][k] : 0 for k < ld, whole
// destination rows written (coalesced on both sides, memory-bound).  Replaces a
// pitched device-to-device cudaMemcpy2D, measured at ~1.5 ms for config 2's
// 262 MB level 6 (this kernel: ~0.1 ms).
constexpr int kPadRowsPerBlock = 16;
// Zero-padded source rows for the full-operator TMA path: rows of n doubles
// -> rows of ld doubles.  Several arrays (the levels of a step) in one launch;
// a warp copies whole rows (coalesced 256-B loads and stores, no division).
struct PadJob {
  double* dst;
  const double* src;
  long long rows;
  long long blk0;  // first block of this job
  int ld, n;
};
constexpr int kMaxPadJobs = 8;
struct PadJobs {
  PadJob j[kMaxPadJobs];
  int n;
};

__global__ void __launch_bounds__(256) k_pad_rows(const PadJobs jobs) {
  int q = 0;
  while (q + 1 < jobs.n && (long long)blockIdx.x >= jobs.j[q + 1].blk0) ++q;
  const PadJob& J = jobs.j[q];
  const long long r0 = ((long long)blockIdx.x - J.blk0) * kPadRowsPerBlock;
  const int nr = int(J.rows - r0 < kPadRowsPerBlock ? J.rows - r0 : kPadRowsPerBlock);
  const int lane = threadIdx.x & 31;
  for (int r = threadIdx.x >> 5; r < nr; r += blockDim.x >> 5) {
    const double* sr = J.src + (r0 + r) * J.n;
    double* dr = J.dst + (r0 + r) * J.ld;
    for (int k = lane; k < J.ld; k += 32) dr[k] = k < J.n ? __ldcs(sr + k) : 0.0;
  }
}

static int64_t launch_pads(const std::vector<PadJob>& in, cudaStream_t s, int threads = 256) {
  int64_t n_launch = 0;
  for (size_t a = 0; a < in.size(); a += kMaxPadJobs) {
    PadJobs jobs{};
    long long blocks = 0;
    for (size_t b = a; b < in.size() && b < a + kMaxPadJobs; ++b) {
      PadJob J = in[b];
      J.blk0 = blocks;
      blocks += (J.rows + kPadRowsPerBlock - 1) / kPadRowsPerBlock;
      jobs.j[jobs.n++] = J;
    }
    if (blocks == 0) continue;
    if (blocks >= (1ll << 31)) throw Error(CFM_ERR_VALUE, "too many rows to pad");
    k_pad_rows<<<unsigned(blocks), threads, 0, s>>>(jobs);
    CUDA_CHECK(cudaGetLastError());
    ++n_launch;
  }
  return n_launch;
}

// rows [r0, r1) of a (rows x n) source array (host or device) into the padded layout
// Returns the kernels launched (0 for a batched job or a host source).
static int64_t xpad_copy(cfm_handler* h, double* dst, int ld, const double* src, int64_t r0, int64_t r1, cudaStream_t s,
                      int threads = 256, std::vector<PadJob>* batch = nullptr) {
  if (r1 <= r0) return 0;
  if (is_device_ptr(src)) {
    const PadJob J{dst + size_t(r0) * ld, src + size_t(r0) * h->n, (long long)(r1 - r0), 0, ld, h->n};
    if (batch) {
      batch->push_back(J);
      return 0;
    }
    return launch_pads({J}, s, threads);
  }
  CUDA_CHECK(cudaMemcpy2DAsync(dst + size_t(r0) * ld, size_t(ld) * sizeof(double), src + size_t(r0) * h->n,
                               size_t(h->n) * sizeof(double), size_t(h->n) * sizeof(double), size_t(r1 - r0),
                               cudaMemcpyDefault, s));
  return 0;
}

static void fill_full(TileParams& p, const cfm_handler* h, const Group& g, const double* xpad, int64_t x_rows) {
  fill_ops(p, g.full, g.fullmap);
  p.nr = h->n;
  p.nk = h->n;
  p.rowtab = nullptr;
  p.invtab = nullptr;
  p.ft = 1;
  p.ft_rows = g.full_rows;
  p.tmap_a = g.full_tmap;
  p.x = xpad;
  p.x_ld = g.full.ld;
  p.x_dc = 1;
  p.x_rows = x_rows;
}

static int64_t run_plan(cfm_handler* h, int level, LevelPlan& lp, const double* d_x, double* d_y, cudaStream_t s) {
  Group& g = group_for_level(h, level);
  const double scale = h->levels[level].second;
  const int dc = lp.dc;
  const int nf = h->n * h->f;
  const long long row_ld = (long long)h->n * (dc == 2 || h->op_complex ? 2 : 1);  // doubles per expansion row
  int64_t launches = 0;
  const int64_t E = lp.hp.n_entries();
  if (lp.hp.n_tiles == 0) return 0;

  TileParams p{};
  p.rowtab = h->rowtab.as<short>();
  p.invtab = h->invtab.as<short>();
  p.zero_row = h->zeros.as<double>();

  if (g.kind == kDense) {
    fill_ops(p, g.dense, g.main);
    fill_plan(p, lp.tile_col, lp.tile_off, lp.entry_code, lp.entry_src, lp.hp.n_tiles);
    p.x = d_x; p.x_ld = row_ld; p.x_dc = dc;
    if (full_mode(g, lp)) {
      const auto off = xpad_layout(h, {{lp.n_rows, g.full.ld}}, s);
      double* xp = h->xpad.as<double>() + off[0];
      launches += xpad_copy(h, xp, g.full.ld, d_x, 0, lp.n_rows, s);
      fill_full(p, h, g, xp, lp.n_rows);
      if (lp.mode == 1) p.entry_ncols = lp.entry_ncols.as<unsigned char>();
      p.n_entries = lp.hp.n_entries();
    }
    if (lp.mode == 1) {
      ensure(h->fbuf, size_t(lp.red.n_frows) * row_ld * sizeof(double));
      p.y = h->fbuf.as<double>(); p.y_ld = row_ld; p.y_dc = dc;
      p.scale = 1.0; p.accumulate = 0; p.pair_out = 1;
      launches += launch_tiles(p, lp.hp.n_tiles, s);
      launches += launch_reduce(lp, h->fbuf.as<double>(), row_ld, d_y, row_ld, int(row_ld), scale, s);
      return launches;
    }
    p.y = d_y; p.y_ld = row_ld; p.y_dc = dc;
    p.scale = scale; p.accumulate = 1;
    if (lp.hyb && full_mode(g, lp)) {
      // hybrid: the kept target tiles, then the leftover targets in pair mode
      const HybridPlan& hy = *lp.hyb;
      fill_plan(p, hy.tile_col, hy.tile_off, hy.entry_code, hy.entry_src, hy.main.n_tiles);
      p.n_entries = hy.main.n_entries();
      launches += launch_tiles(p, hy.main.n_tiles, s);
      const LevelPlan& ax = hy.aux;
      TileParams q = p;
      fill_plan(q, ax.tile_col, ax.tile_off, ax.entry_code, ax.entry_src, ax.hp.n_tiles);
      q.entry_ncols = ax.entry_ncols.as<unsigned char>();
      q.n_entries = ax.hp.n_entries();
      ensure(h->fbuf, size_t(ax.red.n_frows) * row_ld * sizeof(double));
      q.y = h->fbuf.as<double>(); q.y_ld = row_ld; q.y_dc = dc;
      q.scale = 1.0; q.accumulate = 0; q.pair_out = 1;
      launches += launch_tiles(q, ax.hp.n_tiles, s);
      launches += launch_reduce(ax, h->fbuf.as<double>(), row_ld, d_y, row_ld, int(row_ld), scale, s);
      return launches;
    }
    launches += launch_tiles(p, lp.hp.n_tiles, s);
    return launches;
  }

  if (g.kind == kLowRank && lp.ts) {
    // two-stage low-rank: stage 1 Y = V^H x per (source, class segment), stage 2
    // locals += scale * sum U_t Y per target tile (both on the full-operator kernel)
    const int ldx = g.ts_v.ld;
    const auto xo = xpad_layout(h, {{lp.n_rows, ldx}}, s);
    double* xp = h->xpad.as<double>() + xo[0];
    launches += xpad_copy(h, xp, ldx, d_x, 0, lp.n_rows, s);
    if (!lp.ts_y.p) {
      lp.ts_y.alloc(size_t(lp.ts_segs) * 20 * sizeof(double));
      CUDA_CHECK(cudaMemsetAsync(lp.ts_y.p, 0, lp.ts_y.bytes, s));  // segment pads stay zero
    }
    TileParams a{};
    fill_ops(a, g.ts_v, g.main);
    fill_plan(a, lp.ts1_col, lp.ts1_off, lp.ts1_code, lp.ts1_src, lp.ts1.n_tiles);
    a.op_rows = nullptr;
    a.op_klen = nullptr;
    a.nr = 128;
    a.nk = h->n;
    a.code_is_op = 1;
    a.ft = 1;
    a.ft_rows = 128;
    a.tmap_a = g.ts_vmap;
    a.x = xp; a.x_ld = ldx; a.x_dc = 1; a.x_rows = lp.n_rows;
    a.y = lp.ts_y.as<double>(); a.y_ld = 8 * 20; a.y_dc = 1; a.y_seg = 20; a.y_map = lp.ts_map.as<int>();
    a.scale = 1.0; a.accumulate = 0; a.pair_out = 1;
    a.zero_row = h->zeros.as<double>();
    a.n_entries = lp.ts1.n_entries();
    launches += launch_tiles(a, lp.ts1.n_tiles, s);
    TileParams b{};
    fill_ops(b, g.lrf_left, g.main);
    fill_plan(b, lp.ts2_col, lp.ts2_off, lp.ts2_code, lp.ts2_src, lp.ts2.n_tiles);
    b.op_rows = nullptr;
    b.op_klen = nullptr;
    b.nr = h->n;
    b.nk = 16;
    b.code_is_op = 1;
    b.ft = 1;
    b.ft_rows = h->n;
    b.ft_opshift = 1;
    b.ft_colseg = 16;
    b.tmap_a = g.ts_umap;
    b.x = lp.ts_y.as<double>(); b.x_ld = 20; b.x_dc = 1; b.x_rows = lp.ts_segs; b.b_block = 1;
    b.y = d_y; b.y_ld = row_ld; b.y_dc = 1;
    b.scale = scale; b.accumulate = 1; b.pair_out = 0;
    b.zero_row = h->zeros.as<double>();
    b.n_entries = lp.ts2.n_entries();
    {
      const char* e = getenv("CFM_SEG_KSKIP");  // 0: run all 4 k-steps of every segment (A/B)
      b.seg_ksteps = (!e || atoi(e) != 0) ? g.ts_ksteps.as<int>() : nullptr;
    }
    static const bool seg_pair = [] {
      const char* e = getenv("CFM_SEG_PAIR");
      return !e || atoi(e) != 0;
    }();
    launches += seg_pair ? launch_seg_pair(b, lp.ts2.n_tiles, s) : launch_ft16(b, lp.ts2.n_tiles, s);
    return launches;
  }

  if (g.kind == kLowRank) {
    {
      LowRankParams q{};
      q.n_tiles = int(lp.hp.n_tiles);
      q.tile_col = lp.tile_col.as<int>();
      q.tile_off = lp.tile_off.as<int>();
      q.entry_code = lp.entry_code.as<int>();
      q.entry_src = lp.entry_src.as<int>();
      q.code_op = g.main.d_op.as<int>();
      q.code_rperm = g.main.d_rperm.as<int>();
      q.code_cperm = g.pass1.d_cperm.as<int>();
      q.vh = g.right_h.d.as<double>();
      q.vh_stride = g.right_h.stride;
      q.vh_ld = g.right_h.ld;
      q.u = g.left.d.as<double>();
      q.u_stride = g.left.stride;
      q.u_ld = g.left.ld;
      q.rank = g.left.d_klen.as<int>();
      q.n_ops = g.left.n_ops;
      q.nr = g.left.rows;
      q.nk = g.right_h.cols;
      q.rowtab = h->rowtab.as<short>();
      q.invtab = h->invtab.as<short>();
      q.x = d_x; q.x_ld = row_ld; q.x_dc = dc;
      const bool vb = g.has_lrfull && dc == 1;
      if (vb) {
        // per-transfer factors, identity permutations, zero-padded source rows
        const int ldx = g.lrf_right_h.ld;
        const auto xo = xpad_layout(h, {{lp.n_rows, ldx}}, s);
        double* xp = h->xpad.as<double>() + xo[0];
        launches += xpad_copy(h, xp, ldx, d_x, 0, lp.n_rows, s);
        q.code_op = g.fullmap.d_op.as<int>();
        q.code_rperm = g.fullmap.d_rperm.as<int>();
        q.code_cperm = g.fullmap.d_cperm.as<int>();
        q.vh = g.lrf_right_h.d.as<double>();
        q.vh_stride = g.lrf_right_h.stride;
        q.vh_ld = g.lrf_right_h.ld;
        q.u = g.lrf_left.d.as<double>();
        q.u_stride = g.lrf_left.stride;
        q.u_ld = g.lrf_left.ld;
        q.rank = g.lrf_left.d_klen.as<int>();
        q.n_ops = g.lrf_left.n_ops;
        q.x = xp;
        q.x_ld = ldx;
      }
      if (lp.mode == 1) {
        ensure(h->fbuf, size_t(lp.red.n_frows) * row_ld * sizeof(double));
        q.y = h->fbuf.as<double>(); q.y_ld = row_ld; q.y_dc = dc;
        q.scale = 1.0; q.accumulate = 0; q.pair_out = 1;
      } else {
        q.y = d_y; q.y_ld = row_ld; q.y_dc = dc;
        q.scale = scale; q.accumulate = 1; q.pair_out = 0;
      }
      if (launch_lowrank_fused(q, vb ? g.lrf_right_h.rows : g.right_h.rows, 0, lp.hp.n_tiles, s, vb)) {
        ++launches;
        if (lp.mode == 1)
          launches += launch_reduce(lp, h->fbuf.as<double>(), row_ld, d_y, row_ld, int(row_ld), scale, s);
        return launches;
      }
    }
    // chunk tiles so the per-pair intermediate stays bounded
    const int ldy = g.right_h.rows;  // rmax * f
    const size_t max_slots = std::max<size_t>(kBN, (size_t(1) << 30) / (sizeof(double) * std::max(ldy, 1)));
    const std::vector<int>& toff = lp.hp.tile_off;
    if (lp.mode == 1) ensure(h->fbuf, size_t(lp.red.n_frows) * row_ld * sizeof(double));
    int64_t t0 = 0;
    while (t0 < lp.hp.n_tiles) {
      int64_t t1 = t0 + 1;
      while (t1 < lp.hp.n_tiles && size_t(toff[t1 + 1] - toff[t0]) * kBN <= max_slots) ++t1;
      const int64_t e0 = toff[t0], e1 = toff[t1];
      if (e1 > e0) {
        ensure(h->ybuf, size_t(e1 - e0) * kBN * ldy * sizeof(double));
        double* ybase = h->ybuf.as<double>() - (long long)e0 * kBN * ldy;  // slot ids are global
        // pass 1: Y[slot] = right^H P^T w   (tiles = entries)
        TileParams p1 = p;
        fill_ops(p1, g.right_h, g.pass1);
        fill_plan(p1, lp.slot_ids, lp.iota, lp.entry_code, lp.entry_src, E);
        p1.x = d_x; p1.x_ld = row_ld; p1.x_dc = dc;
        p1.y = ybase; p1.y_ld = ldy; p1.y_dc = 1;
        p1.scale = 1.0; p1.accumulate = 0;
        // runs of up to kPass1Run entries per CTA; each entry's Y written when it ends
        p1.tile_off = lp.runs.as<int>();
        p1.pair_out = 1;
        launches += launch_range(p1, lp.run_start[t0], lp.run_start[t1] - lp.run_start[t0], s);
        // pass 2: acc += left[table] Y  (tiles = target tiles, sources = slots)
        TileParams p2 = p;
        fill_ops(p2, g.left, g.main);
        fill_plan(p2, lp.tile_col, lp.tile_off, lp.entry_code, lp.slot_ids, lp.hp.n_tiles);
        p2.x = ybase; p2.x_ld = ldy; p2.x_dc = 1;
        if (lp.mode == 1) {
          p2.y = h->fbuf.as<double>(); p2.y_ld = row_ld; p2.y_dc = dc;
          p2.scale = 1.0; p2.accumulate = 0; p2.pair_out = 1;
        } else {
          p2.y = d_y; p2.y_ld = row_ld; p2.y_dc = dc;
          p2.scale = scale; p2.accumulate = 1;
        }
        launches += launch_range(p2, t0, t1 - t0, s);
      }
      t0 = t1;
    }
    if (lp.mode == 1) launches += launch_reduce(lp, h->fbuf.as<double>(), row_ld, d_y, row_ld, int(row_ld), scale, s);
    return launches;
  }

  // ---- shared basis (sa / sarcmp), m2l.py:366-395
  const int rbf = g.sa_bh.rows;  // r_b * f (realified) rows of B^H
  const int ruf = g.sa_u.cols;   // r_u * f
  // full-operator stage 2 reads W~ rows with bulk copies: rows padded to the
  // cores' leading dimension, padding zeroed when the buffer is (re)allocated
  const bool sa_full = g.has_full && g.any_dense_core && dc == 1;
  const long long wt_ld = sa_full ? (long long)g.dense.ld : (long long)rbf * (dc == 2 ? 2 : 1);
  const long long z_ld = (long long)ruf * (dc == 2 ? 2 : 1);
  {
    const size_t need = std::max<size_t>(size_t(lp.n_rows) * wt_ld * sizeof(double), 16);
    const bool grow = !h->wt.p || need > h->wt.bytes;
    ensure(h->wt, need);
    if (sa_full && (grow || h->wt_ld_zeroed != wt_ld)) {
      CUDA_CHECK(cudaMemsetAsync(h->wt.p, 0, h->wt.bytes, s));
      h->wt_ld_zeroed = wt_ld;
    }
  }
  ensure(h->z, size_t(lp.n_rows) * z_ld * sizeof(double));
  CUDA_CHECK(cudaMemsetAsync(h->z.p, 0, size_t(lp.n_rows) * z_ld * sizeof(double), s));
  // stage 1: W~[src] = B^H M[src]
  {
    TileParams q = p;
    fill_ops(q, g.sa_bh, g.single);
    fill_plan(q, lp.s_tile_col, lp.s_tile_off, lp.s_entry_code, lp.s_entry_src, lp.src_plan.n_tiles);
    q.x = d_x; q.x_ld = row_ld; q.x_dc = dc;
    q.y = h->wt.as<double>(); q.y_ld = wt_ld; q.y_dc = dc;
    q.scale = 1.0; q.accumulate = 0;
    launches += launch_tiles(q, lp.src_plan.n_tiles, s);
  }
  // stage 2 output: Z directly (target tiles) or per-pair rows Fz (pair mode)
  double* z_out = h->z.as<double>();
  int z_pair = 0, z_acc = 1;
  if (lp.mode == 1) {
    ensure(h->fzbuf, size_t(lp.red.n_frows) * z_ld * sizeof(double));
    CUDA_CHECK(cudaMemsetAsync(h->fzbuf.p, 0, size_t(lp.red.n_frows) * z_ld * sizeof(double), s));
    z_out = h->fzbuf.as<double>();
    z_pair = 1;
    z_acc = 0;
  }
  // stage 2a: dense cores Z[tgt] += C_t W~[src]
  if (g.any_dense_core) {
    TileParams q = p;
    fill_ops(q, g.dense, g.main);
    fill_plan(q, lp.tile_col, lp.tile_off, lp.entry_code, lp.entry_src, lp.hp.n_tiles);
    q.x = h->wt.as<double>(); q.x_ld = wt_ld; q.x_dc = dc;
    q.y = z_out; q.y_ld = z_ld; q.y_dc = dc;
    q.scale = 1.0; q.accumulate = z_acc; q.pair_out = z_pair;
    if (sa_full) {
      q.ft = 1;
      q.ft_rows = g.full_rows;
      q.tmap_a = g.full_tmap;
      q.x_rows = lp.n_rows;
      q.rowtab = nullptr;
      q.invtab = nullptr;
      q.n_entries = lp.hp.n_entries();
      if (lp.mode == 1) q.entry_ncols = lp.entry_ncols.as<unsigned char>();
    }
    launches += launch_tiles(q, lp.hp.n_tiles, s);
  }
  // stage 2b: factored cores Z[tgt] += L_t (R_t^H W~[src])
  if (g.any_fac_core) {
    const int ldy = g.right_h.rows;
    ensure(h->ybuf, size_t(E) * kBN * ldy * sizeof(double));
    TileParams p1 = p;
    fill_ops(p1, g.right_h, g.pass1);
    fill_plan(p1, lp.slot_ids, lp.iota, lp.entry_code, lp.entry_src, E);
    p1.x = h->wt.as<double>(); p1.x_ld = wt_ld; p1.x_dc = dc;
    p1.y = h->ybuf.as<double>(); p1.y_ld = ldy; p1.y_dc = 1;
    p1.scale = 1.0; p1.accumulate = 0;
    launches += launch_tiles(p1, E, s);
    TileParams p2 = p;
    fill_ops(p2, g.left, g.sa_fac2);
    fill_plan(p2, lp.tile_col, lp.tile_off, lp.entry_code, lp.slot_ids, lp.hp.n_tiles);
    p2.x = h->ybuf.as<double>(); p2.x_ld = ldy; p2.x_dc = 1;
    p2.y = z_out; p2.y_ld = z_ld; p2.y_dc = dc;
    p2.scale = 1.0; p2.accumulate = z_acc; p2.pair_out = z_pair;
    launches += launch_tiles(p2, lp.hp.n_tiles, s);
  }
  if (lp.mode == 1) launches += launch_reduce(lp, z_out, z_ld, h->z.as<double>(), z_ld, int(z_ld), 1.0, s);
  // stage 3: locals[tgt] += scale * U Z[tgt]
  {
    TileParams q = p;
    fill_ops(q, g.sa_u, g.single);
    fill_plan(q, lp.t_tile_col, lp.t_tile_off, lp.t_entry_code, lp.t_entry_src, lp.tgt_plan.n_tiles);
    q.x = h->z.as<double>(); q.x_ld = z_ld; q.x_dc = dc;
    q.y = d_y; q.y_ld = row_ld; q.y_dc = dc;
    q.scale = scale; q.accumulate = 1;
    launches += launch_tiles(q, lp.tgt_plan.n_tiles, s);
  }
  (void)nf;
  return launches;
}

static void apply_with_buffers(cfm_handler* h, int level, LevelPlan& lp, const double* mpoles, double* locals,
                               cudaStream_t s) {
  const int dc = lp.dc;
  const size_t row_d = size_t(h->n) * (dc == 2 || h->op_complex ? 2 : 1);
  const size_t bytes = size_t(lp.n_rows) * row_d * sizeof(double);
  const bool dev_x = is_device_ptr(mpoles), dev_y = is_device_ptr(locals);
  const double* d_x = mpoles;
  double* d_y = locals;
  if (!dev_x) {
    ensure(h->x_stage, bytes);
    CUDA_CHECK(cudaMemcpyAsync(h->x_stage.p, mpoles, bytes, cudaMemcpyHostToDevice, s));
    d_x = h->x_stage.as<double>();
  }
  if (!dev_y) {
    ensure(h->y_stage, bytes);
    CUDA_CHECK(cudaMemcpyAsync(h->y_stage.p, locals, bytes, cudaMemcpyHostToDevice, s));
    d_y = h->y_stage.as<double>();
  }
  CUDA_CHECK(cudaEventRecord(h->ev0, s));
  h->last_launches = run_plan(h, level, lp, d_x, d_y, s);
  CUDA_CHECK(cudaEventRecord(h->ev1, s));
  if (!dev_y) CUDA_CHECK(cudaMemcpyAsync(locals, d_y, bytes, cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  float ms = 0.f;
  CUDA_CHECK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  h->last_ms = ms;
}

static bool use_merged_pairs() {
  static int v = [] {
    const char* e = getenv("CFM_MERGE_PAIRS");
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}

// Build (or reuse) the merged pair plan of the given pair-mode levels.
static MergedPairPlan& merged_pair_plan(cfm_handler* h, const Group& g, const std::vector<int>& levels,
                                        const std::vector<LevelPlan*>& plans, const std::vector<int64_t>& row_off) {
  std::vector<uint64_t> gens;
  for (auto* P : plans) gens.push_back(P->gen);
  if (h->merged && h->merged->levels == levels && h->merged->gens == gens && h->merged->row_off == row_off)
    return *h->merged;
  auto m = std::make_unique<MergedPairPlan>();
  m->levels = levels;
  m->gens = gens;
  m->row_off = row_off;
  struct Pr {
    int key, code, lvl;
    int src;
    int64_t old_frow;
  };
  std::vector<Pr> pairs;
  std::vector<std::vector<int64_t>> tgt_of(plans.size());
  for (size_t i = 0; i < plans.size(); ++i) {
    const LevelPlan& P = *plans[i];
    const int64_t E = P.hp.n_entries();
    for (int64_t e = 0; e < E; ++e) {
      const int c = P.hp.entry_code[e];
      const int key = std::max(g.main.op[c], 0) + 1;  // the per-level plans' order (build_plan_pairs)
      for (int j = 0; j < kBN; ++j) {
        const int v = P.hp.entry_src[size_t(e) * kBN + j];
        if (v >= 0) pairs.push_back({key, c, int(i), int(v + row_off[i]), e * kBN + j});
      }
    }
  }
  std::stable_sort(pairs.begin(), pairs.end(), [](const Pr& a, const Pr& b) {
    if (a.key != b.key) return a.key < b.key;
    return a.code < b.code;
  });
  std::vector<std::vector<int>> new_frow(plans.size());
  for (size_t i = 0; i < plans.size(); ++i) new_frow[i].assign(size_t(plans[i]->hp.n_entries()) * kBN, -1);
  HostPlan& hp = m->hp;
  hp.dc = 1;
  for (size_t a = 0; a < pairs.size();) {
    size_t b = a;
    while (b < pairs.size() && pairs[b].code == pairs[a].code && pairs[b].key == pairs[a].key) ++b;
    for (size_t q = a; q < b; q += kBN) {
      const int64_t e = hp.n_entries();
      hp.entry_code.push_back(pairs[a].code);
      hp.entry_src.resize(size_t(e + 1) * kBN, -1);
      for (size_t r = q; r < std::min(b, q + kBN); ++r) {
        const int sl = int(r - q);
        hp.entry_src[size_t(e) * kBN + sl] = pairs[r].src;
        new_frow[pairs[r].lvl][pairs[r].old_frow] = int(e * kBN + sl);
      }
    }
    a = b;
  }
  hp.n_pairs = int64_t(pairs.size());
  const int64_t E = hp.n_entries();
  const int nkp = round_up(h->n * h->f, kKC);
  // ~50 MFLOP of row-block work per CTA (measured at l = 9: 2 -> 4 entries per
  // CTA -1.7%), >= 2 CTAs per SM
  int ept = std::max(1, std::min(16, int(5.0e7 / (2.0 * 128 * kBN * nkp))));
  ept = std::min<int64_t>(ept, std::max<int64_t>(1, E / (2 * 148)));
  if (const char* e = getenv("CFM_PAIR_EPT")) ept = std::max(1, atoi(e));
  hp.n_tiles = (E + ept - 1) / ept;
  hp.tile_off.resize(hp.n_tiles + 1);
  for (int64_t t = 0; t <= hp.n_tiles; ++t) hp.tile_off[t] = int(std::min<int64_t>(t * ept, E));
  hp.tile_col.assign(size_t(hp.n_tiles) * kBN, -1);
  push_plan(hp, m->tile_col, m->tile_off, m->entry_code, m->entry_src);
  std::vector<unsigned char> nc(std::max<int64_t>(E, 1), 0);
  for (int64_t e = 0; e < E; ++e)
    for (int c = kBN - 1; c >= 0; --c)
      if (hp.entry_src[size_t(e) * kBN + c] >= 0) {
        nc[e] = static_cast<unsigned char>(c + 1);
        break;
      }
  upload(m->entry_ncols, nc);
  m->red.resize(plans.size());
  m->r_tgt.resize(plans.size());
  m->r_off.resize(plans.size());
  m->r_frow.resize(plans.size());
  for (size_t i = 0; i < plans.size(); ++i) {
    const PairReduce& r0 = plans[i]->red;
    PairReduce& r = m->red[i];
    r.tgt = r0.tgt;
    r.off = r0.off;
    r.frow.resize(r0.frow.size());
    for (size_t q = 0; q < r0.frow.size(); ++q) r.frow[q] = new_frow[i][r0.frow[q]];
    r.n_frows = E * kBN;
    upload(m->r_tgt[i], r.tgt);
    upload(m->r_off[i], r.off);
    upload(m->r_frow[i], r.frow);
  }
  h->merged = std::move(m);
  return *h->merged;
}

// All planned levels of one step in as few launches as possible: dense groups
// go into a single multi-segment launch (levels are independent in M2L, so
// the long per-tile chains of the small levels overlap the big level).
static void apply_levels_impl(cfm_handler* h, int n_levels, const int* levels, const double* const* mpoles,
                              const int64_t* n_rows, double* const* locals, cudaStream_t s) {
  struct Lv {
    int level;
    LevelPlan* lp;
    const double* x;
    double* y;
    double* host_y;
    size_t bytes;
  };
  std::vector<Lv> lv;
  size_t stage_bytes = 0;
  // CFM_TRACE=1: host preparation time and device time before the first launch, to stderr
  static const bool trace = getenv("CFM_TRACE") && atoi(getenv("CFM_TRACE"));
  static cudaEvent_t ev_t = nullptr;
  const auto t_host0 = std::chrono::steady_clock::now();
  if (trace) {
    if (!ev_t) CUDA_CHECK(cudaEventCreate(&ev_t));
    CUDA_CHECK(cudaEventRecord(ev_t, s));
  }
  for (int i = 0; i < n_levels; ++i) {
    auto it = h->plans.find(levels[i]);
    if (it == h->plans.end()) throw Error(CFM_ERR_PRECOMPUTE, "no plan for level " + std::to_string(levels[i]));
    if (it->second.n_rows != n_rows[i]) throw Error(CFM_ERR_VALUE, "row count differs from the planned level");
    group_for_level(h, levels[i]);
    const size_t row_d = size_t(h->n) * (it->second.dc == 2 || h->op_complex ? 2 : 1);
    const size_t bytes = size_t(n_rows[i]) * row_d * sizeof(double);
    lv.push_back({levels[i], &it->second, mpoles[i], locals[i], nullptr, bytes});
    if (!is_device_ptr(mpoles[i])) stage_bytes += bytes;
    if (!is_device_ptr(locals[i])) stage_bytes += bytes;
  }
  std::sort(lv.begin(), lv.end(), [](const Lv& a, const Lv& b) { return a.level < b.level; });
  if (stage_bytes) ensure(h->x_stage, stage_bytes);
  // ---- copy pipeline: large target-mode levels given as host buffers stream
  // their rows in slabs on a copy stream while the kernel runs (flags in device
  // memory, written with cuStreamWriteValue32, gate producers and epilogues;
  // per-slab completion counters gate the D2H slabs via cuStreamWaitValue32)
  bool all_dense_pre = true;
  for (auto& L : lv) all_dense_pre = all_dense_pre && group_for_level(h, L.level).kind == kDense;
  std::vector<int> piped(lv.size(), 0);
  bool any_piped = false;
  if (all_dense_pre && use_copy_pipeline() && lv.size() <= size_t(kMaxSegments)) {
    for (size_t i = 0; i < lv.size(); ++i) {
      if (!is_device_ptr(lv[i].x) && !is_device_ptr(lv[i].y) && lv[i].lp->mode == 0 && lv[i].lp->n_slabs >= 2) {
        piped[i] = 1;
        any_piped = true;
      }
    }
  }
  size_t off = 0;
  std::vector<const double*> host_x(lv.size(), nullptr);
  std::vector<size_t> flag_off(lv.size(), 0);
  std::vector<char> defer_loc(lv.size(), 0);  // locals upload after the first group's multipoles
  // Pipelined full-operator levels with host multipoles: ftl 3 = slabs go H2D
  // contiguously and are padded slab by slab on a side stream by a small
  // kernel that fits beside the running M2L grid (1 CTA/SM, ~7 K registers
  // free); the producers wait on per-slab flags, so the level joins the single
  // launch.  ftl 2 (CFM_PAD_PIPE=0) = the whole level crosses PCIe during the
  // other levels' launch and is padded before its own launch.
  // (measured at config 2: ftl 3 54.0-54.4 ms vs ftl 2 53.6 ms e2e -- the
  // first level-6 tiles wait on their slabs while holding SMs: off by default)
  static const bool pad_pipe = [] {
    const char* e = getenv("CFM_PAD_PIPE");
    return e && atoi(e) != 0;
  }();
  // full-operator levels read zero-padded source rows from h->xpad
  std::vector<int> ftl(lv.size(), 0);
  std::vector<std::pair<int64_t, int>> lay;
  std::vector<size_t> lay_idx(lv.size(), 0);
  if (all_dense_pre) {
    for (size_t i = 0; i < lv.size(); ++i) {
      Group& g = group_for_level(h, lv[i].level);
      if (!full_mode(g, *lv[i].lp)) continue;
      ftl[i] = 1;
      lay_idx[i] = lay.size();
      lay.push_back({lv[i].lp->n_rows, g.full.ld});
    }
  }
  cudaStream_t s_in = s;
  if (any_piped) {
    if (!h->s_h2d) CUDA_CHECK(cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking));
    if (!h->s_d2h) CUDA_CHECK(cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking));
    if (!h->ev_in) CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming));
    if (!h->ev_out) CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_out, cudaEventDisableTiming));
    s_in = h->s_h2d;
    // the copy stream reuses buffers (xpad, stages) that earlier calls' kernels
    // on the caller's stream may still read: start after them
    if (!h->ev_prev) CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_prev, cudaEventDisableTiming));
    CUDA_CHECK(cudaEventRecord(h->ev_prev, s));
    CUDA_CHECK(cudaStreamWaitEvent(s_in, h->ev_prev, 0));
    size_t nflags = 0;
    for (size_t i = 0; i < lv.size(); ++i)
      if (piped[i]) {
        flag_off[i] = nflags;
        nflags += 2 + size_t(lv[i].lp->n_slabs);
      }
    // target-tile levels of the first launch group upload their locals after
    // all first-group multipoles: the launch starts on the multipoles alone and
    // each tile's epilogue waits for its level's locals flag
    static const bool defer_env = [] {
      const char* e = getenv("CFM_DEFER_LOCALS");
      return !e || atoi(e) != 0;
    }();
    for (size_t i = 0; i < lv.size(); ++i)
      if (defer_env && !piped[i] && lv[i].lp->mode == 0 && !is_device_ptr(lv[i].y)) {
        defer_loc[i] = 1;
        flag_off[i] = nflags++;
      }
    ensure(h->pipe_flags, nflags * sizeof(unsigned));
    CUDA_CHECK(cudaMemsetAsync(h->pipe_flags.p, 0, nflags * sizeof(unsigned), s_in));
  }
  // middle launch group (ftl 4): the largest other host-buffer target-tile
  // full-operator level uploads after the first group's data, is padded on
  // its own stream and launched behind the first group (filling its tail)
  std::vector<char> mid(lv.size(), 0);
  if (any_piped && mid_group_enabled() && use_late_stream()) {
    size_t best = lv.size();
    for (size_t i = 0; i < lv.size(); ++i)
      if (ftl[i] == 1 && !piped[i] && lv[i].lp->mode == 0 && !is_device_ptr(lv[i].x) && !is_device_ptr(lv[i].y) &&
          lv[i].lp->n_rows >= 16384 && (best == lv.size() || lv[i].lp->n_rows > lv[best].lp->n_rows))
        best = i;
    if (best < lv.size()) mid[best] = 1;
  }
  std::vector<size_t> xoff;
  std::vector<const double*> staged_x(lv.size(), nullptr);
  std::vector<PadJob> pad_batch;  // the levels' source padding, one launch after the loop
  if (!lay.empty()) xoff = xpad_layout(h, lay, s_in);
  for (size_t i = 0; i < lv.size(); ++i) {
    auto& L = lv[i];
    if (ftl[i]) {
      // host rows go H2D contiguously into the stage (a pitched H2D copy of
      // 1000-B rows runs at 8 GB/s), then device-to-device into xpad.  That
      // copy is an SM kernel (tools/ce_probe.cu): it cannot run while the M2L
      // grid holds every SM, so it is never issued on the copy stream during a
      // launch.  Pipelined levels ("late", ftl = 2) copy their sources H2D
      // while the other levels' launch runs and are padded between the two
      // launches on the compute stream; only their locals stream by slab.
      double* xp = h->xpad.as<double>() + xoff[lay_idx[i]];
      const double* src = L.x;
      if (!is_device_ptr(L.x)) {
        double* d = reinterpret_cast<double*>(static_cast<char*>(h->x_stage.p) + off);
        host_x[i] = L.x;
        staged_x[i] = d;
        if (!piped[i] && !mid[i]) CUDA_CHECK(cudaMemcpyAsync(d, L.x, L.bytes, cudaMemcpyHostToDevice, s_in));
        src = d;
        off += L.bytes;
      }
      if (piped[i])
        ftl[i] = pad_pipe ? 3 : 2;
      else if (mid[i])
        ftl[i] = 4;  // uploaded after the first group's data, padded before its own launch
      else
        xpad_copy(h, xp, lay[lay_idx[i]].second, src, 0, L.lp->n_rows, s_in, 256, &pad_batch);
      L.x = xp;
    } else if (!is_device_ptr(L.x)) {
      double* d = reinterpret_cast<double*>(static_cast<char*>(h->x_stage.p) + off);
      host_x[i] = L.x;
      if (!piped[i]) CUDA_CHECK(cudaMemcpyAsync(d, L.x, L.bytes, cudaMemcpyHostToDevice, s_in));
      L.x = d;
      off += L.bytes;
    }
    if (!is_device_ptr(L.y)) {
      double* d = reinterpret_cast<double*>(static_cast<char*>(h->x_stage.p) + off);
      if (!piped[i] && !defer_loc[i]) CUDA_CHECK(cudaMemcpyAsync(d, L.y, L.bytes, cudaMemcpyHostToDevice, s_in));
      L.host_y = L.y;
      L.y = d;
      off += L.bytes;
    }
  }
  const int64_t pad_launches = launch_pads(pad_batch, s_in);
  if (any_piped) {
    // the kernel may start once the non-pipelined levels and the zeroed flags are in
    CUDA_CHECK(cudaEventRecord(h->ev_in, s_in));
    CUDA_CHECK(cudaStreamWaitEvent(s, h->ev_in, 0));
    CUDA_CHECK(cudaStreamWaitEvent(h->s_d2h, h->ev_in, 0));
    if (std::count(ftl.begin(), ftl.end(), 4)) {
      for (size_t i = 0; i < lv.size(); ++i)
        if (ftl[i] == 4)
          CUDA_CHECK(cudaMemcpyAsync(const_cast<double*>(staged_x[i]), host_x[i], lv[i].bytes, cudaMemcpyHostToDevice,
                                     s_in));
      if (!h->ev_mid) CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_mid, cudaEventDisableTiming));
      CUDA_CHECK(cudaEventRecord(h->ev_mid, s_in));
    }
    for (size_t i = 0; i < lv.size(); ++i) {
      if (!defer_loc[i]) continue;
      CUDA_CHECK(cudaMemcpyAsync(lv[i].y, lv[i].host_y, lv[i].bytes, cudaMemcpyHostToDevice, s_in));
      CUresult r = p_writeValue32(reinterpret_cast<CUstream>(s_in),
                                  reinterpret_cast<CUdeviceptr>(h->pipe_flags.as<unsigned>() + flag_off[i]), 1u, 0);
      if (r != CUDA_SUCCESS) throw Error(CFM_ERR_CUDA, "cuStreamWriteValue32 failed");
    }
    bool any_late = false;
    for (size_t i = 0; i < lv.size(); ++i)
      if (ftl[i] == 2) {
        CUDA_CHECK(cudaMemcpyAsync(const_cast<double*>(staged_x[i]), host_x[i], lv[i].bytes, cudaMemcpyHostToDevice,
                                   s_in));
        any_late = true;
      }
    if (any_late) {
      if (!h->ev_x) CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_x, cudaEventDisableTiming));
      CUDA_CHECK(cudaEventRecord(h->ev_x, s_in));
    }
    unsigned* flags = h->pipe_flags.as<unsigned>();
    for (size_t i = 0; i < lv.size(); ++i) {
      if (!piped[i]) continue;
      const LevelPlan& P = *lv[i].lp;
      const int S = P.n_slabs;
      const size_t row_b = lv[i].bytes / size_t(P.n_rows);
      auto slab_copy = [&](const void* hsrc, void* ddst, int k, cudaMemcpyKind kind, cudaStream_t st) {
        const size_t b0 = size_t(P.slab_row0[k]) * row_b, b1 = size_t(P.slab_row0[k + 1]) * row_b;
        if (b1 > b0)
          CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(ddst) + b0, static_cast<const char*>(hsrc) + b0, b1 - b0,
                                     kind, st));
      };
      auto write_flag = [&](unsigned* f, unsigned v) {
        CUresult r = p_writeValue32(reinterpret_cast<CUstream>(s_in), reinterpret_cast<CUdeviceptr>(f), v, 0);
        if (r != CUDA_SUCCESS) throw Error(CFM_ERR_CUDA, "cuStreamWriteValue32 failed");
      };
      unsigned* mp_ready = flags + flag_off[i];
      unsigned* loc_ready = mp_ready + 1;
      if (ftl[i] == 3) {
        if (!h->s_pad) {
          // highest priority: when an SM frees up, pad blocks are dispatched
          // before the grid's pending CTAs (which may wait on these pads)
          int least = 0, greatest = 0;
          CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
          CUDA_CHECK(cudaStreamCreateWithPriority(&h->s_pad, cudaStreamNonBlocking, greatest));
        }
        if (!h->ev_pad_done) CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_pad_done, cudaEventDisableTiming));
        if (S > 16) throw Error(CFM_ERR_VALUE, "too many slabs");
        for (int k = 0; k < S; ++k)
          if (!h->ev_slab[k]) CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_slab[k], cudaEventDisableTiming));
      }
      // multipole slab k is needed by targets of slab k-1: keep multipoles one slab ahead
      for (int k = 0; k < S; ++k) {
        if (ftl[i] == 3) {
          slab_copy(host_x[i], const_cast<double*>(staged_x[i]), k, cudaMemcpyHostToDevice, s_in);
          CUDA_CHECK(cudaEventRecord(h->ev_slab[k], s_in));
          CUDA_CHECK(cudaStreamWaitEvent(h->s_pad, h->ev_slab[k], 0));
          // 64-thread blocks fit beside a resident M2L CTA (registers)
          xpad_copy(h, const_cast<double*>(lv[i].x), lay[lay_idx[i]].second, staged_x[i], P.slab_row0[k],
                    P.slab_row0[k + 1], h->s_pad, 64);
          CUresult r = p_writeValue32(reinterpret_cast<CUstream>(h->s_pad), reinterpret_cast<CUdeviceptr>(mp_ready),
                                      unsigned(k + 1), 0);
          if (r != CUDA_SUCCESS) throw Error(CFM_ERR_CUDA, "cuStreamWriteValue32 failed");
        } else {
          if (!ftl[i]) slab_copy(host_x[i], const_cast<double*>(lv[i].x), k, cudaMemcpyHostToDevice, s_in);
          write_flag(mp_ready, unsigned(k + 1));
        }
        if (k >= 1) {
          slab_copy(lv[i].host_y, lv[i].y, k - 1, cudaMemcpyHostToDevice, s_in);
          write_flag(loc_ready, unsigned(k));
        }
      }
      slab_copy(lv[i].host_y, lv[i].y, S - 1, cudaMemcpyHostToDevice, s_in);
      write_flag(loc_ready, unsigned(S));
    }
  }
  CUDA_CHECK(cudaEventRecord(h->ev0, s));
  const auto t_host1 = std::chrono::steady_clock::now();
  std::vector<char> copied_early(lv.size(), 0);  // device->host copies already queued
  int64_t launches = pad_launches;
  bool all_dense = true;
  for (auto& L : lv) all_dense = all_dense && group_for_level(h, L.level).kind == kDense;
  if (all_dense) {
    // hybrid levels (LevelPlan::hyb, not host-pipelined): the kept tiles run as
    // the level's segment, the leftover targets as an extra pair-mode "level"
    // sharing the level's padded sources and locals (merged with the other
    // pair-mode levels below)
    std::vector<char> use_hyb(lv.size(), 0);
    {
      const size_t n_real = lv.size();
      for (size_t i = 0; i < n_real; ++i) {
        if (!lv[i].lp->hyb || ftl[i] != 1 || piped[i]) continue;
        // host locals next to a host-pipelined level: the plain tile plan, so
        // the level's locals are final when the first launch ends and go back
        // while the late group runs (no pair reduction after the launch)
        if (any_piped && lv[i].host_y && early_tgt_d2h()) continue;
        use_hyb[i] = 1;
        Lv ax = lv[i];
        ax.lp = &lv[i].lp->hyb->aux;
        ax.host_y = nullptr;
        ax.bytes = 0;
        lv.push_back(ax);
        ftl.push_back(1);
        piped.push_back(0);
        lay_idx.push_back(lay_idx[i]);
        flag_off.push_back(0);
        defer_loc.push_back(0);
        copied_early.push_back(0);
        staged_x.push_back(nullptr);
        host_x.push_back(nullptr);
        use_hyb.push_back(0);
      }
    }
    // one launch: target-mode levels accumulate into locals, pair-mode levels
    // write per-pair rows into their slice of fbuf, reduced right after
    // full-operator pair-mode levels of one group share one merged plan
    std::vector<size_t> mlv;
    for (size_t i = 0; i < lv.size(); ++i)
      if (ftl[i] == 1 && lv[i].lp->mode == 1) mlv.push_back(i);
    MergedPairPlan* mp_plan = nullptr;
    if (use_merged_pairs() && mlv.size() >= 2) {
      const Group* g0 = &group_for_level(h, lv[mlv[0]].level);
      bool one_group = true;
      for (size_t i : mlv) one_group = one_group && &group_for_level(h, lv[i].level) == g0;
      if (one_group) {
        std::vector<int> ml;
        std::vector<LevelPlan*> mp_;
        std::vector<int64_t> roff;
        for (size_t i : mlv) {
          ml.push_back(lv[i].level);
          mp_.push_back(lv[i].lp);
          roff.push_back(int64_t(xoff[lay_idx[i]] / size_t(lay[lay_idx[i]].second)));
        }
        mp_plan = &merged_pair_plan(h, *g0, ml, mp_, roff);
      }
    }
    std::vector<char> merged_lv(lv.size(), 0);
    if (mp_plan)
      for (size_t i : mlv) merged_lv[i] = 1;
    size_t f_total = 0;
    std::vector<size_t> f_off(lv.size(), 0);
    if (mp_plan) f_total = size_t(mp_plan->hp.n_entries()) * kBN * size_t(h->n);
    for (size_t i = 0; i < lv.size(); ++i) {
      if (lv[i].lp->mode != 1 || merged_lv[i]) continue;
      const size_t row_d = size_t(h->n) * (lv[i].lp->dc == 2 || h->op_complex ? 2 : 1);
      f_off[i] = f_total;
      f_total += size_t(lv[i].lp->red.n_frows) * row_d;
    }
    if (f_total) ensure(h->fbuf, f_total * sizeof(double));
    std::vector<TileParams> segs;
    std::vector<int64_t> counts;
    int nr = -1;
    bool same_shape = true;
    for (size_t i = 0; i < lv.size(); ++i) {
      auto& L = lv[i];
      Group& g = group_for_level(h, L.level);
      TileParams p{};
      p.rowtab = h->rowtab.as<short>();
      p.invtab = h->invtab.as<short>();
      p.zero_row = h->zeros.as<double>();
      fill_ops(p, g.dense, g.main);
      if (use_hyb[i])
        fill_plan(p, L.lp->hyb->tile_col, L.lp->hyb->tile_off, L.lp->hyb->entry_code, L.lp->hyb->entry_src,
                  L.lp->hyb->main.n_tiles);
      else
        fill_plan(p, L.lp->tile_col, L.lp->tile_off, L.lp->entry_code, L.lp->entry_src, L.lp->hp.n_tiles);
#ifdef CFM_EXPERIMENTS
      {
        // timing experiments only (results are wrong): CFM_EXP=norow|nocol|noperm drops permutations
        static const char* exp = getenv("CFM_EXP");
        static std::vector<int> neg(kNumCodes, -1);
        static DevBuf d_neg;
        if (exp && !d_neg.p) upload(d_neg, neg);
        if (exp && (!strcmp(exp, "norow") || !strcmp(exp, "noperm"))) p.code_rperm = d_neg.as<int>();
        if (exp && (!strcmp(exp, "nocol") || !strcmp(exp, "noperm"))) p.code_cperm = d_neg.as<int>();
        if (exp && !strcmp(exp, "nowait")) p.debug = 1;
        if (exp && !strcmp(exp, "spin")) p.debug = 2;
        if (exp && !strcmp(exp, "nocopy")) p.debug = 4;
        if (exp && !strcmp(exp, "zfillA")) p.debug = 8;
        if (exp && !strcmp(exp, "zfillB")) p.debug = 16;
        if (exp && !strcmp(exp, "zfillAB")) p.debug = 24;
        if (exp && !strcmp(exp, "noB")) p.debug = 32;
        if (exp && !strcmp(exp, "noA")) p.debug = 64;
      }
#endif
      const long long row_ld = (long long)h->n * (L.lp->dc == 2 || h->op_complex ? 2 : 1);
      p.x = L.x; p.x_ld = row_ld; p.x_dc = L.lp->dc;
      if (ftl[i]) {
        fill_full(p, h, g, L.x, L.lp->n_rows);
        if (L.lp->mode == 1) p.entry_ncols = L.lp->entry_ncols.as<unsigned char>();
        p.n_entries = use_hyb[i] ? L.lp->hyb->main.n_entries() : L.lp->hp.n_entries();
      }
      if (i > 0 && (ftl[i] != 0) != (ftl[0] != 0)) same_shape = false;
      if (L.lp->mode == 1) {
        p.y = h->fbuf.as<double>() + f_off[i]; p.y_ld = row_ld; p.y_dc = L.lp->dc;
        p.scale = 1.0; p.accumulate = 0; p.pair_out = 1;
      } else {
        p.y = L.y; p.y_ld = row_ld; p.y_dc = L.lp->dc;
        p.scale = h->levels[L.level].second;
        p.accumulate = 1;
      }
      if (defer_loc[i]) {
        p.pipe_loc = h->pipe_flags.as<unsigned>() + flag_off[i];
        p.pipe_need_loc = nullptr;  // one flag for the whole level
      }
      if (piped[i]) {
        unsigned* f = h->pipe_flags.as<unsigned>() + flag_off[i];
        p.pipe_mp = (ftl[i] == 0 || ftl[i] == 3) ? f : nullptr;  // ftl 2: sources resident before the launch
        p.pipe_loc = f + 1;
        p.pipe_done = f + 2;
        p.pipe_need_mp = L.lp->p_need_mp.as<int>();
        p.pipe_need_loc = L.lp->p_need_loc.as<int>();
        p.pipe_lo = L.lp->p_lo.as<int>();
        p.pipe_hi = L.lp->p_hi.as<int>();
      }
      if (nr >= 0 && (p.nr != nr)) same_shape = false;
      nr = p.nr;
      segs.push_back(p);
      counts.push_back(merged_lv[i] ? 0 : use_hyb[i] ? L.lp->hyb->n_long : L.lp->hp.n_tiles);  // merged levels run in the merged segment
    }
    // the shorter tiles of hybrid levels: extra segments launched after all
    // levels' long tiles (longest-processing-time order fills the launch tail)
    std::vector<size_t> short_segs;
    for (size_t i = 0; i < lv.size(); ++i) {
      if (!use_hyb[i]) continue;
      const int64_t n_short = lv[i].lp->hyb->main.n_tiles - lv[i].lp->hyb->n_long;
      if (n_short <= 0) continue;
      TileParams p = segs[i];
      p.tile_base = int(lv[i].lp->hyb->n_long);
      short_segs.push_back(segs.size());
      segs.push_back(p);
      counts.push_back(n_short);
    }
    const size_t merged_seg = segs.size();
    if (mp_plan) {
      const size_t i0 = mlv[0];
      Group& g = group_for_level(h, lv[i0].level);
      TileParams p{};
      p.zero_row = h->zeros.as<double>();
      fill_plan(p, mp_plan->tile_col, mp_plan->tile_off, mp_plan->entry_code, mp_plan->entry_src,
                mp_plan->hp.n_tiles);
      fill_full(p, h, g, h->xpad.as<double>(), int64_t(h->xpad.bytes / (sizeof(double) * g.full.ld)));  // global padded source rows
      p.entry_ncols = mp_plan->entry_ncols.as<unsigned char>();
      p.n_entries = mp_plan->hp.n_entries();
      p.y = h->fbuf.as<double>(); p.y_ld = h->n; p.y_dc = 1;
      p.scale = 1.0; p.accumulate = 0; p.pair_out = 1;
      if (p.nr != nr) same_shape = false;
      segs.push_back(p);
      counts.push_back(mp_plan->hp.n_tiles);
    }
    // small pair-mode segments reduce inside the launch (their last CTA)
    std::vector<bool> reduced_inside(lv.size(), false);
    if (same_shape && int(segs.size()) <= kMaxSegments) {  // (one multi-segment launch per group below)
      ensure(h->counters, kMaxSegments * sizeof(unsigned));
      CUDA_CHECK(cudaMemsetAsync(h->counters.p, 0, kMaxSegments * sizeof(unsigned), s));
      for (size_t i = 0; i < lv.size(); ++i) {
        const LevelPlan& P = *lv[i].lp;
        const long long row_ld = (long long)h->n * (P.dc == 2 || h->op_complex ? 2 : 1);
        const double work = double(P.red.frow.size()) * double(row_ld);
        // opt-in (CFM_REDUCE_INSIDE_MAX = elements): a single CTA reducing a
        // level serially measured slower than the separate parallel launch
        // (config 1: 0.92 vs 0.76 ms per step)
        static const double inside_max = [] {
          const char* e = getenv("CFM_REDUCE_INSIDE_MAX");
          return e ? atof(e) : 0.0;
        }();
        if (P.mode == 1 && !merged_lv[i] && work <= inside_max && !P.red.tgt.empty()) {
          TileParams& q = segs[i];
          q.red_counter = h->counters.as<unsigned>() + i;
          q.red_ctas = int(counts[i]) * ((q.nr + 127) / 128);
          q.red_tgt = P.r_tgt.as<long long>();
          q.red_off = P.r_off.as<long long>();
          q.red_frow = P.r_frow.as<int>();
          q.red_n_tgt = int64_t(P.red.tgt.size());
          q.red_y = lv[i].y;
          q.red_ld = row_ld;
          q.red_len = int(row_ld);
          q.red_scale = h->levels[lv[i].level].second;
          reduced_inside[i] = true;
        }
      }
    }
    // launch groups: all levels at once, or -- copy pipeline with late
    // full-operator levels -- the other levels first while the late levels'
    // sources cross PCIe, then the late ones once padded on this stream
    // all pair-mode reductions of the step in one launch (disjoint targets)
    auto reduce_pairs = [&](cudaStream_t rs) {
      MultiReduce mr{};
      long long blocks = 0;
      auto flush = [&] {
        if (mr.n == 0) return;
        mr.start[mr.n] = blocks;
        k_pair_reduce_multi<<<unsigned(blocks), 128, 0, rs>>>(mr);
        CUDA_CHECK(cudaGetLastError());
        ++launches;
        mr = MultiReduce{};
        blocks = 0;
      };
      for (size_t i = 0; i < lv.size(); ++i) {
        if (lv[i].lp->mode != 1 || reduced_inside[i]) continue;
        const long long row_ld = (long long)h->n * (lv[i].lp->dc == 2 || h->op_complex ? 2 : 1);
        ReduceSeg r{};
        if (merged_lv[i]) {
          const size_t k = size_t(std::find(mlv.begin(), mlv.end(), i) - mlv.begin());
          r.F = h->fbuf.as<double>();
          r.tgt = mp_plan->r_tgt[k].as<long long>();
          r.off = mp_plan->r_off[k].as<long long>();
          r.frow = mp_plan->r_frow[k].as<int>();
          r.n_tgt = int64_t(mp_plan->red[k].tgt.size());
        } else {
          const LevelPlan& P = *lv[i].lp;
          r.F = h->fbuf.as<double>() + f_off[i];
          r.tgt = P.r_tgt.as<long long>();
          r.off = P.r_off.as<long long>();
          r.frow = P.r_frow.as<int>();
          r.n_tgt = int64_t(P.red.tgt.size());
        }
        if (r.n_tgt == 0) continue;
        r.f_ld = row_ld;
        r.y = lv[i].y;
        r.y_ld = row_ld;
        r.len = int(row_ld);
        r.scale = h->levels[lv[i].level].second;
        if (mr.n == kMaxReduceSegs || blocks + r.n_tgt >= (1ll << 31)) flush();
        mr.start[mr.n] = blocks;
        mr.seg[mr.n++] = r;
        blocks += r.n_tgt;
      }
      flush();
    };
    bool reduced_early = false;
    // The late group runs on a side stream: it starts (pad, then launch) as
    // soon as its sources are in and its CTAs fill the SMs that the first
    // group's tail leaves idle (levels are independent in M2L); the caller's
    // stream joins it after the launches.
    // Groups: 0 = first launch, 1 = middle (ftl 4, e2e only), 2 = late (ftl 2).
    std::vector<std::vector<size_t>> groups(3);
    for (size_t i = 0; i < lv.size(); ++i)
      if (counts[i]) groups[ftl[i] == 2 ? 2 : ftl[i] == 4 ? 1 : 0].push_back(i);
    for (size_t k : short_segs) groups[0].push_back(k);
    if (mp_plan) groups[0].push_back(merged_seg);
    const bool side = use_late_stream() && !groups[0].empty() && (!groups[1].empty() || !groups[2].empty());
    if (side) {
      if (!h->s_late) CUDA_CHECK(cudaStreamCreateWithFlags(&h->s_late, cudaStreamNonBlocking));
      if (!h->ev_late0) CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_late0, cudaEventDisableTiming));
      if (!h->ev_late1) CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_late1, cudaEventDisableTiming));
      CUDA_CHECK(cudaEventRecord(h->ev_late0, s));  // everything this call (and earlier ones) queued so far
      CUDA_CHECK(cudaStreamWaitEvent(h->s_late, h->ev_late0, 0));
      if (!groups[1].empty()) {
        if (!h->s_mid) CUDA_CHECK(cudaStreamCreateWithFlags(&h->s_mid, cudaStreamNonBlocking));
        if (!h->ev_mid1) CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_mid1, cudaEventDisableTiming));
        CUDA_CHECK(cudaStreamWaitEvent(h->s_mid, h->ev_late0, 0));
      }
    }
    for (size_t gi = 0; gi < groups.size(); ++gi) {
      const auto& grp = groups[gi];
      if (grp.empty()) continue;
      cudaStream_t sg = s;
      if (gi == 1) {
        if (side) sg = h->s_mid;
        CUDA_CHECK(cudaStreamWaitEvent(sg, h->ev_mid, 0));
        std::vector<PadJob> pj;
        for (size_t i : grp) xpad_copy(h, const_cast<double*>(lv[i].x), lay[lay_idx[i]].second, staged_x[i], 0,
                                       lv[i].lp->n_rows, sg, 256, &pj);
        launches += launch_pads(pj, sg);
      }
      if (gi == 2) {
        if (side) sg = h->s_late;
        CUDA_CHECK(cudaStreamWaitEvent(sg, h->ev_x, 0));
        for (size_t i : grp)
          launches += xpad_copy(h, const_cast<double*>(lv[i].x), lay[lay_idx[i]].second, staged_x[i], 0,
                                lv[i].lp->n_rows, sg);
      }
      if (same_shape && int(segs.size()) <= kMaxSegments) {
        std::vector<TileParams> sub;
        std::vector<int64_t> sub_counts;
        for (size_t i : grp) {
          sub.push_back(segs[i]);
          sub_counts.push_back(counts[i]);
        }
        launches += launch_multi(sub, sub_counts, sg);
      } else {
        for (size_t i : grp) launches += launch_range(segs[i], segs[i].tile_base, counts[i], sg);
      }
      static const bool early_d2h = [] {
        const char* e = getenv("CFM_EARLY_D2H");
        return e && atoi(e) != 0;  // measured slower (e2e 54.1 -> 57.5 ms): off
      }();
      if (gi == 0 && side && early_d2h) {
        // the first group's pair reductions and device->host copies go out
        // while the late group still runs
        reduce_pairs(s);
        reduced_early = true;
        CUDA_CHECK(cudaEventRecord(h->ev_out, s));
        CUDA_CHECK(cudaStreamWaitEvent(h->s_d2h, h->ev_out, 0));
        for (size_t i = 0; i < lv.size(); ++i)
          if (!piped[i] && lv[i].host_y && ftl[i] != 4) {
            CUDA_CHECK(cudaMemcpyAsync(lv[i].host_y, lv[i].y, lv[i].bytes, cudaMemcpyDeviceToHost, h->s_d2h));
            copied_early[i] = 1;
          }
      }
      if (gi == 0 && side && !early_d2h && early_tgt_d2h()) {
        // target-tile levels of the first group (no pair reduction pending):
        // their locals download while the late group runs
        bool any = false;
        for (size_t i = 0; i < lv.size(); ++i)
          any = any || (!piped[i] && lv[i].host_y && lv[i].lp->mode == 0 && !use_hyb[i] && ftl[i] != 4);
        if (any) {
          CUDA_CHECK(cudaEventRecord(h->ev_out, s));
          CUDA_CHECK(cudaStreamWaitEvent(h->s_d2h, h->ev_out, 0));
          for (size_t i = 0; i < lv.size(); ++i)
            if (!piped[i] && lv[i].host_y && lv[i].lp->mode == 0 && !use_hyb[i] && ftl[i] != 4) {
              CUDA_CHECK(cudaMemcpyAsync(lv[i].host_y, lv[i].y, lv[i].bytes, cudaMemcpyDeviceToHost, h->s_d2h));
              copied_early[i] = 1;
            }
        }
      }
      if (gi == 1 && side) {
        // the middle group's locals (target tiles, no pair reduction) go back
        // while the late group runs
        CUDA_CHECK(cudaEventRecord(h->ev_mid1, sg));
        CUDA_CHECK(cudaStreamWaitEvent(s, h->ev_mid1, 0));
        if (early_tgt_d2h()) {
          CUDA_CHECK(cudaStreamWaitEvent(h->s_d2h, h->ev_mid1, 0));
          for (size_t i : grp)
            if (i < copied_early.size() && lv[i].host_y && lv[i].lp->mode == 0) {
              CUDA_CHECK(cudaMemcpyAsync(lv[i].host_y, lv[i].y, lv[i].bytes, cudaMemcpyDeviceToHost, h->s_d2h));
              copied_early[i] = 1;
            }
        }
      }
      if (gi == 2 && side) {
        CUDA_CHECK(cudaEventRecord(h->ev_late1, sg));
        CUDA_CHECK(cudaStreamWaitEvent(s, h->ev_late1, 0));
      }
    }
    if (!reduced_early) reduce_pairs(s);
  } else {
    bool all_lr = lv.size() > 1 && use_concurrent_levels();
    for (auto& L : lv) all_lr = all_lr && group_for_level(h, L.level).kind == kLowRank;
    if (!all_lr) {
      for (auto& L : lv) launches += run_plan(h, L.level, *L.lp, L.x, L.y, s);
    } else {
      // low-rank levels are independent and each is a separate launch chain:
      // run them side by side on forked streams, each with its own scratch
      // (per-pair rows, padded sources), so small latency-bound levels overlap
      const size_t nl = lv.size();
      if (h->aux.size() < nl) {
        h->aux.resize(nl);
        h->lvl_scratch.resize(nl);
      }
      if (!h->ev_fork) CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
      CUDA_CHECK(cudaEventRecord(h->ev_fork, s));
      for (size_t k = 0; k < nl; ++k) {
        AuxStream& a = h->aux[k];
        if (!a.s) {
          CUDA_CHECK(cudaStreamCreateWithFlags(&a.s, cudaStreamNonBlocking));
          CUDA_CHECK(cudaEventCreateWithFlags(&a.done, cudaEventDisableTiming));
        }
        CUDA_CHECK(cudaStreamWaitEvent(a.s, h->ev_fork, 0));
        LevelScratch& sc = h->lvl_scratch[k];
        std::swap(h->fbuf, sc.fbuf);
        std::swap(h->xpad, sc.xpad);
        std::swap(h->xpad_sig, sc.xpad_sig);
        std::swap(h->ybuf, sc.ybuf);
        try {
          launches += run_plan(h, lv[k].level, *lv[k].lp, lv[k].x, lv[k].y, a.s);
        } catch (...) {
          std::swap(h->fbuf, sc.fbuf);
          std::swap(h->xpad, sc.xpad);
          std::swap(h->xpad_sig, sc.xpad_sig);
          std::swap(h->ybuf, sc.ybuf);
          throw;
        }
        std::swap(h->fbuf, sc.fbuf);
        std::swap(h->xpad, sc.xpad);
        std::swap(h->xpad_sig, sc.xpad_sig);
        std::swap(h->ybuf, sc.ybuf);
        CUDA_CHECK(cudaEventRecord(a.done, a.s));
        CUDA_CHECK(cudaStreamWaitEvent(s, a.done, 0));
      }
    }
  }
  if (std::count(ftl.begin(), ftl.end(), 3)) {  // join the slab padding stream
    CUDA_CHECK(cudaEventRecord(h->ev_pad_done, h->s_pad));
    CUDA_CHECK(cudaStreamWaitEvent(s, h->ev_pad_done, 0));
  }
  CUDA_CHECK(cudaEventRecord(h->ev1, s));
  if (any_piped) {
    unsigned* flags = h->pipe_flags.as<unsigned>();
    for (size_t i = 0; i < lv.size(); ++i) {
      if (!piped[i]) continue;
      const LevelPlan& P = *lv[i].lp;
      const size_t row_b = lv[i].bytes / size_t(P.n_rows);
      unsigned* done = flags + flag_off[i] + 2;
      for (int k = 0; k < P.n_slabs; ++k) {
        if (P.slab_expected[k]) {
          CUresult r = p_waitValue32(reinterpret_cast<CUstream>(h->s_d2h),
                                           reinterpret_cast<CUdeviceptr>(done + k), P.slab_expected[k],
                                           CU_STREAM_WAIT_VALUE_GEQ);
          if (r != CUDA_SUCCESS) throw Error(CFM_ERR_CUDA, "cuStreamWaitValue32 failed");
        }
        const size_t b0 = size_t(P.slab_row0[k]) * row_b, b1 = size_t(P.slab_row0[k + 1]) * row_b;
        if (b1 > b0)
          CUDA_CHECK(cudaMemcpyAsync(reinterpret_cast<char*>(lv[i].host_y) + b0, reinterpret_cast<char*>(lv[i].y) + b0,
                                     b1 - b0, cudaMemcpyDeviceToHost, h->s_d2h));
      }
    }
    CUDA_CHECK(cudaEventRecord(h->ev_out, s));  // kernel (and reductions) done
    CUDA_CHECK(cudaStreamWaitEvent(h->s_d2h, h->ev_out, 0));
    for (size_t i = 0; i < lv.size(); ++i)
      if (!piped[i] && lv[i].host_y && !copied_early[i])
        CUDA_CHECK(cudaMemcpyAsync(lv[i].host_y, lv[i].y, lv[i].bytes, cudaMemcpyDeviceToHost, h->s_d2h));
    CUDA_CHECK(cudaStreamSynchronize(h->s_d2h));
    CUDA_CHECK(cudaStreamSynchronize(s));
  } else {
    for (auto& L : lv)
      if (L.host_y) CUDA_CHECK(cudaMemcpyAsync(L.host_y, L.y, L.bytes, cudaMemcpyDeviceToHost, s));
  }
  CUDA_CHECK(cudaStreamSynchronize(s));
  float ms = 0.f;
  CUDA_CHECK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  h->last_ms = ms;
  h->last_launches = launches;
  if (trace) {
    float pre = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&pre, ev_t, h->ev0));
    const double prep = std::chrono::duration<double, std::milli>(t_host1 - t_host0).count();
    const double tot = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_host0).count();
    fprintf(stderr, "[cfm trace] host prep %.3f ms, device before launch %.3f ms, launches %.3f ms, call %.3f ms\n",
            prep, pre, ms, tot);
  }
}

// ------------------------------------------------------------------ classifier
struct DeviceLists {
  DevBuf off, src, code;
  int64_t total = 0;
  std::vector<int64_t> h_off;
};

// c_cone_index is per-device __constant__ memory: upload it once per device
// (the caller has selected the device).
static void init_cone_table() {
  static std::mutex mu;
  static std::vector<bool> done;
  int dev = 0;
  CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (size_t(dev) < done.size() && done[dev]) return;
  int8_t tab[kNumCodes];
  std::fill(tab, tab + kNumCodes, int8_t(-1));
  auto cone = full_cone_codes();
  for (size_t i = 0; i < cone.size(); ++i) tab[cone[i]] = int8_t(i);
  CUDA_CHECK(cudaMemcpyToSymbol(c_cone_index, tab, sizeof(tab)));
  if (done.size() <= size_t(dev)) done.resize(dev + 1, false);
  done[dev] = true;
}

// Reusable classifier scratch of the device-output entry points, per calling
// thread AND per device (a buffer allocated on one device is never handed to
// a kernel running on another).
struct ClassifyScratch {
  DevBuf grid, counts;
};
static ClassifyScratch& classify_scratch(int device) {
  static thread_local std::map<int, ClassifyScratch> per_device;
  return per_device[device];
}

static void classify_device(int level, int64_t n_cells, const int32_t* ijk, cudaStream_t s, DeviceLists& out,
                            bool want_codes, int32_t* h_src = nullptr, int8_t* h_t = nullptr, uint8_t* h_rep = nullptr,
                            uint8_t* h_perm = nullptr, const int64_t* given_off = nullptr,
                            const int64_t* target_rows = nullptr, int64_t n_targets = -1) {
  if (level < 0 || level > 9) throw Error(CFM_ERR_VALUE, "classifier supports levels 0..9");
  init_cone_table();
  const int S = 1 << level;
  DevBuf d_ijk, grid, counts, d_tgt;
  const int32_t* dijk = ijk;
  if (!is_device_ptr(ijk)) {
    d_ijk.alloc(std::max<size_t>(size_t(n_cells) * 3 * sizeof(int32_t), 16));
    if (n_cells) CUDA_CHECK(cudaMemcpyAsync(d_ijk.p, ijk, size_t(n_cells) * 12, cudaMemcpyHostToDevice, s));
    dijk = d_ijk.as<int32_t>();
  }
  // validate on host copy (bounds): cheap check on device would need a flag; do it on host data when given
  if (!is_device_ptr(ijk)) {
    for (int64_t i = 0; i < n_cells; ++i)
      for (int a = 0; a < 3; ++a)
        if (ijk[3 * i + a] < 0 || ijk[3 * i + a] >= S) throw Error(CFM_ERR_VALUE, "cell index outside the level grid");
  }
  grid.alloc(size_t(S) * S * S * sizeof(int));
  CUDA_CHECK(cudaMemsetAsync(grid.p, 0xff, grid.bytes, s));
  const int tb = 256;
  if (n_cells) k_grid_scatter<<<unsigned((n_cells + tb - 1) / tb), tb, 0, s>>>(dijk, n_cells, S, grid.as<int>());
  CUDA_CHECK(cudaGetLastError());
  // a subset of the level's cells as targets (a rank's Morton range): the
  // grid holds every occupied cell (sources), the lists are built for the
  // given target rows only
  if (target_rows) {
    if (is_device_ptr(ijk)) throw Error(CFM_ERR_VALUE, "target subsets need host cell arrays");
    std::vector<int32_t> sub(size_t(std::max<int64_t>(n_targets, 0)) * 3);
    for (int64_t k = 0; k < n_targets; ++k) {
      const int64_t r = target_rows[k];
      if (r < 0 || r >= n_cells) throw Error(CFM_ERR_VALUE, "target row out of range");
      std::copy(ijk + 3 * r, ijk + 3 * r + 3, sub.begin() + 3 * k);
    }
    upload(d_tgt, sub);
    dijk = d_tgt.as<int32_t>();
    n_cells = n_targets;
  }
  const unsigned nb = unsigned((n_cells + tb - 1) / tb);
  out.h_off.assign(n_cells + 1, 0);
  if (given_off) {
    std::copy(given_off, given_off + n_cells + 1, out.h_off.begin());
  } else {
    counts.alloc(std::max<size_t>(size_t(n_cells) * sizeof(int), 16));
    if (n_cells && level >= 2)
      k_classify<false><<<nb, tb, 0, s>>>(dijk, n_cells, S, grid.as<int>(), counts.as<int>(), nullptr, nullptr,
                                          nullptr, nullptr, nullptr, nullptr);
    else if (n_cells)
      CUDA_CHECK(cudaMemsetAsync(counts.p, 0, size_t(n_cells) * sizeof(int), s));
    CUDA_CHECK(cudaGetLastError());
    std::vector<int> hc(n_cells);
    if (n_cells) CUDA_CHECK(cudaMemcpyAsync(hc.data(), counts.p, size_t(n_cells) * sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < n_cells; ++i) out.h_off[i + 1] = out.h_off[i] + hc[i];
  }
  out.total = out.h_off[n_cells];
  if (!want_codes && !h_src) return;
  upload(out.off, out.h_off);
  out.src.alloc(std::max<size_t>(size_t(out.total) * sizeof(int), 16));
  DevBuf d_t, d_rep, d_perm;
  if (want_codes) out.code.alloc(std::max<size_t>(size_t(out.total) * sizeof(int16_t), 16));
  if (h_t) d_t.alloc(std::max<size_t>(size_t(out.total) * 3, 16));
  if (h_rep) d_rep.alloc(std::max<size_t>(size_t(out.total), 16));
  if (h_perm) d_perm.alloc(std::max<size_t>(size_t(out.total), 16));
  if (n_cells && level >= 2 && out.total)
    k_classify<true><<<nb, tb, 0, s>>>(dijk, n_cells, S, grid.as<int>(), nullptr, out.off.as<long long>(),
                                       out.src.as<int>(), want_codes ? out.code.as<int16_t>() : nullptr,
                                       h_t ? d_t.as<int8_t>() : nullptr, h_rep ? d_rep.as<uint8_t>() : nullptr,
                                       h_perm ? d_perm.as<uint8_t>() : nullptr);
  CUDA_CHECK(cudaGetLastError());
  if (h_src && out.total) CUDA_CHECK(cudaMemcpyAsync(h_src, out.src.p, size_t(out.total) * 4, cudaMemcpyDeviceToHost, s));
  if (h_t && out.total) CUDA_CHECK(cudaMemcpyAsync(h_t, d_t.p, size_t(out.total) * 3, cudaMemcpyDeviceToHost, s));
  if (h_rep && out.total) CUDA_CHECK(cudaMemcpyAsync(h_rep, d_rep.p, size_t(out.total), cudaMemcpyDeviceToHost, s));
  if (h_perm && out.total) CUDA_CHECK(cudaMemcpyAsync(h_perm, d_perm.p, size_t(out.total), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
}

template <class F>
static int guarded(F&& fn) {
  try {
    g_last_error.clear();
    fn();
    return CFM_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host out of memory";
    return CFM_ERR_INTERNAL;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return CFM_ERR_INTERNAL;
  }
}

// NULL means the CUDA default (legacy) stream, as everywhere in CUDA: work
// stays ordered with the caller's default-stream kernels (e.g. torch's).
// The handler's scratch (padded sources, stages, pair rows) is reused by every
// apply, so an apply on a different stream than the previous one first waits
// for that one's work (calls on one stream are ordered anyway).
static cudaStream_t pick_stream(cfm_handler* h, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  if (h->have_last && h->last_stream != st) CUDA_CHECK(cudaStreamWaitEvent(st, h->ev_last, 0));
  return st;
}
static void mark_stream(cfm_handler* h, cudaStream_t st) {
  if (!h->ev_last) CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_last, cudaEventDisableTiming));
  CUDA_CHECK(cudaEventRecord(h->ev_last, st));
  h->last_stream = st;
  h->have_last = true;
}

// ------------------------------------------------------------------ octree
struct TreeLevel {
  int64_t n = 0;
  DevBuf keys;  // sorted unique lexicographic keys
};

}  // namespace cfm

struct cfm_tree {
  int device = 0, depth = 0;
  int64_t n_points = 0;
  double center[3] = {0, 0, 0}, half = 1.0;
  std::vector<cfm::TreeLevel> levels;  // index = level
  cfm::DevBuf leaf_off, perm;          // leaf particle CSR (int64)
  cfm::DevBuf points;                  // n x 3 on the device (original order)
};

struct cfm_fmm {
  cfm_tree* tree = nullptr;
  int order = 0, n = 0;
  cfm::DevBuf troots, leaf_ijk, leaf_grid, leaf_of_pos;
  cfm::OpStack m2m_ops, l2l_ops;
  cfm::CodeMap octmap;
  std::map<int, cfm::LevelPlan> m2m_plans, l2l_plans;  // key: child level / parent level (x dc)
  // P2P: leaf-sorted positions (built on first use), sorted weights, leaf lists by size class
  cfm::DevBuf px, py, pz, sw, small_leaves, large_leaves;
  int64_t n_small = -1, n_large = 0;
};

namespace cfm {

template <class F>
static void cub_call(F&& f, cudaStream_t s) {
  size_t tmp = 0;
  CUDA_CHECK(f(nullptr, tmp));
  DevBuf t;
  t.alloc(std::max<size_t>(tmp, 16));
  CUDA_CHECK(f(t.p, tmp));
  CUDA_CHECK(cudaStreamSynchronize(s));
}

// sorted unique keys of `in` (n keys, device) -> out (device), returns count; optional run counts
static int64_t sort_unique(const unsigned long long* in, int64_t n, DevBuf& out, DevBuf* counts, int end_bit,
                           cudaStream_t s) {
  DevBuf sorted, nsel;
  sorted.alloc(std::max<size_t>(size_t(n) * 8, 16));
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortKeys(t, b, in, sorted.as<unsigned long long>(), int64_t(n), 0, end_bit, s);
  }, s);
  out.alloc(std::max<size_t>(size_t(n) * 8, 16));
  nsel.alloc(16);
  if (counts) {
    counts->alloc(std::max<size_t>(size_t(n) * 8, 16));
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRunLengthEncode::Encode(t, b, sorted.as<unsigned long long>(), out.as<unsigned long long>(),
                                                counts->as<long long>(), nsel.as<long long>(), int64_t(n), s);
    }, s);
  } else {
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceSelect::Unique(t, b, sorted.as<unsigned long long>(), out.as<unsigned long long>(),
                                       nsel.as<long long>(), int64_t(n), s);
    }, s);
  }
  long long m = 0;
  CUDA_CHECK(cudaMemcpy(&m, nsel.p, 8, cudaMemcpyDeviceToHost));
  return m;
}

static int key_bits(int level) { return std::max(1, 3 * level); }

}  // namespace cfm

// ===================================================================== C ABI
extern "C" {

const char* cfm_last_error(void) { return cfm::g_last_error.c_str(); }

int cfm_abi_version(void) { return 1; }

int cfm_handler_create(int device, int variant, int order, int op_complex, cfm_handler** out) {
  return guarded([&] {
    if (!out) throw Error(CFM_ERR_VALUE, "out is null");
    if (variant < CFM_NA || variant > CFM_IABLK) throw Error(CFM_ERR_VALUE, "unknown M2L variant");
    if (order < 2 || order > 12) throw Error(CFM_ERR_VALUE, "interpolation order must be in [2, 12]");
    int ndev = 0;
    CUDA_CHECK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw Error(CFM_ERR_VALUE, "no such CUDA device");
    CUDA_CHECK(cudaSetDevice(device));
    auto h = std::make_unique<cfm_handler>();
    h->device = device;
    h->variant = variant;
    h->order = order;
    h->op_complex = op_complex ? 1 : 0;
    h->n = order * order * order;
    h->f = op_complex ? 2 : 1;
    h->sym = variant == CFM_NASYM || variant == CFM_NABLK || variant == CFM_IASYM || variant == CFM_IABLK;
    h->lowrank = variant == CFM_IA || variant == CFM_IASYM || variant == CFM_IABLK;
    h->shared = variant == CFM_SA || variant == CFM_SARCMP;
    CUDA_CHECK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    CUDA_CHECK(cudaEventCreate(&h->ev0));
    CUDA_CHECK(cudaEventCreate(&h->ev1));
    build_tables(h.get());
    upload(h->zeros, std::vector<double>(8192, 0.0));
    *out = h.release();
  });
}

int cfm_handler_destroy(cfm_handler* h) {
  return guarded([&] {
    if (!h) return;
    cudaSetDevice(h->device);
    cudaStreamSynchronize(h->stream);
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    if (h->ev_in) cudaEventDestroy(h->ev_in);
    if (h->ev_out) cudaEventDestroy(h->ev_out);
    if (h->ev_prev) cudaEventDestroy(h->ev_prev);
    if (h->ev_x) cudaEventDestroy(h->ev_x);
    if (h->ev_last) cudaEventDestroy(h->ev_last);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    for (auto& a : h->aux) {
      if (a.done) cudaEventDestroy(a.done);
      if (a.s) cudaStreamDestroy(a.s);
    }
    if (h->s_h2d) cudaStreamDestroy(h->s_h2d);
    if (h->s_d2h) cudaStreamDestroy(h->s_d2h);
    if (h->s_late) cudaStreamDestroy(h->s_late);
    if (h->s_pad) cudaStreamDestroy(h->s_pad);
    for (auto& e : h->ev_slab)
      if (e) cudaEventDestroy(e);
    if (h->ev_pad_done) cudaEventDestroy(h->ev_pad_done);
    if (h->ev_late0) cudaEventDestroy(h->ev_late0);
    if (h->ev_late1) cudaEventDestroy(h->ev_late1);
    if (h->s_mid) cudaStreamDestroy(h->s_mid);
    if (h->ev_mid) cudaEventDestroy(h->ev_mid);
    if (h->ev_mid1) cudaEventDestroy(h->ev_mid1);
    cudaStreamDestroy(h->stream);
    delete h;
  });
}

int cfm_set_dense_group(cfm_handler* h, int key, int n_transfers, const int8_t* transfers, int n_ops,
                        const int8_t* op_t, const double* ops) {
  return guarded([&] {
    if (!h) throw Error(CFM_ERR_VALUE, "null handler");
    std::lock_guard<std::mutex> lk(h->mu);
    CUDA_CHECK(cudaSetDevice(h->device));
    if (h->lowrank || h->shared) throw Error(CFM_ERR_VALUE, "dense group on a non-dense variant");
    Group g;
    g.kind = kDense;
    g.n_ops = n_ops;
    map_transfers(h, g, n_transfers, transfers, n_ops, op_t, true, true, g.main);
    g.main.push();
    const int nf = h->n * h->f;
    make_stack(g.dense, n_ops, nf, nf);
    const size_t blk = size_t(h->n) * h->n * (h->op_complex ? 2 : 1);
    std::vector<double> tmp(g.dense.stride);
    for (int i = 0; i < n_ops; ++i) {
      std::fill(tmp.begin(), tmp.end(), 0.0);
      realify_into(ops + i * blk, h->n, h->n, h->op_complex, tmp.data(), g.dense.ld);
      put_stack(g.dense, i, tmp);
    }
    if (use_full_ops(h)) build_full_ops(h, g, n_transfers, transfers, ops);
    h->groups[key] = std::move(g);
    h->plans.clear();
    h->csr_cache.clear();
    h->csr_cache_bytes = 0;
  });
}

int cfm_set_lowrank_group(cfm_handler* h, int key, int n_transfers, const int8_t* transfers, int n_ops,
                          const int8_t* op_t, const int32_t* ranks, const double* left, const double* right) {
  return guarded([&] {
    if (!h) throw Error(CFM_ERR_VALUE, "null handler");
    std::lock_guard<std::mutex> lk(h->mu);
    CUDA_CHECK(cudaSetDevice(h->device));
    if (!h->lowrank) throw Error(CFM_ERR_VALUE, "low-rank group on a non-low-rank variant");
    Group g;
    g.kind = kLowRank;
    g.n_ops = n_ops;
    map_transfers(h, g, n_transfers, transfers, n_ops, op_t, /*rows*/ true, /*cols*/ false, g.main);
    map_transfers(h, g, n_transfers, transfers, n_ops, op_t, /*rows*/ false, /*cols*/ true, g.pass1);
    g.main.push();
    g.pass1.push();
    for (int i = 0; i < n_ops; ++i)
      if (ranks[i] < 0 || ranks[i] > h->n) throw Error(CFM_ERR_VALUE, "rank out of range");
    build_lowrank_stacks(h, g.left, g.right_h, n_ops, ranks, left, right, h->n, h->n);
    if (use_full_ops(h)) build_lowrank_full(h, g, n_transfers, transfers, n_ops, ranks, left, right);
    h->groups[key] = std::move(g);
    h->plans.clear();
    h->csr_cache.clear();
    h->csr_cache_bytes = 0;
  });
}

int cfm_set_shared_group(cfm_handler* h, int key, int r_u, int r_b, const double* u, const double* b, int n_cores,
                         const int8_t* core_t, const int32_t* core_rank, const double* core_data) {
  return guarded([&] {
    if (!h) throw Error(CFM_ERR_VALUE, "null handler");
    std::lock_guard<std::mutex> lk(h->mu);
    CUDA_CHECK(cudaSetDevice(h->device));
    if (!h->shared) throw Error(CFM_ERR_VALUE, "shared group on a non-shared variant");
    if (r_u < 0 || r_b < 0 || r_u > h->n || r_b > h->n) throw Error(CFM_ERR_VALUE, "shared rank out of range");
    const int f = h->f;
    const bool cplx = h->op_complex;
    const int sc = cplx ? 2 : 1;
    Group g;
    g.kind = kShared;
    g.n_ops = n_cores;
    g.r_u = r_u;
    g.r_b = r_b;
    // bases: B^H (r_b f x n f) and U (n f x r_u f)
    make_stack(g.sa_bh, 1, std::max(r_b * f, 1), h->n * f);
    make_stack(g.sa_u, 1, h->n * f, std::max(r_u * f, 1));
    {
      std::vector<double> tmp(g.sa_bh.stride, 0.0);
      if (r_b) realify_into(b, r_b, h->n, cplx, tmp.data(), g.sa_bh.ld, /*conj_t=*/true);
      put_stack(g.sa_bh, 0, tmp);
      std::vector<double> tu(g.sa_u.stride, 0.0);
      if (r_u) realify_into(u, h->n, r_u, cplx, tu.data(), g.sa_u.ld);
      put_stack(g.sa_u, 0, tu);
    }
    g.single.op[0] = 0;
    g.single.push();
    // cores
    std::vector<int> dense_idx, fac_idx, fac_rank;
    std::vector<size_t> off(n_cores);
    size_t o = 0;
    for (int i = 0; i < n_cores; ++i) {
      off[i] = o;
      const int t0 = core_t[3 * i], t1 = core_t[3 * i + 1], t2 = core_t[3 * i + 2];
      if (t0 < -3 || t0 > 3 || t1 < -3 || t1 > 3 || t2 < -3 || t2 > 3)
        throw Error(CFM_ERR_VALUE, "core transfer vector outside [-3,3]^3");
      const int c = tcode(t0, t1, t2);
      g.valid[c] = 1;
      if (core_rank[i] < 0) {
        g.main.op[c] = int(dense_idx.size());
        dense_idx.push_back(i);
        o += size_t(r_u) * r_b * sc;
      } else {
        g.pass1.op[c] = int(fac_idx.size());
        g.sa_fac2.op[c] = int(fac_idx.size());
        fac_idx.push_back(i);
        fac_rank.push_back(core_rank[i]);
        o += size_t(r_u + r_b) * core_rank[i] * sc;
      }
    }
    g.any_dense_core = !dense_idx.empty();
    g.any_fac_core = !fac_idx.empty();
    if (g.any_dense_core) {
      make_stack(g.dense, int(dense_idx.size()), std::max(r_u * f, 1), std::max(r_b * f, 1));
      std::vector<double> tmp(g.dense.stride);
      for (size_t k = 0; k < dense_idx.size(); ++k) {
        std::fill(tmp.begin(), tmp.end(), 0.0);
        realify_into(core_data + off[dense_idx[k]], r_u, r_b, cplx, tmp.data(), g.dense.ld);
        put_stack(g.dense, int(k), tmp);
      }
      // the cores are already one (unpermuted) operator per transfer vector:
      // the full-operator TMA kernel reads them directly (stage 2 of sa / sarcmp)
      static const int full_env = [] {
        const char* e = getenv("CFM_FULL_OPS");
        return e ? atoi(e) : 1;
      }();
      if (full_env && !cplx && r_u > 64 && r_b <= 1024 && resolve_encode_tiled()) {
        const cuuint64_t dims[2] = {cuuint64_t(g.dense.ld), cuuint64_t(g.dense.n_ops) * g.dense.rows};
        const cuuint64_t strides[1] = {cuuint64_t(g.dense.ld) * sizeof(double)};
        const cuuint32_t box[2] = {cuuint32_t(kKC + 4), 128u};
        const cuuint32_t estr[2] = {1u, 1u};
        const CUresult r = resolve_encode_tiled()(&g.full_tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, g.dense.d.p, dims,
                                                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw Error(CFM_ERR_CUDA, "cuTensorMapEncodeTiled failed for the SA cores");
        g.has_full = true;
        g.full_rows = g.dense.rows;
      }
    }
    if (g.any_fac_core) {
      // gather factored blocks contiguously: left blocks then right blocks per core
      std::vector<double> L, R;
      for (size_t k = 0; k < fac_idx.size(); ++k) {
        const double* base = core_data + off[fac_idx[k]];
        const size_t nl = size_t(r_u) * fac_rank[k] * sc, nr = size_t(r_b) * fac_rank[k] * sc;
        L.insert(L.end(), base, base + nl);
        R.insert(R.end(), base + nl, base + nl + nr);
      }
      build_lowrank_stacks(h, g.left, g.right_h, int(fac_idx.size()), fac_rank.data(), L.data(), R.data(), r_u, r_b);
    }
    g.main.push();
    g.pass1.push();
    g.sa_fac2.push();
    h->groups[key] = std::move(g);
    h->plans.clear();
    h->csr_cache.clear();
    h->csr_cache_bytes = 0;
  });
}

int cfm_set_level(cfm_handler* h, int level, int key, double scale) {
  return guarded([&] {
    if (!h) throw Error(CFM_ERR_VALUE, "null handler");
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->groups.count(key)) throw Error(CFM_ERR_VALUE, "unknown group key");
    h->levels[level] = {key, scale};
    h->plans.erase(level);
    for (auto it = h->csr_cache.begin(); it != h->csr_cache.end();) {
      if (it->level == level) {
        h->csr_cache_bytes -= it->host_bytes();
        it = h->csr_cache.erase(it);
      } else {
        ++it;
      }
    }
  });
}

int cfm_plan_level_csr(cfm_handler* h, int level, int64_t n_targets, const int64_t* tgt, const int64_t* off,
                       const int64_t* src, const int8_t* t, int data_complex, int64_t n_rows, int64_t* pair_count_out) {
  return guarded([&] {
    if (!h) throw Error(CFM_ERR_VALUE, "null handler");
    std::lock_guard<std::mutex> lk(h->mu);
    CUDA_CHECK(cudaSetDevice(h->device));
    if (n_targets < 0 || n_rows < 0) throw Error(CFM_ERR_VALUE, "negative size");
    const int64_t P = n_targets ? off[n_targets] : 0;
    auto codes = codes_from_t(P, t);
    LevelPlan& lp = make_plan(h, level, n_targets, tgt, off, src, codes.data(), data_complex, n_rows);
    if (pair_count_out) std::copy(lp.hp.code_count.begin(), lp.hp.code_count.end(), pair_count_out);
  });
}

int cfm_apply_planned(cfm_handler* h, int level, const double* mpoles, int64_t n_rows, double* locals, void* stream) {
  return guarded([&] {
    if (!h) throw Error(CFM_ERR_VALUE, "null handler");
    std::lock_guard<std::mutex> lk(h->mu);
    CUDA_CHECK(cudaSetDevice(h->device));
    auto it = h->plans.find(level);
    if (it == h->plans.end()) throw Error(CFM_ERR_PRECOMPUTE, "no plan for level " + std::to_string(level));
    if (it->second.n_rows != n_rows) throw Error(CFM_ERR_VALUE, "row count differs from the planned level");
    {
      cudaStream_t st = pick_stream(h, stream);
      apply_with_buffers(h, level, it->second, mpoles, locals, st);
      mark_stream(h, st);
    }
  });
}

int cfm_apply_level_csr(cfm_handler* h, int level, int64_t n_targets, const int64_t* tgt, const int64_t* off,
                        const int64_t* src, const int8_t* t, int data_complex, const double* mpoles, int64_t n_rows,
                        double* locals, void* stream, int64_t* pair_count_out) {
  return guarded([&] {
    if (!h) throw Error(CFM_ERR_VALUE, "null handler");
    std::lock_guard<std::mutex> lk(h->mu);
    CUDA_CHECK(cudaSetDevice(h->device));
    if (n_targets < 0 || n_rows < 0) throw Error(CFM_ERR_VALUE, "negative size");
    bool hit = false;
    LevelPlan& lp = csr_plan(h, level, n_targets, tgt, off, src, t, data_complex, n_rows, &hit);
    h->last_csr_hit = hit;
    h->last_csr_mode = lp.mode;
    h->last_csr_two_stage = lp.ts ? 1 : 0;
    if (pair_count_out) std::copy(lp.hp.code_count.begin(), lp.hp.code_count.end(), pair_count_out);
    {
      cudaStream_t st = pick_stream(h, stream);
      apply_with_buffers(h, level, lp, mpoles, locals, st);
      mark_stream(h, st);
    }
  });
}

int cfm_plan_level_cells(cfm_handler* h, int level, int64_t n_cells, const int32_t* ijk, int data_complex,
                         void* stream, int64_t* pair_count_out) {
  return guarded([&] {
    if (!h) throw Error(CFM_ERR_VALUE, "null handler");
    std::lock_guard<std::mutex> lk(h->mu);
    CUDA_CHECK(cudaSetDevice(h->device));
    cudaStream_t s = pick_stream(h, stream);
    DeviceLists dl;
    classify_device(level, n_cells, ijk, s, dl, /*want_codes=*/true);
    std::vector<int32_t> hsrc(dl.total);
    std::vector<int16_t> hcode(dl.total);
    if (dl.total) {
      CUDA_CHECK(cudaMemcpyAsync(hsrc.data(), dl.src.p, size_t(dl.total) * 4, cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaMemcpyAsync(hcode.data(), dl.code.p, size_t(dl.total) * 2, cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
    }
    std::vector<int64_t> tgt(n_cells), src64(hsrc.begin(), hsrc.end());
    std::iota(tgt.begin(), tgt.end(), 0);
    LevelPlan& lp = make_plan(h, level, n_cells, tgt.data(), dl.h_off.data(), src64.data(), hcode.data(),
                              data_complex, n_cells);
    if (pair_count_out) std::copy(lp.hp.code_count.begin(), lp.hp.code_count.end(), pair_count_out);
  });
}

int cfm_apply_levels(cfm_handler* h, int n_levels, const int* levels, const double* const* mpoles,
                     const int64_t* n_rows, double* const* locals, void* stream) {
  return guarded([&] {
    if (!h) throw Error(CFM_ERR_VALUE, "null handler");
    if (n_levels < 0 || (n_levels && (!levels || !mpoles || !n_rows || !locals)))
      throw Error(CFM_ERR_VALUE, "bad level arrays");
    std::lock_guard<std::mutex> lk(h->mu);
    CUDA_CHECK(cudaSetDevice(h->device));
    {
      cudaStream_t st = pick_stream(h, stream);
      apply_levels_impl(h, n_levels, levels, mpoles, n_rows, locals, st);
      mark_stream(h, st);
    }
  });
}

int cfm_plan_level_cells_subset(cfm_handler* h, int level, int64_t n_cells, const int32_t* ijk, int64_t n_targets,
                                const int64_t* target_rows, int data_complex, void* stream, int64_t* pair_count_out,
                                int64_t* n_sources_out, int64_t* sources_out) {
  return guarded([&] {
    if (!h) throw Error(CFM_ERR_VALUE, "null handler");
    if (n_targets < 0 || (n_targets && !target_rows)) throw Error(CFM_ERR_VALUE, "bad target rows");
    std::lock_guard<std::mutex> lk(h->mu);
    CUDA_CHECK(cudaSetDevice(h->device));
    cudaStream_t s = pick_stream(h, stream);
    DeviceLists dl;
    classify_device(level, n_cells, ijk, s, dl, /*want_codes=*/true);
    std::vector<int32_t> hsrc(dl.total);
    std::vector<int16_t> hcode(dl.total);
    if (dl.total) {
      CUDA_CHECK(cudaMemcpyAsync(hsrc.data(), dl.src.p, size_t(dl.total) * 4, cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaMemcpyAsync(hcode.data(), dl.code.p, size_t(dl.total) * 2, cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
    }
    // restrict the CSR to the requested targets (this rank's Morton range)
    std::vector<int64_t> tgt, off(1, 0), src64;
    std::vector<int16_t> codes;
    for (int64_t k = 0; k < n_targets; ++k) {
      const int64_t r = target_rows[k];
      if (r < 0 || r >= n_cells) throw Error(CFM_ERR_VALUE, "target row out of range");
      tgt.push_back(r);
      for (int64_t q = dl.h_off[r]; q < dl.h_off[r + 1]; ++q) {
        src64.push_back(hsrc[q]);
        codes.push_back(hcode[q]);
      }
      off.push_back(int64_t(src64.size()));
    }
    LevelPlan& lp = make_plan(h, level, int64_t(tgt.size()), tgt.data(), off.data(), src64.data(), codes.data(),
                              data_complex, n_cells);
    if (pair_count_out) std::copy(lp.hp.code_count.begin(), lp.hp.code_count.end(), pair_count_out);
    if (n_sources_out) *n_sources_out = int64_t(lp.sources.size());
    if (sources_out) std::copy(lp.sources.begin(), lp.sources.end(), sources_out);
  });
}

int cfm_plan_stats(cfm_handler* h, int level, int64_t* n_tiles, int64_t* n_entries, int64_t* n_pairs,
                   int64_t* n_slots, int64_t* n_targets, int64_t* n_sources) {
  return guarded([&] {
    if (!h) throw Error(CFM_ERR_VALUE, "null handler");
    std::lock_guard<std::mutex> lk(h->mu);
    auto it = h->plans.find(level);
    if (it == h->plans.end()) throw Error(CFM_ERR_PRECOMPUTE, "no plan for level " + std::to_string(level));
    const LevelPlan& lp = it->second;
    if (n_tiles) *n_tiles = lp.hp.n_tiles;
    if (n_entries) *n_entries = lp.hp.n_entries();
    if (n_pairs) *n_pairs = lp.hp.n_pairs;
    if (n_slots) *n_slots = lp.hp.n_entries() * kBN / lp.dc;
    if (n_targets) *n_targets = int64_t(lp.targets.size());
    if (n_sources) *n_sources = int64_t(lp.sources.size());
  });
}

int cfm_plan_info(cfm_handler* h, int level, int* mode, double* target_fill) {
  return guarded([&] {
    if (!h) throw Error(CFM_ERR_VALUE, "null handler");
    std::lock_guard<std::mutex> lk(h->mu);
    auto it = h->plans.find(level);
    if (it == h->plans.end()) throw Error(CFM_ERR_PRECOMPUTE, "no plan for level " + std::to_string(level));
    if (mode) *mode = it->second.mode;
    if (target_fill) *target_fill = it->second.target_fill;
  });
}

int cfm_plan_two_stage(cfm_handler* h, int level, int* two_stage) {
  return guarded([&] {
    if (!h) throw Error(CFM_ERR_VALUE, "null handler");
    std::lock_guard<std::mutex> lk(h->mu);
    auto it = h->plans.find(level);
    if (it == h->plans.end()) throw Error(CFM_ERR_PRECOMPUTE, "no plan for level " + std::to_string(level));
    if (two_stage) *two_stage = it->second.ts ? 1 : 0;
  });
}

int cfm_classify_count(int device, int level, int64_t n_cells, const int32_t* ijk, int64_t* offsets_out,
                       int64_t* total_out) {
  return guarded([&] {
    CUDA_CHECK(cudaSetDevice(device));
    cudaStream_t s;
    CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    DeviceLists dl;
    try {
      classify_device(level, n_cells, ijk, s, dl, false);
    } catch (...) {
      cudaStreamDestroy(s);
      throw;
    }
    cudaStreamDestroy(s);
    if (offsets_out) std::copy(dl.h_off.begin(), dl.h_off.end(), offsets_out);
    if (total_out) *total_out = dl.total;
  });
}

int cfm_classify_fill(int device, int level, int64_t n_cells, const int32_t* ijk, const int64_t* offsets,
                      int32_t* src_out, int8_t* t_out, uint8_t* rep_out, uint8_t* perm_out) {
  return guarded([&] {
    if (!offsets || !src_out) throw Error(CFM_ERR_VALUE, "offsets and src_out are required");
    CUDA_CHECK(cudaSetDevice(device));
    cudaStream_t s;
    CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    DeviceLists dl;
    try {
      classify_device(level, n_cells, ijk, s, dl, false, src_out, t_out, rep_out, perm_out, offsets);
    } catch (...) {
      cudaStreamDestroy(s);
      throw;
    }
    cudaStreamDestroy(s);
  });
}

int cfm_classify_targets_count(int device, int level, int64_t n_cells, const int32_t* ijk, int64_t n_targets,
                               const int64_t* target_rows, int64_t* offsets_out, int64_t* total_out) {
  return guarded([&] {
    if (n_targets < 0 || (n_targets && !target_rows)) throw Error(CFM_ERR_VALUE, "bad target rows");
    CUDA_CHECK(cudaSetDevice(device));
    cudaStream_t s;
    CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    DeviceLists dl;
    try {
      classify_device(level, n_cells, ijk, s, dl, false, nullptr, nullptr, nullptr, nullptr, nullptr, target_rows,
                      n_targets);
    } catch (...) {
      cudaStreamDestroy(s);
      throw;
    }
    cudaStreamDestroy(s);
    if (offsets_out) std::copy(dl.h_off.begin(), dl.h_off.end(), offsets_out);
    if (total_out) *total_out = dl.total;
  });
}

int cfm_classify_targets_fill(int device, int level, int64_t n_cells, const int32_t* ijk, int64_t n_targets,
                              const int64_t* target_rows, const int64_t* offsets, int32_t* src_out, int8_t* t_out) {
  return guarded([&] {
    if (!offsets || !src_out) throw Error(CFM_ERR_VALUE, "offsets and src_out are required");
    if (n_targets < 0 || (n_targets && !target_rows)) throw Error(CFM_ERR_VALUE, "bad target rows");
    CUDA_CHECK(cudaSetDevice(device));
    cudaStream_t s;
    CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    DeviceLists dl;
    try {
      classify_device(level, n_cells, ijk, s, dl, false, src_out, t_out, nullptr, nullptr, offsets, target_rows,
                      n_targets);
    } catch (...) {
      cudaStreamDestroy(s);
      throw;
    }
    cudaStreamDestroy(s);
  });
}

// Row gather for the multi-GPU halo (pack the rows a peer needs into one
// contiguous send buffer): dst[k] = src[rows[k]], rows of `row_doubles`
// doubles.  One warp per row, 16-B loads when the rows allow it.
__global__ void k_gather_rows(const double* __restrict__ src, long long row_doubles,
                              const long long* __restrict__ rows, long long n, double* __restrict__ dst) {
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  const bool vec = (row_doubles & 1) == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  for (long long k = warp; k < n; k += nw) {
    const double* s = src + rows[k] * row_doubles;
    double* d = dst + k * row_doubles;
    if (vec) {
      const double2* s2 = reinterpret_cast<const double2*>(s);
      double2* d2 = reinterpret_cast<double2*>(d);
      for (long long j = lane; j < row_doubles / 2; j += 32) d2[j] = __ldg(s2 + j);
    } else {
      for (long long j = lane; j < row_doubles; j += 32) d[j] = __ldg(s + j);
    }
  }
}

int cfm_gather_rows(int device, const double* src, int64_t row_doubles, const int64_t* rows, int64_t n, double* dst,
                    void* stream) {
  return guarded([&] {
    if (n < 0 || row_doubles <= 0) throw Error(CFM_ERR_VALUE, "bad sizes");
    if (n == 0) return;
    if (!is_device_ptr(src) || !is_device_ptr(rows) || !is_device_ptr(dst))
      throw Error(CFM_ERR_VALUE, "device pointers required");
    CUDA_CHECK(cudaSetDevice(device));
    const int threads = 256;
    const long long blocks = std::min<long long>((n + 7) / 8, 148LL * 16);
    k_gather_rows<<<unsigned(blocks), threads, 0, static_cast<cudaStream_t>(stream)>>>(
        src, row_doubles, reinterpret_cast<const long long*>(rows), n, dst);
    CUDA_CHECK(cudaGetLastError());
  });
}

// Device-output classifier: offsets/sources/codes stay on the device (for a
// device-side pipeline and for timing the kernels alone).  ijk must be device.
int cfm_classify_count_device(int device, int level, int64_t n_cells, const int32_t* ijk, int64_t* offsets_dev,
                              int64_t* total_out, void* stream) {
  return guarded([&] {
    if (level < 2 || level > 9) throw Error(CFM_ERR_VALUE, "classifier supports levels 2..9");
    if (!is_device_ptr(ijk) || !is_device_ptr(offsets_dev)) throw Error(CFM_ERR_VALUE, "device pointers required");
    CUDA_CHECK(cudaSetDevice(device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    init_cone_table();
    const int S = 1 << level;
    ClassifyScratch& scr = classify_scratch(device);
    DevBuf& grid = scr.grid;
    DevBuf& counts = scr.counts;
    grid.alloc(size_t(S) * S * S * sizeof(int));
    counts.alloc(std::max<size_t>(size_t(n_cells + 1) * sizeof(long long), 16));
    CUDA_CHECK(cudaMemsetAsync(grid.p, 0xff, size_t(S) * S * S * sizeof(int), s));
    const unsigned nb = unsigned((n_cells + 255) / 256);
    if (n_cells) {
      k_grid_scatter<<<nb, 256, 0, s>>>(ijk, n_cells, S, grid.as<int>());
      const unsigned nbw = classify_warp_blocks<false>(n_cells, device);
      k_classify_warp<false><<<nbw, 256, 0, s>>>(ijk, n_cells, S, grid.as<int>(), reinterpret_cast<int*>(counts.p),
                                                 nullptr, nullptr, nullptr);
      CUDA_CHECK(cudaGetLastError());
    }
    // offsets = exclusive scan of the counts (int -> int64), n+1 entries
    CUDA_CHECK(cudaMemsetAsync(offsets_dev, 0, sizeof(int64_t), s));
    if (n_cells) {
      size_t tmp = 0;
      const int* cin = reinterpret_cast<const int*>(counts.p);
      CUDA_CHECK(cub::DeviceScan::InclusiveSum(nullptr, tmp, cin, reinterpret_cast<long long*>(offsets_dev) + 1,
                                               int64_t(n_cells), s));
      DevBuf t;
      t.alloc(std::max<size_t>(tmp, 16));
      CUDA_CHECK(cub::DeviceScan::InclusiveSum(t.p, tmp, cin, reinterpret_cast<long long*>(offsets_dev) + 1,
                                               int64_t(n_cells), s));
    }
    long long total = 0;
    CUDA_CHECK(cudaMemcpyAsync(&total, offsets_dev + n_cells, 8, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    if (total_out) *total_out = total;
  });
}

int cfm_classify_fill_device(int device, int level, int64_t n_cells, const int32_t* ijk, const int64_t* offsets_dev,
                             int32_t* src_dev, int16_t* code_dev, void* stream) {
  return guarded([&] {
    if (level < 2 || level > 9) throw Error(CFM_ERR_VALUE, "classifier supports levels 2..9");
    CUDA_CHECK(cudaSetDevice(device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    init_cone_table();
    const int S = 1 << level;
    DevBuf& grid = classify_scratch(device).grid;
    grid.alloc(size_t(S) * S * S * sizeof(int));
    CUDA_CHECK(cudaMemsetAsync(grid.p, 0xff, size_t(S) * S * S * sizeof(int), s));
    const unsigned nb = unsigned((n_cells + 255) / 256);
    if (n_cells) {
      k_grid_scatter<<<nb, 256, 0, s>>>(ijk, n_cells, S, grid.as<int>());
      const unsigned nbw = classify_warp_blocks<true>(n_cells, device);
      k_classify_warp<true><<<nbw, 256, 0, s>>>(ijk, n_cells, S, grid.as<int>(), nullptr,
                                                reinterpret_cast<const long long*>(offsets_dev), src_dev, code_dev);
      CUDA_CHECK(cudaGetLastError());
    }
  });
}

int cfm_tree_build(int device, const double* points, int64_t n, const double* center, double half_width, int depth,
                   cfm_tree** out) {
  return guarded([&] {
    if (!out || !center) throw Error(CFM_ERR_VALUE, "null argument");
    if (depth < 2) throw Error(CFM_ERR_VALUE, "octree depth must be >= 2, got " + std::to_string(depth));
    if (depth > 20) throw Error(CFM_ERR_VALUE, "octree depth must be <= 20");
    if (n < 0) throw Error(CFM_ERR_VALUE, "negative particle count");
    if (!(half_width > 0)) throw Error(CFM_ERR_VALUE, "half_width must be positive");
    CUDA_CHECK(cudaSetDevice(device));
    cudaStream_t s = nullptr;
    auto t = std::make_unique<cfm_tree>();
    t->device = device;
    t->depth = depth;
    t->n_points = n;
    t->levels.resize(depth + 1);
    for (int a = 0; a < 3; ++a) t->center[a] = center[a];
    t->half = half_width;
    t->points.alloc(std::max<size_t>(size_t(n) * 24, 16));
    if (n) CUDA_CHECK(cudaMemcpy(t->points.p, points, size_t(n) * 24, cudaMemcpyDefault));
    const double* dp = t->points.as<double>();
    DevBuf keys, idx, skeys, sidx, bad;
    keys.alloc(std::max<size_t>(size_t(n) * 8, 16));
    idx.alloc(std::max<size_t>(size_t(n) * 8, 16));
    bad.alloc(16);
    CUDA_CHECK(cudaMemset(bad.p, 0, 4));
    const double lx = center[0] - half_width, ly = center[1] - half_width, lz = center[2] - half_width;
    const double width = 2.0 * half_width;
    if (n) {
      k_leaf_keys<<<unsigned((n + 255) / 256), 256, 0, s>>>(dp, n, lx, ly, lz, width, depth,
                                                            keys.as<unsigned long long>(), idx.as<long long>(),
                                                            bad.as<int>());
      CUDA_CHECK(cudaGetLastError());
    }
    int hb = 0;
    CUDA_CHECK(cudaMemcpy(&hb, bad.p, 4, cudaMemcpyDeviceToHost));
    if (hb) throw Error(CFM_ERR_VALUE, "particle outside bounding box");
    // stable sort of (leaf key, particle index): particle indices ascend within a leaf
    skeys.alloc(std::max<size_t>(size_t(n) * 8, 16));
    sidx.alloc(std::max<size_t>(size_t(n) * 8, 16));
    t->perm.alloc(std::max<size_t>(size_t(n) * 8, 16));
    if (n) {
      cub_call([&](void* tp, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(tp, b, keys.as<unsigned long long>(), skeys.as<unsigned long long>(),
                                               idx.as<long long>(), t->perm.as<long long>(), int64_t(n), 0,
                                               key_bits(depth), s);
      }, s);
    }
    // leaves: unique keys and run lengths -> CSR offsets
    DevBuf counts;
    TreeLevel& leaf = t->levels[depth];
    leaf.n = n ? sort_unique(skeys.as<unsigned long long>(), n, leaf.keys, &counts, key_bits(depth), s) : 0;
    std::vector<long long> hc(leaf.n), ho(leaf.n + 1, 0);
    if (leaf.n) CUDA_CHECK(cudaMemcpy(hc.data(), counts.p, size_t(leaf.n) * 8, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < leaf.n; ++i) ho[i + 1] = ho[i] + hc[i];
    upload(t->leaf_off, ho);
    // coarser levels: sorted unique parents
    for (int L = depth; L >= 1; --L) {
      const TreeLevel& c = t->levels[L];
      TreeLevel& pl = t->levels[L - 1];
      if (c.n == 0) {
        pl.n = 0;
        continue;
      }
      DevBuf par;
      par.alloc(size_t(c.n) * 8);
      k_parent_keys<<<unsigned((c.n + 255) / 256), 256, 0, s>>>(c.keys.as<unsigned long long>(), c.n, 1ll << L,
                                                                par.as<unsigned long long>());
      CUDA_CHECK(cudaGetLastError());
      pl.n = sort_unique(par.as<unsigned long long>(), c.n, pl.keys, nullptr, key_bits(L - 1), s);
    }
    *out = t.release();
  });
}

int cfm_tree_level_size(cfm_tree* t, int level, int64_t* n_cells) {
  return guarded([&] {
    if (!t || !n_cells) throw Error(CFM_ERR_VALUE, "null argument");
    if (level < 0 || level > t->depth) throw Error(CFM_ERR_VALUE, "level outside the tree");
    *n_cells = t->levels[level].n;
  });
}

int cfm_tree_level_cells(cfm_tree* t, int level, int32_t* ijk_out) {
  return guarded([&] {
    if (!t || !ijk_out) throw Error(CFM_ERR_VALUE, "null argument");
    if (level < 0 || level > t->depth) throw Error(CFM_ERR_VALUE, "level outside the tree");
    CUDA_CHECK(cudaSetDevice(t->device));
    const TreeLevel& L = t->levels[level];
    if (!L.n) return;
    const bool dev = is_device_ptr(ijk_out);
    DevBuf tmp;
    int* d = ijk_out;
    if (!dev) {
      tmp.alloc(size_t(L.n) * 12);
      d = tmp.as<int>();
    }
    k_keys_to_ijk<<<unsigned((L.n + 255) / 256), 256>>>(L.keys.as<unsigned long long>(), L.n, 1ll << level, d);
    CUDA_CHECK(cudaGetLastError());
    if (!dev) CUDA_CHECK(cudaMemcpy(ijk_out, d, size_t(L.n) * 12, cudaMemcpyDeviceToHost));
    CUDA_CHECK(cudaDeviceSynchronize());
  });
}

int cfm_tree_leaf_particles(cfm_tree* t, int64_t* offsets_out, int64_t* perm_out) {
  return guarded([&] {
    if (!t) throw Error(CFM_ERR_VALUE, "null argument");
    CUDA_CHECK(cudaSetDevice(t->device));
    const int64_t nl = t->levels[t->depth].n;
    if (offsets_out)
      CUDA_CHECK(cudaMemcpy(offsets_out, t->leaf_off.p, size_t(nl + 1) * 8, cudaMemcpyDefault));
    if (perm_out && t->n_points)
      CUDA_CHECK(cudaMemcpy(perm_out, t->perm.p, size_t(t->n_points) * 8, cudaMemcpyDefault));
  });
}

int cfm_tree_destroy(cfm_tree* t) {
  return guarded([&] {
    if (!t) return;
    cudaSetDevice(t->device);
    delete t;
  });
}

// ---------------------------------------------------------------- FMM stages
static FmmGeom fmm_geom(cfm_fmm* f) {
  FmmGeom g{};
  cfm_tree* t = f->tree;
  g.pts = t->points.as<double>();
  g.perm = t->perm.as<long long>();
  g.leaf_off = t->leaf_off.as<long long>();
  g.leaf_ijk = f->leaf_ijk.as<int>();
  g.n_leaves = t->levels[t->depth].n;
  g.depth = t->depth;
  g.lx = t->center[0] - t->half;
  g.ly = t->center[1] - t->half;
  g.lz = t->center[2] - t->half;
  g.leaf_w = 2.0 * t->half / double(1ll << t->depth);
  g.troots = f->troots.as<double>();
  g.order = f->order;
  return g;
}

static std::vector<unsigned long long> host_keys(cfm_tree* t, int level) {
  std::vector<unsigned long long> k(t->levels[level].n);
  if (!k.empty())
    CUDA_CHECK(cudaMemcpy(k.data(), t->levels[level].keys.p, k.size() * 8, cudaMemcpyDeviceToHost));
  return k;
}

// M2M (child level L -> parent L-1) or L2L (parent L-1 -> child L) plan
static LevelPlan& fmm_plan(cfm_fmm* f, int child_level, bool up, int dc) {
  auto& plans = up ? f->m2m_plans : f->l2l_plans;
  const int key = child_level * 4 + dc;
  auto it = plans.find(key);
  if (it != plans.end()) return it->second;
  cfm_tree* t = f->tree;
  auto ck = host_keys(t, child_level);
  auto pk = host_keys(t, child_level - 1);
  const long long cs = 1ll << child_level, ps = cs >> 1;
  const int64_t nc = int64_t(ck.size()), np_ = int64_t(pk.size());
  std::vector<int64_t> parent(nc);
  std::vector<int16_t> oct(nc);
  for (int64_t c = 0; c < nc; ++c) {
    const long long z = ck[c] % cs, y = (ck[c] / cs) % cs, x = ck[c] / (cs * cs);
    const unsigned long long pkey = (unsigned long long)(((x >> 1) * ps + (y >> 1)) * ps + (z >> 1));
    parent[c] = int64_t(std::lower_bound(pk.begin(), pk.end(), pkey) - pk.begin());
    oct[c] = int16_t((x & 1) * 4 + (y & 1) * 2 + (z & 1));
  }
  std::vector<int64_t> tgt, off(1, 0), src;
  std::vector<int16_t> codes;
  if (up) {  // targets = parents, pairs = their children in octant (lexicographic) order
    std::vector<int64_t> ord(nc);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
      return parent[a] != parent[b] ? parent[a] < parent[b] : oct[a] < oct[b];
    });
    for (int64_t i = 0; i < nc;) {
      int64_t j = i;
      tgt.push_back(parent[ord[i]]);
      while (j < nc && parent[ord[j]] == parent[ord[i]]) {
        src.push_back(ord[j]);
        codes.push_back(oct[ord[j]]);
        ++j;
      }
      off.push_back(int64_t(src.size()));
      i = j;
    }
  } else {  // targets = children, one pair each: (parent, octant)
    for (int64_t c = 0; c < nc; ++c) {
      tgt.push_back(c);
      src.push_back(parent[c]);
      codes.push_back(oct[c]);
      off.push_back(int64_t(src.size()));
    }
  }
  std::array<int, kNumCodes> opkey;
  opkey.fill(-1);
  for (int c = 0; c < 8; ++c) opkey[c] = c;
  LevelPlan lp;
  try {
    lp.hp = build_plan_csr(int64_t(tgt.size()), tgt.data(), off.data(), src.data(), codes.data(), dc, opkey,
                           std::max(nc, np_));
  } catch (const PlanError& e) {
    throw Error(CFM_ERR_VALUE, e.what());
  }
  lp.dc = dc;
  lp.n_rows = std::max(nc, np_);
  push_plan(lp.hp, lp.tile_col, lp.tile_off, lp.entry_code, lp.entry_src);
  plans[key] = std::move(lp);
  return plans[key];
}

static void fmm_shift(cfm_fmm* f, int child_level, bool up, const double* x, double* y, int data_complex,
                      cudaStream_t s) {
  if (child_level < 1 || child_level > f->tree->depth) throw Error(CFM_ERR_VALUE, "level outside the tree");
  const int dc = data_complex ? 2 : 1;
  LevelPlan& lp = fmm_plan(f, child_level, up, dc);
  TileParams p{};
  fill_ops(p, up ? f->m2m_ops : f->l2l_ops, f->octmap);
  fill_plan(p, lp.tile_col, lp.tile_off, lp.entry_code, lp.entry_src, lp.hp.n_tiles);
  const long long row_ld = (long long)f->n * dc;
  p.x = x; p.x_ld = row_ld; p.x_dc = dc;
  p.y = y; p.y_ld = row_ld; p.y_dc = dc;
  p.scale = 1.0; p.accumulate = 1;
  launch_tiles(p, lp.hp.n_tiles, s);
}

int cfm_fmm_create(cfm_tree* t, int order, const double* shift_mats, cfm_fmm** out) {
  return guarded([&] {
    if (!t || !out || !shift_mats) throw Error(CFM_ERR_VALUE, "null argument");
    if (order < 2 || order > kMaxOrder) throw Error(CFM_ERR_VALUE, "order must be in [2, 12]");
    if (t->depth > 9) throw Error(CFM_ERR_VALUE, "FMM stages support depth <= 9");
    CUDA_CHECK(cudaSetDevice(t->device));
    auto f = std::make_unique<cfm_fmm>();
    f->tree = t;
    f->order = order;
    f->n = order * order * order;
    const int n = f->n;
    // T_k(root_i), k = 1..l-1 (interp.py:88-103 at the roots)
    std::vector<double> roots(order), tr(size_t(order) * (order - 1));
    const int half = order / 2;
    for (int i = 1; i <= half; ++i) roots[i - 1] = std::cos((2 * i - 1) * M_PI / (2 * order));
    if (order % 2) roots[half] = 0.0;
    for (int i = 0; i < half; ++i) roots[order - half + i] = -roots[half - 1 - i];
    for (int i = 0; i < order; ++i) {
      const double x = roots[i];
      double tm2 = 0, tm1 = 0;
      for (int k = 0; k < order - 1; ++k) {
        double v = (k == 0) ? x : (k == 1 ? 2.0 * x * x - 1.0 : 2.0 * x * tm1 - tm2);
        tr[size_t(i) * (order - 1) + k] = v;
        tm2 = tm1;
        tm1 = v;
      }
    }
    upload(f->troots, tr);
    const int64_t nl = t->levels[t->depth].n;
    f->leaf_ijk.alloc(std::max<size_t>(size_t(nl) * 12, 16));
    if (nl) {
      k_keys_to_ijk<<<unsigned((nl + 255) / 256), 256>>>(t->levels[t->depth].keys.as<unsigned long long>(), nl,
                                                          1ll << t->depth, f->leaf_ijk.as<int>());
      CUDA_CHECK(cudaGetLastError());
    }
    const long long S = 1ll << t->depth;
    f->leaf_grid.alloc(size_t(S * S * S) * sizeof(int));
    CUDA_CHECK(cudaMemset(f->leaf_grid.p, 0xff, f->leaf_grid.bytes));
    if (nl) k_leaf_grid<<<unsigned((nl + 255) / 256), 256>>>(f->leaf_ijk.as<int>(), nl, int(S), f->leaf_grid.as<int>());
    f->leaf_of_pos.alloc(std::max<size_t>(size_t(t->n_points) * 8, 16));
    if (nl) k_leaf_of_pos<<<unsigned((nl + 255) / 256), 256>>>(t->leaf_off.as<long long>(), nl, f->leaf_of_pos.as<long long>());
    CUDA_CHECK(cudaGetLastError());
    // M2M operators: mat (parent x child) per octant; L2L: transposes
    make_stack(f->m2m_ops, 8, n, n);
    make_stack(f->l2l_ops, 8, n, n);
    std::vector<double> blk(f->m2m_ops.stride), blt(f->l2l_ops.stride);
    for (int o = 0; o < 8; ++o) {
      std::fill(blk.begin(), blk.end(), 0.0);
      std::fill(blt.begin(), blt.end(), 0.0);
      const double* m = shift_mats + size_t(o) * n * n;
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          blk[size_t(i) * f->m2m_ops.ld + j] = m[size_t(i) * n + j];
          blt[size_t(j) * f->l2l_ops.ld + i] = m[size_t(i) * n + j];
        }
      put_stack(f->m2m_ops, o, blk);
      put_stack(f->l2l_ops, o, blt);
    }
    for (int c = 0; c < 8; ++c) f->octmap.op[c] = c;
    f->octmap.push();
    CUDA_CHECK(cudaDeviceSynchronize());
    *out = f.release();
  });
}

int cfm_fmm_destroy(cfm_fmm* f) {
  return guarded([&] {
    if (!f) return;
    cudaSetDevice(f->tree->device);
    delete f;
  });
}

int cfm_fmm_p2m(cfm_fmm* f, const double* weights, int data_complex, double* leaf_mpoles, void* stream) {
  return guarded([&] {
    if (!f) throw Error(CFM_ERR_VALUE, "null handle");
    CUDA_CHECK(cudaSetDevice(f->tree->device));
    const int dc = data_complex ? 2 : 1;
    FmmGeom g = fmm_geom(f);
    if (!g.n_leaves) return;
    constexpr int CH = 64;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned nb = unsigned(g.n_leaves);
    const long long ld = (long long)f->n * dc;
    switch (f->order) {
      case 3: k_p2m_t<3, CH><<<nb, 128, 0, st>>>(g, weights, dc, leaf_mpoles, ld); break;
      case 4: k_p2m_t<4, CH><<<nb, 128, 0, st>>>(g, weights, dc, leaf_mpoles, ld); break;
      case 5: k_p2m_t<5, CH><<<nb, 128, 0, st>>>(g, weights, dc, leaf_mpoles, ld); break;
      case 6: k_p2m_t<6, CH><<<nb, 128, 0, st>>>(g, weights, dc, leaf_mpoles, ld); break;
      case 7: k_p2m_t<7, CH><<<nb, 128, 0, st>>>(g, weights, dc, leaf_mpoles, ld); break;
      case 8: k_p2m_t<8, CH><<<nb, 128, 0, st>>>(g, weights, dc, leaf_mpoles, ld); break;
      case 9: k_p2m_t<9, CH><<<nb, 128, 0, st>>>(g, weights, dc, leaf_mpoles, ld); break;
      default: {
        const int threads = f->n <= 1024 ? 128 : 256;
        const size_t smem = size_t(3 * f->order * CH + CH * 2) * sizeof(double);
        k_p2m<CH><<<nb, threads, smem, st>>>(g, weights, dc, leaf_mpoles, ld);
      }
    }
    CUDA_CHECK(cudaGetLastError());
  });
}

int cfm_fmm_m2m(cfm_fmm* f, int child_level, const double* child, double* parent, int data_complex, void* stream) {
  return guarded([&] {
    if (!f) throw Error(CFM_ERR_VALUE, "null handle");
    CUDA_CHECK(cudaSetDevice(f->tree->device));
    fmm_shift(f, child_level, true, child, parent, data_complex, static_cast<cudaStream_t>(stream));
  });
}

int cfm_fmm_l2l(cfm_fmm* f, int parent_level, const double* parent, double* child, int data_complex, void* stream) {
  return guarded([&] {
    if (!f) throw Error(CFM_ERR_VALUE, "null handle");
    CUDA_CHECK(cudaSetDevice(f->tree->device));
    fmm_shift(f, parent_level + 1, false, parent, child, data_complex, static_cast<cudaStream_t>(stream));
  });
}

int cfm_fmm_l2p(cfm_fmm* f, const double* leaf_locals, int data_complex, double* potentials, void* stream) {
  return guarded([&] {
    if (!f) throw Error(CFM_ERR_VALUE, "null handle");
    CUDA_CHECK(cudaSetDevice(f->tree->device));
    const int dc = data_complex ? 2 : 1;
    FmmGeom g = fmm_geom(f);
    const long long np_ = f->tree->n_points;
    if (!np_) return;
    const unsigned nb = unsigned((np_ + 127) / 128);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long* lop = f->leaf_of_pos.as<long long>();
    const long long ld = (long long)f->n * dc;
    switch (f->order) {
      case 3: k_l2p_t<3><<<nb, 128, 0, st>>>(g, lop, leaf_locals, ld, dc, potentials, np_); break;
      case 4: k_l2p_t<4><<<nb, 128, 0, st>>>(g, lop, leaf_locals, ld, dc, potentials, np_); break;
      case 5: k_l2p_t<5><<<nb, 128, 0, st>>>(g, lop, leaf_locals, ld, dc, potentials, np_); break;
      case 6: k_l2p_t<6><<<nb, 128, 0, st>>>(g, lop, leaf_locals, ld, dc, potentials, np_); break;
      case 7: k_l2p_t<7><<<nb, 128, 0, st>>>(g, lop, leaf_locals, ld, dc, potentials, np_); break;
      case 8: k_l2p_t<8><<<nb, 128, 0, st>>>(g, lop, leaf_locals, ld, dc, potentials, np_); break;
      case 9: k_l2p_t<9><<<nb, 128, 0, st>>>(g, lop, leaf_locals, ld, dc, potentials, np_); break;
      default: k_l2p<<<nb, 128, 0, st>>>(g, lop, leaf_locals, ld, dc, potentials, np_);
    }
    CUDA_CHECK(cudaGetLastError());
  });
}

int cfm_fmm_p2p(cfm_fmm* f, int kernel, double wavenumber, const double* weights, int weights_complex,
                double* potentials, int out_complex, void* stream) {
  return guarded([&] {
    if (!f) throw Error(CFM_ERR_VALUE, "null handle");
    if (kernel != 0 && kernel != 1) throw Error(CFM_ERR_VALUE, "kernel must be 0 (Laplace) or 1 (Helmholtz)");
    if (weights_complex && !out_complex) throw Error(CFM_ERR_VALUE, "complex weights need complex potentials");
    if (kernel == 1 && !out_complex) throw Error(CFM_ERR_VALUE, "Helmholtz potentials are complex");
    CUDA_CHECK(cudaSetDevice(f->tree->device));
    FmmGeom g = fmm_geom(f);
    if (!g.n_leaves) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long np_ = f->tree->n_points;
    const unsigned nb = unsigned((np_ + 255) / 256);
    if (f->n_small < 0) {
      // leaf-sorted positions and the two leaf-size classes (<= 64 particles, more)
      f->px.alloc(std::max<size_t>(size_t(np_) * 8, 16));
      f->py.alloc(std::max<size_t>(size_t(np_) * 8, 16));
      f->pz.alloc(std::max<size_t>(size_t(np_) * 8, 16));
      if (np_) k_p2p_sort_pos<<<nb, 256, 0, st>>>(g.pts, g.perm, np_, f->px.as<double>(), f->py.as<double>(),
                                                    f->pz.as<double>());
      CUDA_CHECK(cudaGetLastError());
      std::vector<long long> off(size_t(g.n_leaves) + 1);
      CUDA_CHECK(cudaMemcpy(off.data(), g.leaf_off, off.size() * 8, cudaMemcpyDeviceToHost));
      std::vector<long long> sm, lg;
      for (long long l = 0; l < g.n_leaves; ++l) (off[l + 1] - off[l] <= 64 ? sm : lg).push_back(l);
      upload(f->small_leaves, sm);
      upload(f->large_leaves, lg);
      f->n_small = int64_t(sm.size());
      f->n_large = int64_t(lg.size());
    }
    const int wdc = weights_complex ? 2 : 1;
    f->sw.alloc(std::max<size_t>(size_t(np_) * wdc * 8, 16));
    if (np_) {
      if (wdc == 2) k_p2p_sort_w<2><<<nb, 256, 0, st>>>(weights, g.perm, np_, f->sw.as<double>());
      else k_p2p_sort_w<1><<<nb, 256, 0, st>>>(weights, g.perm, np_, f->sw.as<double>());
      CUDA_CHECK(cudaGetLastError());
    }
    P2PGeom pg{g.leaf_off, g.leaf_ijk, f->leaf_grid.as<int>(), 1 << g.depth, f->px.as<double>(), f->py.as<double>(),
               f->pz.as<double>(), g.perm};
    auto run = [&](auto ker, auto wd, auto od) {
      constexpr int K = decltype(ker)::value, W = decltype(wd)::value, O = decltype(od)::value;
      if (f->n_small)
        k_p2p_small<K, W, O><<<unsigned(f->n_small), 128, 0, st>>>(pg, f->small_leaves.as<long long>(),
                                                                  f->sw.as<double>(), wavenumber, potentials);
      if (f->n_large)
        k_p2p_large<K, W, O><<<unsigned(f->n_large), 128, 0, st>>>(pg, f->large_leaves.as<long long>(),
                                                                  f->sw.as<double>(), wavenumber, potentials);
      CUDA_CHECK(cudaGetLastError());
    };
    using I0 = std::integral_constant<int, 0>;
    using I1 = std::integral_constant<int, 1>;
    using I2 = std::integral_constant<int, 2>;
    if (kernel == 0 && wdc == 1 && !out_complex) run(I0{}, I1{}, I1{});
    else if (kernel == 0 && wdc == 1) run(I0{}, I1{}, I2{});
    else if (kernel == 0) run(I0{}, I2{}, I2{});
    else if (wdc == 1) run(I1{}, I1{}, I2{});
    else run(I1{}, I2{}, I2{});
  });
}

int cfm_assemble_operators(int device, int kernel, double wavenumber, int n, const double* nodes, double width,
                           int n_t, const int8_t* transfers, double* out, void* stream) {
  return guarded([&] {
    if (kernel != 0 && kernel != 1) throw Error(CFM_ERR_VALUE, "kernel must be 0 (Laplace) or 1 (Helmholtz)");
    if (n <= 0 || n > 2048 || n_t < 0) throw Error(CFM_ERR_VALUE, "bad operator size");
    if (!(width > 0.0)) throw Error(CFM_ERR_VALUE, "cell width must be positive");
    if (n_t == 0) return;
    if (!nodes || !transfers || !out) throw Error(CFM_ERR_VALUE, "null pointer");
    for (int t = 0; t < n_t; ++t) {
      const int a = transfers[3 * t], b = transfers[3 * t + 1], c = transfers[3 * t + 2];
      if (a * a + b * b + c * c <= 3) throw Error(CFM_ERR_VALUE, "transfer vector is not admissible (|t| <= sqrt(3))");
    }
    CUDA_CHECK(cudaSetDevice(device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    DevBuf dn, dt;
    dn.alloc(size_t(n) * 3 * sizeof(double));
    dt.alloc(size_t(n_t) * 3);
    CUDA_CHECK(cudaMemcpyAsync(dn.p, nodes, size_t(n) * 3 * sizeof(double), cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaMemcpyAsync(dt.p, transfers, size_t(n_t) * 3, cudaMemcpyHostToDevice, st));
    const long long nn = (long long)n * n;
    dim3 grid(unsigned((nn + 255) / 256), unsigned(n_t));
    k_assemble<<<grid, 256, size_t(n) * 3 * sizeof(double), st>>>(kernel, wavenumber, n, dn.as<double>(), width,
                                                                 dt.as<int8_t>(), out);
    CUDA_CHECK(cudaGetLastError());
    CUDA_CHECK(cudaStreamSynchronize(st));  // the staging buffers are freed on return
  });
}

int cfm_last_csr_plan_info(cfm_handler* h, int* cache_hit, int* mode, int* two_stage) {
  return guarded([&] {
    if (!h) throw Error(CFM_ERR_VALUE, "null handler");
    std::lock_guard<std::mutex> lk(h->mu);
    if (cache_hit) *cache_hit = h->last_csr_hit ? 1 : 0;
    if (mode) *mode = h->last_csr_mode;
    if (two_stage) *two_stage = h->last_csr_two_stage;
  });
}

int cfm_last_apply_stats(cfm_handler* h, double* ms, int64_t* launches) {
  return guarded([&] {
    if (!h) throw Error(CFM_ERR_VALUE, "null handler");
    if (ms) *ms = h->last_ms;
    if (launches) *launches = h->last_launches;
  });
}

}  // extern "C"
