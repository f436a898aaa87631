// Internal declarations shared by the translation units of libchebm2l.so
// (structs of the operator cache, plans and handler; helpers used across
// files).  Not part of the C ABI (include/chebm2l.h is).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
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
#include "plan.hpp"
#include "symmetry.hpp"
#include "tile_gemm.cuh"
#include "tile_gemm_ws.cuh"
#include "lowrank_ws.cuh"


namespace cfm {

extern thread_local std::string g_last_error;

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
inline void upload(DevBuf& d, const std::vector<T>& h) {
  d.alloc(std::max<size_t>(h.size() * sizeof(T), 16));
  if (!h.empty()) CUDA_CHECK(cudaMemcpy(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
}

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

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

inline void realify_into(const double* src, int m, int k, bool cplx, double* dst, int ld, bool conj_t = false) {
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
  CUtensorMap lrf_umap, lrf_vmap;  // box (KC + 4) x 128 over the two stacks (two-pass path on the persistent kernel)
  bool has_lrmaps = false;
  // two-stage low-rank mode (real, dense levels): stage 1 Y = V_t^H x per
  // (source, transfer) for the whole transfer set of the source's class, as a
  // dense GEMM against a per-class stack of V_t^H rows; stage 2 sums U_t Y per
  // target tile.  Classes: per axis the transfer components lie in [-3, 2]
  // (bit 0) or [-2, 3] (bit 1), which holds for every source of an octree
  // level (octree.py:157-175).  Ranks are cut in 16-wide segments (<= 2).
  bool has_ts = false;
  int ts_nb = 0;                 // 128-row blocks per class stack
  std::vector<int> ts_rank;      // per transfer index
  std::vector<int> ts_rho0;      // [8][n_transfers] first row of the transfer's rank rows in the class stack, -1 if absent
  int ts_ldy = 0;                // Y row length: every transfer's rank rows (ceil4) at a fixed column
  DevBuf ts_colmap;              // [8 * ts_nb * 128] class-stack row -> Y column (-1: padding row)
  DevBuf ts_opcol;               // [2 * n_transfers] stage-2 operator 2k + j -> first Y column of its segment
  int ts_ntr = 0;
  OpStack ts_v;                  // 8 * ts_nb blocks of 128 rows x n
  CUtensorMap ts_vmap, ts_umap;  // box 36 x 128 over ts_v; box 20 x 128 over lrf_left
  DevBuf ts_ksteps;              // per stage-2 entry code 2k + j: k-steps holding rank columns (ceil(w / 4))
  // target-major two-stage mode (round 2, default): Y is laid out by TARGET --
  // Y_T[target][rho_T[class(target)][k] + a] = (V_k^H x_source)[a] for the pair
  // (target, source, k) -- with every class's transfers packed back to back at
  // their exact ranks, so stage 2 is one dense GEMM per target class,
  // locals[:, targets] += U_c (n x R_c) Y_T[targets]^T, with K = R_c running
  // over whole 128-column blocks (no per-entry rank padding, contiguous B rows)
  bool has_tsT = false;
  int tsT_nb = 0;                // 128-wide blocks per class (rows of the V stack = columns of the U stack)
  int tsT_nslots = 0;            // transfers per class (189 for octree lists)
  std::vector<int> tsT_rho;      // [8][n_transfers] first packed row of transfer k in class c, -1 if absent
  std::vector<int> tsT_slot;     // [8][n_transfers] index of transfer k among class c's transfers, -1 if absent
  std::vector<int> tsT_nblk;     // [8] blocks holding rank rows of class c
  DevBuf tsT_rowinfo;            // [8 * tsT_nb * 128] V-stack row -> (slot << 8 | a), -1: padding row
  OpStack tsT_v, tsT_u;          // 8 * tsT_nb blocks: V rows (128 x n), U columns (round8(n) x 128)
  CUtensorMap tsT_vmap, tsT_umap;
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
  // rows a host-buffer apply must move: sources [src_lo, src_hi), targets [tgt_lo, tgt_hi)
  int64_t src_lo = 0, src_hi = 0, tgt_lo = 0, tgt_hi = 0;
  uint64_t gen = 0;  // unique per built plan (merged plans remember what they were built from)
  // two-stage low-rank plans (Group::has_ts): stage 1 over source tiles, stage 2 over target tiles
  int ts = 0;  // 0: none, 1: source-major Y + rank-segment stage 2, 2: target-major Y + dense stage 2
  HostPlan ts1, ts2;
  DevBuf ts1_col, ts1_off, ts1_code, ts1_src, ts2_col, ts2_off, ts2_code, ts2_src;
  std::vector<int64_t> ts_tile_tmin;  // per stage-2 tile: smallest target row (tiles are in row order)
  // target-major plans, host-buffer pipeline: rows that must be resident before a tile runs --
  // per stage-1 tile the largest source row of tiles 0..t, per stage-2 tile the largest target row of tiles 0..t
  std::vector<int64_t> ts1_need, ts2_need;
  DevBuf ts_y;          // stage-1 output Y[source row][class-stack row] (n_rows x ts_ldy)
  DevBuf tsT_nbr;       // target-major mode (ts == 2): [n_rows][tsT_nslots] element offset into Y_T of the
                        // (source, class slot)'s rank run, -1 where the source has no such pair
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
  DevBuf fbuf, xpad, ybuf, wt, z, fzbuf;
  std::vector<int64_t> xpad_sig;
  long long wt_ld_zeroed = -1;
};

namespace cfm { struct PinnedStager; }

struct cfm_handler {
  std::unique_ptr<cfm::PinnedStager> stager;  // pageable host buffers (host_stage.hpp)
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
  // host-buffer low-rank pipeline (apply.cu): while set, a two-stage level waits
  // `ts_before_stage2` before stage 2 and runs stage 2 in `ts_chunks` tile
  // chunks, calling ts_after_chunk(rows below this are final) after each
  // ... and a large target-major level streams its rows: stage-1 chunk c starts when
  // multipole rows < x_rows[c + 1] are resident (x_ready[c]; padded chunk by chunk),
  // stage-2 chunk c when the locals of its targets are (y_ready[c])
  struct TsPipe {
    std::vector<int64_t> cut1, cut2;  // tile boundaries of the stage-1 / stage-2 chunks
    std::vector<int64_t> x_rows;      // cut1.size() row boundaries
    std::vector<cudaEvent_t> x_ready, y_ready;
  };
  const TsPipe* ts_pipe = nullptr;
  cudaEvent_t ts_before_stage2 = nullptr;
  int ts_chunks = 1;
  std::function<void(int64_t)> ts_after_chunk;
  std::vector<cudaEvent_t> ev_pool;  // events of the host-buffer low-rank pipeline
  std::vector<cudaEvent_t> ev_late_x;  // per late level: its multipoles are resident (dense host-buffer pipeline)
  bool last_csr_hit = false;  // the last cfm_apply_level_csr reused a cached plan
  int last_csr_mode = -1, last_csr_two_stage = 0;  // and that plan's mode / two-stage flag
  uint64_t last_csr_gen = 0;                        // and its id (unique per built plan)
};


namespace cfm {

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
extern PFN_writeValue32 p_writeValue32;
extern PFN_waitValue32 p_waitValue32;

struct DeviceLists {
  DevBuf off, src, code;
  int64_t total = 0;
  std::vector<int64_t> h_off;
};

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

// Reusable classifier scratch of the device-output entry points, per calling
// thread AND per device (a buffer allocated on one device is never handed to
// a kernel running on another).
struct ClassifyScratch {
  DevBuf grid, counts;
};

// CFM_TRACE=1: host-side stage timings of plans and applies on stderr
inline bool trace_on() {
  static const bool on = getenv("CFM_TRACE") && atoi(getenv("CFM_TRACE"));
  return on;
}
inline double wall_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

uint64_t next_plan_gen();
void set_slab_plan(cfm_handler* h, int level, LevelPlan& lp,
                   const std::function<void(int64_t, int64_t&, int64_t&, int64_t&)>& tile_rows);
bool use_device_plan();
bool device_plan_dense(cfm_handler* h, int level, const Group& g, int64_t n, const int64_t* d_off,
                       const std::vector<int64_t>& h_off, const int32_t* d_src, const int16_t* d_code,
                       int64_t n_rows, cudaStream_t s, LevelPlan& lp);

// ---- functions defined in launch.cu / operators.cu / plan.cu / apply.cu / classify.cu
int tile_kernel_kind(int nk = 0);
bool use_bulk_a(int kc);
void encode_source_map(TileParams& q, int kc);
bool ft_pipe_enabled();
bool use_late_stream();
bool mid_group_enabled();
bool early_tgt_d2h();
bool ktail_enabled();
bool resolve_stream_mem_ops();
bool use_copy_pipeline();
bool use_concurrent_levels();
bool use_fused_lowrank();
bool use_full_ops(const cfm_handler* h);
bool launch_lowrank_fused(const LowRankParams& lp_, int rmax, int64_t first, int64_t count, cudaStream_t s,
                                 bool vb = false);
int64_t launch_multi(const std::vector<TileParams>& segs, const std::vector<int64_t>& counts, cudaStream_t s);
int64_t launch_range(const TileParams& p, int64_t first, int64_t count, cudaStream_t s);
int64_t launch_tiles(const TileParams& p, int64_t n_tiles, cudaStream_t s);
int64_t launch_seg_pair(TileParams q, int64_t n_tiles, cudaStream_t s, int64_t tile_base = 0);
bool use_ts_persistent();
std::vector<int64_t> ts_chunk_cuts(int64_t n_tiles, int chunks, int device);
int64_t launch_ts_gemm(int stage, TileParams q, int64_t n_tiles, int64_t tile_base, int device, cudaStream_t s);
void fill_ops(TileParams& p, const OpStack& s, const CodeMap& m);
void fill_plan(TileParams& p, const DevBuf& col, const DevBuf& toff, const DevBuf& code, const DevBuf& src,
                      int64_t n_tiles);
void push_plan(const HostPlan& hp, DevBuf& col, DevBuf& toff, DevBuf& code, DevBuf& src);
bool is_device_ptr(const void* ptr);
void build_tables(cfm_handler* h);
void map_transfers(cfm_handler* h, Group& g, int n_transfers, const int8_t* transfers, int n_ops,
                          const int8_t* op_t, bool rows_permuted, bool cols_permuted, CodeMap& m);
void build_full_ops(cfm_handler* h, Group& g, int n_transfers, const int8_t* transfers, const double* ops);
void make_stack(OpStack& s, int n_ops, int rows, int cols);
void put_stack(OpStack& s, int i, const std::vector<double>& hostblock);
void set_per_op(OpStack& s, const std::vector<int>& rows, const std::vector<int>& klen);
void build_lowrank_stacks(cfm_handler* h, OpStack& left, OpStack& right_h, int n_ops, const int* ranks,
                                 const double* L, const double* R, int rows_left, int rows_right);
void build_two_stage(cfm_handler* h, Group& g, int n_transfers, const int8_t* transfers,
                            const std::vector<int>& rk, const std::vector<double>& all_v,
                            const std::vector<double>& all_u);
void build_lowrank_full(cfm_handler* h, Group& g, int n_transfers, const int8_t* transfers, int n_ops,
                               const int* ranks, const double* L, const double* R);
std::vector<int16_t> codes_from_t(int64_t P, const int8_t* t);
Group& group_for_level(cfm_handler* h, int level);
void build_two_stage_plan(const Group& g, LevelPlan& lp);
inline bool full_mode(const Group& g, const LevelPlan& lp) { return g.kind == kDense && g.has_full && lp.dc == 1; }
bool use_hybrid();
bool use_two_stage();
bool use_lowrank_full(const cfm_handler* h);
int two_stage_mode();
PFN_encodeTiled resolve_encode_tiled();
void push_pair_plan(LevelPlan& lp);
void build_hybrid_plan(cfm_handler* h, LevelPlan& lp, int64_t n_targets, const int64_t* tgt,
                              const int64_t* off, const int64_t* src, const int16_t* codes,
                              const std::array<int, kNumCodes>& key);
LevelPlan build_level_plan(cfm_handler* h, int level, int64_t n_targets, const int64_t* tgt,
                                  const int64_t* off, const int64_t* src, const int16_t* codes, int data_complex,
                                  int64_t n_rows);
LevelPlan& make_plan(cfm_handler* h, int level, int64_t n_targets, const int64_t* tgt, const int64_t* off,
                            const int64_t* src, const int16_t* codes, int data_complex, int64_t n_rows);
LevelPlan& csr_plan(cfm_handler* h, int level, int64_t n_targets, const int64_t* tgt, const int64_t* off,
                           const int64_t* src, const int8_t* t, int data_complex, int64_t n_rows, bool* hit_out);
inline void ensure(DevBuf& b, size_t bytes) { b.alloc(std::max<size_t>(bytes, 16)); }
int64_t launch_reduce(const LevelPlan& lp, const double* F, long long f_ld, double* y, long long y_ld, int len,
                      double scale, cudaStream_t s);
std::vector<size_t> xpad_layout(cfm_handler* h, const std::vector<std::pair<int64_t, int>>& lay, cudaStream_t s);
int64_t launch_pads(const std::vector<PadJob>& in, cudaStream_t s, int threads = 256);
int64_t xpad_copy(cfm_handler* h, double* dst, int ld, const double* src, int64_t r0, int64_t r1, cudaStream_t s,
                      int threads = 256, std::vector<PadJob>* batch = nullptr);
void fill_full(TileParams& p, const cfm_handler* h, const Group& g, const double* xpad, int64_t x_rows);
int64_t run_plan(cfm_handler* h, int level, LevelPlan& lp, const double* d_x, double* d_y, cudaStream_t s);
void apply_with_buffers(cfm_handler* h, int level, LevelPlan& lp, const double* mpoles, double* locals,
                               cudaStream_t s);
bool use_merged_pairs();
MergedPairPlan& merged_pair_plan(cfm_handler* h, const Group& g, const std::vector<int>& levels,
                                        const std::vector<LevelPlan*>& plans, const std::vector<int64_t>& row_off);
void apply_levels_impl(cfm_handler* h, int n_levels, const int* levels, const double* const* mpoles,
                              const int64_t* n_rows, double* const* locals, cudaStream_t s);
void init_cone_table();
ClassifyScratch& classify_scratch(int device);
void classify_device(int level, int64_t n_cells, const int32_t* ijk, cudaStream_t s, DeviceLists& out,
                            bool want_codes, int32_t* h_src = nullptr, int8_t* h_t = nullptr, uint8_t* h_rep = nullptr,
                            uint8_t* h_perm = nullptr, const int64_t* given_off = nullptr,
                            const int64_t* target_rows = nullptr, int64_t n_targets = -1);

template <class F>
inline int guarded(F&& fn) {
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
inline cudaStream_t pick_stream(cfm_handler* h, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  if (h->have_last && h->last_stream != st) CUDA_CHECK(cudaStreamWaitEvent(st, h->ev_last, 0));
  return st;
}
inline void mark_stream(cfm_handler* h, cudaStream_t st) {
  if (!h->ev_last) CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_last, cudaEventDisableTiming));
  CUDA_CHECK(cudaEventRecord(h->ev_last, st));
  h->last_stream = st;
  h->have_last = true;
}

}  // namespace cfm

#include "host_stage.hpp"
