// Kernel selection and launch helpers of the tile kernels (tile_gemm_ws, seg_pair_gemm, lowrank_ws).
#include "internal.hpp"
#include "seg_gemm.cuh"
#include "ts_gemm.cuh"
#include "step_gemm.cuh"

namespace cfm {


// ------------------------------------------------------------------ launching
// Kernel selection (CFM_TILE_KERNEL): "ws32" warp-specialized KC=32 x 3 stages
// with TMA bulk copies of the operator rows (default, CFM_BULK_A=1), "ws16"
// KC=16 x 5 stages, "sync" the lockstep kernel, "ws16w"
// like ws16 with 16 consumer warps (32x16 warp tiles) on 128-row blocks.
// Default by inner length (measured, profiles/r01_summary.md): KC=32 with bulk
// operator rows up to nk = 512 (l <= 7), KC=16 with cp.async rows above (l = 9).
int tile_kernel_kind(int nk) {
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

bool use_bulk_a(int kc) {
  static int v = [] {
    const char* e = getenv("CFM_BULK_A");
    return e ? atoi(e) : -1;
  }();
  if (v >= 0) return v != 0;
  return kc >= 32;  // 256-B row chunks: bulk copies win; 128-B: cp.async wins
}

// cuTensorMapEncodeTiled, resolved at run time like the stream memory ops.
PFN_encodeTiled resolve_encode_tiled() {
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
void encode_source_map(TileParams& q, int kc) {
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

bool ft_pipe_enabled() {
  static const int v = [] {
    const char* e = getenv("CFM_FT_PIPE");
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}

// CFM_LATE_STREAM=0: later launch groups on the caller's stream, after the first
bool use_late_stream() {
  static const bool v = [] {
    const char* e = getenv("CFM_LATE_STREAM");
    return !e || atoi(e) != 0;
  }();
  return v;
}

// CFM_MID_GROUP=0: with host buffers next to a pipelined level, the largest
// other target-tile level stays in the first launch (its upload then delays
// the first launch; with the middle group it crosses PCIe during that launch)
bool mid_group_enabled() {
  static const bool v = [] {
    const char* e = getenv("CFM_MID_GROUP");
    return !e || atoi(e) != 0;
  }();
  return v;
}

// CFM_EARLY_TGT_D2H=0: first-group target-tile levels download after the whole call
bool early_tgt_d2h() {
  static const bool v = [] {
    const char* e = getenv("CFM_EARLY_TGT_D2H");
    return !e || atoi(e) != 0;
  }();
  return v;
}

// CFM_KTAIL=0: the last k-step of l = 5 operators as a DMMA over zero padding (A/B)
// (read at every launch, so a test can compare both in one process)
bool ktail_enabled() {
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
        {
          // CFM_FT_SKEW=a,b: skew (chunks) of the stage-1 (FTM 3) and the other flat-loop launches
          const char* e = getenv("CFM_FT_SKEW");
          int s3 = 2, s1 = 0;
          if (e) sscanf(e, "%d,%d", &s3, &s1);
          mp.seg[i].ft_skew = q.y_rowblk ? s3 : s1;
        }
      }
      auto kf = q.y_rowblk ? tile_gemm_ws_kernel<BM, BN, WM, WN, KC, 4, SKIP, false, 3>
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
PFN_writeValue32 p_writeValue32 = nullptr;
PFN_waitValue32 p_waitValue32 = nullptr;
bool resolve_stream_mem_ops() {
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

bool use_copy_pipeline() {
  static int v = [] {
    const char* e = getenv("CFM_COPY_PIPELINE");
    return e ? atoi(e) : 1;
  }();
  return v != 0 && resolve_stream_mem_ops();
}

bool use_concurrent_levels() {
  static int v = [] {
    const char* e = getenv("CFM_CONCURRENT_LEVELS");
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}

bool use_fused_lowrank() {  // read per apply (tests switch it)
  const char* e = getenv("CFM_LOWRANK_FUSED");
  return !e || atoi(e) != 0;
}


// Full-operator TMA mode (CFM_FULL_OPS=0 disables): real dense groups with
// 64 < n <= 1024 (l = 5..10); always the 128-row KC=32 kernel.
bool use_full_ops(const cfm_handler* h) {
  static int v = [] {
    const char* e = getenv("CFM_FULL_OPS");
    return e ? atoi(e) : 1;
  }();
  const int nf = h->n * h->f;
  return v != 0 && !h->op_complex && nf > 64 && nf <= 1024 && resolve_encode_tiled() != nullptr;
}

// Per-transfer permuted low-rank factors (fused kernel with contiguous padded
// sources): also for complex operators (realified, CFM_LR_FULL_COMPLEX=0 disables).
bool use_lowrank_full(const cfm_handler* h) {
  if (!h->op_complex) return use_full_ops(h);
  static int v = [] {
    const char* e = getenv("CFM_LR_FULL_COMPLEX");
    return e ? atoi(e) : 1;
  }();
  const int nf = h->n * h->f;
  return v != 0 && nf > 64 && nf <= 1024;
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

bool launch_lowrank_fused(const LowRankParams& lp_, int rmax, int64_t first, int64_t count, cudaStream_t s,
                                 bool vb) {
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

// ---- persistent step kernel (step_gemm.cuh)
// CFM_STEP_PERSIST=0: one CTA per tile on tile_gemm_ws_kernel instead
bool use_step_persistent() {
  const char* e = getenv("CFM_STEP_PERSIST");
  return !e || atoi(e) != 0;
}

// A zeroed work counter for one launch: per device a small pool of counters,
// handed out round-robin and zeroed on the launch's stream right before it
// (256 launches would have to be in flight at once for two to share one).
static unsigned* step_queue_slot(cudaStream_t s) {
  constexpr int kSlots = 256;
  static std::mutex mu;
  static std::map<int, std::pair<unsigned*, int>> pools;
  int dev = 0;
  CUDA_CHECK(cudaGetDevice(&dev));
  unsigned* slot = nullptr;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto& pl = pools[dev];
    if (!pl.first) CUDA_CHECK(cudaMalloc(&pl.first, kSlots * sizeof(unsigned)));
    slot = pl.first + pl.second;
    pl.second = (pl.second + 1) % kSlots;
  }
  CUDA_CHECK(cudaMemsetAsync(slot, 0, sizeof(unsigned), s));
  return slot;
}

// Can these tile lists run on the persistent kernel?  Full-operator staging
// with KC = 32, whole operators (no per-operator row / inner counts), real
// data, every list target tiles, pair entries or a Y_T scatter; dense lists
// only when the last 128-row block wastes less than a warp's rows (l = 5: the
// row-skipping kernel serves l = 7, 9).
static bool step_persistent_ok(const std::vector<TileParams>& segs, const std::vector<int64_t>& counts) {
  if (!use_step_persistent() || segs.empty()) return false;
  int live = 0;
  int64_t tiles = 0;
  const int* code_op = nullptr;
  const TileParams& q0 = segs[0];
  for (size_t i = 0; i < segs.size(); ++i) {
    if (counts[i] == 0) continue;
    const TileParams& q = segs[i];
    ++live;
    tiles += counts[i];
    if (q.no_step || !q.ft || q.op_rows || q.op_klen || q.x_dc != 1 || q.y_dc != 1 || q.red_counter || q.b_block) return false;
    if (q.nk > 1024 || q.nr != q0.nr || q.nk != q0.nk || q.ft_rows != q0.ft_rows || q.ft_opshift) return false;
    if (!q.code_is_op) {
      if (code_op && code_op != q.code_op) return false;
      code_op = q.code_op;
    }
    if (q.pair_out && q.y_rowblk && !q.y_nbr) return false;  // round-1 two-stage layout
    // dead m-tiles in the last row block / empty k-steps in an entry's last chunk (l = 6, 7):
    // the row- and k-step-skipping kernel stays ahead there (measured on the config-2 tree:
    // l = 7 363.3 vs 367.5 ms, l = 6 147.2 vs 147.7 ms with skipping variants of this kernel;
    // its tiles are 2,000+ chunks long, so the per-CTA overhead this kernel removes is < 0.2%)
    // ... but short tiles win far more from losing the per-CTA cost than the empty k-steps cost them
    // (shared-basis cores, K = 203: 7-chunk entries, a dozen per tile)
    const long long chunks_per_tile = (q.n_entries / std::max(q.n_tiles, 1)) * ((q.nk + 31) / 32);
    if (!q.y_rowblk && q.nk % 32 != 0 && q.nk % 32 <= 24 && chunks_per_tile > 500) return false;
    // (dead m-tiles alone -- l = 9: 729 = 22 x 32 + 25 columns, 89-row last block -- run on the MPART variant)
    if (q.pair_out && (q.pipe_mp || q.pipe_loc || q.pipe_done)) return false;
    if (!q.pair_out && !q.accumulate) return false;
  }
  return live > 0 && live <= kStepMaxSegs && tiles * ((q0.nr + 127) / 128) < (int64_t(1) << 31);
}

static int64_t launch_step_persistent(const std::vector<TileParams>& segs, const std::vector<int64_t>& counts,
                                      cudaStream_t s) {
  static StepParams zero{};
  StepParams sp = zero;
  const TileParams* first = nullptr;
  int64_t work = 0;
  for (size_t i = 0; i < segs.size(); ++i) {
    if (counts[i] == 0) continue;
    TileParams q = segs[i];
    if (!first) first = &segs[i];
    encode_source_map(q, kStepKC);
    StepSeg& g = sp.seg[sp.n_seg++];
    const int nrb = (q.nr + 127) / 128;
    g.start = int(work);
    g.tile_base = q.tile_base;
    g.src_row0 = q.x_row0;
    g.mode = !q.pair_out ? 0 : (q.y_rowblk ? 2 : 1);
    g.tile_col = q.tile_col;
    g.tile_off = q.tile_off;
    g.entry_code = q.entry_code;
    g.entry_src = q.entry_src;
    g.y = q.y;
    g.y_ld = q.y_ld;
    g.scale = q.scale;
    g.rowinfo = q.y_colmap;
    g.nbr = q.y_nbr;
    g.nslots = q.y_nslots;
    g.code_is_op = q.code_is_op;
    g.pipe_mp = q.pipe_mp;
    g.pipe_loc = q.pipe_loc;
    g.pipe_done = q.pipe_done;
    g.pipe_need_mp = q.pipe_need_mp;
    g.pipe_need_loc = q.pipe_need_loc;
    g.pipe_lo = q.pipe_lo;
    g.pipe_hi = q.pipe_hi;
    g.tmap_a = q.tmap_a;
    g.tmap_b = q.tmap_b;
    if (!q.code_is_op) sp.code_op = q.code_op;
    work += counts[i] * nrb;
  }
  sp.n_work = int(work);
  sp.nrb = (first->nr + 127) / 128;
  sp.nk = first->nk;
  sp.nr = first->nr;
  sp.a_rows = first->ft_rows;
  const int nch = (sp.nk + kStepKC - 1) / kStepKC;
  {
    const char* e = getenv("CFM_TS_SKEW");
    sp.skew = std::min(e ? atoi(e) : 2, nch - 1);
  }
  sp.queue = step_queue_slot(s);
  int dev = 0, sms = 148;
  CUDA_CHECK(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = int(std::min<int64_t>(work, sms));
  const int smem = step_gemm_smem_bytes();
  bool scatter = false;
  for (int i = 0; i < sp.n_seg; ++i) scatter = scatter || sp.seg[i].mode == 2;
  // MPART: the last row block has dead m-tiles (l = 9: 89 of 128 rows), skipped per warp
  const bool mpart = !scatter && sp.nr % 128 != 0 && 128 - sp.nr % 128 >= 8;
  auto kern = scatter ? step_gemm_kernel<true, false> : mpart ? step_gemm_kernel<false, true> : step_gemm_kernel<false, false>;
  CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<grid, kStepThreads, smem, s>>>(sp);
  CUDA_CHECK(cudaGetLastError());
  return 1;
}

// One launch over several tile lists sharing operator shapes (all levels of a
// homogeneous dense group).  Segments are launched in the given order.
int64_t launch_multi(const std::vector<TileParams>& segs, const std::vector<int64_t>& counts, cudaStream_t s) {
  if (step_persistent_ok(segs, counts)) return launch_step_persistent(segs, counts, s);
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
int64_t launch_range(const TileParams& p, int64_t first, int64_t count, cudaStream_t s) {
  if (count > 0 && first + count < (int64_t(1) << 31)) {
    // single tile lists of per-level applies: the persistent kernel where it is eligible
    TileParams q = p;
    q.tile_base = int(first);
    if (step_persistent_ok({q}, {count})) return launch_step_persistent({q}, {count}, s);
  }
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

int64_t launch_tiles(const TileParams& p, int64_t n_tiles, cudaStream_t s) {
  return launch_range(p, 0, n_tiles, s);
}

// Two-stage low-rank stage 2 on seg_pair_gemm_kernel (two 16-wide rank
// segments per pipeline stage); CFM_SEG_PAIR=0 runs the KC = 16 full-operator
// kernel instead.
int64_t launch_seg_pair(TileParams q, int64_t n_tiles, cudaStream_t s, int64_t tile_base) {
  if (n_tiles <= 0) return 0;
  if (n_tiles + tile_base >= (int64_t(1) << 31)) throw Error(CFM_ERR_VALUE, "too many tiles for one launch");
  q.tile_base = int(tile_base);
  encode_source_map(q, 16);
  const int smem = seg_pair_smem_bytes();
  CUDA_CHECK(cudaFuncSetAttribute(seg_pair_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  seg_pair_gemm_kernel<<<unsigned(n_tiles), 12 * 32, smem, s>>>(q);
  CUDA_CHECK(cudaGetLastError());
  return 1;
}

// Target-major two-stage path: tiles [tile_base, tile_base + n_tiles) of a
// stage-1 (stage = 1) or stage-2 (stage = 2) plan on the persistent kernel
// (ts_gemm.cuh), one CTA per SM.  `q` is the stage's TileParams as the
// one-CTA-per-tile kernel takes it (CFM_TS_PERSIST=0 runs that one instead).
bool use_ts_persistent() {
  const char* e = getenv("CFM_TS_PERSIST");
  return !e || atoi(e) != 0;
}

// Tile boundaries of `chunks` launches over n_tiles uniform tiles, on whole waves
// (one CTA per SM: a chunk of 3.5 waves would run as long as one of 4).
std::vector<int64_t> ts_chunk_cuts(int64_t n_tiles, int chunks, int device) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  std::vector<int64_t> cut{0};
  for (int c = 1; c < chunks; ++c) {
    const int64_t t = std::min<int64_t>(n_tiles, (n_tiles * c / chunks + sms / 2) / sms * sms);
    if (t > cut.back() && t < n_tiles) cut.push_back(t);
  }
  cut.push_back(n_tiles);
  return cut;
}

int64_t launch_ts_gemm(int stage, TileParams q, int64_t n_tiles, int64_t tile_base, int device, cudaStream_t s) {
  if (n_tiles <= 0) return 0;
  {
    // CFM_TS_KERNEL=step: the dynamic-queue step kernel (step_gemm.cuh) instead of the
    // round-robin kernel of ts_gemm.cuh (measured 1.2% slower on these uniform tiles)
    const char* e = getenv("CFM_TS_KERNEL");
    if (e && !strcmp(e, "step")) {
      q.tile_base = int(tile_base);
      return launch_step_persistent({q}, {n_tiles}, s);
    }
  }
  encode_source_map(q, kTsKC);
  TsGemmParams t{};
  t.nrb = (q.nr + 127) / 128;
  if (n_tiles * t.nrb >= (int64_t(1) << 31)) throw Error(CFM_ERR_VALUE, "too many tiles for one launch");
  t.n_work = int(n_tiles * t.nrb);
  t.tile_base = int(tile_base);
  t.tile_col = q.tile_col;
  t.tile_off = q.tile_off;
  t.entry_code = q.entry_code;
  t.code_op = q.code_is_op ? nullptr : q.code_op;
  t.entry_src = q.entry_src;
  t.nk = q.nk;
  t.nr = q.nr;
  t.a_rows = q.ft_rows;
  const int nch = (q.nk + kTsKC - 1) / kTsKC;
  {
    const char* e = getenv("CFM_TS_SKEW");
    t.skew = std::min(e ? atoi(e) : 2, nch - 1);
  }
  t.y = q.y;
  t.rowinfo = q.y_colmap;
  t.nbr = q.y_nbr;
  t.nslots = q.y_nslots;
  t.loc = q.y;
  t.loc_ld = q.y_ld;
  t.scale = q.scale;
  t.tmap_a = q.tmap_a;
  t.tmap_b = q.tmap_b;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int grid = std::min(t.n_work, sms);
  const int smem = ts_gemm_smem_bytes();
  auto kern = stage == 1 ? ts_gemm_kernel<1> : ts_gemm_kernel<2>;
  CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<grid, kTsThreads, smem, s>>>(t);
  CUDA_CHECK(cudaGetLastError());
  return 1;
}

void fill_ops(TileParams& p, const OpStack& s, const CodeMap& m) {
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

void fill_plan(TileParams& p, const DevBuf& col, const DevBuf& toff, const DevBuf& code, const DevBuf& src,
                      int64_t n_tiles) {
  p.n_tiles = int(n_tiles);
  p.tile_col = col.as<int>();
  p.tile_off = toff.as<int>();
  p.entry_code = code.as<int>();
  p.entry_src = src.as<int>();
}

void push_plan(const HostPlan& hp, DevBuf& col, DevBuf& toff, DevBuf& code, DevBuf& src) {
  upload(col, hp.tile_col);
  upload(toff, hp.tile_off);
  upload(code, hp.entry_code);
  upload(src, hp.entry_src);
}

bool is_device_ptr(const void* ptr) {
  if (!ptr) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace cfm
