// Apply: source padding, per-level launch sequences, host-buffer pipelines, multi-level launches.
#include "internal.hpp"
#include "pair_reduce.cuh"

namespace cfm {

// ------------------------------------------------------------------ apply

int64_t launch_reduce(const LevelPlan& lp, const double* F, long long f_ld, double* y, long long y_ld, int len,
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
std::vector<size_t> xpad_layout(cfm_handler* h, const std::vector<std::pair<int64_t, int>>& lay, cudaStream_t s) {
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

int64_t launch_pads(const std::vector<PadJob>& in, cudaStream_t s, int threads) {
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
int64_t xpad_copy(cfm_handler* h, double* dst, int ld, const double* src, int64_t r0, int64_t r1, cudaStream_t s,
                      int threads, std::vector<PadJob>* batch) {
  if (r1 <= r0) return 0;
  const int nsrc = h->n * h->f;  // doubles per source row (complex operators: interleaved re / im)
  if (is_device_ptr(src)) {
    const PadJob J{dst + size_t(r0) * ld, src + size_t(r0) * nsrc, (long long)(r1 - r0), 0, ld, nsrc};
    if (batch) {
      batch->push_back(J);
      return 0;
    }
    return launch_pads({J}, s, threads);
  }
  CUDA_CHECK(cudaMemcpy2DAsync(dst + size_t(r0) * ld, size_t(ld) * sizeof(double), src + size_t(r0) * nsrc,
                               size_t(nsrc) * sizeof(double), size_t(nsrc) * sizeof(double), size_t(r1 - r0),
                               cudaMemcpyDefault, s));
  return 0;
}

void fill_full(TileParams& p, const cfm_handler* h, const Group& g, const double* xpad, int64_t x_rows) {
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

int64_t run_plan(cfm_handler* h, int level, LevelPlan& lp, const double* d_x, double* d_y, cudaStream_t s) {
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

  if (g.kind == kLowRank && lp.ts == 2) {
    // target-major two-stage low rank: stage 1 Y_T[target][rho_T + a] = (V_k^H x_source)[a]
    // (class V stacks on the full-operator kernel, scattered by the pair table),
    // stage 2 locals[targets] += scale * U_c Y_T[targets]^T, a dense GEMM per
    // target class on the step kernel
    const int ldx = g.tsT_v.ld;
    const int nb = g.tsT_nb;
    const auto xo = xpad_layout(h, {{lp.n_rows, ldx}}, s);
    double* xp = h->xpad.as<double>() + xo[0];
    const cfm_handler::TsPipe* pipe = h->ts_pipe;
    if (!pipe) launches += xpad_copy(h, xp, ldx, d_x, 0, lp.n_rows, s);
    if (!lp.ts_y.p) {
      // columns of pairs a target does not have are never written by stage 1;
      // zeroed once, they contribute exact zeros to stage 2 in every step
      lp.ts_y.alloc(size_t(lp.n_rows) * nb * 128 * sizeof(double));
      CUDA_CHECK(cudaMemsetAsync(lp.ts_y.p, 0, lp.ts_y.bytes, s));
    }
    TileParams a{};
    fill_ops(a, g.tsT_v, g.main);
    fill_plan(a, lp.ts1_col, lp.ts1_off, lp.ts1_code, lp.ts1_src, lp.ts1.n_tiles);
    a.op_rows = nullptr;
    a.op_klen = nullptr;
    a.nr = 128;
    a.nk = h->n;
    a.code_is_op = 1;
    a.ft = 1;
    a.ft_rows = 128;
    a.tmap_a = g.tsT_vmap;
    a.x = xp; a.x_ld = ldx; a.x_dc = 1; a.x_rows = lp.n_rows;
    a.y = lp.ts_y.as<double>(); a.y_ld = (long long)nb * 128; a.y_dc = 1; a.y_rowblk = nb;
    a.y_colmap = g.tsT_rowinfo.as<int>();
    a.y_nbr = lp.tsT_nbr.as<int>();
    a.y_nslots = g.tsT_nslots;
    a.scale = 1.0; a.accumulate = 0; a.pair_out = 1;
    a.zero_row = h->zeros.as<double>();
    a.n_entries = lp.ts1.n_entries();
    const bool persist = use_ts_persistent();
    if (pipe) {
      // host-buffer pipeline: stage 1 in chunks of row-ordered tiles, each padded and
      // launched as soon as its multipole rows are resident
      for (size_t c = 0; c + 1 < pipe->cut1.size(); ++c) {
        CUDA_CHECK(cudaStreamWaitEvent(s, pipe->x_ready[c], 0));
        launches += xpad_copy(h, xp, ldx, d_x, pipe->x_rows[c], pipe->x_rows[c + 1], s);
        const int64_t t0 = pipe->cut1[c], t1 = pipe->cut1[c + 1];
        launches += persist ? launch_ts_gemm(1, a, t1 - t0, t0, h->device, s) : launch_range(a, t0, t1 - t0, s);
      }
    } else {
      launches += persist ? launch_ts_gemm(1, a, lp.ts1.n_tiles, 0, h->device, s) : launch_tiles(a, lp.ts1.n_tiles, s);
    }
    TileParams b{};
    fill_ops(b, g.tsT_u, g.main);
    fill_plan(b, lp.ts2_col, lp.ts2_off, lp.ts2_code, lp.ts2_src, lp.ts2.n_tiles);
    b.op_rows = nullptr;
    b.op_klen = nullptr;
    b.nr = h->n;
    b.nk = 128;
    b.code_is_op = 1;
    b.ft = 1;
    b.ft_rows = g.tsT_u.rows;
    b.tmap_a = g.tsT_umap;
    b.x = lp.ts_y.as<double>(); b.x_ld = 128; b.x_dc = 1; b.x_rows = lp.n_rows * nb;
    b.y = d_y; b.y_ld = row_ld; b.y_dc = 1;
    b.scale = scale; b.accumulate = 1; b.pair_out = 0;
    b.zero_row = h->zeros.as<double>();
    b.n_entries = lp.ts2.n_entries();
    const int64_t nt2 = lp.ts2.n_tiles;
    auto run2 = [&](int64_t t0, int64_t t1) {
      launches += persist ? launch_ts_gemm(2, b, t1 - t0, t0, h->device, s) : launch_range(b, t0, t1 - t0, s);
    };
    if (pipe) {
      // stage 2 in chunks of row-ordered tiles: chunk c starts when its targets'
      // locals are resident; after it, every row below the next chunk's smallest
      // target row is final and goes back
      for (size_t c = 0; c + 1 < pipe->cut2.size(); ++c) {
        CUDA_CHECK(cudaStreamWaitEvent(s, pipe->y_ready[c], 0));
        const int64_t t1 = pipe->cut2[c + 1];
        run2(pipe->cut2[c], t1);
        if (h->ts_after_chunk) h->ts_after_chunk(t1 < nt2 ? lp.ts_tile_tmin[t1] : lp.n_rows);
      }
      return launches;
    }
    if (h->ts_before_stage2) CUDA_CHECK(cudaStreamWaitEvent(s, h->ts_before_stage2, 0));
    if (h->ts_chunks > 1 && h->ts_after_chunk && int64_t(lp.ts_tile_tmin.size()) == nt2 && nt2 >= 2 * h->ts_chunks) {
      const std::vector<int64_t> cut = ts_chunk_cuts(nt2, h->ts_chunks, h->device);
      for (size_t c = 0; c + 1 < cut.size(); ++c) {
        run2(cut[c], cut[c + 1]);
        h->ts_after_chunk(cut[c + 1] < nt2 ? lp.ts_tile_tmin[cut[c + 1]] : lp.n_rows);
      }
    } else {
      run2(0, nt2);
    }
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
      // rows of sources no pair reads are never written by stage 1 nor read by
      // stage 2; zeroed once so every Y value a gather can touch is finite
      lp.ts_y.alloc(size_t(lp.n_rows) * g.ts_ldy * sizeof(double));
      CUDA_CHECK(cudaMemsetAsync(lp.ts_y.p, 0, lp.ts_y.bytes, s));
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
    a.y = lp.ts_y.as<double>(); a.y_ld = g.ts_ldy; a.y_dc = 1; a.y_rowblk = g.ts_nb;
    a.y_colmap = g.ts_colmap.as<int>();
#ifdef CFM_EXPERIMENTS
    if (getenv("CFM_EXP") && !strcmp(getenv("CFM_EXP"), "nostore1")) a.debug = 128;  // timing only: no Y stores
#endif
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
    b.x = lp.ts_y.as<double>(); b.x_ld = g.ts_ldy; b.x_dc = 1; b.x_rows = lp.n_rows; b.b_block = 0;
    b.op_col = g.ts_opcol.as<int>();
    b.y = d_y; b.y_ld = row_ld; b.y_dc = 1;
    b.scale = scale; b.accumulate = 1; b.pair_out = 0;
    b.zero_row = h->zeros.as<double>();
    b.n_entries = lp.ts2.n_entries();
    {
      const char* e = getenv("CFM_SEG_KSKIP");  // 0: run all 4 k-steps of every segment (A/B)
      b.seg_ksteps = (!e || atoi(e) != 0) ? g.ts_ksteps.as<int>() : nullptr;
    }
    if (h->ts_before_stage2) CUDA_CHECK(cudaStreamWaitEvent(s, h->ts_before_stage2, 0));
    const int64_t nt2 = lp.ts2.n_tiles;
    if (h->ts_chunks > 1 && h->ts_after_chunk && int64_t(lp.ts_tile_tmin.size()) == nt2 && nt2 >= 2 * h->ts_chunks) {
      // stage 2 in tile chunks (row-ordered tiles): after a chunk, every row
      // below the next chunk's smallest target row is final
      for (int c = 0; c < h->ts_chunks; ++c) {
        const int64_t t0 = nt2 * c / h->ts_chunks, t1 = nt2 * (c + 1) / h->ts_chunks;
        launches += launch_seg_pair(b, t1 - t0, s, t0);
        h->ts_after_chunk(t1 < nt2 ? lp.ts_tile_tmin[t1] : lp.n_rows);
      }
    } else {
      launches += launch_seg_pair(b, nt2, s);
    }
    return launches;
  }

  if (g.kind == kLowRank) {
    // Two passes on the full-operator kernels (CFM_LR_TWOPASS=0: the fused kernel): pass 1 Y[slot] = V_t^H x_src and pass 2 acc += U_t Y[slot] are short-tile
    // GEMMs against the per-transfer permuted factors, which the persistent step kernel
    // runs without per-CTA cost; the fused kernel (both phases in one CTA, Y in shared
    // memory) pays about one shared-memory load per DMMA in its skinny phase 1.
    const char* twopass_e = getenv("CFM_LR_TWOPASS");  // read per apply (tests switch it)
    const int twopass_env = twopass_e ? atoi(twopass_e) : -1;
    const bool ft2 = g.has_lrfull && g.has_lrmaps && dc == 1 && (twopass_env < 0 || twopass_env != 0);
    if (!ft2) {
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
    const int ldy = ft2 ? round_up(g.lrf_right_h.rows, 2) : g.right_h.rows;  // rmax * f (16-B row pitch for TMA)
    double* xp2 = nullptr;
    int ldx2 = 0;
    if (ft2) {
      ldx2 = g.lrf_right_h.ld;
      const auto xo = xpad_layout(h, {{lp.n_rows, ldx2}}, s);
      xp2 = h->xpad.as<double>() + xo[0];
      launches += xpad_copy(h, xp2, ldx2, d_x, 0, lp.n_rows, s);
    }
    const char* ychunk_e = getenv("CFM_Y_CHUNK_MB");  // per-pair intermediate per chunk (default 1024 MB)
    const size_t ychunk = (ychunk_e ? size_t(atoll(ychunk_e)) : size_t(1024)) << 20;
    const size_t max_slots = std::max<size_t>(kBN, ychunk / (sizeof(double) * std::max(ldy, 1)));
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
        if (ft2) {
          fill_ops(p1, g.lrf_right_h, g.fullmap);
          p1.op_rows = nullptr; p1.op_klen = nullptr;  // rows / columns past a rank are exact zeros
          p1.rowtab = nullptr; p1.invtab = nullptr;
          p1.ft = 1; p1.ft_rows = g.lrf_right_h.rows; p1.tmap_a = g.lrf_vmap;
          p1.x = xp2; p1.x_ld = ldx2; p1.x_dc = 1; p1.x_rows = lp.n_rows;
          p1.n_entries = E;
        }
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
        if (ft2) {
          fill_ops(p2, g.lrf_left, g.fullmap);
          p2.op_rows = nullptr; p2.op_klen = nullptr;
          p2.rowtab = nullptr; p2.invtab = nullptr;
          p2.ft = 1; p2.ft_rows = g.lrf_left.rows; p2.tmap_a = g.lrf_umap;
          // the Y map starts at the chunk's first slot (a TMA base below the
          // allocation faults even when every touched row lies inside it)
          p2.x = h->ybuf.as<double>();
          p2.x_row0 = int(e0 * kBN);
          p2.x_rows = (e1 - e0) * kBN;
          p2.n_entries = E;
          if (lp.mode == 1) p2.entry_ncols = lp.entry_ncols.as<unsigned char>();
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
    // (no zeroing: every live pair row is stored once, by the dense-core or the
    // factored-core launch of its entry, and the reduction reads live rows only;
    // at config 3's level 5 the memset was 408 MB per step)
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
    q.no_step = g.any_fac_core ? 1 : 0;  // factored cores' entries carry no operator here: skipped per entry
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

void apply_with_buffers(cfm_handler* h, int level, LevelPlan& lp, const double* mpoles, double* locals,
                        cudaStream_t s) {
  const int dc = lp.dc;
  const size_t row_b = size_t(h->n) * (dc == 2 || h->op_complex ? 2 : 1) * sizeof(double);
  const size_t bytes = size_t(lp.n_rows) * row_b;
  const bool dev_x = is_device_ptr(mpoles), dev_y = is_device_ptr(locals);
  const double* d_x = mpoles;
  double* d_y = locals;
  // host buffers: only the rows the plan reads (sources) and writes (targets)
  // cross PCIe; pageable memory goes through the multi-threaded pinned stager
  auto h2d = [&](void* dst, const void* src, size_t len) {
    if (!len) return;
    if (is_pinned_host(src)) {
      CUDA_CHECK(cudaMemcpyAsync(dst, src, len, cudaMemcpyHostToDevice, s));
    } else {
      if (!h->stager) h->stager = std::make_unique<PinnedStager>();
      h->stager->h2d(dst, src, len, s, h->device);
    }
  };
  if (!dev_x) {
    ensure(h->x_stage, bytes);
    h2d(h->x_stage.as<char>() + lp.src_lo * row_b, reinterpret_cast<const char*>(mpoles) + lp.src_lo * row_b,
        size_t(lp.src_hi - lp.src_lo) * row_b);
    d_x = h->x_stage.as<double>();
  }
  if (!dev_y) {
    ensure(h->y_stage, bytes);
    h2d(h->y_stage.as<char>() + lp.tgt_lo * row_b, reinterpret_cast<const char*>(locals) + lp.tgt_lo * row_b,
        size_t(lp.tgt_hi - lp.tgt_lo) * row_b);
    d_y = h->y_stage.as<double>();
  }
  CUDA_CHECK(cudaEventRecord(h->ev0, s));
  h->last_launches = run_plan(h, level, lp, d_x, d_y, s);
  CUDA_CHECK(cudaEventRecord(h->ev1, s));
  if (!dev_y && lp.tgt_hi > lp.tgt_lo) {
    char* dst = reinterpret_cast<char*>(locals) + lp.tgt_lo * row_b;
    const char* src = reinterpret_cast<const char*>(d_y) + lp.tgt_lo * row_b;
    const size_t len = size_t(lp.tgt_hi - lp.tgt_lo) * row_b;
    if (is_pinned_host(locals)) {
      CUDA_CHECK(cudaMemcpyAsync(dst, src, len, cudaMemcpyDeviceToHost, s));
    } else {
      if (!h->stager) h->stager = std::make_unique<PinnedStager>();
      h->stager->d2h(dst, src, len, s, h->device);
    }
  }
  CUDA_CHECK(cudaStreamSynchronize(s));
  float ms = 0.f;
  CUDA_CHECK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  h->last_ms = ms;
}

static bool use_lr_pipeline() {
  const char* e = getenv("CFM_LR_PIPELINE");
  return !e || atoi(e) != 0;
}

bool use_merged_pairs() {
  static int v = [] {
    const char* e = getenv("CFM_MERGE_PAIRS");
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}

// Build (or reuse) the merged pair plan of the given pair-mode levels.
MergedPairPlan& merged_pair_plan(cfm_handler* h, const Group& g, const std::vector<int>& levels,
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
void apply_levels_impl(cfm_handler* h, int n_levels, const int* levels, const double* const* mpoles,
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
  // ---- low-rank levels from host buffers: multipoles of every level go H2D
  // first, then the locals, on a copy stream; the compute stream starts a
  // level as soon as its multipoles are in, waits for its locals only before
  // the accumulating stage (stage 2 of the two-stage path), and finished rows
  // go back on a second copy stream -- for two-stage levels chunk by chunk of
  // row-ordered stage-2 tiles -- while later work runs (CFM_LR_PIPELINE=0: off)
  bool lr_host = !lv.empty() && use_copy_pipeline() && use_lr_pipeline();
  for (auto& L : lv)
    lr_host = lr_host && group_for_level(h, L.level).kind == kLowRank && !is_device_ptr(L.x) && !is_device_ptr(L.y);
  if (lr_host) {
    if (!h->s_h2d) CUDA_CHECK(cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking));
    if (!h->s_d2h) CUDA_CHECK(cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking));
    if (!h->ev_prev) CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_prev, cudaEventDisableTiming));
    size_t evi = 0;
    auto next_ev = [&]() {
      if (evi == h->ev_pool.size()) {
        cudaEvent_t e;
        CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        h->ev_pool.push_back(e);
      }
      return h->ev_pool[evi++];
    };
    auto fence = [&](cudaStream_t from, cudaStream_t to) {  // `to` waits for the work queued on `from`
      cudaEvent_t e = next_ev();
      CUDA_CHECK(cudaEventRecord(e, from));
      CUDA_CHECK(cudaStreamWaitEvent(to, e, 0));
    };
    const size_t n = lv.size();
    size_t tot = 0;
    for (auto& L : lv) tot += 2 * L.bytes;
    ensure(h->x_stage, tot);
    // the copy streams reuse the staging that earlier work on s may still read
    CUDA_CHECK(cudaEventRecord(h->ev_prev, s));
    CUDA_CHECK(cudaStreamWaitEvent(h->s_h2d, h->ev_prev, 0));
    CUDA_CHECK(cudaStreamWaitEvent(h->s_d2h, h->ev_prev, 0));
    std::vector<char*> dx(n), dy(n);
    std::vector<cudaEvent_t> ex(n), ey(n);
    size_t o = 0;
    for (size_t i = 0; i < n; ++i) {
      dx[i] = static_cast<char*>(h->x_stage.p) + o;
      dy[i] = dx[i] + lv[i].bytes;
      o += 2 * lv[i].bytes;
    }
    // large target-major two-stage levels stream their rows (CFM_TS_SLABS=0: whole arrays):
    // multipoles in the row slabs the stage-1 chunks need, locals in the slabs of the
    // stage-2 chunks, one event per slab
    static const bool ts_slabs = [] {
      const char* e = getenv("CFM_TS_SLABS");
      return !e || atoi(e) != 0;
    }();
    std::vector<cfm_handler::TsPipe> pipes(n);
    std::vector<char> has_pipe(n, 0);
    std::vector<std::vector<int64_t>> y_rows(n);
    for (size_t i = 0; i < n; ++i) {
      const LevelPlan& P = *lv[i].lp;
      if (!ts_slabs || P.ts != 2 || P.n_rows < 65536 || P.ts1_need.empty() || P.ts2_need.empty()) continue;
      cfm_handler::TsPipe& tp = pipes[i];
      tp.cut1 = ts_chunk_cuts(int64_t(P.ts1_need.size()), 8, h->device);
      tp.cut2 = ts_chunk_cuts(int64_t(P.ts2_need.size()), 8, h->device);
      tp.x_rows.assign(1, 0);
      for (size_t c = 1; c < tp.cut1.size(); ++c)
        tp.x_rows.push_back(c + 1 == tp.cut1.size() ? P.n_rows : std::min(P.n_rows, P.ts1_need[tp.cut1[c] - 1] + 1));
      y_rows[i].assign(1, 0);
      for (size_t c = 1; c < tp.cut2.size(); ++c)
        y_rows[i].push_back(c + 1 == tp.cut2.size() ? P.n_rows : std::min(P.n_rows, P.ts2_need[tp.cut2[c] - 1] + 1));
      has_pipe[i] = 1;
    }
    auto upload = [&](size_t i, bool locals) {
      const LevelPlan& P = *lv[i].lp;
      const size_t row_b = lv[i].bytes / size_t(std::max<int64_t>(P.n_rows, 1));
      char* dst = locals ? dy[i] : dx[i];
      const char* src = reinterpret_cast<const char*>(locals ? lv[i].y : lv[i].x);
      if (!has_pipe[i]) {
        CUDA_CHECK(cudaMemcpyAsync(dst, src, lv[i].bytes, cudaMemcpyHostToDevice, h->s_h2d));
        (locals ? ey[i] : ex[i]) = next_ev();
        CUDA_CHECK(cudaEventRecord(locals ? ey[i] : ex[i], h->s_h2d));
        return;
      }
      const std::vector<int64_t>& rows = locals ? y_rows[i] : pipes[i].x_rows;
      std::vector<cudaEvent_t>& evs = locals ? pipes[i].y_ready : pipes[i].x_ready;
      for (size_t c = 0; c + 1 < rows.size(); ++c) {
        if (rows[c + 1] > rows[c])
          CUDA_CHECK(cudaMemcpyAsync(dst + size_t(rows[c]) * row_b, src + size_t(rows[c]) * row_b,
                                     size_t(rows[c + 1] - rows[c]) * row_b, cudaMemcpyHostToDevice, h->s_h2d));
        evs.push_back(next_ev());
        CUDA_CHECK(cudaEventRecord(evs.back(), h->s_h2d));
      }
      (locals ? ey[i] : ex[i]) = evs.back();
    };
    // small levels first (multipoles, then locals): they compute while the streamed
    // levels' multipole slabs cross PCIe; then those slabs, then their locals slabs
    for (int locals = 0; locals < 2; ++locals)
      for (size_t i = 0; i < n; ++i)
        if (!has_pipe[i]) upload(i, locals != 0);
    for (int locals = 0; locals < 2; ++locals)
      for (size_t i = 0; i < n; ++i)
        if (has_pipe[i]) upload(i, locals != 0);
    CUDA_CHECK(cudaEventRecord(h->ev0, s));
    int64_t launches = 0;
    auto reset_hooks = [&] {
      h->ts_pipe = nullptr;
      h->ts_before_stage2 = nullptr;
      h->ts_chunks = 1;
      h->ts_after_chunk = nullptr;
    };
    for (size_t i = 0; i < n; ++i) {
      LevelPlan& P = *lv[i].lp;
      const size_t row_b = lv[i].bytes / size_t(std::max<int64_t>(P.n_rows, 1));
      if (!has_pipe[i]) CUDA_CHECK(cudaStreamWaitEvent(s, ex[i], 0));
      int64_t done = 0;
      auto download = [&](int64_t upto) {  // rows [done, upto) of level i are final
        if (upto <= done) return;
        fence(s, h->s_d2h);
        CUDA_CHECK(cudaMemcpyAsync(reinterpret_cast<char*>(lv[i].y) + done * row_b, dy[i] + done * row_b,
                                   size_t(upto - done) * row_b, cudaMemcpyDeviceToHost, h->s_d2h));
        done = upto;
      };
      if (has_pipe[i]) {
        h->ts_pipe = &pipes[i];
        h->ts_after_chunk = download;
      } else if (P.ts) {
        h->ts_before_stage2 = ey[i];
        h->ts_chunks = P.n_rows >= 65536 ? 8 : 1;
        h->ts_after_chunk = download;
      } else {
        CUDA_CHECK(cudaStreamWaitEvent(s, ey[i], 0));
      }
      try {
        launches += run_plan(h, lv[i].level, P, reinterpret_cast<const double*>(dx[i]),
                             reinterpret_cast<double*>(dy[i]), s);
      } catch (...) {
        reset_hooks();
        throw;
      }
      reset_hooks();
      download(P.n_rows);
    }
    CUDA_CHECK(cudaEventRecord(h->ev1, s));
    fence(h->s_d2h, s);  // the caller's stream joins the downloads
    CUDA_CHECK(cudaStreamSynchronize(s));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    h->last_ms = ms;
    h->last_launches = launches;
    return;
  }
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
  std::vector<size_t> late_order;  // late (ftl 2) levels in upload / launch order
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
    unsigned* flags = h->pipe_flags.as<unsigned>();
    auto upload_slabs = [&](size_t i) {  // the row slabs of pipelined level i (locals; multipoles unless resident)
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
    };
    // late levels, smallest first, each with its own "multipoles resident" event: a smaller
    // late level is launched (and keeps the GPU busy) while a larger one still crosses PCIe
    // (config 4: level 6's 0.7 GB arrive 105 ms before level 7's 5.75 GB)
    late_order.clear();
    for (size_t i = 0; i < lv.size(); ++i)
      if (ftl[i] == 2) late_order.push_back(i);
    std::stable_sort(late_order.begin(), late_order.end(), [&](size_t a, size_t b) { return lv[a].bytes < lv[b].bytes; });
    while (h->ev_late_x.size() < late_order.size()) {
      cudaEvent_t e;
      CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      h->ev_late_x.push_back(e);
    }
    for (size_t j = 0; j < late_order.size(); ++j) {
      const size_t i = late_order[j];
      CUDA_CHECK(cudaMemcpyAsync(const_cast<double*>(staged_x[i]), host_x[i], lv[i].bytes, cudaMemcpyHostToDevice, s_in));
      CUDA_CHECK(cudaEventRecord(h->ev_late_x[j], s_in));
      // ... and its locals slabs right behind, before the next late level's multipoles: its
      // epilogues would otherwise hold the SMs until that (much longer) upload is over
      if (piped[i]) upload_slabs(i);
    }
    for (size_t i = 0; i < lv.size(); ++i)
      if (piped[i] && ftl[i] != 2) upload_slabs(i);
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
    // Groups: 0 = first launch, 1 = middle (ftl 4, e2e only), 2.. = the late levels (ftl 2),
    // one group each in upload order.
    std::vector<std::vector<size_t>> groups(2 + std::max<size_t>(late_order.size(), 1));
    for (size_t i = 0; i < lv.size(); ++i)
      if (counts[i] && ftl[i] != 2) groups[ftl[i] == 4 ? 1 : 0].push_back(i);
    for (size_t j = 0; j < late_order.size(); ++j)
      if (counts[late_order[j]]) groups[2 + j].push_back(late_order[j]);
    for (size_t k : short_segs) groups[0].push_back(k);
    if (mp_plan) groups[0].push_back(merged_seg);
    bool any_late_grp = false;
    size_t last_late = 0;
    for (size_t gi = 2; gi < groups.size(); ++gi)
      if (!groups[gi].empty()) any_late_grp = true, last_late = gi;
    const bool side = use_late_stream() && !groups[0].empty() && (!groups[1].empty() || any_late_grp);
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
      if (gi >= 2) {
        if (side) sg = h->s_late;
        CUDA_CHECK(cudaStreamWaitEvent(sg, h->ev_late_x[gi - 2], 0));
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
      if (gi >= 2 && gi == last_late && side) {
        CUDA_CHECK(cudaEventRecord(h->ev_late1, sg));
        CUDA_CHECK(cudaStreamWaitEvent(s, h->ev_late1, 0));
      }
    }
    if (!reduced_early) reduce_pairs(s);
  } else {
    // low-rank and shared-basis levels: independent per-level launch chains
    bool all_lr = lv.size() > 1 && use_concurrent_levels();
    for (auto& L : lv) {
      const int kind = group_for_level(h, L.level).kind;
      all_lr = all_lr && (kind == kLowRank || kind == kShared);
    }
    if (!all_lr) {
      for (auto& L : lv) launches += run_plan(h, L.level, *L.lp, L.x, L.y, s);
    } else {
      // low-rank / shared-basis levels are independent and each is a separate
      // launch chain: run them side by side on forked streams, each with its
      // own scratch (per-pair rows, padded sources, SA W~ / Z), so small
      // latency-bound levels overlap
      const size_t nl = lv.size();
      if (h->aux.size() < nl) {
        h->aux.resize(nl);
        h->lvl_scratch.resize(nl);
      }
      if (!h->ev_fork) CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
      CUDA_CHECK(cudaEventRecord(h->ev_fork, s));
      // largest level first: its long kernels start at once and the host-side
      // launch work of the small levels (and their short kernels) hides under them
      std::vector<size_t> order(nl);
      std::iota(order.begin(), order.end(), size_t(0));
      std::stable_sort(order.begin(), order.end(),
                       [&](size_t a, size_t b) { return lv[a].lp->n_rows > lv[b].lp->n_rows; });
      for (size_t k : order) {
        AuxStream& a = h->aux[k];
        if (!a.s) {
          CUDA_CHECK(cudaStreamCreateWithFlags(&a.s, cudaStreamNonBlocking));
          CUDA_CHECK(cudaEventCreateWithFlags(&a.done, cudaEventDisableTiming));
        }
        CUDA_CHECK(cudaStreamWaitEvent(a.s, h->ev_fork, 0));
        LevelScratch& sc = h->lvl_scratch[k];
        auto swap_scratch = [&] {
          std::swap(h->fbuf, sc.fbuf);
          std::swap(h->xpad, sc.xpad);
          std::swap(h->xpad_sig, sc.xpad_sig);
          std::swap(h->ybuf, sc.ybuf);
          std::swap(h->wt, sc.wt);
          std::swap(h->z, sc.z);
          std::swap(h->fzbuf, sc.fzbuf);
          std::swap(h->wt_ld_zeroed, sc.wt_ld_zeroed);
        };
        swap_scratch();
        try {
          launches += run_plan(h, lv[k].level, *lv[k].lp, lv[k].x, lv[k].y, a.s);
        } catch (...) {
          swap_scratch();
          throw;
        }
        swap_scratch();
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

}  // namespace cfm
