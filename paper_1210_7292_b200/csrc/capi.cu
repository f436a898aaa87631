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
#include "internal.hpp"

#include <thread>

namespace cfm {
thread_local std::string g_last_error;
}  // namespace cfm

using namespace cfm;

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
    if (use_lowrank_full(h)) build_lowrank_full(h, g, n_transfers, transfers, n_ops, ranks, left, right);
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
    {  // dense full-operator levels with ascending target rows (a rank's shard-local
       // lists): rows without a list get an empty one and the device planner runs
      Group& g = group_for_level(h, level);
      bool ok = use_device_plan() && g.kind == kDense && g.has_full && !data_complex && !h->op_complex &&
                n_rows < (int64_t(1) << 31);
      for (int64_t i = 0; ok && i < n_targets; ++i)
        ok = tgt[i] >= 0 && tgt[i] < n_rows && (i == 0 || tgt[i] > tgt[i - 1]) && off[i + 1] >= off[i];
      for (int64_t q = 0; ok && q < P; ++q) ok = src[q] >= 0 && src[q] < n_rows;
      if (ok) {
        std::vector<int64_t> h_off(n_rows + 1, 0);
        for (int64_t i = 0; i < n_targets; ++i) h_off[tgt[i] + 1] = off[i + 1] - off[i];
        for (int64_t r = 0; r < n_rows; ++r) h_off[r + 1] += h_off[r];
        // pairs are already in row order (targets ascending, lists in CSR order)
        std::vector<int32_t> src32(P);
        for (int64_t q = 0; q < P; ++q) src32[q] = int32_t(src[q]);
        cudaStream_t s = h->stream;
        DevBuf d_off, d_src, d_code;
        upload(d_off, h_off);
        upload(d_src, src32);
        upload(d_code, codes);
        LevelPlan lp;
        if (device_plan_dense(h, level, g, n_rows, d_off.as<int64_t>(), h_off, d_src.as<int32_t>(),
                              d_code.as<int16_t>(), n_rows, s, lp)) {
          lp.gen = next_plan_gen();
          h->plans[level] = std::move(lp);
          const LevelPlan& pl = h->plans[level];
          if (pair_count_out) std::copy(pl.hp.code_count.begin(), pl.hp.code_count.end(), pair_count_out);
          return;
        }
      }
    }
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
    h->last_csr_gen = lp.gen;
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
    const double t0 = trace_on() ? wall_ms() : 0.0;
    DeviceLists dl;
    classify_device(level, n_cells, ijk, s, dl, /*want_codes=*/true);
    const double t1 = trace_on() ? wall_ms() : 0.0;
    {  // dense full-operator levels: the whole plan on the device (plan_device.cu)
      Group& g = group_for_level(h, level);
      if (use_device_plan() && g.kind == kDense && g.has_full && !data_complex && !h->op_complex) {
        LevelPlan lp;
        if (device_plan_dense(h, level, g, n_cells, reinterpret_cast<const int64_t*>(dl.off.p), dl.h_off,
                              dl.src.as<int32_t>(), dl.code.as<int16_t>(), n_cells, s, lp)) {
          lp.gen = next_plan_gen();
          h->plans[level] = std::move(lp);
          const LevelPlan& pl = h->plans[level];
          if (pair_count_out) std::copy(pl.hp.code_count.begin(), pl.hp.code_count.end(), pair_count_out);
          return;
        }
      }
    }
    std::vector<int32_t> hsrc(dl.total);
    std::vector<int16_t> hcode(dl.total);
    if (dl.total) {  // lists to the host through the multi-threaded pinned stager
      if (!h->stager) h->stager = std::make_unique<PinnedStager>();
      h->stager->d2h(hsrc.data(), dl.src.p, size_t(dl.total) * 4, s, h->device);
      h->stager->d2h(hcode.data(), dl.code.p, size_t(dl.total) * 2, s, h->device);
    }
    const double t2 = trace_on() ? wall_ms() : 0.0;
    std::vector<int64_t> tgt(n_cells), src64(dl.total);
    std::iota(tgt.begin(), tgt.end(), 0);
    {  // widen the source rows on several threads
      const int64_t P = dl.total;
      const unsigned nth = unsigned(std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()),
                                                      std::max<int64_t>(1, P / (int64_t(1) << 20))));
      std::vector<std::thread> th;
      auto wid = [&](unsigned w) {
        for (int64_t q = P * w / nth; q < P * (w + 1) / nth; ++q) src64[q] = hsrc[q];
      };
      for (unsigned w = 1; w < nth; ++w) th.emplace_back(wid, w);
      wid(0);
      for (auto& x : th) x.join();
    }
    const double t3 = trace_on() ? wall_ms() : 0.0;
    LevelPlan& lp = make_plan(h, level, n_cells, tgt.data(), dl.h_off.data(), src64.data(), hcode.data(),
                              data_complex, n_cells);
    if (trace_on())
      fprintf(stderr, "[cfm plan L%d] classify %.1f ms, lists D2H %.1f ms, widen %.1f ms, make_plan %.1f ms\n", level,
              t1 - t0, t2 - t1, t3 - t2, wall_ms() - t3);
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

int cfm_last_csr_plan_info(cfm_handler* h, int* cache_hit, int* mode, int* two_stage, uint64_t* plan_id) {
  return guarded([&] {
    if (!h) throw Error(CFM_ERR_VALUE, "null handler");
    std::lock_guard<std::mutex> lk(h->mu);
    if (cache_hit) *cache_hit = h->last_csr_hit ? 1 : 0;
    if (mode) *mode = h->last_csr_mode;
    if (two_stage) *two_stage = h->last_csr_two_stage;
    if (plan_id) *plan_id = h->last_csr_gen;
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
