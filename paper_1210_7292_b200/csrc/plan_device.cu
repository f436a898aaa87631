// Device planner for dense full-operator target-tile plans (the config 2 / 4
// hot path): the plan of plan.hpp's build_plan_csr + plan.cu's row-order tile
// dispatch, slab needs and hybrid split, built on the GPU from the device
// classifier's lists instead of copying 2.3 GB of lists to the host and
// building 1.5 GB of tiles there (config 4 level 7: ~9.7 s on the host).
//
// The plan is the host builder's, entry for entry:
//   1. per target row with pairs: h = sum_q splitmix64(code_q + 1) (mod 2^64,
//      order independent), validity of codes / operators / source rows;
//   2. targets stably sorted by (h, row) -> tiles of 64 / dc consecutive
//      targets;
//   3. tiles stably re-ordered by their smallest target row (row-order
//      dispatch for the host-buffer slab pipeline);
//   4. per tile, one entry per (code, occurrence) -- occurrence = index of the
//      pair among its target's pairs with that code, in list order -- ordered
//      by (operator key, code, occurrence); slot s of entry (c, o) = the o-th
//      pair of code c of the tile's s-th target, or -1;
//   5. hybrid: tiles less than half full leave for a pair-mode sub-plan (built
//      on the host from those targets' lists), the kept tiles re-ordered longest
//      first.
// Levels that plan as pair entries (fill < 0.6, sparse trees) return to the
// host builder.  `test_device_plan_matches_host_plan` checks bitwise equal
// locals and equal plan statistics against the host builder (CFM_DEVICE_PLAN=0).
#include "internal.hpp"

#include <cub/cub.cuh>

namespace cfm {

namespace {

__device__ __forceinline__ unsigned long long splitmix64_d(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// warp per row: multiset hash of the row's codes, non-empty flag, validity
__global__ void k_plan_hash(const long long* __restrict__ off, const int16_t* __restrict__ code,
                            const int* __restrict__ src, long long n, const int* __restrict__ key, long long n_rows,
                            unsigned long long* __restrict__ hash, int* __restrict__ nonempty, int* __restrict__ err) {
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  const long long b = off[w], e = off[w + 1];
  unsigned long long h = 0;
  int bad = 0;
  for (long long q = b + lane; q < e; q += 32) {
    const int c = code[q];
    if (c < 0 || c >= kNumCodes) bad |= 1;
    else if (key[c] < 0) bad |= 2;
    const int s = src[q];
    if (s < 0 || s >= n_rows) bad |= 4;
    h += splitmix64_d((unsigned long long)(c) + 1ull);
  }
  for (int o = 16; o; o >>= 1) {
    h += __shfl_xor_sync(0xffffffffu, h, o);
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if (lane == 0) {
    hash[w] = h;
    nonempty[w] = e > b;
    if (bad) atomicOr(err, bad);
  }
}

// smallest target row of each pre-order tile
__global__ void k_tile_min(const int* __restrict__ uord, long long nu, int tpt, long long nt, int* __restrict__ tmin) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= nt) return;
  int m = 0x7fffffff;
  for (int s = 0; s < tpt; ++s) {
    const long long k = t * tpt + s;
    if (k < nu) m = min(m, uord[k]);
  }
  tmin[t] = m;
}

constexpr int kPlanThreads = 256;
constexpr int kPlanWarps = kPlanThreads / 32;

// Per (final) tile: occurrence maxima per code (in smem `maxocc`), pair count.
// Target s of final tile k = uord[ord[k] * tpt + s].
__device__ void tile_maxocc(long long k, const int* __restrict__ ord, const int* __restrict__ uord, long long nu,
                            int tpt, const long long* __restrict__ off, const int16_t* __restrict__ code, int* maxocc,
                            int* wcnt, long long* cc, int* s_pairs) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = threadIdx.x; c < kNumCodes; c += kPlanThreads) maxocc[c] = 0;
  if (threadIdx.x == 0) *s_pairs = 0;
  int* cnt = wcnt + warp * kNumCodes;
  for (int c = lane; c < kNumCodes; c += 32) cnt[c] = 0;
  __syncthreads();
  const long long base = (long long)ord[k] * tpt;
  int pairs = 0;
  for (int s = warp; s < tpt; s += kPlanWarps) {
    if (base + s >= nu) break;
    const int row = uord[base + s];
    const long long b = off[row], e = off[row + 1];
    pairs += int(e - b);
    for (long long q = b + lane; q < e; q += 32) atomicAdd(&cnt[code[q]], 1);
    __syncwarp();
    for (int c = lane; c < kNumCodes; c += 32) {
      const int v = cnt[c];
      if (v) {
        atomicMax(&maxocc[c], v);
        if (cc) atomicAdd(reinterpret_cast<unsigned long long*>(cc) + c, (unsigned long long)v);
        cnt[c] = 0;
      }
    }
    __syncwarp();
  }
  if (lane == 0) atomicAdd(s_pairs, pairs);
  __syncthreads();
}

__global__ void __launch_bounds__(kPlanThreads) k_plan_count(const int* __restrict__ ord, const int* __restrict__ uord,
                                                               long long nu, int tpt, const long long* __restrict__ off,
                                                               const int16_t* __restrict__ code, long long* __restrict__ n_ent,
                                                               long long* __restrict__ n_pairs, long long* __restrict__ cc) {
  __shared__ int maxocc[kNumCodes];
  __shared__ int wcnt[kPlanWarps * kNumCodes];
  __shared__ int s_pairs;
  const long long k = blockIdx.x;
  tile_maxocc(k, ord, uord, nu, tpt, off, code, maxocc, wcnt, cc, &s_pairs);
  int e = 0;
  for (int c = threadIdx.x; c < kNumCodes; c += kPlanThreads) e += maxocc[c];
  for (int o = 16; o; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  __shared__ int s_e[kPlanWarps];
  if ((threadIdx.x & 31) == 0) s_e[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int w = 0; w < kPlanWarps; ++w) t += s_e[w];
    n_ent[k] = t;
    n_pairs[k] = s_pairs;
  }
}

// Fills tile k of the output plan from source tile src_tile[k] (final order):
// tile_col, entry codes, entry sources (entry_src pre-set to -1).
__global__ void __launch_bounds__(kPlanThreads) k_plan_fill(const int* __restrict__ src_tile, const int* __restrict__ ord,
                                                              const int* __restrict__ uord, long long nu, int tpt,
                                                              const long long* __restrict__ off,
                                                              const int16_t* __restrict__ code,
                                                              const int* __restrict__ src, const int* __restrict__ corder,
                                                              int n_corder, const long long* __restrict__ tile_off,
                                                              int* __restrict__ tile_col, int* __restrict__ entry_code,
                                                              int* __restrict__ entry_src) {
  __shared__ int maxocc[kNumCodes];
  __shared__ int basec[kNumCodes];
  __shared__ int wcnt[kPlanWarps * kNumCodes];
  __shared__ int s_pairs;
  const long long k = blockIdx.x;
  const long long kt = src_tile[k];  // final-order tile whose content goes to slot k
  tile_maxocc(kt, ord, uord, nu, tpt, off, code, maxocc, wcnt, nullptr, &s_pairs);
  if (threadIdx.x == 0) {  // entries ordered by (operator key, code): corder
    int run = 0;
    for (int i = 0; i < n_corder; ++i) {
      const int c = corder[i];
      basec[c] = run;
      run += maxocc[c];
    }
  }
  __syncthreads();
  const long long e0 = tile_off[k];
  for (int c = threadIdx.x; c < kNumCodes; c += kPlanThreads)
    for (int o = 0; o < maxocc[c]; ++o) entry_code[e0 + basec[c] + o] = c;
  const long long base = (long long)ord[kt] * tpt;
  for (int s = threadIdx.x; s < kBN; s += kPlanThreads) {
    const int slot_t = s;  // dc == 1: column s = target slot s
    tile_col[k * kBN + s] = (slot_t < tpt && base + slot_t < nu) ? uord[base + slot_t] : -1;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* run = wcnt + warp * kNumCodes;
  for (int c = lane; c < kNumCodes; c += 32) run[c] = 0;
  __syncwarp();
  for (int s = warp; s < tpt; s += kPlanWarps) {
    if (base + s >= nu) break;
    const int row = uord[base + s];
    const long long b = off[row], e = off[row + 1];
    for (long long q0 = b; q0 < e; q0 += 32) {
      const long long q = q0 + lane;
      const bool live = q < e;
      const unsigned act = __ballot_sync(0xffffffffu, live);
      const int c = live ? int(code[q]) : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, c);
      if (live) {
        const int rank = __popc(peers & ((1u << lane) - 1u));
        const int occ = run[c] + rank;
        entry_src[(e0 + basec[c] + occ) * kBN + s] = src[q];
      }
      __syncwarp();
      if (live && lane == 31 - __clz(peers & act)) run[c] += __popc(peers & act);  // highest peer updates
      __syncwarp();
    }
    for (int c = lane; c < kNumCodes; c += 32) run[c] = 0;
    __syncwarp();
  }
}

// per final tile: min / max target row, min / max source row
__global__ void __launch_bounds__(kPlanThreads) k_plan_tile_rows(const int* __restrict__ ord, const int* __restrict__ uord,
                                                                   long long nu, int tpt, const long long* __restrict__ off,
                                                                   const int* __restrict__ src, int* __restrict__ out) {
  const long long k = blockIdx.x;
  const long long base = (long long)ord[k] * tpt;
  int tlo = 0x7fffffff, thi = -1, slo = 0x7fffffff, shi = -1;
  for (int s = threadIdx.x >> 5; s < tpt; s += kPlanWarps) {
    if (base + s >= nu) break;
    const int row = uord[base + s];
    tlo = min(tlo, row), thi = max(thi, row);
    for (long long q = off[row] + (threadIdx.x & 31); q < off[row + 1]; q += 32) {
      slo = min(slo, src[q]);
      shi = max(shi, src[q]);
    }
  }
  for (int o = 16; o; o >>= 1) {
    tlo = min(tlo, __shfl_xor_sync(0xffffffffu, tlo, o));
    thi = max(thi, __shfl_xor_sync(0xffffffffu, thi, o));
    slo = min(slo, __shfl_xor_sync(0xffffffffu, slo, o));
    shi = max(shi, __shfl_xor_sync(0xffffffffu, shi, o));
  }
  __shared__ int r[4][kPlanWarps];
  if ((threadIdx.x & 31) == 0) {
    const int w = threadIdx.x >> 5;
    r[0][w] = tlo, r[1][w] = thi, r[2][w] = slo, r[3][w] = shi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kPlanWarps; ++w) {
      tlo = min(tlo, r[0][w]), thi = max(thi, r[1][w]), slo = min(slo, r[2][w]), shi = max(shi, r[3][w]);
    }
    out[4 * k] = tlo, out[4 * k + 1] = thi, out[4 * k + 2] = slo, out[4 * k + 3] = shi;
  }
}

__global__ void k_mark_sources(const int* __restrict__ src, long long P, unsigned char* __restrict__ seen) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < P; q += gridDim.x * (long long)blockDim.x)
    seen[src[q]] = 1;
}

// pack the pairs of the given rows (leftover targets of the hybrid split)
__global__ void k_pack_rows(const long long* __restrict__ off, const int* __restrict__ src,
                            const int16_t* __restrict__ code, const int* __restrict__ rows,
                            const long long* __restrict__ out_off, long long n, int* __restrict__ osrc,
                            int16_t* __restrict__ ocode) {
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  const int r = rows[w];
  const long long b = off[r], o = out_off[w];
  for (long long q = b + lane; q < off[r + 1]; q += 32) {
    osrc[o + (q - b)] = src[q];
    ocode[o + (q - b)] = code[q];
  }
}

template <class F>
void cub_run(F&& f, cudaStream_t s) {
  size_t tmp = 0;
  CUDA_CHECK(f(nullptr, tmp));
  DevBuf t;
  t.alloc(std::max<size_t>(tmp, 16));
  CUDA_CHECK(f(t.p, tmp));
}

template <class T>
std::vector<T> to_host(const DevBuf& d, size_t n, cudaStream_t s) {
  std::vector<T> h(n);
  if (n) CUDA_CHECK(cudaMemcpyAsync(h.data(), d.p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  return h;
}

}  // namespace

bool use_device_plan() {  // CFM_DEVICE_PLAN=0: host builder (A/B and the parity test)
  const char* e = getenv("CFM_DEVICE_PLAN");
  return !e || atoi(e) != 0;
}

// Builds lp for a dense full-operator level from device lists (off: n + 1
// int64, src int32, code int16, all on the device; h_off on the host).
// Returns false when the level plans as pair entries (the caller then uses
// the host builder).
bool device_plan_dense(cfm_handler* h, int level, const Group& g, int64_t n, const int64_t* d_off,
                       const std::vector<int64_t>& h_off, const int32_t* d_src, const int16_t* d_code,
                       int64_t n_rows, cudaStream_t s, LevelPlan& lp) {
  const double t0 = trace_on() ? wall_ms() : 0.0;
  constexpr int dc = 1, tpt = kBN;
  std::array<int, kNumCodes> key;
  for (int c = 0; c < kNumCodes; ++c) key[c] = g.valid[c] ? std::max(g.main.op[c], 0) + 1 : -1;
  const int64_t P = h_off[n];
  DevBuf d_key, d_hash, d_ne, d_err, d_rows, d_hash_ne, d_cnt, d_uord, d_hash_sorted;
  upload(d_key, std::vector<int>(key.begin(), key.end()));
  d_hash.alloc(std::max<size_t>(size_t(n) * 8, 16));
  d_ne.alloc(std::max<size_t>(size_t(n) * 4, 16));
  d_err.alloc(16);
  CUDA_CHECK(cudaMemsetAsync(d_err.p, 0, 4, s));
  const long long* off = reinterpret_cast<const long long*>(d_off);
  if (n)
    k_plan_hash<<<unsigned((n * 32 + 255) / 256), 256, 0, s>>>(off, d_code, d_src, n, d_key.as<int>(), n_rows,
                                                               d_hash.as<unsigned long long>(), d_ne.as<int>(),
                                                               d_err.as<int>());
  CUDA_CHECK(cudaGetLastError());
  int err = 0;
  CUDA_CHECK(cudaMemcpyAsync(&err, d_err.p, 4, cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  if (err & 1) throw Error(CFM_ERR_VALUE, "transfer vector outside [-3,3]^3");
  if (err & 4) throw Error(CFM_ERR_VALUE, "source row out of range");
  if (err & 2) throw Error(CFM_ERR_PRECOMPUTE, "no operator for a transfer vector of level " + std::to_string(level));
  // compact the rows with pairs (row order kept), then stable sort by hash
  std::vector<int> iota_rows(n);
  std::iota(iota_rows.begin(), iota_rows.end(), 0);
  DevBuf d_iota;
  upload(d_iota, iota_rows);
  d_rows.alloc(std::max<size_t>(size_t(n) * 4, 16));
  d_hash_ne.alloc(std::max<size_t>(size_t(n) * 8, 16));
  d_cnt.alloc(16);
  cub_run([&](void* t, size_t& b) {
    return cub::DeviceSelect::Flagged(t, b, d_iota.as<int>(), d_ne.as<int>(), d_rows.as<int>(), d_cnt.as<long long>(),
                                      n, s);
  }, s);
  long long nu = 0;
  CUDA_CHECK(cudaMemcpyAsync(&nu, d_cnt.p, 8, cudaMemcpyDeviceToHost, s));
  cub_run([&](void* t, size_t& b) {
    return cub::DeviceSelect::Flagged(t, b, d_hash.as<unsigned long long>(), d_ne.as<int>(),
                                      d_hash_ne.as<unsigned long long>(), d_cnt.as<long long>(), n, s);
  }, s);
  CUDA_CHECK(cudaStreamSynchronize(s));
  d_uord.alloc(std::max<size_t>(size_t(nu) * 4, 16));
  d_hash_sorted.alloc(std::max<size_t>(size_t(nu) * 8, 16));
  cub_run([&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, d_hash_ne.as<unsigned long long>(),
                                           d_hash_sorted.as<unsigned long long>(), d_rows.as<int>(), d_uord.as<int>(),
                                           nu, 0, 64, s);
  }, s);
  const int64_t nt = (nu + tpt - 1) / tpt;
  // tiles in row order of their smallest target (stable)
  DevBuf d_tmin, d_tmin_sorted, d_tiota, d_ord;
  d_tmin.alloc(std::max<size_t>(size_t(nt) * 4, 16));
  d_tmin_sorted.alloc(std::max<size_t>(size_t(nt) * 4, 16));
  d_ord.alloc(std::max<size_t>(size_t(nt) * 4, 16));
  std::vector<int> tio(nt);
  std::iota(tio.begin(), tio.end(), 0);
  upload(d_tiota, tio);
  if (nt) k_tile_min<<<unsigned((nt + 255) / 256), 256, 0, s>>>(d_uord.as<int>(), nu, tpt, nt, d_tmin.as<int>());
  cub_run([&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, d_tmin.as<int>(), d_tmin_sorted.as<int>(), d_tiota.as<int>(),
                                           d_ord.as<int>(), nt, 0, 32, s);
  }, s);
  // entries per tile, code counts
  DevBuf d_nent, d_npairs, d_cc, d_toff;
  d_nent.alloc(std::max<size_t>(size_t(nt + 1) * 8, 16));
  d_npairs.alloc(std::max<size_t>(size_t(nt) * 8, 16));
  d_cc.alloc(kNumCodes * 8);
  CUDA_CHECK(cudaMemsetAsync(d_cc.p, 0, kNumCodes * 8, s));
  if (nt)
    k_plan_count<<<unsigned(nt), kPlanThreads, 0, s>>>(d_ord.as<int>(), d_uord.as<int>(), nu, tpt, off, d_code,
                                                       d_nent.as<long long>(), d_npairs.as<long long>(),
                                                       d_cc.as<long long>());
  CUDA_CHECK(cudaGetLastError());
  std::vector<long long> nent = to_host<long long>(d_nent, nt, s);
  std::vector<long long> npairs = to_host<long long>(d_npairs, nt, s);
  std::vector<long long> cc = to_host<long long>(d_cc, kNumCodes, s);
  int64_t E = 0;
  for (auto v : nent) E += v;
  HostPlan& hp = lp.hp;
  hp.dc = dc;
  hp.n_tiles = nt;
  hp.n_pairs = 0;
  for (int c = 0; c < kNumCodes; ++c) hp.code_count[c] = cc[c], hp.n_pairs += cc[c];
  const double slots = double(E) * kBN;
  lp.target_fill = slots > 0 ? double(hp.n_pairs) * dc / slots : 1.0;
  if (lp.target_fill < 0.6 || getenv("CFM_PLAN_MODE")) return false;  // pair entries: host builder
  if (E > INT32_MAX || E * kBN >= (int64_t(1) << 40)) throw Error(CFM_ERR_VALUE, "plan too large for int32 entry offsets");
  hp.n_entries_dev = E;
  std::vector<int> corder;  // valid codes by (operator key, code)
  for (int c = 0; c < kNumCodes; ++c)
    if (key[c] >= 0) corder.push_back(c);
  std::stable_sort(corder.begin(), corder.end(), [&](int a, int b) { return key[a] < key[b]; });
  DevBuf d_corder;
  upload(d_corder, corder);
  auto fill = [&](const std::vector<int>& tiles, const std::vector<long long>& toff, DevBuf& col, DevBuf& tof,
                  DevBuf& ecode, DevBuf& esrc) {
    const int64_t m = int64_t(tiles.size());
    DevBuf d_tiles, d_toff64;
    upload(d_tiles, tiles);
    upload(d_toff64, toff);
    std::vector<int> toff32(toff.begin(), toff.end());
    upload(tof, toff32);
    const int64_t ne = toff[m];
    col.alloc(std::max<size_t>(size_t(m) * kBN * 4, 16));
    ecode.alloc(std::max<size_t>(size_t(ne) * 4, 16));
    esrc.alloc(std::max<size_t>(size_t(ne) * kBN * 4, 16));
    CUDA_CHECK(cudaMemsetAsync(esrc.p, 0xff, size_t(ne) * kBN * 4, s));
    if (m)
      k_plan_fill<<<unsigned(m), kPlanThreads, 0, s>>>(d_tiles.as<int>(), d_ord.as<int>(), d_uord.as<int>(), nu, tpt,
                                                       off, d_code, d_src, d_corder.as<int>(), int(corder.size()),
                                                       d_toff64.as<long long>(), col.as<int>(), ecode.as<int>(),
                                                       esrc.as<int>());
    CUDA_CHECK(cudaGetLastError());
  };
  {
    std::vector<int> all(nt);
    std::iota(all.begin(), all.end(), 0);
    std::vector<long long> toff(nt + 1, 0);
    for (int64_t t = 0; t < nt; ++t) toff[t + 1] = toff[t] + nent[t];
    fill(all, toff, lp.tile_col, lp.tile_off, lp.entry_code, lp.entry_src);
  }
  // per-tile target / source row ranges: slab needs of the host-buffer pipeline, row spans
  DevBuf d_tr;
  d_tr.alloc(std::max<size_t>(size_t(nt) * 16, 16));
  if (nt)
    k_plan_tile_rows<<<unsigned(nt), kPlanThreads, 0, s>>>(d_ord.as<int>(), d_uord.as<int>(), nu, tpt, off, d_src,
                                                           d_tr.as<int>());
  std::vector<int> tr = to_host<int>(d_tr, size_t(nt) * 4, s);
  lp.dc = dc;
  lp.n_rows = n_rows;
  lp.mode = 0;
  int64_t slo = n_rows, shi = 0, tlo = n_rows, thi = 0;
  for (int64_t t = 0; t < nt; ++t) {
    tlo = std::min<int64_t>(tlo, tr[4 * t]), thi = std::max<int64_t>(thi, tr[4 * t + 1] + 1);
    if (tr[4 * t + 3] >= 0) slo = std::min<int64_t>(slo, tr[4 * t + 2]), shi = std::max<int64_t>(shi, tr[4 * t + 3] + 1);
  }
  lp.src_lo = std::min(slo, shi), lp.src_hi = shi, lp.tgt_lo = std::min(tlo, thi), lp.tgt_hi = thi;
  // targets / sources (plan statistics)
  {
    std::vector<int> uord = to_host<int>(d_uord, size_t(nu), s);
    lp.targets.assign(uord.begin(), uord.end());
    std::sort(lp.targets.begin(), lp.targets.end());
    DevBuf d_seen;
    d_seen.alloc(std::max<size_t>(size_t(n_rows), 16));
    CUDA_CHECK(cudaMemsetAsync(d_seen.p, 0, size_t(n_rows), s));
    if (P) k_mark_sources<<<148 * 8, 256, 0, s>>>(d_src, P, d_seen.as<unsigned char>());
    std::vector<unsigned char> seen = to_host<unsigned char>(d_seen, size_t(n_rows), s);
    for (int64_t r = 0; r < n_rows; ++r)
      if (seen[r]) lp.sources.push_back(r);
  }
  set_slab_plan(h, level, lp, [&](int64_t t, int64_t& tmin, int64_t& tmax, int64_t& smax) {
    tmin = tr[4 * t], tmax = tr[4 * t + 1], smax = tr[4 * t + 3];
  });
  // hybrid: tiles less than half full -> pair sub-plan; kept tiles longest first
  if (use_hybrid() && nt > 0) {
    std::vector<char> left(nt, 0);
    int64_t n_left = 0;
    for (int64_t t = 0; t < nt; ++t)
      if (nent[t] > 0 && 2 * npairs[t] * dc < nent[t] * kBN) left[t] = 1, ++n_left;
    if (n_left > 0 && n_left < nt) {
      auto hy = std::make_shared<HybridPlan>();
      std::vector<int> kept;
      for (int64_t t = 0; t < nt; ++t)
        if (!left[t]) kept.push_back(int(t));
      std::stable_sort(kept.begin(), kept.end(), [&](int a, int b) { return nent[a] > nent[b]; });
      const long long max_e = kept.empty() ? 0 : nent[kept[0]];
      for (int t : kept) hy->n_long += nent[t] * 10 >= max_e * 9;
      std::vector<long long> toff(kept.size() + 1, 0);
      for (size_t i = 0; i < kept.size(); ++i) toff[i + 1] = toff[i] + nent[kept[i]];
      fill(kept, toff, hy->tile_col, hy->tile_off, hy->entry_code, hy->entry_src);
      hy->main.dc = dc;
      hy->main.n_tiles = int64_t(kept.size());
      hy->main.n_entries_dev = toff.back();
      // the leftover targets' lists (row order) -> pair entries on the host
      std::vector<int> uord = to_host<int>(d_uord, size_t(nu), s);
      std::vector<int> ordh = to_host<int>(d_ord, size_t(nt), s);
      std::vector<int> lrows;
      for (int64_t t = 0; t < nt; ++t)
        if (left[t])
          for (int k = 0; k < tpt && int64_t(ordh[t]) * tpt + k < nu; ++k) lrows.push_back(uord[int64_t(ordh[t]) * tpt + k]);
      std::sort(lrows.begin(), lrows.end());
      std::vector<long long> o2(lrows.size() + 1, 0);
      for (size_t i = 0; i < lrows.size(); ++i) o2[i + 1] = o2[i] + (h_off[lrows[i] + 1] - h_off[lrows[i]]);
      DevBuf d_lrows, d_o2, d_s2, d_c2;
      upload(d_lrows, lrows);
      upload(d_o2, o2);
      d_s2.alloc(std::max<size_t>(size_t(o2.back()) * 4, 16));
      d_c2.alloc(std::max<size_t>(size_t(o2.back()) * 2, 16));
      if (!lrows.empty())
        k_pack_rows<<<unsigned((lrows.size() * 32 + 255) / 256), 256, 0, s>>>(
            off, d_src, d_code, d_lrows.as<int>(), d_o2.as<long long>(), int64_t(lrows.size()), d_s2.as<int>(),
            d_c2.as<int16_t>());
      std::vector<int> s2i = to_host<int>(d_s2, size_t(o2.back()), s);
      std::vector<int16_t> c2 = to_host<int16_t>(d_c2, size_t(o2.back()), s);
      std::vector<int64_t> t2(lrows.begin(), lrows.end()), o2l(o2.begin(), o2.end()), s2(s2i.begin(), s2i.end());
      LevelPlan& ax = hy->aux;
      const int nkp = round_up(h->n * h->f, kKC);
      const int64_t e_est = int64_t(s2.size()) / kBN + 1;
      int ept = std::max(1, std::min(16, int(2.5e7 / (2.0 * 128 * kBN * nkp))));
      ept = std::min<int>(ept, int(std::max<int64_t>(1, e_est / (2 * 148))));
      try {
        ax.hp = build_plan_pairs(int64_t(t2.size()), t2.data(), o2l.data(), s2.data(), c2.data(), 1, key, n_rows, ept,
                                 ax.red);
      } catch (const PlanError& e) {
        throw Error(e.code == 2 ? CFM_ERR_PRECOMPUTE : CFM_ERR_VALUE, e.what());
      }
      ax.mode = 1;
      ax.dc = 1;
      ax.n_rows = n_rows;
      push_pair_plan(ax);
      static uint64_t hyb_gen_dev = (uint64_t(1) << 62) + (uint64_t(1) << 61);
      ax.gen = ++hyb_gen_dev;
      lp.hyb = std::move(hy);
    }
  }
  CUDA_CHECK(cudaStreamSynchronize(s));
  if (trace_on())
    fprintf(stderr, "[cfm plan L%d] device planner %.1f ms (%lld tiles, %lld entries)\n", level, wall_ms() - t0,
            (long long)nt, (long long)E);
  return true;
}

}  // namespace cfm
