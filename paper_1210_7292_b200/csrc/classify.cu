// Far-list classifier (octree.py:148-178 + symmetry.py:63-75 on the device) and the halo pack kernel.
#include "internal.hpp"
#include "classify.cuh"
#include <cub/cub.cuh>

namespace cfm {

// ------------------------------------------------------------------ classifier

// c_cone_index is per-device __constant__ memory: upload it once per device
// (the caller has selected the device).
void init_cone_table() {
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
ClassifyScratch& classify_scratch(int device) {
  static thread_local std::map<int, ClassifyScratch> per_device;
  return per_device[device];
}

void classify_device(int level, int64_t n_cells, const int32_t* ijk, cudaStream_t s, DeviceLists& out,
                            bool want_codes, int32_t* h_src, int8_t* h_t, uint8_t* h_rep,
                            uint8_t* h_perm, const int64_t* given_off,
                            const int64_t* target_rows, int64_t n_targets) {
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

}  // namespace cfm

using namespace cfm;

extern "C" {
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

}  // extern "C"
