// Pageable host <-> device copies through pinned staging slots, several host
// threads at once.
//
// The reference's FmmPlan hands apply_level plain np.zeros level arrays
// (engine.py:104-108): pageable memory, which cudaMemcpy stages through the
// driver's internal buffers on one thread (~11 GB/s H2D, ~19 GB/s D2H
// measured on the B200 box, tools/copy_bench.py).  Here T workers each own
// two pinned slots and a stream: a worker copies its chunks (every T-th)
// pageable -> slot with memcpy, then slot -> device with cudaMemcpyAsync on
// its stream, alternating slots so the host copy of one chunk overlaps the
// DMA of the previous one (D2H in reverse).  The caller's stream is ordered
// with the workers by events on both sides.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

namespace cfm {

struct PinnedStager {
  static constexpr size_t kChunk = size_t(8) << 20;  // bytes per chunk
  int n_workers = 0;
  std::vector<void*> slots;             // 2 per worker
  std::vector<cudaStream_t> streams;    // 1 per worker
  std::vector<cudaEvent_t> slot_done;   // 2 per worker: the slot's last DMA finished
  std::vector<cudaEvent_t> worker_done; // 1 per worker
  cudaEvent_t ready = nullptr;

  ~PinnedStager() { release(); }
  void release() {
    for (void* p : slots) cudaFreeHost(p);
    for (auto s : streams) cudaStreamDestroy(s);
    for (auto e : slot_done) cudaEventDestroy(e);
    for (auto e : worker_done) cudaEventDestroy(e);
    if (ready) cudaEventDestroy(ready);
    slots.clear(), streams.clear(), slot_done.clear(), worker_done.clear();
    ready = nullptr;
    n_workers = 0;
  }
  void init() {
    if (n_workers) return;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int T = int(std::min(8u, std::max(1u, hw / 2)));
    for (int w = 0; w < T; ++w) {
      cudaStream_t s;
      CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      streams.push_back(s);
      cudaEvent_t e;
      CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      worker_done.push_back(e);
      for (int k = 0; k < 2; ++k) {
        void* p = nullptr;
        CUDA_CHECK(cudaHostAlloc(&p, kChunk, cudaHostAllocPortable));
        slots.push_back(p);
        CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        slot_done.push_back(e);
      }
    }
    CUDA_CHECK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    n_workers = T;
  }

  // Runs fn(w) on T threads (w = 0 .. T-1), rethrowing the first error.
  template <class F>
  void run(F&& fn) {
    std::vector<std::thread> th;
    std::vector<std::string> err(n_workers);
    std::vector<int> code(n_workers, 0);
    for (int w = 0; w < n_workers; ++w)
      th.emplace_back([&, w] {
        try {
          fn(w);
        } catch (const Error& e) {
          err[w] = e.what();
          code[w] = e.code;
        } catch (const std::exception& e) {
          err[w] = e.what();
          code[w] = CFM_ERR_INTERNAL;
        }
      });
    for (auto& t : th) t.join();
    for (int w = 0; w < n_workers; ++w)
      if (code[w]) throw Error(code[w], err[w]);
  }

  // dst (device) <- src (pageable host); `s` waits for the copies.
  void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s, int device) {
    if (!bytes) return;
    init();
    CUDA_CHECK(cudaEventRecord(ready, s));  // earlier work on s (e.g. the previous apply) may read dst
    const size_t n_chunks = (bytes + kChunk - 1) / kChunk;
    run([&](int w) {
      CUDA_CHECK(cudaSetDevice(device));
      cudaStream_t st = streams[w];
      CUDA_CHECK(cudaStreamWaitEvent(st, ready, 0));
      int k = 0;
      for (size_t c = size_t(w); c < n_chunks; c += size_t(n_workers), k ^= 1) {
        const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
        void* slot = slots[2 * w + k];
        CUDA_CHECK(cudaEventSynchronize(slot_done[2 * w + k]));  // the slot's previous DMA is done
        std::memcpy(slot, static_cast<const char*>(src) + off, len);
        CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(dst) + off, slot, len, cudaMemcpyHostToDevice, st));
        CUDA_CHECK(cudaEventRecord(slot_done[2 * w + k], st));
      }
      CUDA_CHECK(cudaEventRecord(worker_done[w], st));
    });
    for (int w = 0; w < n_workers; ++w) CUDA_CHECK(cudaStreamWaitEvent(s, worker_done[w], 0));
  }

  // dst (pageable host) <- src (device) after the work queued on `s`; returns
  // when dst holds the data.
  void d2h(void* dst, const void* src, size_t bytes, cudaStream_t s, int device) {
    if (!bytes) return;
    init();
    CUDA_CHECK(cudaEventRecord(ready, s));
    const size_t n_chunks = (bytes + kChunk - 1) / kChunk;
    run([&](int w) {
      CUDA_CHECK(cudaSetDevice(device));
      cudaStream_t st = streams[w];
      CUDA_CHECK(cudaStreamWaitEvent(st, ready, 0));
      // two chunks in flight per worker: DMA of chunk c + 1 while c is copied out
      std::vector<size_t> mine;
      for (size_t c = size_t(w); c < n_chunks; c += size_t(n_workers)) mine.push_back(c);
      auto issue = [&](size_t i) {
        const size_t off = mine[i] * kChunk, len = std::min(kChunk, bytes - off);
        CUDA_CHECK(cudaMemcpyAsync(slots[2 * w + (i & 1)], static_cast<const char*>(src) + off, len,
                                   cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaEventRecord(slot_done[2 * w + (i & 1)], st));
      };
      if (!mine.empty()) issue(0);
      for (size_t i = 0; i < mine.size(); ++i) {
        if (i + 1 < mine.size()) issue(i + 1);
        CUDA_CHECK(cudaEventSynchronize(slot_done[2 * w + (i & 1)]));
        const size_t off = mine[i] * kChunk, len = std::min(kChunk, bytes - off);
        std::memcpy(static_cast<char*>(dst) + off, slots[2 * w + (i & 1)], len);
      }
    });
  }
};

// Pinned (page-locked or registered) host memory: plain cudaMemcpyAsync.
inline bool is_pinned_host(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

}  // namespace cfm
