// Consumer-loop microbenchmark: the exact LDS -> DMMA chunk loop of
// tile_gemm_ws_kernel (BM=128, BN=64, 4x2 consumer warps, KC chunks, STAGES
// ring in shared memory), without producers, to find what caps the DMMA pipe.
//   mode 0: chunk loop over the ring (q % STAGES addressing), no barriers
//   mode 1: + mbarrier try_wait per chunk on an already-completed barrier
//   mode 2: + __syncwarp + lane-0 arrive per chunk (as the consumers do)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int KC, int STAGES, int MODE>
__global__ void __launch_bounds__(256, 1) k_loop(double* out, int chunks) {
  constexpr int BM = 128, BN = 64, LDA = KC + 4, LDB = KC + 4, MT = 4, NTL = 4;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = As + STAGES * BM * LDA;
  uint64_t* bar = reinterpret_cast<uint64_t*>(Bs + STAGES * BN * LDB);
  for (int i = threadIdx.x; i < STAGES * (BM + BN) * LDA; i += blockDim.x) smem[i] = 1e-3 * (i % 13);
  if (threadIdx.x == 0) {
    unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(1));
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(a) : "memory");
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tg = lane & 3, wm = warp % 4, wn = warp / 4;
  double acc[MT][NTL][2] = {};
  for (int q = 0; q < chunks; ++q) {
    const int s = q % STAGES;
    if (MODE >= 1) {
      unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
      asm volatile(
          "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(a),
          "r"(0)
          : "memory");
    }
    const double* as = As + s * BM * LDA + (wm * 32 + g) * LDA + tg;
    const double* bs = Bs + s * BN * LDB + (wn * 32 + g) * LDB + tg;
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
        for (int nj = 0; nj < NTL; ++nj) dmma(acc[mi][nj][0], acc[mi][nj][1], a[mi], b[nj]);
    }
    if (MODE >= 2) {
      __syncwarp();
      if (lane == 0) {
        unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar + 1));
        (void)a;
      }
    }
  }
  double sum = 0;
  for (int mi = 0; mi < MT; ++mi)
    for (int nj = 0; nj < NTL; ++nj) sum += acc[mi][nj][0] + acc[mi][nj][1];
  if (sum == 1234.5) out[0] = sum;
}

template <int KC, int STAGES, int MODE>
void run(const char* name, double* out, int nsm) {
  const int smem = STAGES * (128 + 64) * (KC + 4) * 8 + 64;
  auto k = k_loop<KC, STAGES, MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int chunks = 4000;
  k<<<nsm, 256, smem>>>(out, 100);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<nsm * 4, 256, smem>>>(out, chunks);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double flops = double(nsm) * 4 * 8 * chunks * (KC / 4) * 16 * 512.0;
  printf("{\"test\":\"%s\",\"KC\":%d,\"ms\":%.3f,\"tflops\":%.3f,\"err\":\"%s\"}\n", name, KC, ms, flops / ms * 1e-9,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 64);
  run<16, 5, 0>("ring_nobar", out, nsm);
  run<16, 5, 1>("ring_trywait", out, nsm);
  run<16, 5, 2>("ring_trywait_sync", out, nsm);
  run<32, 3, 0>("ring32_nobar", out, nsm);
  run<64, 2, 0>("ring64_nobar", out, nsm);
  return 0;
}
