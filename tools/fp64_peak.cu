// FP64 throughput microbenchmark for the M2L roofline denominator.
//
// MEASURED_PEAKS.json carries HBM and bf16 peaks only; the M2L full-rank path
// is FP64-bound, so its peak is measured here on the box:
//   * DMMA  : mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 (SASS DMMA.8x8x4)
//   * DFMA  : scalar fp64 fused multiply-add
//   * smem-fed DMMA: the same with operands loaded from shared memory each step
// Output: one JSON line per test.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int NACC>
__global__ void k_dmma(double* out, int iters, double a, double b) {
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  double av = a + threadIdx.x * 1e-9, bv = b - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(c[i][0], c[i][1], av, bv);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = threadIdx.x * 1e-3 + i;
  double av = a + threadIdx.x * 1e-9, bv = b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(av, c[i], bv);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

// DMMA fed from shared memory: warp tile 32x32 (4x4 mma tiles), k-steps of 4,
// A/B fragments loaded via LDS each step, mirroring the M2L tile kernel's inner loop.
__global__ void k_dmma_smem(double* out, int iters) {
  __shared__ double As[64 * 36];
  __shared__ double Bs[64 * 36];
  for (int i = threadIdx.x; i < 64 * 36; i += blockDim.x) { As[i] = 1e-3 * (i % 17); Bs[i] = 1e-3 * (i % 13); }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp & 1) * 32, wn = ((warp >> 1) & 1) * 32;
  double c[4][4][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k0 = 0; k0 < 32; k0 += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[(wm + i * 8 + g) * 36 + k0 + t];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[(wn + j * 8 + g) * 36 + k0 + t];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(c[i][j][0], c[i][j][1], a[i], b[j]);
    }
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += c[i][j][0] + c[i][j][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double* out;
  CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int iters = 4096;
  for (int blocks_per_sm : {1, 2, 4}) {
    for (int threads : {256, 512}) {
      dim3 grid(nsm * blocks_per_sm);
      // DMMA: 512 flops per warp-instruction
      for (int rep = 0; rep < 2; ++rep) k_dmma<8><<<grid, threads>>>(out, iters / 8, 1.0, 1.0);
      CK(cudaEventRecord(e0));
      k_dmma<8><<<grid, threads>>>(out, iters, 1.0000001, 0.9999999);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      double flops = double(grid.x) * (threads / 32) * iters * 8 * 512.0;
      printf("{\"test\":\"dmma_m8n8k4\",\"blocks_per_sm\":%d,\"threads\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n",
             blocks_per_sm, threads, ms, flops / ms * 1e-9);
      for (int rep = 0; rep < 2; ++rep) k_dfma<8><<<grid, threads>>>(out, iters / 8, 1.0, 1.0);
      CK(cudaEventRecord(e0));
      k_dfma<8><<<grid, threads>>>(out, iters, 0.9999999, 1e-7);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      flops = double(grid.x) * threads * iters * 8 * 2.0;
      printf("{\"test\":\"dfma\",\"blocks_per_sm\":%d,\"threads\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n",
             blocks_per_sm, threads, ms, flops / ms * 1e-9);
    }
  }
  for (int blocks_per_sm : {1, 2}) {
    dim3 grid(nsm * blocks_per_sm);
    const int threads = 256, it2 = 512;
    k_dmma_smem<<<grid, threads>>>(out, it2 / 8);
    CK(cudaEventRecord(e0));
    k_dmma_smem<<<grid, threads>>>(out, it2);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    double flops = double(grid.x) * 8 * it2 * 8 * 16 * 512.0;
    printf("{\"test\":\"dmma_smem_fed_32x32\",\"blocks_per_sm\":%d,\"threads\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n",
           blocks_per_sm, threads, ms, flops / ms * 1e-9);
  }
  printf("{\"sm_count\":%d,\"clock_khz_attr\":%d}\n", nsm, clk);
  CK(cudaGetLastError());
  return 0;
}
