// Do DMMA (mma.sync m8n8k4 f64) and DFMA share one FP64 pipe on B200?
// Runs the two instruction kinds concurrently (same warp interleaved, and
// split across warps of one CTA) and reports the combined FP64 rate.  If the
// sum stays at the single-kind peak (~37 TF/s), the pipe is shared and DFMA
// can only replace padded DMMA work, not add to it.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// every warp: ND dmma chains and NF dfma chains per iteration
template <int ND, int NF>
__global__ void k_mix(double* out, int iters, double a, double b) {
  double c[ND > 0 ? ND : 1][2];
  double f[NF > 0 ? NF : 1];
#pragma unroll
  for (int i = 0; i < (ND > 0 ? ND : 1); ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
#pragma unroll
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) f[i] = threadIdx.x * 1e-3 + i;
  double av = a + threadIdx.x * 1e-9, bv = b - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ND; ++i) dmma(c[i][0], c[i][1], av, bv);
#pragma unroll
    for (int i = 0; i < NF; ++i) f[i] = fma(av, f[i], bv);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < (ND > 0 ? ND : 1); ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) s += f[i];
  if (s == 12345.678) out[0] = s;
}

// warps 0..dw-1 run DMMA, the rest DFMA (iters scaled so both halves finish together if independent)
__global__ void k_split(double* out, int iters_d, int iters_f, int dw, double a, double b) {
  const int warp = threadIdx.x >> 5;
  double av = a + threadIdx.x * 1e-9, bv = b - threadIdx.x * 1e-9;
  double s = 0;
  if (warp < dw) {
    double c[8][2] = {};
    for (int it = 0; it < iters_d; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], av, bv);
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  } else {
    double f[8];
    for (int i = 0; i < 8; ++i) f[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters_f; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = fma(av, f[i], bv);
    for (int i = 0; i < 8; ++i) s += f[i];
  }
  if (s == 12345.678) out[0] = s;
}

template <int ND, int NF>
int run(double* out, int nsm, cudaEvent_t e0, cudaEvent_t e1) {
  const int threads = 256, iters = 4096;
  dim3 grid(nsm * 2);
  k_mix<ND, NF><<<grid, threads>>>(out, iters / 8, 1.0, 1.0);
  CK(cudaEventRecord(e0));
  k_mix<ND, NF><<<grid, threads>>>(out, iters, 1.0000001, 0.9999999);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  const double warps = double(grid.x) * (threads / 32) * iters;
  const double fd = warps * ND * 512.0, ff = warps * NF * 64.0;
  printf("{\"test\":\"mix\",\"dmma_chains\":%d,\"dfma_chains\":%d,\"ms\":%.3f,\"dmma_tflops\":%.2f,\"dfma_tflops\":%.2f,\"total_tflops\":%.2f}\n",
         ND, NF, ms, fd / ms * 1e-9, ff / ms * 1e-9, (fd + ff) / ms * 1e-9);
  return 0;
}

int main() {
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  double* out;
  CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  if (run<8, 0>(out, nsm, e0, e1)) return 1;
  if (run<0, 8>(out, nsm, e0, e1)) return 1;
  if (run<8, 8>(out, nsm, e0, e1)) return 1;
  if (run<8, 16>(out, nsm, e0, e1)) return 1;
  if (run<8, 64>(out, nsm, e0, e1)) return 1;
  if (run<4, 32>(out, nsm, e0, e1)) return 1;
  // split warps: 4 DMMA warps + 4 DFMA warps per CTA, 2 CTAs/SM
  for (int fr : {1, 4, 8}) {
    const int threads = 256, id = 2048, iff = id * fr;
    dim3 grid(nsm * 2);
    k_split<<<grid, threads>>>(out, id / 8, iff / 8, 4, 1.0, 1.0);
    CK(cudaEventRecord(e0));
    k_split<<<grid, threads>>>(out, id, iff, 4, 1.0000001, 0.9999999);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    const double w = double(grid.x) * 4;
    const double fd = w * id * 8 * 512.0, ff = w * iff * 8 * 64.0;
    printf("{\"test\":\"split\",\"dfma_iter_ratio\":%d,\"ms\":%.3f,\"dmma_tflops_if_alone\":%.2f,\"dfma_tflops_if_alone\":%.2f,\"total_tflops\":%.2f}\n",
           fr, ms, fd / ms * 1e-9, ff / ms * 1e-9, (fd + ff) / ms * 1e-9);
  }
  CK(cudaGetLastError());
  return 0;
}
