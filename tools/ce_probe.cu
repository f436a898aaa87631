// Does a copy need an SM?  A grid that fills every SM (one CTA per SM with
// ~200 KB of shared memory) spins until a flag written after the copy on a
// second stream arrives (1024 threads x 64 registers fill the register file); if the copy runs as a kernel it cannot start and the
// spinners time out.  nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/ce_probe tools/ce_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

__global__ void __launch_bounds__(1024, 1) spin(const unsigned* flag, int* timed_out) {
  extern __shared__ char sm[];
  sm[threadIdx.x] = 0;
  // keep ~56 registers live so the CTA holds the whole register file
  double r[26];
#pragma unroll
  for (int i = 0; i < 26; ++i) r[i] = (double)(threadIdx.x * (i + 1)) * (double)*(volatile const unsigned*)flag;
  const long long t0 = clock64();
  while (*(volatile const unsigned*)flag == 0u) {
#pragma unroll
    for (int i = 0; i < 26; ++i) r[i] = r[i] * 1.0000001 + 1.0;
    if (clock64() - t0 > 4000000000ll) {  // ~2 s
      if (threadIdx.x == 0) atomicAdd(timed_out, 1);
      break;
    }
  }
  double acc = 0;
#pragma unroll
  for (int i = 0; i < 26; ++i) acc += r[i];
  if (acc == 12345.0) sm[0] = 1;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t rows = 262144, n = 125, ld = 128;
  double *src, *dst, *hsrc;
  cudaMalloc(&src, rows * n * 8);
  cudaMalloc(&dst, rows * ld * 8);
  cudaMallocHost(&hsrc, rows * n * 8);
  unsigned* flag;
  int* to;
  cudaMalloc(&flag, 4);
  cudaMalloc(&to, 4);
  cudaStream_t a, b;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  const int smem = 227 * 1024;
  cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"memcpy2D D2D pitched", "memcpy 1D D2D", "memcpy2D H2D pitched", "memcpy 1D H2D"};
  for (int mode = 0; mode < 4; ++mode) {
    cudaMemset(flag, 0, 4);
    cudaMemset(to, 0, 4);
    cudaDeviceSynchronize();
    spin<<<nsm, 1024, smem, a>>>(flag, to);  // every thread slot and all shared memory of each SM
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, b);
    if (mode == 0) cudaMemcpy2DAsync(dst, ld * 8, src, n * 8, n * 8, rows, cudaMemcpyDeviceToDevice, b);
    if (mode == 1) cudaMemcpyAsync(dst, src, rows * n * 8, cudaMemcpyDeviceToDevice, b);
    if (mode == 2) cudaMemcpy2DAsync(dst, ld * 8, hsrc, n * 8, n * 8, rows, cudaMemcpyHostToDevice, b);
    if (mode == 3) cudaMemcpyAsync(dst, hsrc, rows * n * 8, cudaMemcpyHostToDevice, b);
    cudaEventRecord(e1, b);
    cuStreamWriteValue32(reinterpret_cast<CUstream>(b), reinterpret_cast<CUdeviceptr>(flag), 1, 0);
    cudaError_t err = cudaDeviceSynchronize();
    int h_to = 0;
    cudaMemcpy(&h_to, to, 4, cudaMemcpyDeviceToHost);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-24s spinners timed out: %d of %d  copy %.3f ms (%.1f GB/s)  %s\n", names[mode], h_to, nsm, ms,
           rows * n * 8 / (ms * 1e6), cudaGetErrorString(err));
  }
  return 0;
}
