// Partially pivoted adaptive cross approximation on the device, one CTA per
// operator (compression="aca": lowrank.py:65-160 `aca`, called per operator
// by m2l.py:206-214 / 241-255 through aca_plus_svd).
//
// The loop is the reference's, step for step: the pivot-row probe order
// ([next_row] + the first four unused rows), the residual row / column
// updates in cross order with separately rounded products and differences
// (no FMA contraction, as numpy evaluates `trial -= u[c] * v`), first-index
// argmax of |.| with used rows / columns masked, the running Frobenius norm
// estimate and the stopping test inc^2 <= eps^2 * norm^2, the zero-pivot
// stagnation exit and the for-else "full rank reached".  Only the dot
// products' summation order differs from BLAS (it enters the stopping test
// at the 1e-16 level).  The entries come from the device-assembled operator
// stack, which equals the reference's node evaluator (kernels.py:75-93).
// The QR + SVD recompression of aca_plus_svd (lowrank.py:163-184) runs on the
// host from the crosses returned here.
#include "internal.hpp"

namespace cfm {

constexpr int kAcaThreads = 256;
constexpr int kAcaMaxN = 1024;

template <bool C>
struct Num;
template <>
struct Num<false> {
  using T = double;
  static __device__ T load(const double* p, long long i) { return p[i]; }
  static __device__ void store(double* p, long long i, T v) { p[i] = v; }
  static __device__ T mul(T a, T b) { return __dmul_rn(a, b); }
  static __device__ T sub(T a, T b) { return __dsub_rn(a, b); }
  static __device__ T div(T a, T b) { return __ddiv_rn(a, b); }
  static __device__ double absv(T a) { return fabs(a); }
  static __device__ bool nz(T a) { return a != 0.0; }
  static __device__ T conj(T a) { return a; }
  static __device__ double re(T a) { return a; }
  static __device__ T zero() { return 0.0; }
};
template <>
struct Num<true> {
  using T = double2;
  static __device__ T load(const double* p, long long i) { return make_double2(p[2 * i], p[2 * i + 1]); }
  static __device__ void store(double* p, long long i, T v) { p[2 * i] = v.x, p[2 * i + 1] = v.y; }
  static __device__ T mul(T a, T b) {  // numpy: (ac - bd) + (ad + bc) i
    return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                        __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
  }
  static __device__ T sub(T a, T b) { return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y)); }
  static __device__ T div(T a, T b) {  // Smith's algorithm (numpy's complex division)
    if (fabs(b.x) >= fabs(b.y)) {
      const double rat = b.y / b.x, scl = 1.0 / (b.x + b.y * rat);
      return make_double2((a.x + a.y * rat) * scl, (a.y - a.x * rat) * scl);
    }
    const double rat = b.x / b.y, scl = 1.0 / (b.y + b.x * rat);
    return make_double2((a.x * rat + a.y) * scl, (a.y * rat - a.x) * scl);
  }
  static __device__ double absv(T a) { return hypot(a.x, a.y); }
  static __device__ bool nz(T a) { return a.x != 0.0 || a.y != 0.0; }
  static __device__ T conj(T a) { return make_double2(a.x, -a.y); }
  static __device__ double re(T a) { return a.x; }
  static __device__ T zero() { return make_double2(0.0, 0.0); }
};

// block reductions (kAcaThreads threads)
__device__ double block_sum(double v, double* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < kAcaThreads / 32; ++w) s += red[w];
  return s;
}
// first index of the maximum of a (values < 0 never win)
__device__ int block_argmax(double a, int idx, double* redv, int* redi) {
  for (int o = 16; o; o >>= 1) {
    const double b = __shfl_xor_sync(0xffffffffu, a, o);
    const int j = __shfl_xor_sync(0xffffffffu, idx, o);
    if (b > a || (b == a && j < idx)) a = b, idx = j;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) redv[threadIdx.x >> 5] = a, redi[threadIdx.x >> 5] = idx;
  __syncthreads();
  double bv = redv[0];
  int bi = redi[0];
  for (int w = 1; w < kAcaThreads / 32; ++w)
    if (redv[w] > bv || (redv[w] == bv && redi[w] < bi)) bv = redv[w], bi = redi[w];
  return bi;
}

// ops: [T][n][n] (row i = target node); U, V: [T][kmax][n] crosses (V holds
// v, not conj(v)); rank[T]; flag[T]: 1 converged, 0 stagnated (zero pivot /
// zero residual rows before the tolerance), 2 cross cap kmax reached.
template <bool C>
__global__ void __launch_bounds__(kAcaThreads) k_aca(const double* __restrict__ ops, int n, double eps, int kmax,
                                                      double* __restrict__ Ug, double* __restrict__ Vg,
                                                      int* __restrict__ rank_out, int* __restrict__ flag_out) {
  using N = Num<C>;
  using T = typename N::T;
  const int op = blockIdx.x, tid = threadIdx.x;
  const int f = C ? 2 : 1;
  const double* K = ops + (long long)op * n * n * f;
  double* U = Ug + (long long)op * kmax * n * f;
  double* V = Vg + (long long)op * kmax * n * f;
  __shared__ T row[kAcaMaxN], col[kAcaMaxN];
  __shared__ unsigned used_r[kAcaMaxN / 32], used_c[kAcaMaxN / 32];
  __shared__ double redv[kAcaThreads / 32];
  __shared__ int redi[kAcaThreads / 32];
  __shared__ int s_cand[5], s_nc, s_row;
  for (int i = tid; i < kAcaMaxN / 32; i += kAcaThreads) used_r[i] = used_c[i] = 0u;
  __syncthreads();
  auto used = [&](const unsigned* m, int i) { return (m[i >> 5] >> (i & 31)) & 1u; };
  double norm_sq = 0.0;
  int next_row = 0, k = 0, flag = -1;
  const double eps2 = eps * eps;
  for (int it = 0; it < n; ++it) {
    if (k == kmax) {
      flag = 2;
      break;
    }
    // candidate pivot rows: [next_row] + the first 4 unused rows (lowrank.py:103)
    if (tid == 0) {
      int nc = 0;
      s_cand[nc++] = next_row;
      for (int r = 0, m = 0; r < n && m < 4; ++r)
        if (!used(used_r, r)) s_cand[nc++] = r, ++m;
      s_nc = nc;
      s_row = -1;
    }
    __syncthreads();
    for (int ci = 0; ci < s_nc; ++ci) {
      const int cand = s_cand[ci];
      if (used(used_r, cand)) continue;  // uniform
      double mx = 0.0;
      for (int j = tid; j < n; j += kAcaThreads) {
        T tr = N::load(K, (long long)cand * n + j);
        for (int q = 0; q < k; ++q) tr = N::sub(tr, N::mul(N::load(U, (long long)q * n + cand), N::load(V, (long long)q * n + j)));
        row[j] = tr;
        mx = fmax(mx, N::absv(tr));
      }
      for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      __syncthreads();
      if ((tid & 31) == 0) redv[tid >> 5] = mx;
      __syncthreads();
      double bm = 0.0;
      for (int w = 0; w < kAcaThreads / 32; ++w) bm = fmax(bm, redv[w]);
      if (bm > 0.0) {
        if (tid == 0) s_row = cand;
        break;
      }
    }
    __syncthreads();
    if (s_row < 0) {
      flag = k > 0 ? 1 : 0;
      break;
    }
    next_row = s_row;
    if (tid == 0) used_r[next_row >> 5] |= 1u << (next_row & 31);
    // pivot column: argmax |row| over unused columns
    double best = -1.0;
    int bj = 0x7fffffff;
    for (int j = tid; j < n; j += kAcaThreads) {
      const double a = used(used_c, j) ? 0.0 : N::absv(row[j]);
      if (a > best) best = a, bj = j;
    }
    const int j = block_argmax(best, bj, redv, redi);
    const T pivot = row[j];
    if (!N::nz(pivot)) {
      flag = 0;
      break;
    }
    __syncthreads();
    if (tid == 0) used_c[j >> 5] |= 1u << (j & 31);
    // v_new = row / pivot; u_new = K[:, j] - sum_q v_q[j] u_q
    for (int jj = tid; jj < n; jj += kAcaThreads) N::store(V, (long long)k * n + jj, N::div(row[jj], pivot));
    for (int i = tid; i < n; i += kAcaThreads) {
      T c = N::load(K, (long long)i * n + j);
      for (int q = 0; q < k; ++q) c = N::sub(c, N::mul(N::load(V, (long long)q * n + j), N::load(U, (long long)q * n + i)));
      col[i] = c;
      N::store(U, (long long)k * n + i, c);
    }
    __syncthreads();
    // running ||S_k||_F^2 (lowrank.py:131-134)
    double cross_re = 0.0;
    for (int q = 0; q < k; ++q) {
      T du = N::zero(), dv = N::zero();
      for (int i = tid; i < n; i += kAcaThreads) {
        const T a = N::mul(N::conj(N::load(U, (long long)q * n + i)), N::load(U, (long long)k * n + i));
        const T b = N::mul(N::conj(N::load(V, (long long)q * n + i)), N::load(V, (long long)k * n + i));
        if constexpr (C) {
          du.x += a.x, du.y += a.y, dv.x += b.x, dv.y += b.y;
        } else {
          du += a, dv += b;
        }
      }
      if constexpr (C) {
        const double ur = block_sum(du.x, redv), ui = block_sum(du.y, redv);
        const double vr = block_sum(dv.x, redv), vi = block_sum(dv.y, redv);
        cross_re += ur * vr - ui * vi;
      } else {
        const double ur = block_sum(du, redv), vr = block_sum(dv, redv);
        cross_re += ur * vr;
      }
    }
    double uu = 0.0, vv = 0.0;
    for (int i = tid; i < n; i += kAcaThreads) {
      const T a = N::load(U, (long long)k * n + i), b = N::load(V, (long long)k * n + i);
      uu += N::re(N::mul(N::conj(a), a));
      vv += N::re(N::mul(N::conj(b), b));
    }
    uu = block_sum(uu, redv);
    vv = block_sum(vv, redv);
    const double inc_sq = uu * vv;
    norm_sq = fmax(norm_sq + 2.0 * cross_re + inc_sq, 0.0);
    ++k;
    if (inc_sq <= eps2 * norm_sq) {
      flag = 1;
      break;
    }
    // next pivot row: argmax |col| over unused rows
    best = -1.0;
    bj = 0x7fffffff;
    for (int i = tid; i < n; i += kAcaThreads) {
      const double a = used(used_r, i) ? 0.0 : N::absv(col[i]);
      if (a > best) best = a, bj = i;
    }
    next_row = block_argmax(best, bj, redv, redi);
    __syncthreads();
  }
  if (flag < 0) flag = 1;  // for-else: full rank reached
  if (tid == 0) rank_out[op] = k, flag_out[op] = flag;
}

}  // namespace cfm

using namespace cfm;

extern "C" {

int cfm_aca_batch(int device, int n, int data_complex, int n_ops, const double* ops, double eps, int kmax,
                  double* u_out, double* v_out, int* rank_out, int* flag_out, void* stream) {
  return guarded([&] {
    if (n <= 0 || n > kAcaMaxN) throw Error(CFM_ERR_VALUE, "ACA supports 1 <= n <= 1024 nodes");
    if (n_ops < 0 || kmax <= 0) throw Error(CFM_ERR_VALUE, "bad sizes");
    if (!(eps > 0.0 && eps < 1.0)) throw Error(CFM_ERR_VALUE, "accuracy must lie in (0, 1)");
    if (!n_ops) return;
    if (!is_device_ptr(ops) || !is_device_ptr(u_out) || !is_device_ptr(v_out))
      throw Error(CFM_ERR_VALUE, "device pointers required");
    CUDA_CHECK(cudaSetDevice(device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DevBuf d_rank, d_flag;
    d_rank.alloc(size_t(n_ops) * sizeof(int));
    d_flag.alloc(size_t(n_ops) * sizeof(int));
    if (data_complex)
      k_aca<true><<<unsigned(n_ops), kAcaThreads, 0, s>>>(ops, n, eps, kmax, u_out, v_out, d_rank.as<int>(),
                                                          d_flag.as<int>());
    else
      k_aca<false><<<unsigned(n_ops), kAcaThreads, 0, s>>>(ops, n, eps, kmax, u_out, v_out, d_rank.as<int>(),
                                                           d_flag.as<int>());
    CUDA_CHECK(cudaGetLastError());
    CUDA_CHECK(cudaMemcpyAsync(rank_out, d_rank.p, size_t(n_ops) * sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaMemcpyAsync(flag_out, d_flag.p, size_t(n_ops) * sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

}  // extern "C"
