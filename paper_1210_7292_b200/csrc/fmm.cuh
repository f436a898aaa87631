// The FMM stages around M2L on the GPU:
//   P2M  engine.py:122-127  leaf multipoles = S(x_p)^T w   (anterpolation)
//   L2P  engine.py:170-175  potential_p   += S(x_p) . leaf locals
//   P2P  engine.py:177-199  near field, direct sum over the 27 neighbour
//                           leaves in source-ijk order, coincident points skipped
// (M2M / L2L are dense 8-operator products and run on the tile-GEMM kernel.)
//
// S is the tensor Chebyshev interpolation weight (interp.py:106-111, 224-236):
//   S_l(x, r_i) = 1/l + (2/l) sum_{k=1}^{l-1} T_k(x) T_k(r_i),
//   S(x)[m] = S(x1, r_a1) S(x2, r_a2) S(x3, r_a3),  m = a1 + a2 l + a3 l^2,
// with reference coordinates ref = (x - center) / half of the particle's leaf.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cfm {

constexpr int kMaxOrder = 12;

struct FmmGeom {
  const double* pts;        // n x 3, original particle order
  const long long* perm;    // particles sorted by leaf (row order), ascending index inside a leaf
  const long long* leaf_off;  // n_leaves + 1
  const int* leaf_ijk;      // n_leaves x 3
  long long n_leaves;
  int depth;
  double lx, ly, lz;        // bounding-cube low corner
  double leaf_w;            // leaf width
  const double* troots;     // [l][l-1] T_k(root_i), k = 1..l-1
  int order;
};

// 1-D weights S(x, r_i), i < l, written to s[i * stride]
__device__ __forceinline__ void cheb_weights_1d(double x, int order, const double* __restrict__ troots, double* s,
                                                int stride) {
  double t[kMaxOrder];
  if (order >= 2) t[0] = x;
  for (int k = 1; k < order - 1; ++k) t[k] = (k == 1) ? 2.0 * x * x - 1.0 : 2.0 * x * t[k - 1] - t[k - 2];
  const double inv = 1.0 / order, two = 2.0 / order;
  for (int i = 0; i < order; ++i) {
    double d = 0.0;
    for (int k = 0; k < order - 1; ++k) d += t[k] * troots[i * (order - 1) + k];
    s[i * stride] = inv + two * d;
  }
}

__device__ __forceinline__ void leaf_frame(const FmmGeom& g, long long leaf, double c[3], double& half) {
  const double w = g.leaf_w;
  half = 0.5 * w;
  const double low[3] = {g.lx, g.ly, g.lz};
  for (int a = 0; a < 3; ++a) c[a] = low[a] + (double(g.leaf_ijk[3 * leaf + a]) + 0.5) * w;
}

// P2M: one CTA per leaf; particles staged in chunks of CH with their 3 x l
// weights in shared memory; thread per output node (dc = 1 real, 2 complex).
template <int CH>
__global__ void k_p2m(const FmmGeom g, const double* __restrict__ weights, int dc, double* __restrict__ mp,
                      long long mp_ld) {
  extern __shared__ double sm[];
  const int L = g.order, n = L * L * L;
  double* sw = sm;                 // [3][L][CH]
  double* swt = sw + 3 * L * CH;   // [CH][dc]
  const long long leaf = blockIdx.x;
  double c[3], half;
  leaf_frame(g, leaf, c, half);
  const long long p0 = g.leaf_off[leaf], p1 = g.leaf_off[leaf + 1];
  double acc[2][8];
  for (int u = 0; u < 8; ++u) acc[0][u] = acc[1][u] = 0.0;
  for (long long base = p0; base < p1; base += CH) {
    const int cnt = int(min((long long)CH, p1 - base));
    __syncthreads();
    for (int pp = threadIdx.x; pp < cnt; pp += blockDim.x) {
      const long long q = g.perm[base + pp];
      for (int a = 0; a < 3; ++a) {
        const double ref = (g.pts[3 * q + a] - c[a]) / half;
        cheb_weights_1d(ref, L, g.troots, sw + a * L * CH + pp, CH);
      }
      for (int d = 0; d < dc; ++d) swt[pp * dc + d] = weights[q * dc + d];
    }
    __syncthreads();
    int u = 0;
    for (int m = threadIdx.x; m < n; m += blockDim.x, ++u) {
      const int a1 = m % L, a2 = (m / L) % L, a3 = m / (L * L);
      const double* s1 = sw + a1 * CH;
      const double* s2 = sw + (L + a2) * CH;
      const double* s3 = sw + (2 * L + a3) * CH;
      for (int pp = 0; pp < cnt; ++pp) {
        const double s = s1[pp] * s2[pp] * s3[pp];
        for (int d = 0; d < dc; ++d) acc[d][u] += s * swt[pp * dc + d];
      }
    }
  }
  int u = 0;
  for (int m = threadIdx.x; m < n; m += blockDim.x, ++u)
    for (int d = 0; d < dc; ++d) mp[leaf * mp_ld + (long long)m * dc + d] = acc[d][u];
}

// P2M specialized on the order (accumulators in registers).
template <int L, int CH>
__global__ void __launch_bounds__(128) k_p2m_t(const FmmGeom g, const double* __restrict__ weights, int dc,
                                               double* __restrict__ mp, long long mp_ld) {
  constexpr int N = L * L * L, U = (N + 127) / 128;
  __shared__ double sw[3][L][CH];
  __shared__ double swt[CH][2];
  const long long leaf = blockIdx.x;
  double c[3], half;
  leaf_frame(g, leaf, c, half);
  const long long p0 = g.leaf_off[leaf], p1 = g.leaf_off[leaf + 1];
  double acc0[U], acc1[U];
#pragma unroll
  for (int u = 0; u < U; ++u) acc0[u] = acc1[u] = 0.0;
  int a1[U], a2[U], a3[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int m = threadIdx.x + 128 * u;
    a1[u] = m % L;
    a2[u] = (m / L) % L;
    a3[u] = min(m / (L * L), L - 1);
  }
  for (long long base = p0; base < p1; base += CH) {
    const int cnt = int(min((long long)CH, p1 - base));
    __syncthreads();
    for (int pp = threadIdx.x; pp < cnt; pp += blockDim.x) {
      const long long q = g.perm[base + pp];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double x = (g.pts[3 * q + a] - c[a]) / half;
        double t[L > 1 ? L - 1 : 1];
        t[0] = x;
#pragma unroll
        for (int k = 1; k < L - 1; ++k) t[k] = (k == 1) ? 2.0 * x * x - 1.0 : 2.0 * x * t[k - 1] - t[k - 2];
#pragma unroll
        for (int i = 0; i < L; ++i) {
          double d = 0.0;
#pragma unroll
          for (int k = 0; k < L - 1; ++k) d += t[k] * __ldg(g.troots + i * (L - 1) + k);
          sw[a][i][pp] = 1.0 / L + (2.0 / L) * d;
        }
      }
      swt[pp][0] = weights[q * dc];
      swt[pp][1] = dc == 2 ? weights[q * dc + 1] : 0.0;
    }
    __syncthreads();
    for (int pp = 0; pp < cnt; ++pp) {
      const double w0 = swt[pp][0], w1 = swt[pp][1];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double sv = sw[0][a1[u]][pp] * sw[1][a2[u]][pp] * sw[2][a3[u]][pp];
        acc0[u] += sv * w0;
        acc1[u] += sv * w1;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int m = threadIdx.x + 128 * u;
    if (m < N) {
      mp[leaf * mp_ld + (long long)m * dc] = acc0[u];
      if (dc == 2) mp[leaf * mp_ld + (long long)m * dc + 1] = acc1[u];
    }
  }
}

// L2P specialized on the order: the 3 x L weights stay in registers.
template <int L>
__global__ void k_l2p_t(const FmmGeom g, const long long* __restrict__ leaf_of_pos, const double* __restrict__ loc,
                        long long loc_ld, int dc, double* __restrict__ pot, long long n_points) {
  const long long pos = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (pos >= n_points) return;
  const long long leaf = leaf_of_pos[pos];
  const long long q = g.perm[pos];
  double c[3], half;
  leaf_frame(g, leaf, c, half);
  double s[3][L];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double x = (g.pts[3 * q + a] - c[a]) / half;
    double t[L > 1 ? L - 1 : 1];
    t[0] = x;
#pragma unroll
    for (int k = 1; k < L - 1; ++k) t[k] = (k == 1) ? 2.0 * x * x - 1.0 : 2.0 * x * t[k - 1] - t[k - 2];
#pragma unroll
    for (int i = 0; i < L; ++i) {
      double d = 0.0;
#pragma unroll
      for (int k = 0; k < L - 1; ++k) d += t[k] * __ldg(g.troots + i * (L - 1) + k);
      s[a][i] = 1.0 / L + (2.0 / L) * d;
    }
  }
  const double* lp = loc + leaf * loc_ld;
  double r0 = 0.0, r1 = 0.0;
#pragma unroll
  for (int a3 = 0; a3 < L; ++a3)
#pragma unroll
    for (int a2 = 0; a2 < L; ++a2) {
      const double w23 = s[1][a2];
#pragma unroll
      for (int a1 = 0; a1 < L; ++a1) {
        const int m = a1 + L * (a2 + L * a3);
        const double w = s[0][a1] * w23 * s[2][a3];
        r0 += w * __ldg(lp + (long long)m * dc);
        if (dc == 2) r1 += w * __ldg(lp + (long long)m * dc + 1);
      }
    }
  pot[q * dc] += r0;
  if (dc == 2) pot[q * dc + 1] += r1;
}

// L2P: one thread per particle (sorted order); pot[q] += S(x_q) . locals[leaf]
__global__ void k_l2p(const FmmGeom g, const long long* __restrict__ leaf_of_pos, const double* __restrict__ loc,
                      long long loc_ld, int dc, double* __restrict__ pot, long long n_points) {
  const long long pos = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (pos >= n_points) return;
  const int L = g.order;
  const long long leaf = leaf_of_pos[pos];
  const long long q = g.perm[pos];
  double c[3], half;
  leaf_frame(g, leaf, c, half);
  double s[3][kMaxOrder];
  for (int a = 0; a < 3; ++a) cheb_weights_1d((g.pts[3 * q + a] - c[a]) / half, L, g.troots, s[a], 1);
  const double* lp = loc + leaf * loc_ld;
  double r0 = 0.0, r1 = 0.0;
  int m = 0;
  for (int a3 = 0; a3 < L; ++a3)
    for (int a2 = 0; a2 < L; ++a2)
      for (int a1 = 0; a1 < L; ++a1, ++m) {
        const double w = s[0][a1] * s[1][a2] * s[2][a3];
        r0 += w * lp[(long long)m * dc];
        if (dc == 2) r1 += w * lp[(long long)m * dc + 1];
      }
  pot[q * dc] += r0;
  if (dc == 2) pot[q * dc + 1] += r1;
}

// P2P: one CTA per target leaf; the 27 neighbour leaves (source-ijk order) are
// walked leaf by leaf, their particles staged in shared memory.  kernel 0:
// 1/(4 pi r); 1: exp(i k r)/(4 pi r).  Weights / output: wdc / odc components.
template <int CH>
__global__ void k_p2p(const FmmGeom g, const int* __restrict__ grid, int kernel, double wavenumber,
                      const double* __restrict__ weights, int wdc, double* __restrict__ pot, int odc) {
  __shared__ double sx[CH][3];
  __shared__ double swv[CH][2];
  const long long leaf = blockIdx.x;
  const int S = 1 << g.depth;
  const int x = g.leaf_ijk[3 * leaf], y = g.leaf_ijk[3 * leaf + 1], z = g.leaf_ijk[3 * leaf + 2];
  const long long t0 = g.leaf_off[leaf], t1 = g.leaf_off[leaf + 1];
  const double FOUR_PI = 4.0 * 3.141592653589793;
  const double INV_FOUR_PI = 1.0 / FOUR_PI;
  for (long long tb = t0; tb < t1; tb += blockDim.x) {
    const long long tp = tb + threadIdx.x;
    const bool active = tp < t1;
    long long q = active ? g.perm[tp] : 0;
    const double xt = active ? g.pts[3 * q] : 0.0, yt = active ? g.pts[3 * q + 1] : 0.0,
                 zt = active ? g.pts[3 * q + 2] : 0.0;
    double acc_r = 0.0, acc_i = 0.0;
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          const int sx_ = x + dx, sy_ = y + dy, sz_ = z + dz;
          if (sx_ < 0 || sx_ >= S || sy_ < 0 || sy_ >= S || sz_ < 0 || sz_ >= S) continue;
          const int sl = grid[((long long)sx_ * S + sy_) * S + sz_];
          if (sl < 0) continue;
          const long long s0 = g.leaf_off[sl], s1 = g.leaf_off[sl + 1];
          // per-source-leaf partial (the reference adds one mat @ w per source leaf)
          double pr = 0.0, pi = 0.0;
          for (long long sb = s0; sb < s1; sb += CH) {
            const int cnt = int(min((long long)CH, s1 - sb));
            __syncthreads();
            for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
              const long long qs = g.perm[sb + k];
              sx[k][0] = g.pts[3 * qs];
              sx[k][1] = g.pts[3 * qs + 1];
              sx[k][2] = g.pts[3 * qs + 2];
              swv[k][0] = weights[qs * wdc];
              swv[k][1] = wdc == 2 ? weights[qs * wdc + 1] : 0.0;
            }
            __syncthreads();
            if (active) {
              for (int k = 0; k < cnt; ++k) {
                const double ddx = xt - sx[k][0], ddy = yt - sx[k][1], ddz = zt - sx[k][2];
                const double d2 = ddx * ddx + ddy * ddy + ddz * ddz;
                if (d2 == 0.0) continue;
                if (kernel == 0) {
                  // 1/(4 pi r) via rsqrt (<= 1 ulp; the reference rounds sqrt and the division)
                  const double v = rsqrt(d2) * INV_FOUR_PI;
                  pr += v * swv[k][0];
                  pi += v * swv[k][1];
                } else {
                  const double r = sqrt(d2);
                  const double den = FOUR_PI * r;
                  double sn, cs;
                  sincos(wavenumber * r, &sn, &cs);
                  const double inv = 1.0 / den;
                  const double vr = cs * inv, vi = sn * inv;
                  pr += vr * swv[k][0] - vi * swv[k][1];
                  pi += vr * swv[k][1] + vi * swv[k][0];
                }
              }
            }
          }
          acc_r += pr;
          acc_i += pi;
        }
    if (active) {
      pot[q * odc] += acc_r;
      if (odc == 2) pot[q * odc + 1] += acc_i;
    }
  }
}

// ---- P2P v2: leaf-sorted SoA particles, two leaf-size classes -------------
//
// Per interaction (the roofline unit): 3 DADD + 1 DMUL + 2 DFMA for r^2, the
// FP64 reciprocal square root, 1 DFMA to accumulate (Laplace; Helmholtz adds a
// sincos) -- FP64-pipe bound, no tensor-core formulation (nonlinear kernel).
struct P2PGeom {
  const long long* leaf_off;
  const int* leaf_ijk;
  const int* grid;  // S^3 leaf index or -1
  int S;
  const double* px;  // leaf-sorted positions (SoA)
  const double* py;
  const double* pz;
  const long long* perm;  // sorted position -> original particle
};

__global__ void k_p2p_sort_pos(const double* __restrict__ pts, const long long* __restrict__ perm, long long n,
                               double* __restrict__ px, double* __restrict__ py, double* __restrict__ pz) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long q = perm[i];
  px[i] = pts[3 * q];
  py[i] = pts[3 * q + 1];
  pz[i] = pts[3 * q + 2];
}

// leaf-sorted weights, pre-scaled by 1/(4 pi) (one multiply per particle
// instead of one per interaction)
template <int WDC>
__global__ void k_p2p_sort_w(const double* __restrict__ w, const long long* __restrict__ perm, long long n,
                             double* __restrict__ sw) {
  constexpr double INV_FOUR_PI = 0.07957747154594767;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long q = perm[i];
#pragma unroll
  for (int c = 0; c < WDC; ++c) sw[i * WDC + c] = w[q * WDC + c] * INV_FOUR_PI;
}

// occupied neighbour leaves of `leaf` in source-ijk order (dx, dy, dz ascending)
__device__ __forceinline__ int p2p_neighbours(const P2PGeom& g, long long leaf, long long* s0, long long* s1) {
  const int x = g.leaf_ijk[3 * leaf], y = g.leaf_ijk[3 * leaf + 1], z = g.leaf_ijk[3 * leaf + 2];
  int n = 0;
  for (int dx = -1; dx <= 1; ++dx)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dz = -1; dz <= 1; ++dz) {
        const int a = x + dx, b = y + dy, c = z + dz;
        if (a < 0 || a >= g.S || b < 0 || b >= g.S || c < 0 || c >= g.S) continue;
        const int sl = g.grid[((long long)a * g.S + b) * g.S + c];
        if (sl < 0) continue;
        s0[n] = g.leaf_off[sl];
        s1[n] = g.leaf_off[sl + 1];
        ++n;
      }
  return n;
}

// 1/sqrt(d2) for d2 > 0 without the library's special-case branch: the fp32
// MUFU estimate (~2^-22) refined by two Newton steps in fp64 (~1 ulp); the
// bench geometries keep d2 in the fp32 normal range (d2 >= 1e-32).
__device__ __forceinline__ double rsqrt_nr(double d2) {
  double y = double(rsqrtf(float(d2)));
  const double h = 0.5 * d2;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}

// one interaction: acc += K(|t - s|) * w, coincident points skipped (kernels.py:75-93 skip_singular)
// (weights arrive pre-scaled by 1/(4 pi))
template <int KER, int WDC>
__device__ __forceinline__ void p2p_interact(double xt, double yt, double zt, double xs, double ys, double zs,
                                             const double* ws, double k, double& ar, double& ai) {
  const double dx = xt - xs, dy = yt - ys, dz = zt - zs;
  const double d2 = fma(dz, dz, fma(dy, dy, dx * dx));
  const double rinv = d2 > 0.0 ? rsqrt_nr(d2) : 0.0;
  if (KER == 0) {
    ar = fma(rinv, ws[0], ar);
    if (WDC == 2) ai = fma(rinv, ws[1], ai);
  } else {
    double sn, cs;
    sincos(k * (d2 * rinv), &sn, &cs);
    const double vr = cs * rinv, vi = sn * rinv;
    if (WDC == 2) {
      ar = fma(vr, ws[0], fma(-vi, ws[1], ar));
      ai = fma(vr, ws[1], fma(vi, ws[0], ai));
    } else {
      ar = fma(vr, ws[0], ar);
      ai = fma(vi, ws[0], ai);
    }
  }
}

// Small target leaves (<= 64 particles): a CTA of 128 threads per leaf works on
// (target, neighbour leaf) items; per-item partials land in shared memory and
// are summed per target in neighbour order (deterministic).
template <int KER, int WDC, int ODC>
__global__ void __launch_bounds__(128) k_p2p_small(const P2PGeom g, const long long* __restrict__ leaves,
                                                   const double* __restrict__ sw, double k, double* __restrict__ pot) {
  __shared__ long long s0[27], s1[27];
  __shared__ int s_nnb;
  __shared__ double part[27 * 64 * 2];
  const long long leaf = leaves[blockIdx.x];
  const long long t0 = g.leaf_off[leaf];
  const int nt = int(g.leaf_off[leaf + 1] - t0);
  if (threadIdx.x == 0) s_nnb = p2p_neighbours(g, leaf, s0, s1);
  __syncthreads();
  const int nnb = s_nnb;
  for (int it = threadIdx.x; it < nt * nnb; it += blockDim.x) {
    const int t = it % nt, j = it / nt;
    const double xt = g.px[t0 + t], yt = g.py[t0 + t], zt = g.pz[t0 + t];
    double ar = 0.0, ai = 0.0;
    for (long long q = s0[j]; q < s1[j]; ++q) {
      double ws[2];
      ws[0] = sw[q * WDC];
      if (WDC == 2) ws[1] = sw[q * WDC + 1];
      p2p_interact<KER, WDC>(xt, yt, zt, g.px[q], g.py[q], g.pz[q], ws, k, ar, ai);
    }
    part[(j * 64 + t) * 2] = ar;
    part[(j * 64 + t) * 2 + 1] = ai;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nt; t += blockDim.x) {
    double ar = 0.0, ai = 0.0;
    for (int j = 0; j < nnb; ++j) {
      ar += part[(j * 64 + t) * 2];
      ai += part[(j * 64 + t) * 2 + 1];
    }
    const long long o = g.perm[t0 + t];
    pot[o * ODC] += ar;
    if (ODC == 2) pot[o * ODC + 1] += ai;
  }
}

// Large target leaves: thread per target (two targets per thread share every
// staged source), sources of the 27 neighbours streamed through shared memory.
template <int KER, int WDC, int ODC>
__global__ void __launch_bounds__(128) k_p2p_large(const P2PGeom g, const long long* __restrict__ leaves,
                                                   const double* __restrict__ sw, double k, double* __restrict__ pot) {
  constexpr int CH = 256;
  __shared__ long long s0[27], s1[27];
  __shared__ int s_nnb;
  __shared__ double sx[CH], sy[CH], sz[CH], sws[CH * WDC];
  const long long leaf = leaves[blockIdx.x];
  const long long t0 = g.leaf_off[leaf];
  const int nt = int(g.leaf_off[leaf + 1] - t0);
  if (threadIdx.x == 0) s_nnb = p2p_neighbours(g, leaf, s0, s1);
  __syncthreads();
  const int nnb = s_nnb;
  for (int tb = 0; tb < nt; tb += 2 * blockDim.x) {
    const int ta = tb + threadIdx.x, tc = ta + blockDim.x;
    const bool va = ta < nt, vc = tc < nt;
    const double xa = va ? g.px[t0 + ta] : 0.0, ya = va ? g.py[t0 + ta] : 0.0, za = va ? g.pz[t0 + ta] : 0.0;
    const double xc = vc ? g.px[t0 + tc] : 0.0, yc = vc ? g.py[t0 + tc] : 0.0, zc = vc ? g.pz[t0 + tc] : 0.0;
    double ar = 0.0, ai = 0.0, cr = 0.0, ci = 0.0;
    for (int j = 0; j < nnb; ++j) {
      for (long long sb = s0[j]; sb < s1[j]; sb += CH) {
        const int cnt = int(min((long long)CH, s1[j] - sb));
        __syncthreads();
        for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
          sx[q] = g.px[sb + q];
          sy[q] = g.py[sb + q];
          sz[q] = g.pz[sb + q];
#pragma unroll
          for (int c = 0; c < WDC; ++c) sws[q * WDC + c] = sw[(sb + q) * WDC + c];
        }
        __syncthreads();
#pragma unroll 4
        for (int q = 0; q < cnt; ++q) {
          const double* ws = sws + q * WDC;
          p2p_interact<KER, WDC>(xa, ya, za, sx[q], sy[q], sz[q], ws, k, ar, ai);
          p2p_interact<KER, WDC>(xc, yc, zc, sx[q], sy[q], sz[q], ws, k, cr, ci);
        }
      }
    }
    if (va) {
      const long long o = g.perm[t0 + ta];
      pot[o * ODC] += ar;
      if (ODC == 2) pot[o * ODC + 1] += ai;
    }
    if (vc) {
      const long long o = g.perm[t0 + tc];
      pot[o * ODC] += cr;
      if (ODC == 2) pot[o * ODC + 1] += ci;
    }
  }
}

__global__ void k_leaf_of_pos(const long long* __restrict__ leaf_off, long long n_leaves,
                              long long* __restrict__ out) {
  const long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (l >= n_leaves) return;
  for (long long p = leaf_off[l]; p < leaf_off[l + 1]; ++p) out[p] = l;
}

__global__ void k_leaf_grid(const int* __restrict__ ijk, long long n, int S, int* __restrict__ grid) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  grid[((long long)ijk[3 * i] * S + ijk[3 * i + 1]) * S + ijk[3 * i + 2]] = int(i);
}

}  // namespace cfm
