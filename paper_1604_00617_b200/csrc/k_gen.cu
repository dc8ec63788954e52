// On-device problem generators for the BASELINE configurations (SURVEY.md
// 8(f) row 1; formulas of 8(d), emitted in the reference's input format,
// reference problems.py:88-133).
//
//   k_gen_const    constant five-point stencils (configs 1, 3, 4): every band
//                  is one value computed on the host exactly as numpy does.
//   k_gen_field /  configs 2 and 5: a(x, y) = exp(sum_k c_k cos(2 pi (p_k x +
//   k_gen_varcoef  q_k y) + phi_k)) on the (n+2)^2 nodes including the boundary
//                  ring, harmonic-mean faces, finite-volume bands.  Every
//                  product / sum is rounded as numpy evaluates it (no FMA
//                  contraction); cos and exp are CUDA's (<= 2 ulp), so bands
//                  agree with the numpy generator to a few ulp.
//   k_gen_uniform  Uniform[low, high) draws of numpy's default Generator
//                  (PCG64, XSL-RR 128/64, next_double = (x >> 11) 2^-53) from a
//                  given 128-bit state and increment: each thread jumps ahead
//                  (LCG advance, O(log k)) to its first draw, so the stream is
//                  bitwise numpy's.  Draw d of a (k, N) sample lands in
//                  out[(d % N) * k + d / N] (the transposed N x k layout).
#include <cuda_runtime.h>

#include "acr_launch.h"

namespace acr {

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

__device__ __forceinline__ u128 pcg_advance(u128 st, u128 inc, unsigned long long delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta) {
    if (delta & 1ull) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * st + acc_plus;
}

__device__ __forceinline__ unsigned long long pcg_next(u128& st, u128 inc) {
  st = st * pcg_mult() + inc;
  const unsigned long long hi = (unsigned long long)(st >> 64), lo = (unsigned long long)st;
  const unsigned rot = (unsigned)(st >> 122);
  const unsigned long long x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

static constexpr int GEN_PER = 64;   // draws per thread

__global__ void k_gen_uniform(unsigned long long st_hi, unsigned long long st_lo,
                              unsigned long long inc_hi, unsigned long long inc_lo,
                              long long N, int k, double low, double range, double* out) {
  const long long total = N * (long long)k;
  const long long d0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * GEN_PER;
  if (d0 >= total) return;
  const u128 inc = ((u128)inc_hi << 64) | inc_lo;
  u128 st = pcg_advance(((u128)st_hi << 64) | st_lo, inc, (unsigned long long)d0);
  const long long d1 = d0 + GEN_PER < total ? d0 + GEN_PER : total;
  for (long long d = d0; d < d1; ++d) {
    const unsigned long long x = pcg_next(st, inc);
    const double u = (double)(x >> 11) * (1.0 / 9007199254740992.0);
    const long long col = d / N, row = d - col * N;
    out[row * k + col] = __dadd_rn(low, __dmul_rn(range, u));
  }
}

__global__ void k_gen_const(int m, int n, double sub, double diag, double sup, double e,
                            double f, double* D_sub, double* D_diag, double* D_sup, double* E,
                            double* F) {
  const long long tot = (long long)m * n;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(idx / n), i = (int)(idx - (long long)j * n);
    D_diag[idx] = diag;
    if (i < n - 1) {
      D_sub[(long long)j * (n - 1) + i] = sub;
      D_sup[(long long)j * (n - 1) + i] = sup;
    }
    if (j < m - 1) {
      E[idx] = e;
      F[idx] = f;
    }
  }
}

// a on the (n+2)^2 nodes, row y (grid line), column x; t_i = i h
__global__ void k_gen_field(int n, GenField P, double* a) {
  const int w = n + 2;
  const long long tot = (long long)w * w;
  const double h = 1.0 / (n + 1);
  const double two_pi = 6.283185307179586;   // 2.0 * np.pi
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    const int y = (int)(idx / w), x = (int)(idx - (long long)y * w);
    const double X = __dmul_rn((double)x, h), Y = __dmul_rn((double)y, h);
    double expo = 0.0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const double arg = __dadd_rn(
          __dmul_rn(two_pi, __dadd_rn(__dmul_rn((double)P.p[t], X), __dmul_rn((double)P.q[t], Y))),
          P.phi[t]);
      expo = __dadd_rn(expo, __dmul_rn(P.c[t], cos(arg)));
    }
    a[idx] = exp(expo);
  }
}

__device__ __forceinline__ double gen_hmean(double p, double q) {
  return __ddiv_rn(__dmul_rn(__dmul_rn(2.0, p), q), __dadd_rn(p, q));
}

__global__ void k_gen_varcoef(int n, const double* __restrict__ a, double* D_sub, double* D_diag,
                              double* D_sup, double* E, double* F) {
  const int w = n + 2;
  const double h = 1.0 / (n + 1);
  const double h2 = __dmul_rn(h, h);
  const long long tot = (long long)n * n;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(idx / n), i = (int)(idx - (long long)j * n);
    // node (i, j) of the interior is a[j + 1][i + 1]
    const double* r0 = a + (long long)j * w;         // line j - 1
    const double* r1 = r0 + w;                       // line j
    const double* r2 = r1 + w;                       // line j + 1
    const double aW = gen_hmean(r1[i], r1[i + 1]);
    const double aE = gen_hmean(r1[i + 1], r1[i + 2]);
    const double aS = gen_hmean(r0[i + 1], r1[i + 1]);
    const double aN = gen_hmean(r1[i + 1], r2[i + 1]);
    D_diag[idx] = __ddiv_rn(__dadd_rn(__dadd_rn(__dadd_rn(aW, aE), aS), aN), h2);
    if (i < n - 1) D_sup[(long long)j * (n - 1) + i] = __ddiv_rn(-aE, h2);
    if (i > 0) D_sub[(long long)j * (n - 1) + i - 1] = __ddiv_rn(-aW, h2);
    if (j < n - 1) F[idx] = __ddiv_rn(-aN, h2);
    if (j > 0) E[idx - n] = __ddiv_rn(-aS, h2);
  }
}

static int gen_grid(long long tot) {
  long long b = (tot + 255) / 256;
  return (int)(b < 148LL * 64 ? (b < 1 ? 1 : b) : 148LL * 64);
}

cudaError_t launch_gen_const(int m, int n, const double* v, double* D_sub, double* D_diag,
                             double* D_sup, double* E, double* F, cudaStream_t st) {
  k_gen_const<<<gen_grid((long long)m * n), 256, 0, st>>>(m, n, v[0], v[1], v[2], v[3], v[4],
                                                         D_sub, D_diag, D_sup, E, F);
  return cudaGetLastError();
}

cudaError_t launch_gen_varcoef(int n, const GenField& P, double* work, double* D_sub,
                               double* D_diag, double* D_sup, double* E, double* F,
                               cudaStream_t st) {
  const long long w = n + 2;
  k_gen_field<<<gen_grid(w * w), 256, 0, st>>>(n, P, work);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_gen_varcoef<<<gen_grid((long long)n * n), 256, 0, st>>>(n, work, D_sub, D_diag, D_sup, E,
                                                            F);
  return cudaGetLastError();
}

cudaError_t launch_gen_uniform(const unsigned long long* state, long long N, int k, double low,
                               double high, double* out, cudaStream_t st) {
  const long long total = N * (long long)k;
  if (total <= 0) return cudaSuccess;
  const long long threads = (total + GEN_PER - 1) / GEN_PER;
  const int blocks = (int)((threads + 255) / 256);
  k_gen_uniform<<<blocks, 256, 0, st>>>(state[0], state[1], state[2], state[3], N, k, low,
                                        high - low, out);
  return cudaGetLastError();
}

}  // namespace acr
