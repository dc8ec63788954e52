// Dense cutoff solve and I/O kernels.
//   k_todense        HBlockTridiag.to_dense (reference reduction.py:66-75,
//                    hodlr.py:146-155) for the cutoff assembly / export
//   lu_factor/solve  dense LU with partial pivoting (reference oracles.py:20-31,
//                    scipy getrf/getrs semantics: first max pivot, singular if
//                    a U diagonal entry is exactly 0)
//   k_residual       ||A u - f|| / ||f|| from the bands (oracles.py:34-49)
#include "acr_types.cuh"
#include "acr_launch.h"

namespace acr {

// one CTA per (dense block, row chunk); A row-major with leading dim ld
__global__ void k_todense(TreeDev T, const HB* blk, const int* rowblk,
                          const int* colblk, double* A, int ld) {
  const int b = blockIdx.y, n = T.n, bw = T.bw;
  const HB h = blk[b];
  double* Ab = A + (long long)rowblk[b] * n * ld + (long long)colblk[b] * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
       idx < (long long)n * n; idx += (long long)gridDim.x * blockDim.x) {
    int i = (int)(idx / n), j = (int)(idx - (long long)i * n);
    int v = 0;
    double val = 0.0;
    while (true) {
      if (T.isleaf[v]) {
        val = h.leaf[(long long)i * bw + (j - T.lo[v])];
        break;
      }
      int mid = T.mid[v];
      bool ti = i < mid, tj = j < mid;
      if (ti == tj) {
        v = ti ? T.c0[v] : T.c1[v];
        continue;
      }
      int side = ti ? 0 : 1;   // (top,bot) -> off12
      int r = h.rk[v * 2 + side];
      const double* U = h.U + (long long)T.depth[v] * h.R * n;
      const double* V = h.V + (long long)T.depth[v] * h.R * n;
      double s = 0.0;
      for (int c = 0; c < r; ++c) s += U[(long long)c * n + i] * V[(long long)c * n + j];
      val = s;
      break;
    }
    Ab[(long long)i * ld + j] = val;
  }
}

cudaError_t launch_todense(const TreeDev& T, const HB* blk, int nblk,
                           const int* rowblk, const int* colblk, double* A,
                           int ld, cudaStream_t st) {
  if (!nblk) return cudaSuccess;
  int bx = (T.n * T.n + 255) / 256;
  if (bx > 1024) bx = 1024;
  k_todense<<<dim3(bx, nblk), 256, 0, st>>>(T, blk, rowblk, colblk, A, ld);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// blocked right-looking LU, nb = 32, row-major N x N
// ---------------------------------------------------------------------------
static constexpr int LU_NB = 32;
static constexpr int LU_PT = 1024;

__global__ void __launch_bounds__(LU_PT) k_lu_panel(double* A, int N, int j0,
                                                    int jb, int* piv, int* info) {
  __shared__ double bv[LU_PT / 32];
  __shared__ int bi[LU_PT / 32];
  __shared__ int sp;
  __shared__ double spv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int j = j0; j < j0 + jb; ++j) {
    double best = -1.0;
    int bidx = j;
    for (int i = j + tid; i < N; i += LU_PT) {
      double v = fabs(A[(long long)i * N + j]);
      if (v > best) { best = v; bidx = i; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (ov > best || (ov == best && oi < bidx)) { best = ov; bidx = oi; }
    }
    if (lane == 0) { bv[warp] = best; bi[warp] = bidx; }
    __syncthreads();
    if (tid == 0) {
      double b = bv[0];
      int ix = bi[0];
      for (int w = 1; w < LU_PT / 32; ++w)
        if (bv[w] > b || (bv[w] == b && bi[w] < ix)) { b = bv[w]; ix = bi[w]; }
      sp = ix;
      piv[j] = ix;
      spv = A[(long long)ix * N + j];
      if (spv == 0.0 && *info == 0) *info = j + 1;
    }
    __syncthreads();
    const int p = sp;
    if (p != j)
      for (int c = tid; c < N; c += LU_PT) {
        double t = A[(long long)j * N + c];
        A[(long long)j * N + c] = A[(long long)p * N + c];
        A[(long long)p * N + c] = t;
      }
    __syncthreads();
    const double pvv = spv;
    if (pvv != 0.0) {
      const double rinv = 1.0 / pvv;
      for (int i = j + 1 + tid; i < N; i += LU_PT) A[(long long)i * N + j] *= rinv;
    }
    __syncthreads();
    // rank-1 update inside the panel: lane -> column, warp -> row stride
    const int w = j0 + jb - j - 1;
    if (w > 0 && lane < w) {
      const int c = j + 1 + lane;
      const double ajc = A[(long long)j * N + c];
      constexpr int ST = LU_PT / 32;
      int i = j + 1 + warp;
      for (; i + 3 * ST < N; i += 4 * ST) {      // 4 independent rows in flight
        double l0 = A[(long long)i * N + j], l1 = A[(long long)(i + ST) * N + j];
        double l2 = A[(long long)(i + 2 * ST) * N + j], l3 = A[(long long)(i + 3 * ST) * N + j];
        double a0 = A[(long long)i * N + c], a1 = A[(long long)(i + ST) * N + c];
        double a2 = A[(long long)(i + 2 * ST) * N + c], a3 = A[(long long)(i + 3 * ST) * N + c];
        A[(long long)i * N + c] = a0 - l0 * ajc;
        A[(long long)(i + ST) * N + c] = a1 - l1 * ajc;
        A[(long long)(i + 2 * ST) * N + c] = a2 - l2 * ajc;
        A[(long long)(i + 3 * ST) * N + c] = a3 - l3 * ajc;
      }
      for (; i < N; i += ST) A[(long long)i * N + c] -= A[(long long)i * N + j] * ajc;
    }
    __syncthreads();
  }
}

// A12 := L11^{-1} A12 (unit lower), one thread per column, L11 in smem
__global__ void k_lu_trsm(double* A, int N, int j0, int jb) {
  __shared__ double L[LU_NB][LU_NB + 1];
  for (int idx = threadIdx.x; idx < jb * jb; idx += blockDim.x) {
    int i = idx / jb, k = idx - i * jb;
    L[i][k] = A[(long long)(j0 + i) * N + j0 + k];
  }
  __syncthreads();
  int c = j0 + jb + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  double x[LU_NB];
#pragma unroll
  for (int i = 0; i < LU_NB; ++i)
    x[i] = i < jb ? A[(long long)(j0 + i) * N + c] : 0.0;
#pragma unroll
  for (int i = 0; i < LU_NB; ++i) {
    double v = x[i];
#pragma unroll
    for (int k = 0; k < i; ++k) v -= L[i][k] * x[k];
    x[i] = v;
  }
#pragma unroll
  for (int i = 0; i < LU_NB; ++i)
    if (i < jb) A[(long long)(j0 + i) * N + c] = x[i];
}

// A22 -= A21 A12, 64x64 tiles, k = jb <= 32
__global__ void __launch_bounds__(256) k_lu_gemm(double* A, int N, int j0, int jb) {
  __shared__ double sa[64][LU_NB + 1];
  __shared__ double sb[LU_NB][64 + 1];
  const int r0 = j0 + jb + blockIdx.y * 64, c0 = j0 + jb + blockIdx.x * 64;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < 64 * jb; idx += 256) {
    int i = idx / jb, k = idx - i * jb;
    int r = r0 + i;
    sa[i][k] = r < N ? A[(long long)r * N + j0 + k] : 0.0;
  }
  for (int idx = tid; idx < jb * 64; idx += 256) {
    int k = idx / 64, j = idx - k * 64;
    int c = c0 + j;
    sb[k][j] = c < N ? A[(long long)(j0 + k) * N + c] : 0.0;
  }
  __syncthreads();
  const int tx = tid & 15, ty = tid >> 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int k = 0; k < jb; ++k) {
    double av[4], bv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) av[a] = sa[ty + 16 * a][k];
#pragma unroll
    for (int b = 0; b < 4; ++b) bv[b] = sb[k][tx + 16 * b];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] += av[a] * bv[b];
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      int r = r0 + ty + 16 * a, c = c0 + tx + 16 * b;
      if (r < N && c < N) A[(long long)r * N + c] -= acc[a][b];
    }
}

cudaError_t lu_factor(double* A, int N, int* piv, int* info, cudaStream_t st) {
  cudaMemsetAsync(info, 0, sizeof(int), st);
  for (int j0 = 0; j0 < N; j0 += LU_NB) {
    int jb = N - j0 < LU_NB ? N - j0 : LU_NB;
    k_lu_panel<<<1, LU_PT, 0, st>>>(A, N, j0, jb, piv, info);
    int rest = N - j0 - jb;
    if (rest > 0) {
      k_lu_trsm<<<(rest + 63) / 64, 64, 0, st>>>(A, N, j0, jb);
      dim3 g((rest + 63) / 64, (rest + 63) / 64);
      k_lu_gemm<<<g, 256, 0, st>>>(A, N, j0, jb);
    }
  }
  return cudaGetLastError();
}

// solve with B column-major (N x nrhs, ld N), one CTA per column
__global__ void __launch_bounds__(1024) k_lu_solve(const double* A, int N,
                                                   const int* piv, double* B) {
  double* b = B + (long long)blockIdx.x * N;
  const int tid = threadIdx.x;
  if (tid == 0)
    for (int j = 0; j < N; ++j) {
      int p = piv[j];
      if (p != j) { double t = b[j]; b[j] = b[p]; b[p] = t; }
    }
  __syncthreads();
  for (int j = 0; j < N; ++j) {
    double bj = b[j];
    for (int i = j + 1 + tid; i < N; i += blockDim.x) b[i] -= A[(long long)i * N + j] * bj;
    __syncthreads();
  }
  for (int j = N - 1; j >= 0; --j) {
    if (tid == 0) b[j] = b[j] / A[(long long)j * N + j];
    __syncthreads();
    double bj = b[j];
    for (int i = tid; i < j; i += blockDim.x) b[i] -= A[(long long)i * N + j] * bj;
    __syncthreads();
  }
}

cudaError_t lu_solve(const double* A, int N, const int* piv, double* B,
                     int nrhs, cudaStream_t st) {
  if (!nrhs) return cudaSuccess;
  k_lu_solve<<<nrhs, 1024, 0, st>>>(A, N, piv, B);
  return cudaGetLastError();
}

// user RHS (m*n, k) row-major  <->  panels [m][k][n]
__global__ void k_rhs_in(const double* rhs, int N, int k, int n, double* P) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
       idx < (long long)N * k; idx += (long long)gridDim.x * blockDim.x) {
    long long row = idx / k;
    int c = (int)(idx - row * k);
    long long blk = row / n;
    int i = (int)(row - blk * n);
    P[(blk * k + c) * n + i] = rhs[idx];
  }
}

cudaError_t launch_rhs_in(const double* rhs, int N, int k, int n, double* P,
                          cudaStream_t st) {
  long long tot = (long long)N * k;
  int bx = (int)((tot + 255) / 256);
  if (bx > 4096) bx = 4096;
  k_rhs_in<<<bx, 256, 0, st>>>(rhs, N, k, n, P);
  return cudaGetLastError();
}

__global__ void k_u_out(const double* P, int N, int k, int n, double* u) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
       idx < (long long)N * k; idx += (long long)gridDim.x * blockDim.x) {
    long long row = idx / k;
    int c = (int)(idx - row * k);
    long long blk = row / n;
    int i = (int)(row - blk * n);
    u[idx] = P[(blk * k + c) * n + i];
  }
}

cudaError_t launch_u_out(const double* P, int N, int k, int n, double* u,
                         cudaStream_t st) {
  long long tot = (long long)N * k;
  int bx = (int)((tot + 255) / 256);
  if (bx > 4096) bx = 4096;
  k_u_out<<<bx, 256, 0, st>>>(P, N, k, n, u);
  return cudaGetLastError();
}

// partial[(part*k + c)*2 + {0,1}] = sum over this part's rows of r^2 and f^2
__global__ void k_residual(int m, int n, int k, const double* sub,
                           const double* diag, const double* sup, const double* E,
                           const double* F, const double* u, const double* f,
                           double* partial) {
  __shared__ double red[2][8][32];
  const long long N = (long long)m * n;
  const int c = blockIdx.y;
  double sr = 0.0, sf = 0.0;
  for (long long row = blockIdx.x * (long long)blockDim.x + threadIdx.x; row < N;
       row += (long long)gridDim.x * blockDim.x) {
    long long b = row / n;
    int i = (int)(row - b * n);
    double y = diag[row] * u[row * k + c];
    if (i + 1 < n) y += sup[b * (n - 1) + i] * u[(row + 1) * k + c];
    if (i > 0) y += sub[b * (n - 1) + i - 1] * u[(row - 1) * k + c];
    if (b > 0) y += E[(b - 1) * n + i] * u[(row - n) * k + c];
    if (b + 1 < m) y += F[b * n + i] * u[(row + n) * k + c];
    double fv = f[row * k + c];
    double r = y - fv;
    sr += r * r;
    sf += fv * fv;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sr += __shfl_xor_sync(0xffffffffu, sr, o);
    sf += __shfl_xor_sync(0xffffffffu, sf, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { red[0][w][0] = sr; red[1][w][0] = sf; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, bsum = 0.0;
    for (int x = 0; x < (int)(blockDim.x >> 5); ++x) { a += red[0][x][0]; bsum += red[1][x][0]; }
    partial[((long long)blockIdx.x * k + c) * 2] = a;
    partial[((long long)blockIdx.x * k + c) * 2 + 1] = bsum;
  }
}

cudaError_t launch_residual(int m, int n, int k, const double* sub,
                            const double* diag, const double* sup,
                            const double* E, const double* F, const double* u,
                            const double* f, double* partial, int nparts,
                            cudaStream_t st) {
  k_residual<<<dim3(nparts, k), 256, 0, st>>>(m, n, k, sub, diag, sup, E, F, u, f,
                                             partial);
  return cudaGetLastError();
}

}  // namespace acr
