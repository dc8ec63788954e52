// HODLR x panel products over subtrees (reference algebra.py:52-83,
// hodlr.py:89-99) and the small "panel x (panel^T panel)" products of
// invert / multiply (algebra.py:152-156, 214-225).
//
// hmat, phase A: for every branch node beta below a subtree root mu and both
//   sides, t = V^T X[rows V]  (trans: U^T X[rows U])      -> tbuf
// hmat, phase B: per leaf lambda below mu,
//   Y[rows lambda] = L X[rows lambda]  (+ U t of each ancestor inside the
//   subtree, deepest first -- the reference's recursion order)
#include "acr_types.cuh"
#include "acr_launch.h"

namespace acr {

static constexpr int HT = 128;

__device__ __forceinline__ double hwarp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int mm_slot(const TreeDev& T, int mu) {
  return mu == 0 ? 0 : T.depth[T.parent[mu]];
}

__device__ __forceinline__ int mm_cols(const MMJob& J, const TreeDev& T, int g,
                                       int mu) {
  if (J.cols_fixed >= 0) return J.cols_fixed;
  int p = T.parent[mu];
  int ci = (mu == T.c0[p]) ? 0 : 1;
  return rank_base(J.cols, g)[p * 2 + (ci ^ J.swap)];
}

struct MMJobs2 {
  MMJob j[2];
};

__global__ void __launch_bounds__(HT) k_hmatA(TreeDev T, MMJobs2 JJ) {
  const MMJob& J = JJ.j[blockIdx.z];
  if ((int)blockIdx.x >= J.nA) return;
  const int g = blockIdx.y, n = T.n;
  const int e0 = T.startA[J.mu0];
  const int* ent = T.listA + (e0 + blockIdx.x) * 3;
  const int mu = ent[0], beta = ent[1], side = ent[2];
  const int c = mm_cols(J, T, g, mu);
  if (!c) return;
  const HB h = J.H[g];
  const int r = h.rk[beta * 2 + side];
  if (!r) return;
  const int lo = T.lo[beta], hi = T.hi[beta], mid = T.mid[beta];
  // non-trans: V rows (other half); trans: U rows
  int row, len;
  const double* F;
  const long long fs = (long long)T.depth[beta] * h.R * n;
  if (!J.trans) {
    row = side ? lo : mid;
    len = side ? mid - lo : hi - mid;
    F = h.V + fs + row;
  } else {
    row = side ? mid : lo;
    len = side ? hi - mid : mid - lo;
    F = h.U + fs + row;
  }
  const double* X = src_col(J.X, n, g, mm_slot(T, mu), 0) + row;
  double* t = J.tbuf + ((long long)g * J.nA + blockIdx.x) * J.RT * J.CT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int p = warp; p < r * c; p += HT / 32) {
    int a = p / c, b = p - a * c;
    const double* fa = F + (long long)a * n;
    const double* xb = X + (long long)b * n;
    double s = 0.0;
    for (int i = lane; i < len; i += 32) s += fa[i] * xb[i];
    s = hwarp_sum(s);
    if (lane == 0) t[a * J.CT + b] = s;
  }
}

__global__ void __launch_bounds__(HT) k_hmatB(TreeDev T, MMJobs2 JJ, int nBmax) {
  extern __shared__ double sm[];
  const MMJob& J = JJ.j[blockIdx.z];
  const int b0 = T.startB[J.mu0], nB = T.startB[J.mu1] - b0;
  if ((int)blockIdx.x >= nB) return;
  const int g = blockIdx.y, n = T.n, bw = T.bw;
  const int mu = T.listB[(b0 + blockIdx.x) * 2], lam = T.listB[(b0 + blockIdx.x) * 2 + 1];
  const int c = mm_cols(J, T, g, mu);
  if (!c) return;
  const HB h = J.H[g];
  const int lo = T.lo[lam], s = T.hi[lam] - lo;
  const int slot = mm_slot(T, mu);
  const int ld = s + 1;            // padded: conflict-free column reads
  double* L = sm;                 // s x ld
  double* X = L + s * ld;         // c x s (column-major panel)
  const double* Lg = h.leaf + (long long)lo * bw;
  for (int idx = threadIdx.x; idx < s * s; idx += HT) {
    int i = idx / s, j = idx - i * s;
    L[i * ld + j] = Lg[(long long)i * bw + j];
  }
  for (int idx = threadIdx.x; idx < s * c; idx += HT) {
    int b = idx / s, i = idx - b * s;
    X[idx] = src_col(J.X, n, g, slot, b)[lo + i];
  }
  __syncthreads();
  const int eA0 = T.startA[J.mu0];
  for (int idx = threadIdx.x; idx < s * c; idx += HT) {
    int b = idx / s, i = idx - b * s;
    double y = 0.0;
    if (!J.trans)
      for (int j = 0; j < s; ++j) y += L[i * ld + j] * X[b * s + j];
    else
      for (int j = 0; j < s; ++j) y += L[j * ld + i] * X[b * s + j];
    for (int be = lam; be != mu;) {
      be = T.parent[be];
      int bmid = T.mid[be];
      bool top = lo < bmid;
      int sd = J.trans ? (top ? 1 : 0) : (top ? 0 : 1);
      int r = h.rk[be * 2 + sd];
      if (!r) continue;
      int e = T.startA[mu] + 2 * T.posA[mu * T.nnodes + be] + sd - eA0;
      const double* t = J.tbuf + ((long long)g * J.nA + e) * J.RT * J.CT;
      const double* F = (J.trans ? h.V : h.U) + (long long)T.depth[be] * h.R * n + lo + i;
      double z = 0.0;
      for (int a = 0; a < r; ++a) z += F[(long long)a * n] * t[a * J.CT + b];
      y = y + z;
    }
    src_col(J.Y, n, g, slot, b)[lo + i] = J.alpha * y;
  }
}

// Phase B for jobs whose subtree roots are every non-root node (multiply M1):
// one CTA per (leaf, element, job) serves all roots mu on the leaf's path, so
// the leaf block is read once instead of once per ancestor.
__global__ void __launch_bounds__(HT) k_hmatB_path(TreeDev T, MMJobs2 JJ) {
  extern __shared__ double sm[];
  const MMJob& J = JJ.j[blockIdx.z];
  const int g = blockIdx.y, n = T.n, bw = T.bw;
  const int lam = T.listB[(T.startB[0] + blockIdx.x) * 2 + 1];
  const int lo = T.lo[lam], s = T.hi[lam] - lo;
  const HB h = J.H[g];
  const int* an = T.anc + lam * (T.maxdepth + 1);
  const int dl = T.depth[lam];
  const int ld = s + 1;            // padded: conflict-free column reads
  double* L = sm;
  double* X = L + s * ld;
  // columns of each root on the path (t = 0: lam itself ... dl-1)
  int cnt = 0;
  int off[16], cols[16], mus[16];
  for (int t = 0; t < dl && t < 16; ++t) {
    const int mu = an[t];
    if (mu < J.mu0 || mu >= J.mu1) continue;
    const int c = mm_cols(J, T, g, mu);
    mus[cnt] = mu;
    cols[cnt] = c;
    off[cnt] = cnt == 0 ? 0 : off[cnt - 1] + cols[cnt - 1];
    ++cnt;
  }
  const int ctot = cnt ? off[cnt - 1] + cols[cnt - 1] : 0;
  if (!ctot) return;
  const double* Lg = h.leaf + (long long)lo * bw;
  for (int idx = threadIdx.x; idx < s * s; idx += HT) {
    int i = idx / s, j = idx - i * s;
    L[i * ld + j] = Lg[(long long)i * bw + j];
  }
  for (int q = 0; q < cnt; ++q) {
    const int slot = mm_slot(T, mus[q]);
    for (int idx = threadIdx.x; idx < s * cols[q]; idx += HT) {
      int b = idx / s, i = idx - b * s;
      X[(off[q] + b) * s + i] = src_col(J.X, n, g, slot, b)[lo + i];
    }
  }
  __syncthreads();
  const int eA0 = T.startA[J.mu0];
  for (int idx = threadIdx.x; idx < s * ctot; idx += HT) {
    const int bb = idx / s, i = idx - bb * s;
    int q = 0;
    while (q + 1 < cnt && off[q + 1] <= bb) ++q;
    const int mu = mus[q], b = bb - off[q];
    double y = 0.0;
    const double* xb = X + bb * s;
    if (!J.trans)
      for (int j = 0; j < s; ++j) y += L[i * ld + j] * xb[j];
    else
      for (int j = 0; j < s; ++j) y += L[j * ld + i] * xb[j];
    for (int be = lam; be != mu;) {
      be = T.parent[be];
      const int bmid = T.mid[be];
      const bool top = lo < bmid;
      const int sd = J.trans ? (top ? 1 : 0) : (top ? 0 : 1);
      const int r = h.rk[be * 2 + sd];
      if (!r) continue;
      const int e = T.startA[mu] + 2 * T.posA[mu * T.nnodes + be] + sd - eA0;
      const double* t = J.tbuf + ((long long)g * J.nA + e) * J.RT * J.CT;
      const double* F = (J.trans ? h.V : h.U) + (long long)T.depth[be] * h.R * n + lo + i;
      double z = 0.0;
      for (int a = 0; a < r; ++a) z += F[(long long)a * n] * t[a * J.CT + b];
      y = y + z;
    }
    src_col(J.Y, n, g, mm_slot(T, mu), b)[lo + i] = J.alpha * y;
  }
}

cudaError_t launch_hmat(const TreeDev& T, const MMJob* jobs, int njobs,
                        int nelem, cudaStream_t st) {
  if (!nelem || !njobs) return cudaSuccess;
  MMJobs2 JJ;
  JJ.j[0] = jobs[0];
  JJ.j[1] = njobs > 1 ? jobs[1] : jobs[0];
  int nA = 0, nB = 0, cmax = 0;
  for (int k = 0; k < njobs; ++k) {
    nA = jobs[k].nA > nA ? jobs[k].nA : nA;
    nB = jobs[k].nB > nB ? jobs[k].nB : nB;
    cmax = jobs[k].CT > cmax ? jobs[k].CT : cmax;
  }
  if (nA > 0) {
    dim3 g(nA, nelem, njobs);
    k_hmatA<<<g, HT, 0, st>>>(T, JJ);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_hmatB, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    cudaFuncSetAttribute(k_hmatB_path, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  if (jobs[0].mu0 == 1 && jobs[0].mu1 == T.nnodes && T.maxdepth <= 16) {
    size_t smem = ((size_t)T.bw * (T.bw + 1) + (size_t)T.bw * cmax * T.maxdepth) * 8;
    dim3 g(T.nleaves, nelem, njobs);
    k_hmatB_path<<<g, HT, smem, st>>>(T, JJ);
    return cudaGetLastError();
  }
  size_t smem = ((size_t)T.bw * (T.bw + 1) + (size_t)T.bw * cmax) * 8;
  dim3 g(nB, nelem, njobs);
  k_hmatB<<<g, HT, smem, st>>>(T, JJ, nB);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Z[rows hw] = alpha * W[rows hw] (X[rows hx]^T Y[rows hx]) per branch node
// ---------------------------------------------------------------------------
struct GPJobs2 {
  GPJob j[2];
};

__global__ void __launch_bounds__(HT) k_gp(TreeDev T, GPJobs2 JJ, const int* nodes) {
  extern __shared__ double K[];
  const GPJob& J = JJ.j[blockIdx.z];
  const int g = blockIdx.y, n = T.n;
  const int nu = nodes[blockIdx.x];
  const int rx = rank_base(J.rx, g)[nu * 2 + J.sx];
  const int ry = rank_base(J.ry, g)[nu * 2 + J.sy];
  if (!rx || !ry) {
    if (J.orank && threadIdx.x == 0) J.orank[g * J.ors + nu * 2 + J.oside] = 0;
    return;
  }
  const int lo = T.lo[nu], hi = T.hi[nu], mid = T.mid[nu];
  const int slot = T.depth[nu];
  const int r1 = J.hx ? mid : lo, l1 = J.hx ? hi - mid : mid - lo;
  const int r2 = J.hw ? mid : lo, l2 = J.hw ? hi - mid : mid - lo;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int p = warp; p < rx * ry; p += HT / 32) {
    int a = p / ry, b = p - a * ry;
    const double* xa = src_col(J.X, n, g, slot, a) + r1;
    const double* yb = src_col(J.Y, n, g, slot, b) + r1;
    double s = 0.0;
    for (int i = lane; i < l1; i += 32) s += xa[i] * yb[i];
    s = hwarp_sum(s);
    if (lane == 0) K[a * ry + b] = s;
  }
  __syncthreads();
  // thread per output row: W[i][:] loaded once, all ry outputs of the row
  for (int i = threadIdx.x; i < l2; i += HT) {
    double w[32];
    for (int a0 = 0; a0 < rx; a0 += 32) {
      const int na = rx - a0 < 32 ? rx - a0 : 32;
#pragma unroll
      for (int a = 0; a < 32; ++a)
        if (a < na) w[a] = src_col(J.W, n, g, slot, a0 + a)[r2 + i];
      for (int b = 0; b < ry; ++b) {
        double z = 0.0;
#pragma unroll
        for (int a = 0; a < 32; ++a)
          if (a < na) z += w[a] * K[(a0 + a) * ry + b];
        if (a0 == 0) src_col(J.Z, n, g, slot, b)[r2 + i] = J.alpha * z;
        else src_col(J.Z, n, g, slot, b)[r2 + i] += J.alpha * z;
      }
    }
  }
  if (J.orank && threadIdx.x == 0) J.orank[g * J.ors + nu * 2 + J.oside] = ry;
}

cudaError_t launch_gp(const TreeDev& T, const GPJob* jobs, int njobs,
                      const int* nodes, int nnodes, int nelem, int kcap,
                      cudaStream_t st) {
  if (!nelem || !njobs || !nnodes) return cudaSuccess;
  GPJobs2 JJ;
  JJ.j[0] = jobs[0];
  JJ.j[1] = njobs > 1 ? jobs[1] : jobs[0];
  size_t smem = (size_t)kcap * 8;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  dim3 g(nnodes, nelem, njobs);
  k_gp<<<g, HT, smem, st>>>(T, JJ, nodes);
  return cudaGetLastError();
}

// out = (f - a) - b  over count panels of len doubles (reference
// reduction.py:204-216 and 249-253 order); a or b may be null
__global__ void k_rhs_combine(const double* f, long long fs, const double* a,
                              long long as, const double* b, long long bs,
                              double* out, long long os, int len) {
  const int e = blockIdx.y;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len;
       i += gridDim.x * blockDim.x) {
    double v = f[e * fs + i];
    if (a) v = v - a[e * as + i];
    if (b) v = v - b[e * bs + i];
    out[e * os + i] = v;
  }
}

cudaError_t launch_rhs_combine(const double* f, long long fs, const double* a,
                               long long as, const double* b, long long bs,
                               double* out, long long os, int count, int len,
                               cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  int bx = (len + 255) / 256;
  if (bx > 64) bx = 64;
  k_rhs_combine<<<dim3(bx, count), 256, 0, st>>>(f, fs, a, as, b, bs, out, os, len);
  return cudaGetLastError();
}

}  // namespace acr
