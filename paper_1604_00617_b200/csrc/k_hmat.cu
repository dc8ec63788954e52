// HODLR x panel products over subtrees (reference algebra.py:52-83,
// hodlr.py:89-99) and the small "panel x (panel^T panel)" products of
// invert / multiply (algebra.py:152-156, 214-225).
//
// hmat, phase A: for every branch node beta below a subtree root mu and both
//   sides, t = V^T X[rows V]  (trans: U^T X[rows U])      -> tbuf
// hmat, phase B: per leaf lambda below mu,
//   Y[rows lambda] = L X[rows lambda]  (+ U t of each ancestor inside the
//   subtree, deepest first -- the reference's recursion order)
//   k_hmatB_tc (FP64 tensor pipe, leaves of at most 64 rows) / k_hmatB_sm
#include "acr_types.cuh"
#include "acr_launch.h"
#include "acr_pdl.cuh"
#include <cstdlib>

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

template <bool LAT>
__global__ void __launch_bounds__(HT) k_hmatA(TreeDev T, MMJobs2 JJ) {
  ACR_PDL_ENTRY();
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
  if (LAT && c <= 16) {
    // latency-bound launches (few elements): one warp per factor column a, all c panel columns at once: the factor
    // element is loaded once for every column and the 16 accumulation chains
    // (and their loads) are independent, so a long node's dot products keep
    // many loads in flight instead of one serial chain per output
    for (int a = warp; a < r; a += HT / 32) {
      const double* fa = F + (long long)a * n;
      double acc[16];
#pragma unroll
      for (int b = 0; b < 16; ++b) acc[b] = 0.0;
      for (int i = lane; i < len; i += 32) {
        const double f = fa[i];
#pragma unroll
        for (int b = 0; b < 16; ++b)
          if (b < c) acc[b] += f * X[(long long)b * n + i];
      }
#pragma unroll
      for (int b = 0; b < 16; ++b)
        if (b < c) {
          const double v = hwarp_sum(acc[b]);
          if (lane == b) t[a * J.CT + b] = v;
        }
    }
    return;
  }
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

// Phase A on the FP64 tensor pipe: t = F^T X (r x c) over the node's rows,
// rows split over the warps, every 8 x 8 tile of t accumulated with
// mma.sync m8n8k4, the warps' partial tiles summed in a fixed order through
// shared memory (same structure as k_gp_tc).  TMAX: tiles per side.
template <int NT, int TMAX>
__global__ void __launch_bounds__(NT) k_hmatA_tc(TreeDev T, MMJobs2 JJ) {
  ACR_PDL_ENTRY();
  constexpr int NW = NT / 32;
  extern __shared__ double part[];   // NW * TMAX * TMAX * 64
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
  const int gi = lane >> 2, ti = lane & 3;
  const int ta = (r + 7) >> 3, tb = (c + 7) >> 3;
  double acc[TMAX][TMAX][2];
#pragma unroll
  for (int a = 0; a < TMAX; ++a)
#pragma unroll
    for (int b = 0; b < TMAX; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const double* fc[TMAX];
  const double* xc[TMAX];
#pragma unroll
  for (int a = 0; a < TMAX; ++a) {
    const int ca = a * 8 + gi;
    fc[a] = (a < ta && ca < r) ? F + (long long)ca * n : nullptr;
    xc[a] = (a < tb && ca < c) ? X + (long long)ca * n : nullptr;
  }
  // UL row chunks of a warp in flight: their loads are issued together (one
  // trip to L2 per UL chunks instead of one per chunk); chunks past the end
  // contribute exact zeros, the order of the sums is unchanged
  constexpr int UL = TMAX >= 4 ? 2 : 4;
  for (int k0 = warp * 4; k0 < len; k0 += NW * 4 * UL) {
    double av[UL][TMAX], bv[UL][TMAX];
#pragma unroll
    for (int u = 0; u < UL; ++u) {
      const int k = k0 + u * NW * 4 + ti;
#pragma unroll
      for (int a = 0; a < TMAX; ++a) {
        av[u][a] = (fc[a] && k < len) ? fc[a][k] : 0.0;
        bv[u][a] = (xc[a] && k < len) ? xc[a][k] : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < UL; ++u)
#pragma unroll
      for (int a = 0; a < TMAX; ++a)
#pragma unroll
        for (int b = 0; b < TMAX; ++b)
          if (a < ta && b < tb)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 "
                         "{%0, %1}, {%2}, {%3}, {%0, %1};\n"
                         : "+d"(acc[a][b][0]), "+d"(acc[a][b][1])
                         : "d"(av[u][a]), "d"(bv[u][b]));
  }
#pragma unroll
  for (int a = 0; a < TMAX; ++a)
#pragma unroll
    for (int b = 0; b < TMAX; ++b)
      if (a < ta && b < tb) {
        double* pt = part + ((warp * TMAX + a) * TMAX + b) * 64;
        pt[gi * 8 + 2 * ti] = acc[a][b][0];
        pt[gi * 8 + 2 * ti + 1] = acc[a][b][1];
      }
  __syncthreads();
  for (int e = threadIdx.x; e < r * c; e += NT) {
    const int x = e / c, y = e - x * c;
    const int a = x >> 3, b = y >> 3, off = (x & 7) * 8 + (y & 7);
    double sacc = 0.0;
    for (int w = 0; w < NW; ++w) sacc += part[((w * TMAX + a) * TMAX + b) * 64 + off];
    t[x * J.CT + y] = sacc;
  }
}

// Phase A for throughput-bound launches (hundreds of thousands of (entry,
// element) pairs, each a few dozen rows by a handful of columns): one WARP per
// pair, eight pairs per CTA.  k_hmatA_tc spends one 128-thread CTA per pair --
// at 800 k CTAs per launch the CTA dispatch rate, not the arithmetic, set its
// duration (1.8 ms for the level-1 products).  A warp walks all the rows of
// its pair, 4 per mma.sync m8n8k4, so there is no cross-warp reduction either.
template <int TMAX>
__global__ void __launch_bounds__(256) k_hmatA_tcw(TreeDev T, MMJobs2 JJ) {
  ACR_PDL_ENTRY();
  const MMJob& J = JJ.j[blockIdx.z];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ei = blockIdx.x * 8 + warp;
  if (ei >= J.nA) return;
  const int g = blockIdx.y, n = T.n;
  const int e0 = T.startA[J.mu0];
  const int* ent = T.listA + (e0 + ei) * 3;
  const int mu = ent[0], beta = ent[1], side = ent[2];
  const int c = mm_cols(J, T, g, mu);
  if (!c) return;
  const HB h = J.H[g];
  const int r = h.rk[beta * 2 + side];
  if (!r) return;
  const int lo = T.lo[beta], hi = T.hi[beta], mid = T.mid[beta];
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
  double* t = J.tbuf + ((long long)g * J.nA + ei) * J.RT * J.CT;
  const int gi = lane >> 2, ti = lane & 3;
  const int ta = (r + 7) >> 3, tb = (c + 7) >> 3;
  double acc[TMAX][TMAX][2];
#pragma unroll
  for (int a = 0; a < TMAX; ++a)
#pragma unroll
    for (int b = 0; b < TMAX; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const double* fc[TMAX];
  const double* xc[TMAX];
#pragma unroll
  for (int a = 0; a < TMAX; ++a) {
    const int ca = a * 8 + gi;
    fc[a] = (a < ta && ca < r) ? F + (long long)ca * n : nullptr;
    xc[a] = (a < tb && ca < c) ? X + (long long)ca * n : nullptr;
  }
  for (int k0 = 0; k0 < len; k0 += 4) {
    const int k = k0 + ti;
    double av[TMAX], bv[TMAX];
#pragma unroll
    for (int a = 0; a < TMAX; ++a) {
      av[a] = (fc[a] && k < len) ? fc[a][k] : 0.0;
      bv[a] = (xc[a] && k < len) ? xc[a][k] : 0.0;
    }
#pragma unroll
    for (int a = 0; a < TMAX; ++a)
#pragma unroll
      for (int b = 0; b < TMAX; ++b)
        if (a < ta && b < tb)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 "
                       "{%0, %1}, {%2}, {%3}, {%0, %1};\n"
                       : "+d"(acc[a][b][0]), "+d"(acc[a][b][1]) : "d"(av[a]), "d"(bv[b]));
  }
  // accumulator fragment: row gi, columns 2 ti, 2 ti + 1 of every 8 x 8 tile
#pragma unroll
  for (int a = 0; a < TMAX; ++a)
#pragma unroll
    for (int b = 0; b < TMAX; ++b)
      if (a < ta && b < tb) {
        const int x = a * 8 + gi, y = b * 8 + 2 * ti;
        if (x < r && y < c) t[x * J.CT + y] = acc[a][b][0];
        if (x < r && y + 1 < c) t[x * J.CT + y + 1] = acc[a][b][1];
      }
}

// Fallback phase B (trees deeper than 16; k_hmatB_sm below is the main path).
// Register tile of phase B: one thread = one leaf row i x HB_CB columns of
// one subtree root.  The leaf row and every ancestor U (V) row element are
// loaded once per HB_CB columns; X is row-major [j][cp] in shared memory with
// its columns zero-padded to a multiple of HB_CB (double2 broadcast loads).
// Every output keeps the scalar summation order (leaf terms j = 0..s-1, then
// y = y + z per ancestor, deepest first), so results are unchanged bitwise.
static constexpr int HB_CB = 8;   // padding unit (largest tile)

template <int CB>
__device__ __forceinline__ void hmatB_tile(const TreeDev& T, const MMJob& J, const HB& h,
                                           int g, int mu, int lam, int lo, int s, int ld,
                                           const double* L, const double* Xr, int cp,
                                           int i, int b0, int nb, int eA0, int slot) {
  const int n = T.n;
  double y[CB];
#pragma unroll
  for (int u = 0; u < CB; ++u) y[u] = 0.0;
  for (int j = 0; j < s; ++j) {
    const double l = J.trans ? L[j * ld + i] : L[i * ld + j];
    const double2* x = reinterpret_cast<const double2*>(Xr + j * cp + b0);
#pragma unroll
    for (int u = 0; u < CB / 2; ++u) {
      const double2 xv = x[u];
      y[2 * u] += l * xv.x;
      y[2 * u + 1] += l * xv.y;
    }
  }
  for (int be = lam; be != mu;) {
    be = T.parent[be];
    const int bmid = T.mid[be];
    const bool top = lo < bmid;
    const int sd = J.trans ? (top ? 1 : 0) : (top ? 0 : 1);
    const int r = h.rk[be * 2 + sd];
    if (!r) continue;
    const int e = T.startA[mu] + 2 * T.posA[mu * T.nnodes + be] + sd - eA0;
    const double* t = J.tbuf + ((long long)g * J.nA + e) * J.RT * J.CT + b0;
    const double* F = (J.trans ? h.V : h.U) + (long long)T.depth[be] * h.R * n + lo + i;
    double z[CB];
#pragma unroll
    for (int u = 0; u < CB; ++u) z[u] = 0.0;
    for (int a = 0; a < r; ++a) {
      const double f = F[(long long)a * n];
      const double* ta = t + a * J.CT;
#pragma unroll
      for (int u = 0; u < CB; ++u)
        if (u < nb) z[u] += f * __ldg(ta + u);
    }
#pragma unroll
    for (int u = 0; u < CB; ++u) y[u] = y[u] + z[u];
  }
#pragma unroll
  for (int u = 0; u < CB; ++u)
    if (u < nb) src_col(J.Y, n, g, slot, b0 + u)[lo + i] = J.alpha * y[u];
}

template <int CB>
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
  const int cp = (c + HB_CB - 1) / HB_CB * HB_CB;
  double* L = sm;                 // s x ld
  double* X = L + ((s * ld + 1) & ~1);   // s x cp, row-major, 16-byte aligned
  const double* Lg = h.leaf + (long long)lo * bw;
  for (int idx = threadIdx.x; idx < s * s; idx += HT) {
    int i = idx / s, j = idx - i * s;
    L[i * ld + j] = Lg[(long long)i * bw + j];
  }
  for (int idx = threadIdx.x; idx < s * cp; idx += HT) {
    int b = idx / s, i = idx - b * s;
    X[i * cp + b] = b < c ? src_col(J.X, n, g, slot, b)[lo + i] : 0.0;
  }
  __syncthreads();
  const int eA0 = T.startA[J.mu0];
  const int nch = (c + CB - 1) / CB;
  for (int idx = threadIdx.x; idx < s * nch; idx += HT) {
    const int q = idx / s, i = idx - q * s;
    const int bb = q * CB, nb = c - bb < CB ? c - bb : CB;
    hmatB_tile<CB>(T, J, h, g, mu, lam, lo, s, ld, L, X, cp, i, bb, nb, eA0, slot);
  }
}

// Phase B for jobs whose subtree roots are every non-root node (multiply M1):
// one CTA per (leaf, element, job) serves all roots mu on the leaf's path, so
// the leaf block is read once instead of once per ancestor.
template <int CB>
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
  // columns of each root on the path, each padded to a multiple of HB_CB
  int cnt = 0;
  int off[16], cols[16], mus[16];
  for (int t = 0; t < dl && t < 16; ++t) {
    const int mu = an[t];
    if (mu < J.mu0 || mu >= J.mu1) continue;
    const int c = mm_cols(J, T, g, mu);
    if (!c) continue;
    mus[cnt] = mu;
    cols[cnt] = c;
    off[cnt] = cnt == 0 ? 0 : off[cnt - 1] + (cols[cnt - 1] + HB_CB - 1) / HB_CB * HB_CB;
    ++cnt;
  }
  if (!cnt) return;
  const int cp = off[cnt - 1] + (cols[cnt - 1] + HB_CB - 1) / HB_CB * HB_CB;
  double* L = sm;
  double* X = L + ((s * ld + 1) & ~1);
  const double* Lg = h.leaf + (long long)lo * bw;
  for (int idx = threadIdx.x; idx < s * s; idx += HT) {
    int i = idx / s, j = idx - i * s;
    L[i * ld + j] = Lg[(long long)i * bw + j];
  }
  for (int q = 0; q < cnt; ++q) {
    const int slot = mm_slot(T, mus[q]);
    const int w = (cols[q] + HB_CB - 1) / HB_CB * HB_CB;
    for (int idx = threadIdx.x; idx < s * w; idx += HT) {
      int b = idx / s, i = idx - b * s;
      X[i * cp + off[q] + b] = b < cols[q] ? src_col(J.X, n, g, slot, b)[lo + i] : 0.0;
    }
  }
  __syncthreads();
  const int eA0 = T.startA[J.mu0];
  const int nch = cp / CB;
  for (int idx = threadIdx.x; idx < s * nch; idx += HT) {
    const int ch = idx / s, i = idx - ch * s;
    const int pos = ch * CB;
    int q = 0;
    while (q + 1 < cnt && off[q + 1] <= pos) ++q;
    const int bb = pos - off[q], nb = cols[q] - bb < CB ? cols[q] - bb : CB;
    if (nb <= 0) continue;   // padding chunk of a root
    hmatB_tile<CB>(T, J, h, g, mus[q], lam, lo, s, ld, L, X + off[q], cp, i, bb, nb, eA0,
               mm_slot(T, mus[q]));
  }
}

// Phase B, column-pair tiles.  A CTA serves one leaf lam and either the single
// listB root (plain jobs) or every root on the leaf's path (M1).  Each thread
// computes two adjacent columns of one root for one leaf row; X is staged
// row-major [j][cp] (pairs 16-byte aligned, odd widths zero-padded) so one
// double2 broadcast load feeds two FMAs.  Summation order per output is the
// scalar one: leaf terms j = 0..s-1, then y = y + z per ancestor deepest
// first (z = sum over a in order) -- equal bitwise to k_hmatB.
struct HBRoots {
  int lam, cnt, cp;
  int off[16], cols[16], mus[16];
  int steps[16];              // mu = anc(lam, steps)
  int slot[16];               // mm_slot(mu): output panel slot of the root
};

// The root table of a CTA, built once in shared memory by its first warp: in
// path mode lane t looks at ancestor t of the leaf (the tree-metadata and rank
// loads of all ancestors are issued together instead of one dependent chain
// per ancestor in every thread), the nonzero roots are compacted in t order
// (ballot) and their column offsets formed by a warp scan: the same table,
// in the same order, as the sequential walk of hb_roots.
__device__ __forceinline__ void hb_roots_shared(const TreeDev& T, const MMJob& J, int g,
                                                int path, HBRoots& R) {
  const int lane = threadIdx.x & 31;
  if (path) {
    const int lam = T.listB[(T.startB[0] + blockIdx.x) * 2 + 1];
    const int dl = T.depth[lam];
    int mu = -1, c = 0, slot = 0;
    if (lane < dl && lane < 16) {
      mu = T.anc[lam * (T.maxdepth + 1) + lane];
      if (mu >= J.mu0 && mu < J.mu1) {
        c = mm_cols(J, T, g, mu);
        slot = mm_slot(T, mu);
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, c != 0);
    const int pos = __popc(m & ((1u << lane) - 1u));
    const int padded = c ? ((c + 1) & ~1) : 0;
    int incl = padded;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (c) {
      R.mus[pos] = mu;
      R.cols[pos] = c;
      R.steps[pos] = lane;
      R.off[pos] = incl - padded;
      R.slot[pos] = slot;
    }
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    if (lane == 0) {
      R.lam = lam;
      R.cnt = __popc(m);
      R.cp = tot;
    }
  } else if (lane == 0) {
    R.cnt = 0;
    const int b0 = T.startB[J.mu0], nB = T.startB[J.mu1] - b0;
    if ((int)blockIdx.x < nB) {
      const int mu = T.listB[(b0 + blockIdx.x) * 2];
      R.lam = T.listB[(b0 + blockIdx.x) * 2 + 1];
      const int c = mm_cols(J, T, g, mu);
      if (c) {
        R.mus[0] = mu;
        R.cols[0] = c;
        R.off[0] = 0;
        R.steps[0] = T.depth[R.lam] - T.depth[mu];
        R.slot[0] = mm_slot(T, mu);
        R.cnt = 1;
        R.cp = (c + 1) & ~1;
      }
    }
  }
}


// ancestor walk of every root, tabulated once per CTA (k = steps above lam)
struct HBAnc {
  int r[17];
  long long F[17];
  const double* t[16][17];
};

__device__ __forceinline__ void hb_anc_tables(const TreeDev& T, const MMJob& J, const HB& h,
                                              int g, const HBRoots& R, int lo, HBAnc& A) {
  const int* an = T.anc + R.lam * (T.maxdepth + 1);
  const int dl = T.depth[R.lam];
  const int eA0 = T.startA[J.mu0];
  for (int p = threadIdx.x; p < 17 * (R.cnt + 1); p += blockDim.x) {
    const int q = p / 17 - 1, k = p % 17;
    if (k < 1 || k > dl) continue;
    const int be = an[k];
    const bool top = lo < T.mid[be];
    const int sd = J.trans ? (top ? 1 : 0) : (top ? 0 : 1);
    if (q < 0) {
      A.r[k] = h.rk[be * 2 + sd];
      A.F[k] = (long long)T.depth[be] * h.R * T.n + lo;
    } else if (k <= R.steps[q]) {
      const int mu = R.mus[q];
      const int e = T.startA[mu] + 2 * T.posA[mu * T.nnodes + be] + sd - eA0;
      A.t[q][k] = J.tbuf + ((long long)g * J.nA + e) * J.RT * J.CT;
    }
  }
}

__device__ __forceinline__ void hb_finish_tab(const TreeDev& T, const MMJob& J, const HB& h,
                                              int g, int q, const HBRoots& R, const HBAnc& A,
                                              int lo, int i, int b0, int nb, double y0,
                                              double y1) {
  const int n = T.n;
  const double* base = (J.trans ? h.V : h.U) + i;
  const int nst = R.steps[q];
  for (int k = 1; k <= nst; ++k) {
    const int r = A.r[k];
    if (!r) continue;
    const double* t = A.t[q][k] + b0;
    const double* F = base + A.F[k];
    double z0 = 0.0, z1 = 0.0;
#pragma unroll 4
    for (int a = 0; a < r; ++a) {
      const double f = F[(long long)a * n];
      z0 += f * __ldg(t + a * J.CT);
      if (nb > 1) z1 += f * __ldg(t + a * J.CT + 1);
    }
    y0 = y0 + z0;
    y1 = y1 + z1;
  }
  const int slot = R.slot[q];
  src_col(J.Y, n, g, slot, b0)[lo + i] = J.alpha * y0;
  if (nb > 1) src_col(J.Y, n, g, slot, b0 + 1)[lo + i] = J.alpha * y1;
}

// Leaf in padded shared memory (few registers, high occupancy);
// X staged in windows of at most xc columns (bounded shared memory)
template <int NTB>
__global__ void __launch_bounds__(NTB) k_hmatB_sm(TreeDev T, MMJobs2 JJ, int path, int xc) {
  ACR_PDL_ENTRY();
  extern __shared__ double sm[];
  const MMJob& J = JJ.j[blockIdx.z];
  const int g = blockIdx.y, bw = T.bw;
  __shared__ HBRoots R;
  if (threadIdx.x < 32) hb_roots_shared(T, J, g, path, R);
  __syncthreads();
  if (!R.cnt) return;
  const HB h = J.H[g];
  const int lam = R.lam, lo = T.lo[lam], s = T.hi[lam] - lo, cp = R.cp;
  const int ld = s + 1;
  double* L = sm;                               // s x ld
  double* X = L + ((s * ld + 1) & ~1);          // s x (window width), pairs aligned
  const double* Lg = h.leaf + (long long)lo * bw;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // asynchronous staging: warp per row, lanes along the row (no divisions)
  for (int ii = warp; ii < s; ii += NTB / 32)
    for (int j = lane; j < s; j += 32) cp_async8(L + ii * ld + j, Lg + (long long)ii * bw + j, true);
  __shared__ HBAnc A;
  hb_anc_tables(T, J, h, g, R, lo, A);
  for (int w0 = 0; w0 < cp; w0 += xc) {
    const int wc = cp - w0 < xc ? cp - w0 : xc;
    for (int q = 0; q < R.cnt; ++q) {
      const int slot = R.slot[q];
      const int q0 = R.off[q], q1 = q0 + ((R.cols[q] + 1) & ~1);
      const int c0 = q0 > w0 ? q0 : w0, c1 = q1 < w0 + wc ? q1 : w0 + wc;
      for (int pos = c0 + warp; pos < c1; pos += NTB / 32) {
        const int b = pos - q0;
        const bool ok = b < R.cols[q];
        const double* src = src_col(J.X, T.n, g, slot, ok ? b : 0) + lo;
        for (int ii = lane; ii < s; ii += 32) cp_async8(X + ii * wc + (pos - w0), src + ii, ok);
      }
    }
    cp_async_wait_all();
    __syncthreads();
    const int npairs = wc >> 1;
    for (int idx = threadIdx.x; idx < s * npairs; idx += NTB) {
      const int pr = idx / s, i = idx - pr * s;
      const int pos = w0 + pr * 2;
      int q = 0;
      while (q + 1 < R.cnt && R.off[q + 1] <= pos) ++q;
      const int b0 = pos - R.off[q];
      const int nb = R.cols[q] - b0 < 2 ? R.cols[q] - b0 : 2;
      if (nb <= 0) continue;
      double y0 = 0.0, y1 = 0.0;
      const double2* x = reinterpret_cast<const double2*>(X + pr * 2);
      const int li = J.trans ? i : i * ld, lj = J.trans ? ld : 1;
      for (int j = 0; j < s; ++j) {
        const double l = L[li + j * lj];
        const double2 xv = x[j * npairs];
        y0 += l * xv.x;
        y1 += l * xv.y;
      }
      hb_finish_tab(T, J, h, g, q, R, A, lo, i, b0, nb, y0, y1);
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void hb_dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 "
               "{%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// Phase B on the FP64 tensor pipe (leaves of at most 64 rows).  The leaf is
// staged in shared memory once (16-byte cp.async, one warp request per row;
// row pitch = 4 mod 16 doubles so the mma.sync m8n8k4 fragment reads -- 8 rows
// x 4 columns, or 4 x 8 transposed -- touch 16 distinct bank pairs per half
// warp).  Warp w owns rows 8w .. 8w+7.  The columns of ALL roots are packed
// into one list cut into 8-column tiles (a root of three columns does not pay
// for eight: the FP64 tensor pipe is only as fast as the FMA pipe, padding is
// not free); X is staged per window of W tiles, column-major with the leaf's
// pitch, and every warp takes the window's tiles two at a time (independent
// DMMA chains).  The ancestors' terms sum_k U_k t_k are one product over the
// concatenated inner index (k, a) -- a flat table, so the loads of a tile are
// independent of one another; a column stops contributing at its own root
// (zero B fragments above it) -- chained onto the same accumulators, deepest
// ancestor first.
static constexpr int HB_FLAT = 512;
static constexpr int HB_COLS = 256;

template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_hmatB_tc(TreeDev T, MMJobs2 JJ, int path, int W,
                                                        int ldl, int zskip) {
  ACR_PDL_ENTRY();
  constexpr bool AREG = MINB < 5;       // leaf fragments kept in registers
  extern __shared__ double sm[];
  const MMJob& J = JJ.j[blockIdx.z];
  const int g = blockIdx.y, bw = T.bw, n = T.n;
  __shared__ HBRoots R;
  __shared__ HBAnc A;
  __shared__ int fl_n[17];              // flat inner length of the ancestors 1 .. k
  __shared__ int fl_ka[HB_FLAT];        // (k << 16) | a
  __shared__ int col_qb[HB_COLS];       // packed column -> (root q << 16) | column of the root
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gi = lane >> 2, ti = lane & 3;
  if (threadIdx.x < 32) hb_roots_shared(T, J, g, path, R);
  __syncthreads();
  if (!R.cnt) return;
  double* L = sm;                 // bw x ldl
  double* X = L + bw * ldl;       // 8 W x ldl, column-major
  const HB h = J.H[g];
  const int lam = R.lam, lo = T.lo[lam], s = T.hi[lam] - lo;
  // zskip (the lifted level's inversion: panels with a single nonzero row):
  // when every X row of this leaf is an exact zero the leaf product is zero,
  // and neither the leaf nor X is fetched -- only the ancestors' terms remain
  bool have_leaf = true;
  if (zskip) {
    int nzx = 0;
    for (int q = 0; q < R.cnt; ++q) {
      const int slot = R.slot[q], nc = R.cols[q];
      for (int idx = threadIdx.x; idx < nc * s; idx += 256) {
        const int b = idx / s, ii = idx - b * s;
        nzx |= src_col(J.X, n, g, slot, b)[lo + ii] != 0.0;
      }
    }
    have_leaf = __syncthreads_or(nzx) != 0;
  }
  if (have_leaf) {
    const double* Lg = h.leaf + (long long)lo * bw;
    if (!(s & 1)) {
      // warp per row, a 16-byte chunk per lane
      for (int ii = warp; ii < s; ii += 8)
        for (int c = 2 * lane; c < s; c += 64)
          cp_async16(L + ii * ldl + c, Lg + (long long)ii * bw + c);
    } else {
      for (int ii = warp; ii < s; ii += 8)
        for (int j = lane; j < s; j += 32)
          cp_async8(L + ii * ldl + j, Lg + (long long)ii * bw + j, true);
    }
  }
  hb_anc_tables(T, J, h, g, R, lo, A);
  int ntot = 0;
  for (int q = 0; q < R.cnt; ++q) {
    const int nc = R.cols[q];
    for (int b = threadIdx.x; b < nc; b += 256)
      if (ntot + b < HB_COLS) col_qb[ntot + b] = (q << 16) | b;
    ntot += nc;
  }
  if (ntot > HB_COLS) ntot = HB_COLS;   // (the launcher keeps maxdepth * cmax <= HB_COLS)
  __syncthreads();
  {
    // flat (k, a) table of the ancestors' inner index, k ascending
    const int dl = T.depth[lam];
    int pre = 0;
    for (int k = 1; k <= dl && k < 17; ++k) {
      const int r = A.r[k];
      for (int a2 = threadIdx.x; a2 < r; a2 += 256)
        if (pre + a2 < HB_FLAT) fl_ka[pre + a2] = (k << 16) | a2;
      pre += r;
      if (threadIdx.x == 0) fl_n[k] = pre < HB_FLAT ? pre : HB_FLAT;
    }
    if (threadIdx.x == 0) fl_n[0] = 0;
  }
  const int i = warp * 8 + gi;
  const bool rowok = i < s;
  const double* Fb = (J.trans ? h.V : h.U) + i;
  const double* La = J.trans ? L + i : L + i * ldl;
  const int lj = J.trans ? ldl : 1;
  double a[AREG ? 16 : 1];
  for (int w0 = 0; w0 < ntot; w0 += 8 * W) {
    const int wn = ntot - w0 < 8 * W ? ntot - w0 : 8 * W;
    for (int j = warp; j < wn && have_leaf; j += 8) {
      const int qb = col_qb[w0 + j];
      const double* src = src_col(J.X, n, g, R.slot[qb >> 16], qb & 0xffff) + lo;
      for (int ii = lane; ii < s; ii += 32) cp_async8(X + j * ldl + ii, src + ii, true);
    }
    cp_async_wait_all();
    __syncthreads();
    if (AREG && w0 == 0 && have_leaf) {
#pragma unroll
      for (int kk = 0; kk < (AREG ? 16 : 1); ++kk) {
        const int j = kk * 4 + ti;
        a[kk] = (rowok && j < s) ? La[j * lj] : 0.0;
      }
    }
    if (warp * 8 < s && wn <= 2) {
      // one or two columns in all (rank-1 levels): an 8-column tile would be
      // mostly padding, so the same lane layout runs on the FMA pipe -- lane
      // (gi, ti) sums the inner indices = ti mod 4, two shuffles finish a row
      const int qb0 = col_qb[w0], qb1 = col_qb[w0 + wn - 1];
      const double* x1 = X + (wn - 1) * ldl;
      double p0 = 0.0, p1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const int j = kk * 4 + ti;
        if (j < s && have_leaf) {
          double av;
          if constexpr (AREG) av = a[kk];
          else av = rowok ? La[j * lj] : 0.0;
          p0 = fma(av, X[j], p0);
          p1 = fma(av, x1[j], p1);
        }
      }
      const int f0 = fl_n[R.steps[qb0 >> 16]], f1 = fl_n[R.steps[qb1 >> 16]];
      const int fm = f0 > f1 ? f0 : f1;
      const double* const* tp0 = A.t[qb0 >> 16];
      const double* const* tp1 = A.t[qb1 >> 16];
      const int c0 = qb0 & 0xffff, c1 = qb1 & 0xffff;
#pragma unroll 2
      for (int idx = ti; idx < fm; idx += 4) {
        const int ka = fl_ka[idx];
        const int k = ka >> 16, aa = ka & 0xffff;
        const double f = rowok ? Fb[A.F[k] + (long long)aa * n] : 0.0;
        if (idx < f0) p0 = fma(f, __ldg(tp0[k] + aa * J.CT + c0), p0);
        if (idx < f1) p1 = fma(f, __ldg(tp1[k] + aa * J.CT + c1), p1);
      }
      p0 += __shfl_xor_sync(0xffffffffu, p0, 1);
      p1 += __shfl_xor_sync(0xffffffffu, p1, 1);
      p0 += __shfl_xor_sync(0xffffffffu, p0, 2);
      p1 += __shfl_xor_sync(0xffffffffu, p1, 2);
      if (rowok && ti == 0)
        src_col(J.Y, n, g, R.slot[qb0 >> 16], c0)[lo + i] = J.alpha * p0;
      if (rowok && ti == 1 && wn > 1)
        src_col(J.Y, n, g, R.slot[qb1 >> 16], c1)[lo + i] = J.alpha * p1;
    } else if (warp * 8 < s) {
      for (int t0 = 0; t0 < wn; t0 += 16) {
        const bool two = t0 + 8 < wn;
        const int jA = t0 + gi, jB = t0 + 8 + gi;
        const bool okA = jA < wn, okB = jB < wn;
        const int qbA = col_qb[w0 + (okA ? jA : t0)], qbB = col_qb[w0 + (okB ? jB : t0)];
        const double* xA = X + (okA ? jA : t0) * ldl;
        const double* xB = X + (okB ? jB : t0) * ldl;
        double y00 = 0.0, y01 = 0.0, y10 = 0.0, y11 = 0.0;
        if (!have_leaf) {
          // zero leaf product: the accumulators start from the ancestors' terms
        } else if (s == 64 && !J.trans && !AREG) {
          // full 64-row leaf, plain product: no predicates, immediate offsets
          // (unstaged X columns of a ragged last tile are never stored)
          const double* la = La + ti;
          const double* xa = xA + ti;
          const double* xb = xB + ti;
          if (two) {
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) {
              const double av = la[kk * 4];
              hb_dmma(y00, y01, av, okA ? xa[kk * 4] : 0.0);
              hb_dmma(y10, y11, av, okB ? xb[kk * 4] : 0.0);
            }
          } else {
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) hb_dmma(y00, y01, la[kk * 4], okA ? xa[kk * 4] : 0.0);
          }
        } else {
#pragma unroll
          for (int kk = 0; kk < 16; ++kk) {
            const int j = kk * 4 + ti;
            if (kk * 4 < s) {
              double av;
              if constexpr (AREG) av = a[kk];
              else av = (rowok && j < s) ? La[j * lj] : 0.0;
              const double b0 = (okA && j < s) ? xA[j] : 0.0;
              hb_dmma(y00, y01, av, b0);
              if (two) {
                const double b1 = (okB && j < s) ? xB[j] : 0.0;
                hb_dmma(y10, y11, av, b1);
              }
            }
          }
        }
        // per-lane column: its root's flat length and t panels
        const int fA = okA ? fl_n[R.steps[qbA >> 16]] : 0;
        const int fB = okB ? fl_n[R.steps[qbB >> 16]] : 0;
        const int fm = __reduce_max_sync(0xffffffffu, fA > fB ? fA : fB);
        const double* const* tA = A.t[qbA >> 16];
        const double* const* tB = A.t[qbB >> 16];
        const int cA = qbA & 0xffff, cB = qbB & 0xffff;
#pragma unroll 2
        for (int a0 = 0; a0 < fm; a0 += 4) {
          const int idx = a0 + ti;
          const int ka = idx < fm ? fl_ka[idx] : (1 << 16);
          const int k = ka >> 16, aa = ka & 0xffff;
          const double f = (idx < fm && rowok) ? Fb[A.F[k] + (long long)aa * n] : 0.0;
          const double t0v = idx < fA ? __ldg(tA[k] + aa * J.CT + cA) : 0.0;
          hb_dmma(y00, y01, f, t0v);
          if (two) {
            const double t1v = idx < fB ? __ldg(tB[k] + aa * J.CT + cB) : 0.0;
            hb_dmma(y10, y11, f, t1v);
          }
        }
        if (rowok) {
          const int c = t0 + 2 * ti;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int j = c + (e & 1) + (e >> 1) * 8;
            if (j < wn) {
              const int qb = col_qb[w0 + j];
              const double y = e == 0 ? y00 : e == 1 ? y01 : e == 2 ? y10 : y11;
              src_col(J.Y, n, g, R.slot[qb >> 16], qb & 0xffff)[lo + i] = J.alpha * y;
            }
          }
        }
      }
    }
    __syncthreads();
  }
}

// HODLR x panel with a DIAGONAL HODLR operand (level 0: E, F lifted from the
// bands, diagonal leaves, rank-0 factors): every subtree product reduces to a
// row scaling, Y[slot(mu)][:, rows(mu)] = alpha diag(H) X[slot(mu)][:, rows(mu)],
// for every root mu in [mu0, mu1) -- bitwise the dense leaf product (the
// off-diagonal leaf entries are exact zeros and the factor terms vanish),
// reading n diagonal values instead of the n x bw leaf panel.
__global__ void k_hmat_diag(TreeDev T, MMJob J) {
  ACR_PDL_ENTRY();
  const int g = blockIdx.y, n = T.n, bw = T.bw;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const HB h = J.H[g];
  // leaf of row i and the chain of nodes above it
  int node = 0, path[17], np = 0;
  while (!T.isleaf[node] && np < 16) {
    path[np++] = node;
    node = i < T.mid[node] ? T.c0[node] : T.c1[node];
  }
  path[np] = node;
  const double d = h.leaf[(long long)i * bw + (i - T.lo[node])];
  for (int q = 0; q <= np; ++q) {               // mu = path[q], slot = depth(parent) (root: 0)
    const int mu = path[q];
    if (mu < J.mu0 || mu >= J.mu1) continue;
    const int c = mm_cols(J, T, g, mu);
    const int slot = mm_slot(T, mu);
    for (int b = 0; b < c; ++b)
      src_col(J.Y, n, g, slot, b)[i] = J.alpha * (d * src_col(J.X, n, g, slot, b)[i]);
  }
}

cudaError_t launch_hmat_diag(const TreeDev& T, const MMJob& job, int nelem, cudaStream_t st) {
  if (!nelem) return cudaSuccess;
  CK_PDL(launch_pdl(k_hmat_diag, dim3((T.n + 255) / 256, nelem), dim3(256), 0, st, T, job));
  return cudaGetLastError();
}

cudaError_t launch_hmat(const TreeDev& T, const MMJob* jobs, int njobs,
                        int nelem, cudaStream_t st, int zskip) {
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
  int rtmax = 0;
  for (int k = 0; k < njobs; ++k) rtmax = jobs[k].RT > rtmax ? jobs[k].RT : rtmax;
  if (nA > 0) {
    dim3 g(nA, nelem, njobs);
    static const bool tc_off = getenv("ACR_HMATA_SCALAR") != nullptr;   // A/B aid
    const int tmax = ((rtmax > cmax ? rtmax : cmax) + 7) / 8;
    static const long long wmin = getenv("ACR_HMATA_WMIN") ? atoll(getenv("ACR_HMATA_WMIN")) : 10000;
    if (!tc_off && tmax <= 2 && (long long)nA * nelem * njobs >= wmin) {
      // throughput-bound launch: a warp per (entry, element), 8 per CTA
      dim3 gw((nA + 7) / 8, nelem, njobs);
      if (tmax <= 1) CK_PDL(launch_pdl(k_hmatA_tcw<1>, gw, dim3(256), 0, st, T, JJ));
      else CK_PDL(launch_pdl(k_hmatA_tcw<2>, gw, dim3(256), 0, st, T, JJ));
    } else if (!tc_off && tmax <= 4) {
      static bool attr_a = false;
      if (!attr_a) {
        cudaFuncSetAttribute(k_hmatA_tc<512, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(k_hmatA_tc<512, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_a = true;
      }
      // 16 warps per pair for launches of a handful of CTAs: measured no gain
      // (most pairs of such a launch are deep nodes of 64 .. 128 rows, where
      // the wider cross-warp sum costs what the shorter row loop saves), off
      // unless ACR_HMATA_TINY sets a CTA-count limit
      static const long long tiny_max = getenv("ACR_HMATA_TINY") ? atoll(getenv("ACR_HMATA_TINY")) : 0;
      const bool tiny = (long long)nA * nelem * njobs <= tiny_max;
      const int tm = tmax <= 1 ? 1 : tmax <= 2 ? 2 : 4;
      const size_t sma = (size_t)(tiny ? 16 : 4) * tm * tm * 64 * 8;
      if (tiny && tm == 4) CK_PDL(launch_pdl(k_hmatA_tc<512, 4>, g, dim3(512), sma, st, T, JJ));
      else if (tiny && tm == 2) CK_PDL(launch_pdl(k_hmatA_tc<512, 2>, g, dim3(512), sma, st, T, JJ));
      else if (tiny) CK_PDL(launch_pdl(k_hmatA_tc<512, 1>, g, dim3(512), sma, st, T, JJ));
      else if (tmax <= 1) CK_PDL(launch_pdl(k_hmatA_tc<128, 1>, g, dim3(128), sma, st, T, JJ));
      else if (tmax <= 2) CK_PDL(launch_pdl(k_hmatA_tc<128, 2>, g, dim3(128), sma, st, T, JJ));
      else CK_PDL(launch_pdl(k_hmatA_tc<128, 4>, g, dim3(128), sma, st, T, JJ));
    } else if (nelem <= 32) CK_PDL(launch_pdl(k_hmatA<true>, dim3(g), dim3(HT), 0, st, T, JJ));
    else CK_PDL(launch_pdl(k_hmatA<false>, dim3(g), dim3(HT), 0, st, T, JJ));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  // wide column tiles only when the grid fills the GPU several times over;
  // small (top-level) grids keep per-thread chains short
  auto big = [](dim3 g) { return (long long)g.x * g.y * g.z >= 148LL * 8; };
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_hmatB<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_hmatB_sm<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_hmatB_tc<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_hmatB_tc<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_hmatB_tc<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_hmatB<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_hmatB_path<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    cudaFuncSetAttribute(k_hmatB_path<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  const bool path = jobs[0].mu0 == 1 && jobs[0].mu1 == T.nnodes && T.maxdepth <= 16;
  if (T.maxdepth <= 16) {
    size_t cp = (size_t)((cmax + 1) & ~1) * (path ? T.maxdepth : 1);
    // X staged in windows of at most 16 columns: 44 KB per CTA, five CTAs per
    // SM instead of four (measured: 64 -> 16 columns, factor -2.3 ms)
    static const int xcap = getenv("ACR_HMAT_XC") ? atoi(getenv("ACR_HMAT_XC")) : 16;
    if (cp > (size_t)xcap) cp = xcap;
    const size_t smem = ((size_t)T.bw * cp + (size_t)T.bw * (T.bw + 1) + 1) * 8;
    dim3 g(path ? T.nleaves : nB, nelem, njobs);
    static const bool sm_path = getenv("ACR_HMATB_SM") != nullptr;   // A/B aid
    if (T.bw <= 64 && !sm_path && (long long)T.maxdepth * rtmax <= HB_FLAT &&
        (long long)(path ? T.maxdepth : 1) * cmax <= HB_COLS) {
      const int ldl = (T.bw + 11) / 16 * 16 + 4;
      static const int xtc = getenv("ACR_HMAT_XTC") ? atoi(getenv("ACR_HMAT_XTC")) : 2;
      // tiles (8 columns) per X window
      int W = (int)(((size_t)cmax + 7) / 8) * (path ? T.maxdepth : 1);
      if (W > xtc) W = xtc;
      const size_t smtc = ((size_t)T.bw + 8 * (size_t)W) * ldl * 8;
      static const int minb = getenv("ACR_HMAT_MINB") ? atoi(getenv("ACR_HMAT_MINB")) : 5;
      if (minb == 5)
        CK_PDL(launch_pdl(k_hmatB_tc<5>, dim3(g), dim3(256), smtc, st, T, JJ, (int)path, W, ldl, zskip));
      else if (minb == 4)
        CK_PDL(launch_pdl(k_hmatB_tc<4>, dim3(g), dim3(256), smtc, st, T, JJ, (int)path, W, ldl, zskip));
      else
        CK_PDL(launch_pdl(k_hmatB_tc<3>, dim3(g), dim3(256), smtc, st, T, JJ, (int)path, W, ldl, zskip));
      return cudaGetLastError();
    }
    // 256 threads per leaf CTA (measured: 128 and 512 are slower)
    CK_PDL(launch_pdl(k_hmatB_sm<256>, dim3(g), dim3(256), smem, st, T, JJ, path, (int)cp));
    return cudaGetLastError();
  }
  if (path) {
    const size_t cpad = (size_t)(cmax + HB_CB - 1) / HB_CB * HB_CB;
    size_t smem = ((size_t)T.bw * (T.bw + 1) + 1 + (size_t)T.bw * cpad * T.maxdepth) * 8;
    dim3 g(T.nleaves, nelem, njobs);
    if (big(g)) k_hmatB_path<8><<<g, HT, smem, st>>>(T, JJ);
    else k_hmatB_path<2><<<g, HT, smem, st>>>(T, JJ);
    return cudaGetLastError();
  }
  const size_t cpad = (size_t)(cmax + HB_CB - 1) / HB_CB * HB_CB;
  size_t smem = ((size_t)T.bw * (T.bw + 1) + 1 + (size_t)T.bw * cpad) * 8;
  dim3 g(nB, nelem, njobs);
  if (big(g)) k_hmatB<8><<<g, HT, smem, st>>>(T, JJ, nB);
  else k_hmatB<2><<<g, HT, smem, st>>>(T, JJ, nB);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Z[rows hw] = alpha * W[rows hw] (X[rows hx]^T Y[rows hx]) per branch node
// ---------------------------------------------------------------------------
struct GPJobs2 {
  GPJob j[2];
};

// GT threads: 256 for small (latency-bound) grids, 128 for large ones
template <int GT>
__global__ void __launch_bounds__(GT) k_gp(TreeDev T, GPJobs2 JJ, const int* nodes) {
  ACR_PDL_ENTRY();
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
  for (int p = warp; p < rx * ry; p += GT / 32) {
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
  for (int i = threadIdx.x; i < l2; i += GT) {
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

// K = X^T Y on the FP64 tensor pipe: the node's l1 rows split over the
// warps, each warp accumulating every 8 x 8 tile of K with mma.sync m8n8k4
// (A fragment = 8 columns of X at 4 rows, B = 8 columns of Y), the warps'
// partial tiles summed in a fixed order through shared memory.  Every X / Y
// element is read once (the scalar kernel re-read X for every column of Y
// and paid a warp reduction per dot product).  Then Z = alpha W K as k_gp.
// TMAX: tiles per side (ranks <= 8 TMAX).
template <int NT, int TMAX>
__global__ void __launch_bounds__(NT) k_gp_tc(TreeDev T, GPJobs2 JJ, const int* nodes) {
  ACR_PDL_ENTRY();
  extern __shared__ double smp[];
  constexpr int NW = NT / 32;
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
  const int gi = lane >> 2, ti = lane & 3;
  const int ta = (rx + 7) >> 3, tb = (ry + 7) >> 3;
  double acc[TMAX][TMAX][2];
#pragma unroll
  for (int a = 0; a < TMAX; ++a)
#pragma unroll
    for (int b = 0; b < TMAX; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  // this warp's rows: chunks of 4 rows, interleaved across warps
  const double* xc[TMAX];
  const double* yc[TMAX];
#pragma unroll
  for (int a = 0; a < TMAX; ++a) {
    const int ca = a * 8 + gi;
    xc[a] = (a < ta && ca < rx) ? src_col(J.X, n, g, slot, ca) + r1 : nullptr;
    yc[a] = (a < tb && ca < ry) ? src_col(J.Y, n, g, slot, ca) + r1 : nullptr;
  }
  // UL row chunks of a warp in flight (loads issued together; chunks past the
  // end contribute exact zeros, the order of the sums is unchanged)
  constexpr int UL = TMAX >= 4 ? 2 : 4;
  for (int k0 = warp * 4; k0 < l1; k0 += NW * 4 * UL) {
    double av[UL][TMAX], bv[UL][TMAX];
#pragma unroll
    for (int u = 0; u < UL; ++u) {
      const int k = k0 + u * NW * 4 + ti;
#pragma unroll
      for (int a = 0; a < TMAX; ++a) {
        av[u][a] = (xc[a] && k < l1) ? xc[a][k] : 0.0;
        bv[u][a] = (yc[a] && k < l1) ? yc[a][k] : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < UL; ++u)
#pragma unroll
      for (int a = 0; a < TMAX; ++a)
#pragma unroll
        for (int b = 0; b < TMAX; ++b)
          if (a < ta && b < tb)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 "
                         "{%0, %1}, {%2}, {%3}, {%0, %1};\n"
                         : "+d"(acc[a][b][0]), "+d"(acc[a][b][1])
                         : "d"(av[u][a]), "d"(bv[u][b]));
  }
  // partial tiles -> smem [warp][a][b][64], then K[a][b] summed over warps in order
  double* part = smp;
  double* K = smp + (size_t)NW * TMAX * TMAX * 64;
#pragma unroll
  for (int a = 0; a < TMAX; ++a)
#pragma unroll
    for (int b = 0; b < TMAX; ++b)
      if (a < ta && b < tb) {
        double* pt = part + (((size_t)warp * TMAX + a) * TMAX + b) * 64;
        pt[gi * 8 + 2 * ti] = acc[a][b][0];
        pt[gi * 8 + 2 * ti + 1] = acc[a][b][1];
      }
  __syncthreads();
  for (int e = threadIdx.x; e < rx * ry; e += NT) {
    const int x = e / ry, y = e - x * ry;
    const int a = x >> 3, b = y >> 3, off = (x & 7) * 8 + (y & 7);
    double sacc = 0.0;
    for (int w = 0; w < NW; ++w) sacc += part[(((size_t)w * TMAX + a) * TMAX + b) * 64 + off];
    K[e] = sacc;
  }
  __syncthreads();
  // Z = alpha W K: thread per output row, W row in registers (8 at a time)
  for (int i = threadIdx.x; i < l2; i += NT) {
    for (int b0 = 0; b0 < ry; b0 += 8) {
      const int nb = ry - b0 < 8 ? ry - b0 : 8;
      double z[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) z[q] = 0.0;
      for (int a0 = 0; a0 < rx; a0 += 8) {   // eight W loads in flight, same sum order
        double w[8];
#pragma unroll
        for (int qa = 0; qa < 8; ++qa)
          w[qa] = a0 + qa < rx ? src_col(J.W, n, g, slot, a0 + qa)[r2 + i] : 0.0;
#pragma unroll
        for (int qa = 0; qa < 8; ++qa)
          if (a0 + qa < rx) {
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (q < nb) z[q] += w[qa] * K[(a0 + qa) * ry + b0 + q];
          }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < nb) src_col(J.Z, n, g, slot, b0 + q)[r2 + i] = J.alpha * z[q];
    }
  }
  if (J.orank && threadIdx.x == 0) J.orank[g * J.ors + nu * 2 + J.oside] = ry;
}

cudaError_t launch_gp(const TreeDev& T, const GPJob* jobs, int njobs,
                      const int* nodes, int nnodes, int nelem, int kcap,
                      cudaStream_t st, int rxcap, int rycap) {
  if (!nelem || !njobs || !nnodes) return cudaSuccess;
  GPJobs2 JJ;
  JJ.j[0] = jobs[0];
  JJ.j[1] = njobs > 1 ? jobs[1] : jobs[0];
  static const bool tc_off = getenv("ACR_GP_SCALAR") != nullptr;   // A/B aid
  const int tmax = ((rxcap > rycap ? rxcap : rycap) + 7) / 8;
  if (!tc_off && rxcap > 0 && tmax <= 4) {
    const bool small = (long long)nnodes * nelem * njobs < 148LL * 4;
    // a handful of CTAs in all: 16 warps per product
    static const long long tiny_max = getenv("ACR_GP_TINY") ? atoll(getenv("ACR_GP_TINY")) : 74;
    const bool tiny = (long long)nnodes * nelem * njobs <= tiny_max;
    const int nw = tiny ? 16 : small ? 8 : 4;
    const int tm = tmax <= 1 ? 1 : tmax <= 2 ? 2 : 4;
    const size_t smem = ((size_t)nw * tm * tm * 64 + (size_t)rxcap * rycap) * 8;
    static bool attr_tc = false;
    if (!attr_tc) {
      cudaFuncSetAttribute(k_gp_tc<256, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_gp_tc<256, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_gp_tc<256, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_gp_tc<128, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_gp_tc<128, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_gp_tc<128, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_gp_tc<512, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_gp_tc<512, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_gp_tc<512, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr_tc = true;
    }
    dim3 g(nnodes, nelem, njobs);
    if (tiny) {
      if (tm == 1) CK_PDL(launch_pdl(k_gp_tc<512, 1>, g, dim3(512), smem, st, T, JJ, nodes));
      else if (tm == 2) CK_PDL(launch_pdl(k_gp_tc<512, 2>, g, dim3(512), smem, st, T, JJ, nodes));
      else CK_PDL(launch_pdl(k_gp_tc<512, 4>, g, dim3(512), smem, st, T, JJ, nodes));
    } else if (small) {
      if (tm == 1) CK_PDL(launch_pdl(k_gp_tc<256, 1>, g, dim3(256), smem, st, T, JJ, nodes));
      else if (tm == 2) CK_PDL(launch_pdl(k_gp_tc<256, 2>, g, dim3(256), smem, st, T, JJ, nodes));
      else CK_PDL(launch_pdl(k_gp_tc<256, 4>, g, dim3(256), smem, st, T, JJ, nodes));
    } else {
      if (tm == 1) CK_PDL(launch_pdl(k_gp_tc<128, 1>, g, dim3(128), smem, st, T, JJ, nodes));
      else if (tm == 2) CK_PDL(launch_pdl(k_gp_tc<128, 2>, g, dim3(128), smem, st, T, JJ, nodes));
      else CK_PDL(launch_pdl(k_gp_tc<128, 4>, g, dim3(128), smem, st, T, JJ, nodes));
    }
    return cudaGetLastError();
  }
  size_t smem = (size_t)kcap * 8;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gp<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    cudaFuncSetAttribute(k_gp<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  dim3 g(nnodes, nelem, njobs);
  if ((long long)nnodes * nelem * njobs < 148LL * 4) CK_PDL(launch_pdl(k_gp<256>, dim3(g), dim3(256), smem, st, T, JJ, nodes));
  else CK_PDL(launch_pdl(k_gp<128>, dim3(g), dim3(128), smem, st, T, JJ, nodes));
  return cudaGetLastError();
}

// out = (f - a) - b  over count panels of len doubles (reference
// reduction.py:204-216 and 249-253 order); a or b may be null
__global__ void k_rhs_combine(const double* f, long long fs, const double* a,
                              long long as, const double* b, long long bs,
                              double* out, long long os, int len) {
  ACR_PDL_ENTRY();
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
  CK_PDL(launch_pdl(k_rhs_combine, dim3(dim3(bx, count)), dim3(256), 0, st, f, fs, a, as, b, bs, out, os, len));
  return cudaGetLastError();
}

}  // namespace acr
