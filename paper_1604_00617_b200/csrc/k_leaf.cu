// Dense-leaf kernels of the batched HODLR arithmetic.
//   k_leafinv   leaf inverse, reference algebra.py:199-207 (np.linalg.solve(L, I)
//               with partial pivoting; singular / non-finite flagged per block);
//               k_leafinv_tri: the same for the exactly tridiagonal leaves of
//               the lifted level (banded elimination, getrf's pivot rule)
//   k_leafgemm  leaf products of multiply (algebra.py:162-163) followed by the
//               ancestors' cross terms, deepest first (algebra.py:165-168 via
//               add_lowrank's exact dense update, algebra.py:134-135)
//   k_leaflr    add_lowrank at the leaves of one subtree (algebra.py:134-135)
//   k_leafadd   add() at the leaves (algebra.py:104-105)
//   k_negate    scale(H, -1) (algebra.py:115-125)
//   k_lift*     exact lift of the bands (hodlr.py:242-314)
#include <climits>
#include <cstdlib>
#include "acr_types.cuh"
#include "acr_launch.h"
#include "acr_pdl.cuh"

namespace acr {

static constexpr int LT = 256;

// ---------------------------------------------------------------------------
// leaf inverse: in-place Gauss-Jordan with row partial pivoting (the pivot
// sequence equals getrf's: first index of the largest |a_ik|), column swaps
// undone at the end.  256 threads; thread t owns column (t mod cp) of rows
// (t / cp) + k*rs, so no runtime division in the O(s^3) loop.
// ---------------------------------------------------------------------------
static constexpr int IT = 256;

__global__ void __launch_bounds__(IT) k_leafinv(TreeDev T, const HB* H, int leaf,
                                                int* sing) {
  extern __shared__ double sm[];
  const int g = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  const int lo = T.lo[leaf], s = T.hi[leaf] - lo, bw = T.bw;
  const int ld = s + 1;
  double* A = sm;
  double* colk = A + s * ld;
  int* piv = reinterpret_cast<int*>(colk + s);
  __shared__ double pv, akk;
  __shared__ int pidx, bad;
  const int cp = s <= 32 ? 32 : (s <= 64 ? 64 : 128);
  const int rs = IT / cp;
  const int tj = tid & (cp - 1), ti0 = tid / cp;
  double* L = H[g].leaf + (long long)lo * bw;
  if (tj < s)
    for (int i = ti0; i < s; i += rs) A[i * ld + tj] = L[(long long)i * bw + tj];
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int k = 0; k < s; ++k) {
    if (tid < 32) {
      double best = -1.0;
      int bi = k;
      for (int i = k + lane; i < s; i += 32) {
        double v = fabs(A[i * ld + k]);
        if (v > best) { best = v; bi = i; }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, best, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if (lane == 0) {
        pidx = bi;
        piv[k] = bi;
        pv = A[bi * ld + k];
        akk = A[k * ld + k];
        if (pv == 0.0) bad = 1;
      }
    }
    __syncthreads();
    if (bad) break;
    const int p = pidx;
    const double inv = 1.0 / pv;
    // swap rows k <-> p and scale the new pivot row; save column k
    for (int j = tid; j < s; j += IT) {
      double rk = A[k * ld + j], rp = A[p * ld + j];
      if (p != k) A[p * ld + j] = rk;
      A[k * ld + j] = (j == k) ? inv : rp * inv;
    }
    for (int i = tid; i < s; i += IT)
      colk[i] = (i == k) ? 0.0 : (i == p ? akk : A[i * ld + k]);
    __syncthreads();
    if (tj < s) {
      const double akj = A[k * ld + tj];
      for (int i = ti0; i < s; i += rs) {
        if (i == k) continue;
        if (tj != k) A[i * ld + tj] -= colk[i] * akj;
        else A[i * ld + k] = -colk[i] * akj;
      }
    }
    __syncthreads();
  }
  if (!bad) {
    for (int k = s - 1; k >= 0; --k) {
      int p = piv[k];
      if (p != k)
        for (int i = tid; i < s; i += IT) {
          double t = A[i * ld + k];
          A[i * ld + k] = A[i * ld + p];
          A[i * ld + p] = t;
        }
      __syncthreads();
    }
    int nf = 0;
    if (tj < s)
      for (int i = ti0; i < s; i += rs) {
        double v = A[i * ld + tj];
        if (!isfinite(v)) nf = 1;
        L[(long long)i * bw + tj] = v;
      }
    if (__syncthreads_or(nf) && tid == 0) bad = 1;
  }
  __syncthreads();
  if (bad && tid == 0) {
    // leaves are numbered by row order; the reference stops at the first
    int pos = 0;
    for (int v = 0; v < T.nnodes; ++v)
      if (T.isleaf[v] && T.lo[v] < lo) ++pos;
    atomicMin(sing + g, pos);
  }
}

// Register-tiled Gauss-Jordan for leaves of size <= S (S in {16, 32, 64})
// with implicit row pivoting: rows never move; step k's pivot row is the
// unused row with the largest |a_ik| (first physical index on ties -- the
// same candidates as getrf's remaining rows), and the permutation is applied
// when the inverse is stored.  Every element does one FMA
// x -= a_rk * (row_p / pivot) (the owner of column k zeroes it first, the
// pivot row becomes the scaled row).  Shared memory carries the pivot column
// (published with the pivot search by its owner group) and the pivot row:
// two barriers per step, no full-matrix copy.
// TR x TC register tiles, S/TR row groups (<= 32: one warp segment holds a
// column group) x S/TC column groups; (4, 4) with 256 threads for batched
// (throughput) launches, (2, 2) with 1024 threads for launches with fewer
// leaves than SMs, where the pivot chain's latency is the cost.
template <int S, int TR, int TC, int MINB>
__global__ void __launch_bounds__((S / TR) * (S / TC), MINB) k_leafinv_v2(TreeDev T, const HB* H,
                                                                       int leaf, int* sing) {
  ACR_PDL_ENTRY();
  constexpr int TGY = S / TR, TGX = S / TC, NT = TGX * TGY;
  static_assert(TGY <= 32, "a column group must fit one warp");
  constexpr unsigned MASK = TGY >= 32 ? 0xffffffffu : (NT >= 32 ? 0xffffffffu : (1u << NT) - 1u);
  __shared__ double colbuf[2][S], rowP[S];
  __shared__ int piv[S + 1], kpos[S];
  const int g = blockIdx.x, tid = threadIdx.x;
  const int tx = tid / TGY, ty = tid - tx * TGY;   // column group, row group
  const int lo = T.lo[leaf], s = T.hi[leaf] - lo, bw = T.bw;
  double* L = H[g].leaf + (long long)lo * bw;
  double x[TR][TC];
#pragma unroll
  for (int a = 0; a < TR; ++a)
#pragma unroll
    for (int b = 0; b < TC; ++b) {
      const int r = ty * TR + a, c = tx * TC + b;
      x[a][b] = (r < s && c < s) ? L[(long long)r * bw + c] : 0.0;
    }
  // column 0 and its pivot: the warp holding column group 0 (every lane takes
  // part in the shuffles; only column group 0 publishes)
  if (tid < 32) {
    double best = -1.0;
    int pb = 0;
#pragma unroll
    for (int a = 0; a < TR; ++a) {
      const int r = ty * TR + a;
      if (tx == 0) colbuf[0][r] = x[a][0];
      const double v = fabs(x[a][0]);
      if (r < s && v > best) { best = v; pb = r; }
    }
#pragma unroll
    for (int o = TGY / 2; o; o >>= 1) {
      const double ov = __shfl_xor_sync(MASK, best, o);
      const int oi = __shfl_xor_sync(MASK, pb, o);
      if (ov > best || (ov == best && oi < pb)) { best = ov; pb = oi; }
    }
    if (tx == 0 && ty == 0) piv[0] = pb;
  }
  bool bad = false;
  unsigned used = 0;                            // bit a: row ty TR + a has been a pivot
  for (int k = 0; k < s; ++k) {
    __syncthreads();                            // colbuf[k & 1], piv[k]
    const int p = piv[k];
    const double* cb = colbuf[k & 1];
    const double pv = cb[p];
    if (pv == 0.0) { bad = true; break; }       // uniform
    if (ty == p / TR) {                         // pivot row p (select chain: x stays in registers)
      const int ap = p % TR;
#pragma unroll
      for (int b = 0; b < TC; ++b) {
        double v = x[0][b];
#pragma unroll
        for (int a = 1; a < TR; ++a) v = ap == a ? x[a][b] : v;
        rowP[tx * TC + b] = v;
      }
      used |= 1u << ap;
    }
    __syncthreads();
    const double inv = 1.0 / pv;
    double rk[TC];
#pragma unroll
    for (int b = 0; b < TC; ++b) {
      const int c = tx * TC + b;
      rk[b] = (c == k) ? inv : rowP[c] * inv;   // the pivot row, scaled
    }
    if (tx == k / TC) {                         // column k acts as zero
      const int bk = k % TC;
#pragma unroll
      for (int a = 0; a < TR; ++a)
#pragma unroll
        for (int b = 0; b < TC; ++b) x[a][b] = bk == b ? 0.0 : x[a][b];
    }
#pragma unroll
    for (int a = 0; a < TR; ++a) {
      const double f = cb[ty * TR + a];
      const bool isp = ty * TR + a == p;
#pragma unroll
      for (int b = 0; b < TC; ++b) x[a][b] = isp ? rk[b] : x[a][b] - f * rk[b];
    }
    const int kn = k + 1;                       // next pivot by column kn's owners
    if (kn < s && (tid >> 5) == ((kn / TC) * TGY) >> 5) {
      const bool own = tx == kn / TC;
      const int bn = kn % TC;
      double best = -1.0;
      int pb = kn;
#pragma unroll
      for (int a = 0; a < TR; ++a) {
        double v = x[a][0];
#pragma unroll
        for (int b = 1; b < TC; ++b) v = bn == b ? x[a][b] : v;
        const int r = ty * TR + a;
        if (own) colbuf[kn & 1][r] = v;
        if (!((used >> a) & 1u) && r < s && fabs(v) > best) { best = fabs(v); pb = r; }
      }
#pragma unroll
      for (int o = TGY / 2; o; o >>= 1) {
        const double ov = __shfl_xor_sync(MASK, best, o);
        const int oi = __shfl_xor_sync(MASK, pb, o);
        if (ov > best || (ov == best && oi < pb)) { best = ov; pb = oi; }
      }
      if (own && ty == 0) piv[kn] = pb;
    }
  }
  if (bad) {
    if (tid == 0) {
      int ps = 0;
      for (int v = 0; v < T.nnodes; ++v)
        if (T.isleaf[v] && T.lo[v] < lo) ++ps;
      atomicMin(sing + g, ps);
    }
    return;
  }
  __syncthreads();
  // implicit pivoting: step k used physical row piv[k], so
  // A^{-1}[kpos(r)][piv(c)] = X[r][c] with kpos(piv[k]) = k
  for (int j = tid; j < s; j += NT) kpos[piv[j]] = j;
  __syncthreads();
  int nf = 0;
#pragma unroll
  for (int a = 0; a < TR; ++a)
#pragma unroll
    for (int b = 0; b < TC; ++b) {
      const int r = ty * TR + a, c = tx * TC + b;
      if (r < s && c < s) {
        if (!isfinite(x[a][b])) nf = 1;
        L[(long long)kpos[r] * bw + piv[c]] = x[a][b];
      }
    }
  if (__syncthreads_or(nf) && tid == 0) {
    int ps = 0;
    for (int v = 0; v < T.nnodes; ++v)
      if (T.isleaf[v] && T.lo[v] < lo) ++ps;
    atomicMin(sing + g, ps);
  }
}

// ---------------------------------------------------------------------------
// Blocked Gauss-Jordan leaf inverse for 33..64-row leaves, trailing updates
// on the FP64 tensor pipe (mma.sync.m8n8k4.f64 -> DMMA).  Same pivot rule
// and implicit row pivoting as k_leafinv_v2 (step k's pivot is the unused row
// with the largest |x_ik|, first index on ties; rows never move; the
// permutation is applied at the store).  Columns are taken in panels of 8:
//   1. one warp runs the 8 unblocked Gauss-Jordan steps on the 64 x 8 panel
//      (rows lane and lane + 32 in registers, warp-shuffle pivot search and
//      pivot-row broadcast: no CTA barrier on the pivot chain);
//   2. T = the panel's pivot rows of every other column (8 x 64, copied);
//   3. every other 8 x 8 tile: X <- (X with the panel's pivot rows zeroed)
//      + P T, two DMMAs per tile (k = 8) -- the 8 elementary GJ transforms
//      composed, E = I + (E - I)[:, pivots], whose columns are exactly the
//      panel's final values (in-place GJ stores E e_p in column k).
// The non-panel columns therefore get one rank-8 update per panel instead of
// eight rank-1 updates: the same algorithm up to the FP summation order.
// ---------------------------------------------------------------------------
static constexpr int BGJ_LD = 68;       // padded row stride (doubles)

// one 8-column panel of unblocked Gauss-Jordan steps by one warp (see above)
__device__ __forceinline__ void bgj_panel(double* X, int pq, int s, int lane, unsigned& used,
                                          int* piv, int* pflag, int* s_bad) {
  const int kq = pq * 8;
      double x[2][8];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < 8; ++c) x[h][c] = X[(lane + 32 * h) * BGJ_LD + kq + c];
      bool bad = false;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        if (kq + t < s && !bad) {
          // warp argmax of |x| over the unused rows, first index on ties, by
          // integer warp reductions on the bit pattern (monotone for
          // non-negative doubles): max of the high words, then of the low
          // words among the lanes holding that high word, then the smallest
          // row index holding both -- exact, no floating compares on the chain
          double best = -1.0;
          int pi = 64;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = lane + 32 * h;
            const double v = fabs(x[h][t]);
            if (r < s && !((used >> h) & 1u) && v > best) { best = v; pi = r; }
          }
          const unsigned long long bb = best < 0.0 ? 0ull : (unsigned long long)__double_as_longlong(best) + 1ull;
          const unsigned hi = (unsigned)(bb >> 32), lw = (unsigned)bb;
          const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
          const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lw : 0u);
          pi = (int)__reduce_min_sync(0xffffffffu, (hi == mhi && lw == mlo) ? (unsigned)pi : 64u);
          const int hp = pi >> 5, lp = pi & 31;
          double rowp[8];
#pragma unroll
          for (int c = 0; c < 8; ++c)
            rowp[c] = __shfl_sync(0xffffffffu, hp ? x[1][c] : x[0][c], lp);
          const double pv = rowp[t];
          if (pv == 0.0) {
            bad = true;                     // uniform
          } else {
            const double inv = __drcp_rn(pv);   // == 1.0 / pv (both correctly rounded)
            double rk[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) rk[c] = c == t ? inv : rowp[c] * inv;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const bool isp = lane + 32 * h == pi;
              const double f = x[h][t];
              x[h][t] = 0.0;
#pragma unroll
              for (int c = 0; c < 8; ++c) x[h][c] = isp ? rk[c] : x[h][c] - f * rk[c];
            }
            if (lane == lp) used |= 1u << hp;
            if (lane == 0) {
              piv[kq + t] = pi;
              pflag[pi] = pq;
            }
          }
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < 8; ++c) X[(lane + 32 * h) * BGJ_LD + kq + c] = x[h][c];
      if (bad && lane == 0) *s_bad = 1;
    }

template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_leafinv_bgj(TreeDev T, const HB* H, int leaf,
                                                         int* sing) {
  ACR_PDL_ENTRY();
  constexpr int NW = NT / 32;
  __shared__ __align__(16) double X[64 * BGJ_LD];
  __shared__ __align__(16) double Tb[8 * BGJ_LD];
  __shared__ int piv[64], kpos[64], pflag[64];
  __shared__ int s_bad;
  const int g = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lo = T.lo[leaf], s = T.hi[leaf] - lo, bw = T.bw;
  double* L = H[g].leaf + (long long)lo * bw;
  {
    // every load of a thread in flight before the first shared store (a
    // load-store loop kept one global round trip per element on the chain)
    constexpr int PT = 64 * 64 / NT;
    double v[PT];
#pragma unroll
    for (int u = 0; u < PT; ++u) {
      const int idx = tid + u * NT, r = idx >> 6, c = idx & 63;
      v[u] = (r < s && c < s) ? __ldg(L + (long long)r * bw + c) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < PT; ++u) {
      const int idx = tid + u * NT;
      X[(idx >> 6) * BGJ_LD + (idx & 63)] = v[u];
    }
  }
  if (tid < 64) pflag[tid] = -1;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  unsigned used = 0;                        // warp 0: bit h = row lane + 32 h pivoted
  const int gi = lane >> 2, ti = lane & 3;
  const int npan = (s + 7) / 8;
  if (warp == 0) bgj_panel(X, 0, s, lane, used, piv, pflag, &s_bad);
  __syncthreads();
  for (int pb = 0; pb < npan && !s_bad; ++pb) {
    const int k0 = pb * 8;
    // ---- T = pivot rows of panel pb in every other column ----
    const int np = s - k0 < 8 ? s - k0 : 8;
    for (int idx = tid; idx < 8 * 64; idx += NT) {
      const int t = idx >> 6, c = idx & 63;
      Tb[t * BGJ_LD + c] = t < np ? X[piv[k0 + t] * BGJ_LD + c] : 0.0;
    }
    __syncthreads();
    // rank-8 update of tile (rb, cb) on DMMA: X <- (X, panel pb's pivot rows
    // zeroed) + P T
    auto upd = [&](int rb, int cb) {
      const int r = rb * 8 + gi, c = cb * 8 + 2 * ti;
      const bool zr = pflag[r] == pb;
      double d0 = zr ? 0.0 : X[r * BGJ_LD + c];
      double d1 = zr ? 0.0 : X[r * BGJ_LD + c + 1];
#pragma unroll
      for (int kk = 0; kk < 8; kk += 4) {
        const double av = X[r * BGJ_LD + k0 + kk + ti];
        const double bv = Tb[(kk + ti) * BGJ_LD + cb * 8 + gi];
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 "
                     "{%0, %1}, {%2}, {%3}, {%0, %1};\n"
                     : "+d"(d0), "+d"(d1) : "d"(av), "d"(bv));
      }
      X[r * BGJ_LD + c] = d0;
      X[r * BGJ_LD + c + 1] = d1;
    };
    if (pb + 1 < npan && NW == 8) {
      // look-ahead: the next panel's column block first (one tile per warp),
      // then warp 0 factors panel pb + 1 while the other warps update the rest
      upd(warp, pb + 1);
      __syncthreads();
      if (warp == 0) {
        bgj_panel(X, pb + 1, s, lane, used, piv, pflag, &s_bad);
      } else {
        for (int tl = warp - 1; tl < 64; tl += NW - 1) {
          const int rb = tl >> 3, cb = tl & 7;
          if (cb != pb && cb != pb + 1) upd(rb, cb);
        }
      }
    } else {
      for (int tl = warp; tl < 64; tl += NW) {
        const int rb = tl >> 3, cb = tl & 7;
        if (cb != pb) upd(rb, cb);
      }
      __syncthreads();
      if (pb + 1 < npan && warp == 0) bgj_panel(X, pb + 1, s, lane, used, piv, pflag, &s_bad);
    }
    __syncthreads();
  }
  if (s_bad) {
    if (tid == 0) {
      int ps = 0;
      for (int v = 0; v < T.nnodes; ++v)
        if (T.isleaf[v] && T.lo[v] < lo) ++ps;
      atomicMin(sing + g, ps);
    }
    return;
  }
  for (int j = tid; j < s; j += NT) kpos[piv[j]] = j;
  __syncthreads();
  int nf = 0;
  for (int idx = tid; idx < s * s; idx += NT) {
    const int r = idx / s, c = idx - r * s;
    const double v = X[r * BGJ_LD + c];
    if (!isfinite(v)) nf = 1;
    L[(long long)kpos[r] * bw + piv[c]] = v;
  }
  if (__syncthreads_or(nf) && tid == 0) {
    int ps = 0;
    for (int v = 0; v < T.nnodes; ++v)
      if (T.isleaf[v] && T.lo[v] < lo) ++ps;
    atomicMin(sing + g, ps);
  }
}

template <int S>
static cudaError_t leafinv_reg(const TreeDev& T, const HB* H, int nelem, int leaf,
                               int* sing, cudaStream_t st) {
  CK_PDL(launch_pdl(k_leafinv_v2<S, 4, 4, 3>, dim3(nelem), dim3((S / 4) * (S / 4)), 0, st, T, H, leaf, sing));
  return cudaGetLastError();
}

// Inverse of a TRIDIAGONAL leaf (the lifted level: D is given by its three
// bands and the Schur complements of its inversion only change a corner
// entry, so every leaf a level-0 inversion meets is exactly tridiagonal).
// Elimination with partial pivoting restricted to the band -- the pivot choice
// of getrf on such a matrix (rows k and k+1 are the only candidates, the
// first maximum wins), LAPACK dgttrf's recurrences -- by one thread, then
// thread j solves for column j of the inverse (dgtts2).  O(s^2) per leaf
// instead of 2 s^3.  The structure is checked while the leaf is read: any
// nonzero off the band raises `fail` (the level is then redone with the
// dense kernel), so a wrong assumption cannot produce a wrong inverse.
static constexpr int TRI_FAIL = 1 << 28;

__global__ void __launch_bounds__(64) k_leafinv_tri(TreeDev T, const HB* H, int leaf, int* sing,
                                                    int* fail) {
  ACR_PDL_ENTRY();
  const int g = blockIdx.x, tid = threadIdx.x, bw = T.bw;
  const int lo = T.lo[leaf], s = T.hi[leaf] - lo;
  double* L = H[g].leaf + (long long)lo * bw;
  __shared__ double dl[64], dd[64], du[64], du2[64], rd[64];
  __shared__ int ip[64];
  __shared__ int s_bad;
  // read the leaf by rows (coalesced), keep the band, check the rest
  bool nz = false;
  if (tid == 0) s_bad = 0;
  if (tid < s) { dl[tid] = 0.0; du[tid] = 0.0; du2[tid] = 0.0; }
  __syncthreads();
  // (all the loads of a 32-row half issued before any of them is used: one
  // trip to memory per half instead of one per row)
#pragma unroll
  for (int h0 = 0; h0 < 64; h0 += 32) {
    double v[32];
#pragma unroll
    for (int q = 0; q < 32; ++q)
      v[q] = (tid < s && h0 + q < s) ? L[(long long)(h0 + q) * bw + tid] : 0.0;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int r = h0 + q;
      if (r < s) {
        if (tid == r) dd[r] = v[q];
        else if (tid == r - 1) dl[tid] = v[q];   // sub-diagonal entry (r, r-1) -> dl[r-1]
        else if (tid == r + 1) du[r] = v[q];     // super-diagonal entry (r, r+1) -> du[r]
        else if (v[q] != 0.0) nz = true;
      }
    }
  }
  if (__syncthreads_or(nz)) {
    if (tid == 0) atomicMax(fail, TRI_FAIL);
    return;
  }
  if (tid == 0) {
    // the running diagonal and super-diagonal entries stay in registers (the
    // chain of a step is one division and one FMA; the band loads of the next
    // step do not depend on it)
    int bad = 0;
    double dk = dd[0], uk = s > 1 ? du[0] : 0.0;        // d(k), du(k) as updated so far
    for (int k = 0; k + 1 < s; ++k) {
      const double lk = dl[k], dn = dd[k + 1];
      const double un = k + 2 < s ? du[k + 1] : 0.0;
      if (fabs(dk) >= fabs(lk)) {                // no interchange
        ip[k] = 0;
        double dn2 = dn;
        if (dk != 0.0) {
          const double f = lk / dk;
          dl[k] = f;
          dn2 = dn - f * uk;
        } else {
          bad = 1;
        }
        dd[k] = dk;
        du[k] = uk;
        du2[k] = 0.0;
        dk = dn2;
        uk = un;
      } else {                                   // rows k, k+1 interchanged
        const double f = dk / lk;
        dd[k] = lk;
        dl[k] = f;
        du[k] = dn;
        du2[k] = un;                             // (zero beyond the band's end)
        ip[k] = 1;
        dk = uk - f * dn;
        uk = -f * un;
      }
    }
    if (s > 0) dd[s - 1] = dk;
    for (int k = 0; k < s; ++k)
      if (dd[k] == 0.0) bad = 1;
    s_bad = bad;
  }
  __syncthreads();
  if (s_bad) {
    if (tid == 0) {
      int ps = 0;
      for (int v = 0; v < T.nnodes; ++v)
        if (T.isleaf[v] && T.lo[v] < lo) ++ps;
      atomicMin(sing + g, ps);
    }
    return;
  }
  if (tid < s) rd[tid] = 1.0 / dd[tid];
  __syncthreads();
  int nf = 0;
  if (tid < s) {
    // The right-hand side e_tid lives in column tid of the leaf itself (every
    // thread has read what it needs of the input; a store by this thread is
    // only ever read back by this thread): no shared-memory copy, so a dozen
    // CTAs fit an SM.
    double* b = L + tid;                         // b(i) = L[i * bw + tid]
    // forward: L and the interchanges; entries above tid - 1 are zero (not
    // stored), the running entry b(k) is carried in a register
    const int k0 = tid > 0 ? tid - 1 : 0;
    double bk = k0 == tid ? 1.0 : 0.0;           // b(k0)
    for (int k = k0; k + 1 < s; ++k) {
      const double bn = k + 1 == tid ? 1.0 : 0.0;   // b(k+1) before the step (untouched so far)
      if (!ip[k]) {
        b[(long long)k * bw] = bk;
        bk = bn - dl[k] * bk;
      } else {
        b[(long long)k * bw] = bn;
        bk = bk - dl[k] * bn;
      }
    }
    // back: U with two super-diagonals, x(i+1) and x(i+2) carried in
    // registers; the forward results come back 16 rows at a time
    double x1 = bk * rd[s - 1], x2 = 0.0;
    if (!isfinite(x1)) nf = 1;
    b[(long long)(s - 1) * bw] = x1;
    for (int i0 = s - 2; i0 >= 0; i0 -= 16) {
      double y[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int i = i0 - q;
        y[q] = (i >= k0) ? b[(long long)i * bw] : 0.0;   // i >= k0 >= 0
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int i = i0 - q;
        if (i >= 0) {
          const double x = (y[q] - du[i] * x1 - du2[i] * x2) * rd[i];
          if (!isfinite(x)) nf = 1;
          b[(long long)i * bw] = x;
          x2 = x1;
          x1 = x;
        }
      }
    }
  }
  if (__syncthreads_or(nf) && tid == 0) {
    int ps = 0;
    for (int v = 0; v < T.nnodes; ++v)
      if (T.isleaf[v] && T.lo[v] < lo) ++ps;
    atomicMin(sing + g, ps);
  }
}

cudaError_t launch_leafinv_tri(const TreeDev& T, const HB* H, int nelem, int leaf, int* sing,
                               int* fail, cudaStream_t st) {
  if (!nelem) return cudaSuccess;
  if (T.bw > 64) return cudaErrorInvalidValue;
  CK_PDL(launch_pdl(k_leafinv_tri, dim3(nelem), dim3(64), 0, st, T, H, leaf, sing, fail));
  return cudaGetLastError();
}

cudaError_t launch_leafinv(const TreeDev& T, const HB* H, int nelem, int leaf,
                           int* sing, cudaStream_t st) {
  if (!nelem) return cudaSuccess;
  int s = T.bw;
  if (s <= 16) return leafinv_reg<16>(T, H, nelem, leaf, sing, st);
  if (s <= 32) return leafinv_reg<32>(T, H, nelem, leaf, sing, st);
  if (s <= 64) {
    static const int bgj = getenv("ACR_LEAFINV_GJ") ? 0 : 1;   // A/B aid: 0 = unblocked v2
    if (bgj && s > 32) {
      // 256 threads, three CTAs per SM (measured: 128-thread CTAs at five per
      // SM are slower for batched launches too, 126 vs 85 us per 1024 leaves)
      // ... except when the batch would take a third wave at three per SM
      // (444 CTAs) and not at four: 64 registers, a few spills, one wave less
      static const int four = getenv("ACR_LEAFINV_4") ? atoi(getenv("ACR_LEAFINV_4")) : 445;
      if (four > 0 && nelem >= four)
        CK_PDL(launch_pdl(k_leafinv_bgj<256, 4>, dim3(nelem), dim3(256), 0, st, T, H, leaf, sing));
      else
        CK_PDL(launch_pdl(k_leafinv_bgj<256, 3>, dim3(nelem), dim3(256), 0, st, T, H, leaf, sing));
      return cudaGetLastError();
    }
    return leafinv_reg<64>(T, H, nelem, leaf, sing, st);
  }
  size_t smem = (size_t)s * (s + 1) * 8 + (size_t)s * 8 + (size_t)s * 4 + 16;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_leafinv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  k_leafinv<<<nelem, IT, smem, st>>>(T, H, leaf, sing);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// leaf GEMM + ancestor cross terms
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(LT) k_leafgemm(TreeDev T, const HB* A,
                                                 const HB* B, const HB* C,
                                                 Src PX, RankRef xr) {
  extern __shared__ double sm[];
  const int g = blockIdx.y, tid = threadIdx.x;
  const int lam = T.listB[(T.startB[0] + blockIdx.x) * 2 + 1];
  const int lo = T.lo[lam], s = T.hi[lam] - lo, bw = T.bw, n = T.n;
  double* a = sm;
  double* b = a + s * s;
  const double* La = A[g].leaf + (long long)lo * bw;
  const double* Lb = B[g].leaf + (long long)lo * bw;
  for (int idx = tid; idx < s * s; idx += LT) {
    int i = idx / s, j = idx - i * s;
    a[idx] = La[(long long)i * bw + j];
    b[idx] = Lb[(long long)i * bw + j];
  }
  __syncthreads();
  const HB bb = B[g];
  const int* cr = rank_base(xr, g);
  double* Lc = C[g].leaf + (long long)lo * bw;
  for (int idx = tid; idx < s * s; idx += LT) {
    int i = idx / s, j = idx - i * s;
    double acc = 0.0;
    for (int l = 0; l < s; ++l) acc += a[i * s + l] * b[l * s + j];
    int child = lam;
    for (int al = T.parent[lam]; al >= 0; child = al, al = T.parent[al]) {
      int r = cr[al * 2 + (child == T.c0[al] ? 0 : 1)];
      if (!r) continue;
      int slot = T.depth[al];
      const double* P = src_col(PX, n, g, slot, 0) + lo;
      const double* Q = bb.V + (long long)slot * bb.R * n + lo;
      double z = 0.0;
      for (int c = 0; c < r; ++c) z += P[(long long)c * n + i] * Q[(long long)c * n + j];
      acc = acc + z;
    }
    Lc[(long long)i * bw + j] = acc;
  }
}

// ---------------------------------------------------------------------------
// leaf GEMM on the FP64 tensor pipe: mma.sync.m8n8k4.f64 (SASS DMMA).
// One CTA of 8 warps per (leaf, element); the leaf is zero-padded to S (a
// multiple of 8, <= 64) in shared memory, A row-major and B column-major so
// both fragments are 8x4 row-contiguous reads.  Ancestor cross terms
// (P Q^T, rank r, deepest first) are separate tensor-core products added to
// C one at a time, the reference's order (algebra.py:165-168, 134-135).
// diag: 1 = A diagonal, 2 = B diagonal (level 0, exact fast path).
// ---------------------------------------------------------------------------
static constexpr int GT = 256;
static constexpr int GLD = 68;           // padded leading dimension (doubles)

// TMA bulk copies (cp.async.bulk, global -> shared, completion counted in
// bytes on an mbarrier) for the leaf staging of k_leafgemm_tc
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
      ::"r"(d), "l"(src), "r"(bytes), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done) : "r"(a), "r"(phase) : "memory");
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 "
               "{%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// warp tile block: 2 x 4 tiles of 8x8 (16 x 32 outputs); 8 warps cover 64x64.
// A fragment: A[r][k] (row-major sa), B fragment: B[k][c] (row-major sb).
__device__ __forceinline__ void dmma_block(double (&acc)[2][4][2], const double* sa,
                                           const double* sb, int r0, int c0, int K,
                                           int gi, int ti, int K0 = 0) {
  for (int k = K0; k < K; k += 4) {
    double a0 = sa[(r0 + gi) * GLD + k + ti];
    double a1 = sa[(r0 + 8 + gi) * GLD + k + ti];
    double b[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) b[q] = sb[(k + ti) * GLD + c0 + q * 8 + gi];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      dmma(acc[0][q][0], acc[0][q][1], a0, b[q]);
      dmma(acc[1][q][0], acc[1][q][1], a1, b[q]);
    }
  }
}

__global__ void __launch_bounds__(GT, 2) k_leafgemm_tc(TreeDev T, const HB* A, const HB* B,
                                                      const HB* C, Src PX, RankRef xr,
                                                      int diag) {
  ACR_PDL_ENTRY();
  extern __shared__ double sm[];
  double* sa = sm;                 // [64][GLD]  A rows       (P for cross terms)
  double* sb = sa + 64 * GLD;      // [64][GLD]  B rows       (Q^T for cross terms)
  const int g = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lam = T.listB[(T.startB[0] + blockIdx.x) * 2 + 1];
  const int lo = T.lo[lam], s = T.hi[lam] - lo, bw = T.bw, n = T.n;
  const int S = (s + 7) & ~7;
  const double* La = A[g].leaf + (long long)lo * bw;
  const double* Lb = B[g].leaf + (long long)lo * bw;
  double* Lc = C[g].leaf + (long long)lo * bw;
  if (diag) {                      // exact: C = diag(a) B or A diag(b)
    if (s == 64 && (bw & 1) == 0) {  // 16-byte rows, shifts instead of divisions
      // the diagonal operand's 64 values staged once (each was otherwise a
      // separate sector load repeated by every thread of its row / column)
      const double* Ld = diag == 1 ? La : Lb;
      if (tid < 64) sa[tid] = Ld[(long long)tid * bw + tid];
      __syncthreads();
      const double* Lm = diag == 1 ? Lb : La;
      for (int idx = tid; idx < 64 * 32; idx += GT) {
        const int i = idx >> 5, j = (idx & 31) * 2;
        const double2 x = *reinterpret_cast<const double2*>(Lm + (long long)i * bw + j);
        const double2 v = diag == 1 ? make_double2(sa[i] * x.x, sa[i] * x.y)
                                    : make_double2(x.x * sa[j], x.y * sa[j + 1]);
        *reinterpret_cast<double2*>(Lc + (long long)i * bw + j) = v;
      }
      return;
    }
    for (int idx = tid; idx < s * s; idx += GT) {
      const int i = idx / s, j = idx - i * s;
      Lc[(long long)i * bw + j] = diag == 1
          ? La[(long long)i * bw + i] * Lb[(long long)i * bw + j]
          : La[(long long)i * bw + j] * Lb[(long long)j * bw + j];
    }
    return;                        // level-0 couplings have rank-0 factors
  }
  __shared__ __align__(8) unsigned long long lbar;
  const bool tma = s == 64 && (bw & 1) == 0;
  if (tma) {
    // TMA: one 512-byte bulk copy per leaf row into the padded rows (GLD:
    // conflict-free DMMA fragment reads), 128 copies on one mbarrier that
    // counts the 64 KB of both leaves, issued by 16 lanes of every warp
    if (tid == 32) {
      mbar_init(&lbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (tid == 32) mbar_expect_tx(&lbar, 2u * 64u * 64u * 8u);
    if (lane < 16) {                 // 128 row copies issued by 8 warps x 16 lanes
      const int i = warp * 8 + (lane & 7);
      if (lane < 8) bulk_g2s(sa + i * GLD, La + (long long)i * bw, 512u, &lbar);
      else bulk_g2s(sb + i * GLD, Lb + (long long)i * bw, 512u, &lbar);
    }
  } else {
    for (int idx = tid; idx < 64 * 64; idx += GT) {
      const int i = idx >> 6, j = idx & 63;
      const bool in = i < s && j < s;
      cp_async8(sa + i * GLD + j, in ? La + (long long)i * bw + j : La, in);
      cp_async8(sb + i * GLD + j, in ? Lb + (long long)i * bw + j : Lb, in);
    }
  }
  // ancestor table (parent first), built once per CTA by the first warp while
  // the leaves land: lane t holds ancestor t + 1 of the leaf; its rank, slot
  // and staging offset (prefix of padded ranks over the nonzero ones)
  __shared__ int a_r[32], a_slot[32], a_off[32], a_cnt, a_tot;
  const int* cr = rank_base(xr, g);
  if (warp == 0) {
    const int* an = T.anc + lam * (T.maxdepth + 1);
    const int dl = T.depth[lam];
    int r = 0, slot = 0;
    if (lane < dl) {
      const int al = an[lane + 1], ch = an[lane];
      r = cr[al * 2 + (ch == T.c0[al] ? 0 : 1)];
      slot = T.depth[al];
    }
    const unsigned m = __ballot_sync(0xffffffffu, r != 0);
    const int pos = __popc(m & ((1u << lane) - 1u));
    const int rp = (r + 3) & ~3;
    int incl = rp;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (r) {
      a_r[pos] = r;
      a_slot[pos] = slot;
      a_off[pos] = incl - rp;
    }
    if (lane == 31) {
      a_cnt = __popc(m);
      a_tot = incl;
    }
  }
  cp_async_wait_all();
  if (tma) mbar_wait(&lbar, 0);
  __syncthreads();
  const int gi = lane >> 2, ti = lane & 3;
  const int r0 = (warp >> 1) * 16, c0 = (warp & 1) * 32;   // 4 x 2 warp grid
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[a][q][0] = acc[a][q][1] = 0.0;
  dmma_block(acc, sa, sb, r0, c0, S, gi, ti);
  // ancestor cross terms, parent first: acc += P Q^T, one ancestor at a time
  const HB bb = B[g];
  // every ancestor's P and Q^T in one staging phase when their padded ranks
  // fit the 64 columns of sa / sb (the usual case); the products are still
  // formed and added one ancestor at a time, parent first
  const int tot = a_tot, na = a_cnt;
  if (tot > 0 && tot <= 64) {
    __syncthreads();                             // main product done with sa / sb
    for (int t = 0; t < na; ++t) {
      const int r = a_r[t], rp = (r + 3) & ~3, slot = a_slot[t], off = a_off[t];
      const double* P = src_col(PX, n, g, slot, 0) + lo;
      const double* Q = bb.V + (long long)slot * bb.R * n + lo;
      for (int idx = tid; idx < 64 * rp; idx += GT) {
        const int c = idx / 64, i = idx - c * 64;
        const bool in = i < s && c < r;
        cp_async8(sa + i * GLD + off + c, in ? P + (long long)c * n + i : P, in);
        cp_async8(sb + (off + c) * GLD + i, in ? Q + (long long)c * n + i : Q, in);
      }
    }
    cp_async_wait_all();
    __syncthreads();
    for (int t = 0; t < na; ++t) {
      const int rp = (a_r[t] + 3) & ~3, off = a_off[t];
      double z[2][4][2];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int q = 0; q < 4; ++q) z[a][q][0] = z[a][q][1] = 0.0;
      dmma_block(z, sa, sb, r0, c0, off + rp, gi, ti, off);
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc[a][q][0] = acc[a][q][0] + z[a][q][0];
          acc[a][q][1] = acc[a][q][1] + z[a][q][1];
        }
    }
  }
  int child = lam;
  for (int al = T.parent[lam]; tot > 64 && al >= 0; child = al, al = T.parent[al]) {
    const int r = cr[al * 2 + (child == T.c0[al] ? 0 : 1)];
    if (!r) continue;
    const int slot = T.depth[al];
    const double* P = src_col(PX, n, g, slot, 0) + lo;
    const double* Q = bb.V + (long long)slot * bb.R * n + lo;
    double z[2][4][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int q = 0; q < 4; ++q) z[a][q][0] = z[a][q][1] = 0.0;
    for (int k0 = 0; k0 < r; k0 += 64) {       // ranks above 64 in chunks
      const int kr = r - k0 < 64 ? r - k0 : 64;
      const int rp = (kr + 3) & ~3;
      __syncthreads();
      for (int idx = tid; idx < 64 * rp; idx += GT) {
        const int c = idx / 64, i = idx - c * 64;             // coalesced in i
        const bool in = i < s && c < kr;
        cp_async8(sa + i * GLD + c, in ? P + (long long)(k0 + c) * n + i : P, in);   // P[i][c]
        cp_async8(sb + c * GLD + i, in ? Q + (long long)(k0 + c) * n + i : Q, in);   // Q^T[c][i]
      }
      cp_async_wait_all();
      __syncthreads();
      dmma_block(z, sa, sb, r0, c0, rp, gi, ti);
    }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[a][q][0] = acc[a][q][0] + z[a][q][0];
        acc[a][q][1] = acc[a][q][1] + z[a][q][1];
      }
  }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = r0 + a * 8 + gi, j = c0 + q * 8 + ti * 2;
      if (i < s) {
        if (j < s) Lc[(long long)i * bw + j] = acc[a][q][0];
        if (j + 1 < s) Lc[(long long)i * bw + j + 1] = acc[a][q][1];
      }
    }
}

// level-0 leaf products with an exact diagonal operand (E, F lifted from the
// bands: rank-0 factors, diagonal leaves): C = diag(a) B (diag 1) or
// A diag(b) (diag 2), a streaming kernel (no tensor work, small footprint so
// that many CTAs per SM keep the HBM busy)
__global__ void __launch_bounds__(256) k_leafgemm_diag(TreeDev T, const HB* A, const HB* B,
                                                       const HB* C, int diag) {
  ACR_PDL_ENTRY();
  __shared__ double dv[128];
  const int g = blockIdx.y, tid = threadIdx.x;
  const int lam = T.listB[(T.startB[0] + blockIdx.x) * 2 + 1];
  const int lo = T.lo[lam], s = T.hi[lam] - lo, bw = T.bw;
  const double* La = A[g].leaf + (long long)lo * bw;
  const double* Lb = B[g].leaf + (long long)lo * bw;
  double* Lc = C[g].leaf + (long long)lo * bw;
  const double* Ld = diag == 1 ? La : Lb;
  const double* Lm = diag == 1 ? Lb : La;
  if (tid < s) dv[tid] = Ld[(long long)tid * bw + tid];
  __syncthreads();
  if ((s & 1) == 0) {                          // bw is even: 16-byte rows
    const int h = s >> 1;
    for (int idx = tid; idx < s * h; idx += 256) {
      const int i = idx / h, j = 2 * (idx - i * h);
      const double2 x = *reinterpret_cast<const double2*>(Lm + (long long)i * bw + j);
      const double2 v = diag == 1 ? make_double2(dv[i] * x.x, dv[i] * x.y)
                                  : make_double2(x.x * dv[j], x.y * dv[j + 1]);
      *reinterpret_cast<double2*>(Lc + (long long)i * bw + j) = v;
    }
    return;
  }
  for (int idx = tid; idx < s * s; idx += 256) {
    const int i = idx / s, j = idx - i * s;
    const double x = Lm[(long long)i * bw + j];
    Lc[(long long)i * bw + j] = diag == 1 ? dv[i] * x : x * dv[j];
  }
}

cudaError_t launch_leafgemm(const TreeDev& T, const HB* A, const HB* B,
                            const HB* C, int nelem, Src PX, RankRef xr, int diag,
                            cudaStream_t st) {
  if (!nelem) return cudaSuccess;
  dim3 grid(T.nleaves, nelem);
  if (diag && T.bw <= 128) {
    CK_PDL(launch_pdl(k_leafgemm_diag, dim3(grid), dim3(256), 0, st, T, A, B, C, diag));
    return cudaGetLastError();
  }
  if (T.bw <= 64) {
    const size_t smem = 2ull * 64 * GLD * 8;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_leafgemm_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      attr = true;
    }
    CK_PDL(launch_pdl(k_leafgemm_tc, dim3(grid), dim3(GT), smem, st, T, A, B, C, PX, xr, diag));
    return cudaGetLastError();
  }
  size_t smem = 2ull * T.bw * T.bw * 8;
  static bool attr2 = false;
  if (!attr2) {
    cudaFuncSetAttribute(k_leafgemm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr2 = true;
  }
  k_leafgemm<<<grid, LT, smem, st>>>(T, A, B, C, PX, xr);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// add_lowrank at the leaves of subtree(mu): L += U V^T (exact dense update)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(LT) k_leaflr(TreeDev T, const HB* H, int mu,
                                               Src Us, Src Vs, RankRef rr,
                                               int node, int fside) {
  ACR_PDL_ENTRY();
  extern __shared__ double sm[];
  const int g = blockIdx.y, tid = threadIdx.x, n = T.n, bw = T.bw;
  const int* rb = rank_base(rr, g);
  int r = rb[node * 2 + fside];
  if (rb[node * 2 + 1 - fside] == 0) r = 0;
  if (!r) return;
  const int lam = T.listB[(T.startB[mu] + blockIdx.x) * 2 + 1];
  const int lo = T.lo[lam], s = T.hi[lam] - lo;
  const int slot = T.depth[node];
  const double* U = src_col(Us, n, g, slot, 0) + lo;
  const double* V = src_col(Vs, n, g, slot, 0) + lo;
  // stage the leaf rows of U and V (r columns) once: u[c][i], v[c][j];
  // loads issued in batches of 4 before their shared-memory stores
  double* u = sm;
  double* v = u + r * s;
  int nzu = 0, nzv = 0;
  for (int base = tid; base < r * s; base += 4 * LT) {
    double a[4], b[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = base + q * LT;
      const int c = idx / s, i = idx - c * s;
      a[q] = idx < r * s ? U[(long long)c * n + i] : 0.0;
      b[q] = idx < r * s ? V[(long long)c * n + i] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = base + q * LT;
      if (idx < r * s) { u[idx] = a[q]; v[idx] = b[q]; }
      nzu |= a[q] != 0.0;
      nzv |= b[q] != 0.0;
    }
  }
  // the leaf's rows of U, or of V, are exact zeros (the lifted level: a Schur
  // update W V12^T touches one corner entry of one leaf): the update adds
  // exact zeros, the leaf is neither read nor written
  if (!__syncthreads_or(nzu)) return;
  if (!__syncthreads_or(nzv)) return;
  // leaf += u v^T: 8 leaf entries per thread in flight (same sum order)
  double* L = H[g].leaf + (long long)lo * bw;
  for (int base = tid; base < s * s; base += 8 * LT) {
    double lv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int idx = base + q * LT;
      const int i = idx / s, j = idx - i * s;
      lv[q] = idx < s * s ? L[(long long)i * bw + j] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int idx = base + q * LT;
      if (idx < s * s) {
        const int i = idx / s, j = idx - i * s;
        double z = 0.0;
        for (int c = 0; c < r; ++c) z += u[c * s + i] * v[c * s + j];
        L[(long long)i * bw + j] = lv[q] + z;
      }
    }
  }
}

cudaError_t launch_leaflr_n(const TreeDev& T, const HB* H, int nelem, int mu,
                            int nleaf, Src U, Src V, RankRef rr, int node,
                            int fside, cudaStream_t st) {
  if (!nelem || !nleaf) return cudaSuccess;
  dim3 grid(nleaf, nelem);
  const int cap = U.kind >= 2 ? 256 : (U.C > 0 ? U.C : 256);   // rank bound
  size_t smem = 2ull * T.bw * (size_t)cap * 8;
  if (smem > 200 * 1024) smem = 200 * 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_leaflr, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  CK_PDL(launch_pdl(k_leaflr, dim3(grid), dim3(LT), smem, st, T, H, mu, U, V, rr, node, fside));
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Fused Schur step at a branch node nu whose children are both leaves -- the
// bottom of invert's recursion (algebra.py:214-238).  With the inverse X of
// leaf rho just computed (in place in H), one CTA per block does what the
// general path does in three launches (HODLR x panel, panel product, leaf
// update):
//   P1[rho] = X A,  P2[rho] = X^T B           A = U_nu[rho], B = V_nu[rho]
//   K = B^T (X A);  W = alpha Lp K;  leaf(rho') += W Rp^T
// half 0: rho = left leaf, Lp = U_nu[rho'], Rp = V_nu[rho'], alpha = -1
//         (the Schur complement S = H22 - H21 x11 H12)
// half 1: rho = right leaf, Lp = P1[rho'] (T), Rp = P2[rho'] (Hh), alpha = +1
//         (b11 = x11 + x11 H12 sinv H21 x11)
// A has rank(nu, half) columns, B rank(nu, 1 - half); a zero rank skips what
// the general path skips.  Fixed summation order: reproducible.
// ---------------------------------------------------------------------------
static constexpr int ST = 512;   // threads of k_schur_leaf

__global__ void __launch_bounds__(ST) k_schur_leaf(TreeDev T, const HB* H, int nu, int half,
                                                   Src P1, Src P2) {
  ACR_PDL_ENTRY();
  extern __shared__ double sm[];
  const int g = blockIdx.x, tid = threadIdx.x, n = T.n, bw = T.bw;
  const HB hb = H[g];
  const int r12 = hb.rk[nu * 2], r21 = hb.rk[nu * 2 + 1];
  const int ca = half ? r21 : r12, cb = half ? r12 : r21;
  if (!ca && !cb) return;
  const int lo = T.lo[nu], mid = T.mid[nu], hi = T.hi[nu];
  const int r0 = half ? mid : lo, sr = half ? hi - mid : mid - lo;    // rho
  const int q0 = half ? lo : mid, sp = half ? mid - lo : hi - mid;    // rho'
  const int slot = T.depth[nu];
  const int ldx = sr + 1, lr = sr | 1, lp = sp | 1;
  const double* Ug = hb.U + (long long)slot * hb.R * n;
  const double* Vg = hb.V + (long long)slot * hb.R * n;
  double* X = sm;                                   // [sr][ldx]
  double* A = X + (long long)sr * ldx;              // [ca][lr]
  double* B = A + (long long)ca * lr;               // [cb][lr]
  double* TA = B + (long long)cb * lr;              // [ca][lr]
  double* K = TA + (long long)ca * lr;              // [cb][ca]
  double* Lp = K + (long long)cb * ca;              // [cb][lp]
  double* Rp = Lp + (long long)cb * lp;             // [ca][lp]
  double* Wp = Rp + (long long)ca * lp;             // [ca][lp]
  const bool upd = ca > 0 && cb > 0;
  {
    const double* Lg = hb.leaf + (long long)r0 * bw;
    for (int idx = tid; idx < sr * sr; idx += ST) {
      const int i = idx / sr, j = idx - i * sr;
      X[i * ldx + j] = Lg[(long long)i * bw + j];
    }
    for (int idx = tid; idx < ca * sr; idx += ST) {
      const int c = idx / sr, j = idx - c * sr;
      A[c * lr + j] = Ug[(long long)c * n + r0 + j];
    }
    for (int idx = tid; idx < cb * sr; idx += ST) {
      const int c = idx / sr, j = idx - c * sr;
      B[c * lr + j] = Vg[(long long)c * n + r0 + j];
    }
    if (upd) {
      for (int idx = tid; idx < cb * sp; idx += ST) {
        const int c = idx / sp, j = idx - c * sp;
        Lp[c * lp + j] = half ? src_col(P1, n, g, slot, c)[q0 + j] : Ug[(long long)c * n + q0 + j];
      }
      for (int idx = tid; idx < ca * sp; idx += ST) {
        const int c = idx / sp, j = idx - c * sp;
        Rp[c * lp + j] = half ? src_col(P2, n, g, slot, c)[q0 + j] : Vg[(long long)c * n + q0 + j];
      }
    }
  }
  __syncthreads();
  // TA = X A (kept for K, and to P1[rho]); X^T B to P2[rho]
  for (int idx = tid; idx < (ca + cb) * sr; idx += ST) {
    const int c = idx / sr, i = idx - c * sr;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (c < ca) {
      const double* xi = X + i * ldx;
      const double* ac = A + c * lr;
      int j = 0;
#pragma unroll 2
      for (; j + 3 < sr; j += 4) {
        a0 = fma(xi[j], ac[j], a0);
        a1 = fma(xi[j + 1], ac[j + 1], a1);
        a2 = fma(xi[j + 2], ac[j + 2], a2);
        a3 = fma(xi[j + 3], ac[j + 3], a3);
      }
      for (; j < sr; ++j) a0 = fma(xi[j], ac[j], a0);
      const double v = (a0 + a1) + (a2 + a3);
      TA[c * lr + i] = v;
      src_col(P1, n, g, slot, c)[r0 + i] = v;
    } else {
      const double* bc = B + (c - ca) * lr;
      int j = 0;
#pragma unroll 2
      for (; j + 3 < sr; j += 4) {
        a0 = fma(X[j * ldx + i], bc[j], a0);
        a1 = fma(X[(j + 1) * ldx + i], bc[j + 1], a1);
        a2 = fma(X[(j + 2) * ldx + i], bc[j + 2], a2);
        a3 = fma(X[(j + 3) * ldx + i], bc[j + 3], a3);
      }
      for (; j < sr; ++j) a0 = fma(X[j * ldx + i], bc[j], a0);
      src_col(P2, n, g, slot, c - ca)[r0 + i] = (a0 + a1) + (a2 + a3);
    }
  }
  if (!upd) return;
  __syncthreads();
  // K = B^T TA (cb x ca)
  for (int idx = tid; idx < cb * ca; idx += ST) {
    const int b = idx / ca, a = idx - b * ca;
    const double* bb = B + b * lr;
    const double* ta = TA + a * lr;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int i = 0;
#pragma unroll 2
    for (; i + 3 < sr; i += 4) {
      a0 = fma(bb[i], ta[i], a0);
      a1 = fma(bb[i + 1], ta[i + 1], a1);
      a2 = fma(bb[i + 2], ta[i + 2], a2);
      a3 = fma(bb[i + 3], ta[i + 3], a3);
    }
    for (; i < sr; ++i) a0 = fma(bb[i], ta[i], a0);
    K[idx] = (a0 + a1) + (a2 + a3);
  }
  __syncthreads();
  // W = alpha Lp K (sp x ca)
  const double alpha = half ? 1.0 : -1.0;
  for (int idx = tid; idx < ca * sp; idx += ST) {
    const int a = idx / sp, i = idx - a * sp;
    double z = 0.0;
    for (int b = 0; b < cb; ++b) z = fma(Lp[b * lp + i], K[b * ca + a], z);
    Wp[a * lp + i] = alpha * z;
  }
  __syncthreads();
  // leaf(rho') += W Rp^T
  double* Lq = hb.leaf + (long long)q0 * bw;
  for (int base = tid; base < sp * sp; base += 4 * ST) {
    double lv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = base + q * ST;
      const int i = idx / sp, j = idx - i * sp;
      lv[q] = idx < sp * sp ? Lq[(long long)i * bw + j] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = base + q * ST;
      if (idx < sp * sp) {
        const int i = idx / sp, j = idx - i * sp;
        double z = 0.0;
        for (int a = 0; a < ca; ++a) z = fma(Wp[a * lp + i], Rp[a * lp + j], z);
        Lq[(long long)i * bw + j] = lv[q] + z;
      }
    }
  }
}

// shared memory (bytes) of k_schur_leaf for leaves of at most bw rows and
// ranks of at most R
size_t schur_leaf_smem(int bw, int R) {
  const size_t l = (size_t)bw | 1;
  return 8 * ((size_t)bw * (bw + 1) + 6 * (size_t)R * l + (size_t)R * R);
}

cudaError_t launch_schur_leaf(const TreeDev& T, const HB* H, int nelem, int nu, int half,
                              Src P1, Src P2, int R, cudaStream_t st) {
  if (!nelem) return cudaSuccess;
  const size_t smem = schur_leaf_smem(T.bw, R);
  static size_t attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(k_schur_leaf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  CK_PDL(launch_pdl(k_schur_leaf, dim3(nelem), dim3(ST), smem, st, T, H, nu, half, P1, P2));
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// elementwise leaf ops
// ---------------------------------------------------------------------------
__global__ void k_leafadd(int len, const HB* A, const HB* B, const HB* C,
                          double sb) {
  ACR_PDL_ENTRY();
  const int g = blockIdx.y;
  const double* a = A[g].leaf;
  const double* b = B[g].leaf;
  double* c = C[g].leaf;
  const double2* a2 = reinterpret_cast<const double2*>(a);
  const double2* b2 = reinterpret_cast<const double2*>(b);
  double2* c2 = reinterpret_cast<double2*>(c);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len / 2;
       i += gridDim.x * blockDim.x) {
    const double2 x = a2[i], y = b2[i];
    c2[i] = make_double2(x.x + sb * y.x, x.y + sb * y.y);
  }
}

cudaError_t launch_leafadd(const TreeDev& T, const HB* A, const HB* B,
                           const HB* C, double sb, int nelem, cudaStream_t st) {
  if (!nelem) return cudaSuccess;
  int len = T.n * T.bw;
  int bx = (len + 255) / 256;
  if (bx > 64) bx = 64;
  CK_PDL(launch_pdl(k_leafadd, dim3(dim3(bx, nelem)), dim3(256), 0, st, len, A, B, C, sb));
  return cudaGetLastError();
}

__global__ void k_negate(TreeDev T, const HB* H) {
  ACR_PDL_ENTRY();
  const int g = blockIdx.y, n = T.n;
  const HB h = H[g];
  const int len = n * T.bw;
  double2* h2 = reinterpret_cast<double2*>(h.leaf);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len / 2;
       i += gridDim.x * blockDim.x) {
    const double2 x = h2[i];
    h2[i] = make_double2(-1.0 * x.x, -1.0 * x.y);
  }
  // factors: U columns below the rank, per branch node and side
  for (int v = blockIdx.x; v < T.nnodes; v += gridDim.x) {
    if (T.isleaf[v]) continue;
    int lo = T.lo[v], hi = T.hi[v], mid = T.mid[v];
    long long slot = (long long)T.depth[v] * h.R * n;
    for (int side = 0; side < 2; ++side) {
      int r = h.rk[v * 2 + side];
      int row = side ? mid : lo, len2 = side ? hi - mid : mid - lo;
      for (int idx = threadIdx.x; idx < r * len2; idx += blockDim.x) {
        int c = idx / len2, i = idx - c * len2;
        double* p = h.U + slot + (long long)c * n + row + i;
        *p = -1.0 * *p;
      }
    }
  }
}

__global__ void k_copy_i32(int* __restrict__ dst, const int* __restrict__ src, long long n) {
  ACR_PDL_ENTRY();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

__global__ void k_fill_i32(int* dst, int v, long long n) {
  ACR_PDL_ENTRY();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = v;
}

cudaError_t launch_copy_i32(int* dst, const int* src, long long n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const long long b = (n + 255) / 256;
  CK_PDL(launch_pdl(k_copy_i32, dim3((int)(b < 592 ? b : 592)), dim3(256), 0, st, dst, src, n));
  return cudaGetLastError();
}

cudaError_t launch_fill_i32(int* dst, int v, long long n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const long long b = (n + 255) / 256;
  CK_PDL(launch_pdl(k_fill_i32, dim3((int)(b < 592 ? b : 592)), dim3(256), 0, st, dst, v, n));
  return cudaGetLastError();
}

cudaError_t launch_negate(const TreeDev& T, const HB* H, int nelem,
                          cudaStream_t st) {
  if (!nelem) return cudaSuccess;
  CK_PDL(launch_pdl(k_negate, dim3(dim3(32, nelem)), dim3(256), 0, st, T, H));
  return cudaGetLastError();
}

__global__ void k_copyhb(TreeDev T, const HB* S, const HB* D, int* overflow) {
  ACR_PDL_ENTRY();
  const int g = blockIdx.y, n = T.n;
  const HB s = S[g], d = D[g];
  const int len = n * T.bw;
  {
    const double2* s2 = reinterpret_cast<const double2*>(s.leaf);
    double2* d2 = reinterpret_cast<double2*>(d.leaf);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len / 2;
         i += gridDim.x * blockDim.x)
      d2[i] = s2[i];
  }
  for (int v = blockIdx.x; v < T.nnodes; v += gridDim.x) {
    if (T.isleaf[v]) {
      if (threadIdx.x < 2) d.rk[v * 2 + threadIdx.x] = 0;
      continue;
    }
    int lo = T.lo[v], hi = T.hi[v], mid = T.mid[v];
    long long ss = (long long)T.depth[v] * s.R * n, ds = (long long)T.depth[v] * d.R * n;
    for (int side = 0; side < 2; ++side) {
      int r = s.rk[v * 2 + side];
      if (r > d.R) {
        if (threadIdx.x == 0) atomicMax(overflow, r);
        r = d.R;
      }
      int ur = side ? mid : lo, ul = side ? hi - mid : mid - lo;
      int vr = side ? lo : mid, vl = side ? mid - lo : hi - mid;
      for (int idx = threadIdx.x; idx < r * ul; idx += blockDim.x) {
        int c = idx / ul, i = idx - c * ul;
        d.U[ds + (long long)c * n + ur + i] = s.U[ss + (long long)c * n + ur + i];
      }
      for (int idx = threadIdx.x; idx < r * vl; idx += blockDim.x) {
        int c = idx / vl, i = idx - c * vl;
        d.V[ds + (long long)c * n + vr + i] = s.V[ss + (long long)c * n + vr + i];
      }
      if (threadIdx.x == 0) d.rk[v * 2 + side] = r;
    }
  }
}

cudaError_t launch_copyhb(const TreeDev& T, const HB* S, const HB* D, int nelem,
                          int* overflow, cudaStream_t st) {
  if (!nelem) return cudaSuccess;
  CK_PDL(launch_pdl(k_copyhb, dim3(dim3(32, nelem)), dim3(256), 0, st, T, S, D, overflow));
  return cudaGetLastError();
}

__global__ void k_zerohb(TreeDev T, const HB* D) {
  ACR_PDL_ENTRY();
  const int g = blockIdx.y;
  const HB d = D[g];
  const int len = T.n * T.bw;
  double2* d2 = reinterpret_cast<double2*>(d.leaf);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len / 2;
       i += gridDim.x * blockDim.x)
    d2[i] = make_double2(0.0, 0.0);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * T.nnodes;
       i += gridDim.x * blockDim.x)
    d.rk[i] = 0;
}

cudaError_t launch_zerohb(const TreeDev& T, const HB* D, int nelem,
                          cudaStream_t st) {
  if (!nelem) return cudaSuccess;
  CK_PDL(launch_pdl(k_zerohb, dim3(dim3(16, nelem)), dim3(256), 0, st, T, D));
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// lift (hodlr.py:242-314): bands -> leaves + rank<=1 corner factors
// ---------------------------------------------------------------------------
// row -> (first row, size) of its leaf for every row of the block, in shared
// memory, built once per CTA from the leaf list
__device__ __forceinline__ void leaf_map(const TreeDev& T, int* mlo, int* msz) {
  const int b0 = T.startB[0], nb = T.startB[1] - b0;
  for (int q = threadIdx.x; q < nb; q += blockDim.x) {
    const int v = T.listB[(b0 + q) * 2 + 1];
    const int lo = T.lo[v], hi = T.hi[v];
    for (int i = lo; i < hi; ++i) {
      mlo[i] = lo;
      msz[i] = hi - lo;
    }
  }
  __syncthreads();
}

// exact lift of the tridiagonal bands (hodlr.py:242-291): dense tridiagonal
// leaves (two columns per thread, 16-byte stores) and, at every branch depth,
// factor column 0 zero except the corners off12 = a e_{mid-1} e_mid^T,
// off21 = b e_mid e_{mid-1}^T (a = sup[mid-1], b = sub[mid-1]; rank 0 if 0)
__global__ void k_lift(TreeDev T, const double* sub, const double* diag,
                       const double* sup, const HB* D) {
  ACR_PDL_ENTRY();
  extern __shared__ int lmap[];
  const int g = blockIdx.y, n = T.n, bw = T.bw;
  const HB d = D[g];
  const double* sb = sub + (long long)g * (n - 1);
  const double* dg = diag + (long long)g * n;
  const double* sp = sup + (long long)g * (n - 1);
  int* mlo = lmap;
  int* msz = lmap + n;
  leaf_map(T, mlo, msz);
  double2* L2 = reinterpret_cast<double2*>(d.leaf);
  const int half = bw >> 1;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n * half;
       idx += gridDim.x * blockDim.x) {
    const int i = idx / half, jj = 2 * (idx - i * half);
    const int lo = mlo[i], s = msz[i];
    double v2[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = lo + jj + q;
      v2[q] = jj + q >= s ? 0.0 : j == i ? dg[i] : j == i + 1 ? sp[i] : j == i - 1 ? sb[j] : 0.0;
    }
    L2[idx] = make_double2(v2[0], v2[1]);
  }
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < T.nd * n;
       idx += gridDim.x * blockDim.x) {
    const int k = idx / n, i = idx - k * n;
    int node = 0;                               // the depth-k node holding row i
    for (int t = 0; t < k && !T.isleaf[node]; ++t)
      node = i < T.mid[node] ? T.c0[node] : T.c1[node];
    double u = 0.0, v = 0.0;
    if (!T.isleaf[node] && T.depth[node] == k) {
      const int mid = T.mid[node];
      const double a = sp[mid - 1], b = sb[mid - 1];
      if (i == mid - 1) { u = a; v = b != 0.0 ? 1.0 : 0.0; }
      if (i == mid) { u = b; v = a != 0.0 ? 1.0 : 0.0; }
    }
    const long long slot = (long long)k * d.R * n;
    d.U[slot + i] = u;
    d.V[slot + i] = v;
  }
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < T.nnodes;
       v += gridDim.x * blockDim.x) {
    if (T.isleaf[v]) {
      d.rk[v * 2] = d.rk[v * 2 + 1] = 0;
      continue;
    }
    const int mid = T.mid[v];
    d.rk[v * 2] = sp[mid - 1] != 0.0 ? 1 : 0;
    d.rk[v * 2 + 1] = sb[mid - 1] != 0.0 ? 1 : 0;
  }
}

cudaError_t launch_lift(const TreeDev& T, const double* sub, const double* diag,
                        const double* sup, const HB* D, int nelem,
                        cudaStream_t st) {
  if (!nelem) return cudaSuccess;
  CK_PDL(launch_pdl(k_lift, dim3(dim3(8, nelem)), dim3(256), 2 * T.n * sizeof(int), st, T, sub, diag, sup, D));
  return cudaGetLastError();
}

// exact diagonal block (hodlr.py:294-314): dense diagonal leaves, rank 0
__global__ void k_liftdiag(TreeDev T, const double* dd, const HB* D) {
  ACR_PDL_ENTRY();
  extern __shared__ int lmap[];
  const int g = blockIdx.y, n = T.n, bw = T.bw;
  const HB d = D[g];
  const double* dg = dd + (long long)g * n;
  int* mlo = lmap;
  int* msz = lmap + n;
  leaf_map(T, mlo, msz);
  double2* L2 = reinterpret_cast<double2*>(d.leaf);
  const int half = bw >> 1;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n * half;
       idx += gridDim.x * blockDim.x) {
    const int i = idx / half, jj = 2 * (idx - i * half);
    const int c = i - mlo[i];                   // the diagonal's column in the leaf
    L2[idx] = make_double2(c == jj ? dg[i] : 0.0, c == jj + 1 ? dg[i] : 0.0);
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * T.nnodes;
       i += gridDim.x * blockDim.x)
    d.rk[i] = 0;
}

cudaError_t launch_liftdiag(const TreeDev& T, const double* d, const HB* D,
                            int nelem, cudaStream_t st) {
  if (!nelem) return cudaSuccess;
  CK_PDL(launch_pdl(k_liftdiag, dim3(dim3(8, nelem)), dim3(256), 2 * T.n * sizeof(int), st, T, d, D));
  return cudaGetLastError();
}

// HB table for a strided set of blocks: tab[i] = block (first + i*step)
__global__ void k_build_tab(HB* tab, HB base, long long sl, long long sf,
                            long long sr, int first, int step, int count) {
  ACR_PDL_ENTRY();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  long long e = first + (long long)i * step;
  HB h = base;
  h.leaf = base.leaf + e * sl;
  h.U = base.U + e * sf;
  h.V = base.V + e * sf;
  h.rk = base.rk + e * sr;
  tab[i] = h;
}

cudaError_t launch_build_tab(HB* tab, HB base, long long sl, long long sf,
                             long long sr, int first, int step, int count,
                             cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  CK_PDL(launch_pdl(k_build_tab, dim3((count + 127) / 128), dim3(128), 0, st, tab, base, sl, sf, sr, first,
                                                  step, count));
  return cudaGetLastError();
}

}  // namespace acr
