// Development harness: one 64x64 leaf inverse per launch, timed with events
#include <cstdio>
#include <vector>
#include <cstdlib>
#include "../../paper_1604_00617_b200/csrc/k_leaf.cu"
namespace acr {
template <int S, int TR, int TC, int MINB>
__global__ void __launch_bounds__((S / TR) * (S / TC), MINB) li_noupd(TreeDev T, const HB* H,
                                                                       int leaf, int* sing) {
  constexpr int TGY = S / TR, TGX = S / TC, NT = TGX * TGY;
  static_assert(TGY <= 32, "a column group must fit one warp");
  constexpr unsigned MASK = TGY >= 32 ? 0xffffffffu : (NT >= 32 ? 0xffffffffu : (1u << NT) - 1u);
  __shared__ double colbuf[2][S], rowP[S], rowK[S];
  __shared__ int piv[S + 1], inv_[S];
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
  for (int k = 0; k < s; ++k) {
    __syncthreads();                            // colbuf[k & 1], piv[k]
    const int p = piv[k];
    const double* cb = colbuf[k & 1];
    const double pv = cb[p];
    if (pv == 0.0) { bad = true; break; }       // uniform
    if (ty == p / TR) {                         // old row p (select chain: x stays in registers)
      const int ap = p % TR;
#pragma unroll
      for (int b = 0; b < TC; ++b) {
        double v = x[0][b];
#pragma unroll
        for (int a = 1; a < TR; ++a) v = ap == a ? x[a][b] : v;
        rowP[tx * TC + b] = v;
      }
    }
    if (ty == k / TR) {                         // old row k
      const int ak = k % TR;
#pragma unroll
      for (int b = 0; b < TC; ++b) {
        double v = x[0][b];
#pragma unroll
        for (int a = 1; a < TR; ++a) v = ak == a ? x[a][b] : v;
        rowK[tx * TC + b] = v;
      }
    }
    __syncthreads();
    const double inv = 1.0 / pv;
    double rk[TC];
#pragma unroll
    for (int b = 0; b < TC; ++b) {
      const int c = tx * TC + b;
      rk[b] = (c == k) ? inv : rowP[c] * inv;   // new row k = old row p / pv
    }
    if (tx == k / TC) {                         // column k acts as zero
      const int bk = k % TC;
#pragma unroll
      for (int a = 0; a < TR; ++a)
#pragma unroll
        for (int b = 0; b < TC; ++b) x[a][b] = bk == b ? 0.0 : x[a][b];
    }

    if (ty == k / TR || ty == p / TR) {
      const double fk = cb[k];                  // old a_kk: row k moves to p
#pragma unroll
      for (int a = 0; a < TR; ++a) {
        const int r = ty * TR + a;
        if (r == p && p != k) {
#pragma unroll
          for (int b = 0; b < TC; ++b) {
            const int c = tx * TC + b;
            const double ok = (c == k) ? 0.0 : rowK[c];
            x[a][b] = ok - fk * rk[b];
          }
        }
        if (r == k) {
#pragma unroll
          for (int b = 0; b < TC; ++b) x[a][b] = rk[b];
        }
      }
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
        if (r >= kn && r < s && fabs(v) > best) { best = fabs(v); pb = r; }
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
  // A^{-1} = X P: undo the column swaps in reverse order
  if (tid == 0) {
    int* pos = reinterpret_cast<int*>(rowP);   // S ints fit in S doubles
    for (int j = 0; j < s; ++j) pos[j] = j;
    for (int k = s - 1; k >= 0; --k) {
      const int t = pos[k];
      pos[k] = pos[piv[k]];
      pos[piv[k]] = t;
    }
    for (int j = 0; j < s; ++j) inv_[pos[j]] = j;
  }
  __syncthreads();
  int nf = 0;
#pragma unroll
  for (int a = 0; a < TR; ++a)
#pragma unroll
    for (int b = 0; b < TC; ++b) {
      const int r = ty * TR + a, c = tx * TC + b;
      if (r < s && c < s) {
        if (!isfinite(x[a][b])) nf = 1;
        L[(long long)r * bw + inv_[c]] = x[a][b];
      }
    }
  if (__syncthreads_or(nf) && tid == 0) {
    int ps = 0;
    for (int v = 0; v < T.nnodes; ++v)
      if (T.isleaf[v] && T.lo[v] < lo) ++ps;
    atomicMin(sing + g, ps);
  }
}
template <int S, int TR, int TC, int MINB>
__global__ void __launch_bounds__((S / TR) * (S / TC), MINB) li_nosync2(TreeDev T, const HB* H,
                                                                       int leaf, int* sing) {
  constexpr int TGY = S / TR, TGX = S / TC, NT = TGX * TGY;
  static_assert(TGY <= 32, "a column group must fit one warp");
  constexpr unsigned MASK = TGY >= 32 ? 0xffffffffu : (NT >= 32 ? 0xffffffffu : (1u << NT) - 1u);
  __shared__ double colbuf[2][S], rowP[S], rowK[S];
  __shared__ int piv[S + 1], inv_[S];
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
  for (int k = 0; k < s; ++k) {
    __syncthreads();                            // colbuf[k & 1], piv[k]
    const int p = piv[k];
    const double* cb = colbuf[k & 1];
    const double pv = cb[p];
    if (pv == 0.0) { bad = true; break; }       // uniform
    if (ty == p / TR) {                         // old row p (select chain: x stays in registers)
      const int ap = p % TR;
#pragma unroll
      for (int b = 0; b < TC; ++b) {
        double v = x[0][b];
#pragma unroll
        for (int a = 1; a < TR; ++a) v = ap == a ? x[a][b] : v;
        rowP[tx * TC + b] = v;
      }
    }
    if (ty == k / TR) {                         // old row k
      const int ak = k % TR;
#pragma unroll
      for (int b = 0; b < TC; ++b) {
        double v = x[0][b];
#pragma unroll
        for (int a = 1; a < TR; ++a) v = ak == a ? x[a][b] : v;
        rowK[tx * TC + b] = v;
      }
    }
    const double inv = 1.0 / pv;
    double rk[TC];
#pragma unroll
    for (int b = 0; b < TC; ++b) {
      const int c = tx * TC + b;
      rk[b] = (c == k) ? inv : rowP[c] * inv;   // new row k = old row p / pv
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
#pragma unroll
      for (int b = 0; b < TC; ++b) x[a][b] -= f * rk[b];
    }
    if (ty == k / TR || ty == p / TR) {
      const double fk = cb[k];                  // old a_kk: row k moves to p
#pragma unroll
      for (int a = 0; a < TR; ++a) {
        const int r = ty * TR + a;
        if (r == p && p != k) {
#pragma unroll
          for (int b = 0; b < TC; ++b) {
            const int c = tx * TC + b;
            const double ok = (c == k) ? 0.0 : rowK[c];
            x[a][b] = ok - fk * rk[b];
          }
        }
        if (r == k) {
#pragma unroll
          for (int b = 0; b < TC; ++b) x[a][b] = rk[b];
        }
      }
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
        if (r >= kn && r < s && fabs(v) > best) { best = fabs(v); pb = r; }
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
  // A^{-1} = X P: undo the column swaps in reverse order
  if (tid == 0) {
    int* pos = reinterpret_cast<int*>(rowP);   // S ints fit in S doubles
    for (int j = 0; j < s; ++j) pos[j] = j;
    for (int k = s - 1; k >= 0; --k) {
      const int t = pos[k];
      pos[k] = pos[piv[k]];
      pos[piv[k]] = t;
    }
    for (int j = 0; j < s; ++j) inv_[pos[j]] = j;
  }
  __syncthreads();
  int nf = 0;
#pragma unroll
  for (int a = 0; a < TR; ++a)
#pragma unroll
    for (int b = 0; b < TC; ++b) {
      const int r = ty * TR + a, c = tx * TC + b;
      if (r < s && c < s) {
        if (!isfinite(x[a][b])) nf = 1;
        L[(long long)r * bw + inv_[c]] = x[a][b];
      }
    }
  if (__syncthreads_or(nf) && tid == 0) {
    int ps = 0;
    for (int v = 0; v < T.nnodes; ++v)
      if (T.isleaf[v] && T.lo[v] < lo) ++ps;
    atomicMin(sing + g, ps);
  }
}
template <int S, int TR, int TC, int MINB>
__global__ void __launch_bounds__((S / TR) * (S / TC), MINB) li_nodiv(TreeDev T, const HB* H,
                                                                       int leaf, int* sing) {
  constexpr int TGY = S / TR, TGX = S / TC, NT = TGX * TGY;
  static_assert(TGY <= 32, "a column group must fit one warp");
  constexpr unsigned MASK = TGY >= 32 ? 0xffffffffu : (NT >= 32 ? 0xffffffffu : (1u << NT) - 1u);
  __shared__ double colbuf[2][S], rowP[S], rowK[S];
  __shared__ int piv[S + 1], inv_[S];
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
  for (int k = 0; k < s; ++k) {
    __syncthreads();                            // colbuf[k & 1], piv[k]
    const int p = piv[k];
    const double* cb = colbuf[k & 1];
    const double pv = cb[p];
    if (pv == 0.0) { bad = true; break; }       // uniform
    if (ty == p / TR) {                         // old row p (select chain: x stays in registers)
      const int ap = p % TR;
#pragma unroll
      for (int b = 0; b < TC; ++b) {
        double v = x[0][b];
#pragma unroll
        for (int a = 1; a < TR; ++a) v = ap == a ? x[a][b] : v;
        rowP[tx * TC + b] = v;
      }
    }
    if (ty == k / TR) {                         // old row k
      const int ak = k % TR;
#pragma unroll
      for (int b = 0; b < TC; ++b) {
        double v = x[0][b];
#pragma unroll
        for (int a = 1; a < TR; ++a) v = ak == a ? x[a][b] : v;
        rowK[tx * TC + b] = v;
      }
    }
    __syncthreads();
    const double inv = pv * 1e-3;
    double rk[TC];
#pragma unroll
    for (int b = 0; b < TC; ++b) {
      const int c = tx * TC + b;
      rk[b] = (c == k) ? inv : rowP[c] * inv;   // new row k = old row p / pv
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
#pragma unroll
      for (int b = 0; b < TC; ++b) x[a][b] -= f * rk[b];
    }
    if (ty == k / TR || ty == p / TR) {
      const double fk = cb[k];                  // old a_kk: row k moves to p
#pragma unroll
      for (int a = 0; a < TR; ++a) {
        const int r = ty * TR + a;
        if (r == p && p != k) {
#pragma unroll
          for (int b = 0; b < TC; ++b) {
            const int c = tx * TC + b;
            const double ok = (c == k) ? 0.0 : rowK[c];
            x[a][b] = ok - fk * rk[b];
          }
        }
        if (r == k) {
#pragma unroll
          for (int b = 0; b < TC; ++b) x[a][b] = rk[b];
        }
      }
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
        if (r >= kn && r < s && fabs(v) > best) { best = fabs(v); pb = r; }
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
  // A^{-1} = X P: undo the column swaps in reverse order
  if (tid == 0) {
    int* pos = reinterpret_cast<int*>(rowP);   // S ints fit in S doubles
    for (int j = 0; j < s; ++j) pos[j] = j;
    for (int k = s - 1; k >= 0; --k) {
      const int t = pos[k];
      pos[k] = pos[piv[k]];
      pos[piv[k]] = t;
    }
    for (int j = 0; j < s; ++j) inv_[pos[j]] = j;
  }
  __syncthreads();
  int nf = 0;
#pragma unroll
  for (int a = 0; a < TR; ++a)
#pragma unroll
    for (int b = 0; b < TC; ++b) {
      const int r = ty * TR + a, c = tx * TC + b;
      if (r < s && c < s) {
        if (!isfinite(x[a][b])) nf = 1;
        L[(long long)r * bw + inv_[c]] = x[a][b];
      }
    }
  if (__syncthreads_or(nf) && tid == 0) {
    int ps = 0;
    for (int v = 0; v < T.nnodes; ++v)
      if (T.isleaf[v] && T.lo[v] < lo) ++ps;
    atomicMin(sing + g, ps);
  }
}
template <int S, int TR, int TC, int MINB>
__global__ void __launch_bounds__((S / TR) * (S / TC), MINB) li_norows(TreeDev T, const HB* H,
                                                                       int leaf, int* sing) {
  constexpr int TGY = S / TR, TGX = S / TC, NT = TGX * TGY;
  static_assert(TGY <= 32, "a column group must fit one warp");
  constexpr unsigned MASK = TGY >= 32 ? 0xffffffffu : (NT >= 32 ? 0xffffffffu : (1u << NT) - 1u);
  __shared__ double colbuf[2][S], rowP[S], rowK[S];
  __shared__ int piv[S + 1], inv_[S];
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
  for (int k = 0; k < s; ++k) {
    __syncthreads();                            // colbuf[k & 1], piv[k]
    const int p = piv[k];
    const double* cb = colbuf[k & 1];
    const double pv = cb[p];
    if (pv == 0.0) { bad = true; break; }       // uniform
    if (false) {
      const int ap = p % TR;
#pragma unroll
      for (int b = 0; b < TC; ++b) {
        double v = x[0][b];
#pragma unroll
        for (int a = 1; a < TR; ++a) v = ap == a ? x[a][b] : v;
        rowP[tx * TC + b] = v;
      }
    }
    if (false) {
      const int ak = k % TR;
#pragma unroll
      for (int b = 0; b < TC; ++b) {
        double v = x[0][b];
#pragma unroll
        for (int a = 1; a < TR; ++a) v = ak == a ? x[a][b] : v;
        rowK[tx * TC + b] = v;
      }
    }
    __syncthreads();
    const double inv = 1.0 / pv;
    double rk[TC];
#pragma unroll
    for (int b = 0; b < TC; ++b) {
      const int c = tx * TC + b;
      rk[b] = (c == k) ? inv : rowP[c] * inv;   // new row k = old row p / pv
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
#pragma unroll
      for (int b = 0; b < TC; ++b) x[a][b] -= f * rk[b];
    }
    if (false) {
      const double fk = cb[k];                  // old a_kk: row k moves to p
#pragma unroll
      for (int a = 0; a < TR; ++a) {
        const int r = ty * TR + a;
        if (r == p && p != k) {
#pragma unroll
          for (int b = 0; b < TC; ++b) {
            const int c = tx * TC + b;
            const double ok = (c == k) ? 0.0 : rowK[c];
            x[a][b] = ok - fk * rk[b];
          }
        }
        if (r == k) {
#pragma unroll
          for (int b = 0; b < TC; ++b) x[a][b] = rk[b];
        }
      }
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
        if (r >= kn && r < s && fabs(v) > best) { best = fabs(v); pb = r; }
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
  // A^{-1} = X P: undo the column swaps in reverse order
  if (tid == 0) {
    int* pos = reinterpret_cast<int*>(rowP);   // S ints fit in S doubles
    for (int j = 0; j < s; ++j) pos[j] = j;
    for (int k = s - 1; k >= 0; --k) {
      const int t = pos[k];
      pos[k] = pos[piv[k]];
      pos[piv[k]] = t;
    }
    for (int j = 0; j < s; ++j) inv_[pos[j]] = j;
  }
  __syncthreads();
  int nf = 0;
#pragma unroll
  for (int a = 0; a < TR; ++a)
#pragma unroll
    for (int b = 0; b < TC; ++b) {
      const int r = ty * TR + a, c = tx * TC + b;
      if (r < s && c < s) {
        if (!isfinite(x[a][b])) nf = 1;
        L[(long long)r * bw + inv_[c]] = x[a][b];
      }
    }
  if (__syncthreads_or(nf) && tid == 0) {
    int ps = 0;
    for (int v = 0; v < T.nnodes; ++v)
      if (T.isleaf[v] && T.lo[v] < lo) ++ps;
    atomicMin(sing + g, ps);
  }
}
template <int S, int TR, int TC, int MINB>
__global__ void __launch_bounds__((S / TR) * (S / TC), MINB) li_nopiv(TreeDev T, const HB* H,
                                                                       int leaf, int* sing) {
  constexpr int TGY = S / TR, TGX = S / TC, NT = TGX * TGY;
  static_assert(TGY <= 32, "a column group must fit one warp");
  constexpr unsigned MASK = TGY >= 32 ? 0xffffffffu : (NT >= 32 ? 0xffffffffu : (1u << NT) - 1u);
  __shared__ double colbuf[2][S], rowP[S], rowK[S];
  __shared__ int piv[S + 1], inv_[S];
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
  for (int k = 0; k < s; ++k) {
    __syncthreads();                            // colbuf[k & 1], piv[k]
    const int p = piv[k];
    const double* cb = colbuf[k & 1];
    const double pv = cb[p];
    if (pv == 0.0) { bad = true; break; }       // uniform
    if (ty == p / TR) {                         // old row p (select chain: x stays in registers)
      const int ap = p % TR;
#pragma unroll
      for (int b = 0; b < TC; ++b) {
        double v = x[0][b];
#pragma unroll
        for (int a = 1; a < TR; ++a) v = ap == a ? x[a][b] : v;
        rowP[tx * TC + b] = v;
      }
    }
    if (ty == k / TR) {                         // old row k
      const int ak = k % TR;
#pragma unroll
      for (int b = 0; b < TC; ++b) {
        double v = x[0][b];
#pragma unroll
        for (int a = 1; a < TR; ++a) v = ak == a ? x[a][b] : v;
        rowK[tx * TC + b] = v;
      }
    }
    __syncthreads();
    const double inv = 1.0 / pv;
    double rk[TC];
#pragma unroll
    for (int b = 0; b < TC; ++b) {
      const int c = tx * TC + b;
      rk[b] = (c == k) ? inv : rowP[c] * inv;   // new row k = old row p / pv
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
#pragma unroll
      for (int b = 0; b < TC; ++b) x[a][b] -= f * rk[b];
    }
    if (ty == k / TR || ty == p / TR) {
      const double fk = cb[k];                  // old a_kk: row k moves to p
#pragma unroll
      for (int a = 0; a < TR; ++a) {
        const int r = ty * TR + a;
        if (r == p && p != k) {
#pragma unroll
          for (int b = 0; b < TC; ++b) {
            const int c = tx * TC + b;
            const double ok = (c == k) ? 0.0 : rowK[c];
            x[a][b] = ok - fk * rk[b];
          }
        }
        if (r == k) {
#pragma unroll
          for (int b = 0; b < TC; ++b) x[a][b] = rk[b];
        }
      }
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
        if (r >= kn && r < s && fabs(v) > best) { best = fabs(v); pb = r; }
      }
      if (own && ty == 0) piv[kn] = kn;
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
  // A^{-1} = X P: undo the column swaps in reverse order
  if (tid == 0) {
    int* pos = reinterpret_cast<int*>(rowP);   // S ints fit in S doubles
    for (int j = 0; j < s; ++j) pos[j] = j;
    for (int k = s - 1; k >= 0; --k) {
      const int t = pos[k];
      pos[k] = pos[piv[k]];
      pos[piv[k]] = t;
    }
    for (int j = 0; j < s; ++j) inv_[pos[j]] = j;
  }
  __syncthreads();
  int nf = 0;
#pragma unroll
  for (int a = 0; a < TR; ++a)
#pragma unroll
    for (int b = 0; b < TC; ++b) {
      const int r = ty * TR + a, c = tx * TC + b;
      if (r < s && c < s) {
        if (!isfinite(x[a][b])) nf = 1;
        L[(long long)r * bw + inv_[c]] = x[a][b];
      }
    }
  if (__syncthreads_or(nf) && tid == 0) {
    int ps = 0;
    for (int v = 0; v < T.nnodes; ++v)
      if (T.isleaf[v] && T.lo[v] < lo) ++ps;
    atomicMin(sing + g, ps);
  }
}

}
using namespace acr;
__global__ void li_empty() {}
int main() {
  const int s = 64;
  std::vector<double> h(s * s);
  srand(1);
  for (int i = 0; i < s * s; ++i) h[i] = (rand() / (double)RAND_MAX - 0.5) + ((i / s == i % s) ? 8.0 : 0.0);
  double* d; cudaMalloc(&d, 8 * s * s);
  int tree[8] = {0, s, s / 2, 0, -1, -1, -1, 1};
  int* dt; cudaMalloc(&dt, sizeof(tree)); cudaMemcpy(dt, tree, sizeof(tree), cudaMemcpyHostToDevice);
  TreeDev T; memset(&T, 0, sizeof(T));
  T.n = s; T.bw = s; T.nnodes = 1; T.nleaves = 1;
  T.lo = dt; T.hi = dt + 1; T.mid = dt + 2; T.depth = dt + 3; T.parent = dt + 4; T.c0 = dt + 5; T.c1 = dt + 6; T.isleaf = dt + 7;
  HB hb; memset(&hb, 0, sizeof(hb)); hb.leaf = d; hb.R = 1;
  HB* dhb; cudaMalloc(&dhb, sizeof(HB)); cudaMemcpy(dhb, &hb, sizeof(HB), cudaMemcpyHostToDevice);
  int* sg; cudaMalloc(&sg, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int v = 0; v < 8; ++v) {
    float best = 1e9;
    for (int rep = 0; rep < 20; ++rep) {
      cudaMemcpy(d, h.data(), 8 * s * s, cudaMemcpyHostToDevice);
      cudaEventRecord(e0);
      if (v == 0) k_leafinv_v2<64, 2, 2, 1><<<1, 1024>>>(T, dhb, 0, sg);
      else if (v == 1) k_leafinv_v2<64, 4, 4, 3><<<1, 256>>>(T, dhb, 0, sg);
      else if (v == 2) li_nopiv<64, 2, 2, 1><<<1, 1024>>>(T, dhb, 0, sg);
      else if (v == 3) li_nopiv<64, 4, 4, 3><<<1, 256>>>(T, dhb, 0, sg);
      else if (v == 4) li_noupd<64, 2, 2, 1><<<1, 1024>>>(T, dhb, 0, sg);
      else if (v == 5) li_nosync2<64, 2, 2, 1><<<1, 1024>>>(T, dhb, 0, sg);
      else if (v == 6) li_nodiv<64, 2, 2, 1><<<1, 1024>>>(T, dhb, 0, sg);
      else li_norows<64, 2, 2, 1><<<1, 1024>>>(T, dhb, 0, sg);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const char* nm[] = {"2x2/1024", "4x4/256", "2x2/1024 nopivsearch", "4x4/256 nopivsearch", "2x2 noupdate", "2x2 nosync2", "2x2 nodiv", "2x2 norowsel"};
    printf("%-24s %.1f us  (%s)\n", nm[v], best * 1e3, cudaGetErrorString(cudaGetLastError()));
  }
  { float best = 1e9; for (int rep = 0; rep < 20; ++rep) { cudaEventRecord(e0); li_empty<<<1, 1024>>>(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; } printf("empty launch %.1f us\n", best * 1e3); }
  return 0;
}
