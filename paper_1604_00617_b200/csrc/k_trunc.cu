// Batched low-rank recompression: reference hodlr.py:176-200
// (truncate_factor) and algebra.py:90-97 (_combine), one CTA per
// (task, element).
//
//   combine(F, G): rank-0 operand -> the other passes through untouched;
//                  otherwise truncate([F | G]).
//   truncate(F):   R = #columns; R == 0 -> F; R == 1 -> F if U != 0 and
//                  V != 0 else 0; otherwise Householder QR of U and V
//                  (LAPACK dgeqr2 / dlarfg conventions), one-sided Jacobi
//                  SVD of the core Ru Rv^T, noise guard
//                  s1 <= R eps64 |Ru|_F |Rv|_F -> 0, keep s_i >= eps s1,
//                  optional cap, U' = Qu (W s), V' = Qv Z.
// All reductions are fixed-order (warp shuffles + 4-way smem) so results are
// bitwise reproducible run to run and independent of elimination order.
#include <cooperative_groups.h>

#include "acr_types.cuh"
#include "acr_launch.h"
#include "acr_pdl.cuh"

namespace acr {

static constexpr int TT = 512;   // threads per block-path truncation CTA
static constexpr int NWB = TT / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Two warp sums for the price of one and a half: after the first exchange the
// lower half-warp carries a, the upper half b; four single-value rounds; one
// broadcast each.  Every value is summed over the same tree as warp_sum
// (lane l + lane l ^ 16 first, then 8, 4, 2, 1): bitwise the same results.
__device__ __forceinline__ void warp_sum2(double& a, double& b, int lane) {
  const bool hi = lane & 16;
  const double send = hi ? a : b;                 // what the other half needs
  const double got = __shfl_xor_sync(0xffffffffu, send, 16);
  double v = (hi ? b : a) + got;                  // lower: a_l + a_{l+16}; upper: b_l + b_{l-16}
  v += __shfl_xor_sync(0xffffffffu, v, 8);
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  a = __shfl_sync(0xffffffffu, v, 0);
  b = __shfl_sync(0xffffffffu, v, 16);
}

// N (2, 4 or 8) warp sums at once by halving: at every exchange half the
// lanes keep one half of the values, so N sums cost N - 1 exchanges, the
// remaining single-value rounds and N broadcasts instead of 5 N exchanges.
// Every value is summed over the same tree as warp_sum: bitwise the same.
template <int N>
__device__ __forceinline__ void warp_sum_multi(double (&v)[N], int lane) {
  static_assert(N == 2 || N == 4 || N == 8, "N");
  int o = 16;
#pragma unroll
  for (int n = N; n > 1; n >>= 1, o >>= 1) {
    const bool hi = lane & o;
#pragma unroll
    for (int k = 0; k < n / 2; ++k) {
      const double send = hi ? v[k] : v[k + n / 2];
      const double got = __shfl_xor_sync(0xffffffffu, send, o);
      v[k] = (hi ? v[k + n / 2] : v[k]) + got;
    }
  }
  for (; o; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
  // lane bits 4, 3, 2 (for N = 8) name the value a lane ended up with
  const double mine = v[0];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    int src = 0;
    if (N >= 2 && (i & (N / 2))) src |= 16;
    if (N >= 4 && (i & (N / 4))) src |= 8;
    if (N >= 8 && (i & (N / 8))) src |= 4;
    v[i] = __shfl_sync(0xffffffffu, mine, src);
  }
}

// Householder reflector of a column with head alpha and tail norm^2 ss > 0
// (LAPACK dlarfg convention): beta = -sign(alpha) r, r = |(alpha, tail)|,
// tau = (beta - alpha) / beta = 1 + |alpha| / r, tail scale 1 / (alpha - beta)
// = sign(alpha) / (|alpha| + r); reciprocal square roots only on the chain.
__device__ __forceinline__ void householder(double alpha, double ss, double& beta,
                                            double& scal, double& tau) {
  const double r2 = fma(alpha, alpha, ss);
  const double ir = rsqrt(r2);
  const double r = r2 * ir;
  const double ix = rsqrt(fabs(alpha) + r);
  beta = -copysign(r, alpha);
  scal = copysign(ix * ix, alpha);
  tau = fma(fabs(alpha), ir, 1.0);
}

// Jacobi rotation (cos, sin) annihilating the off-diagonal 2c of the 2x2
// Gram block [a c; c b], d = b - a, e = 2c: the smaller rotation angle,
// tan(2 theta) = e / d, from the half-angle identities
//   cos^2 = (1 + |d|/r) / 2,  sin = sign(d) (e/r) / (2 cos),  r = |(d, e)|,
// two reciprocal square roots on the dependent chain (no sqrt, no division).
__device__ __forceinline__ void jacobi_rot(double d, double e, double& cs, double& sn) {
  const double ir = rsqrt(d * d + e * e);
  const double h = fma(0.5 * fabs(d), ir, 0.5);
  const double ih = rsqrt(h);
  cs = h * ih;
  sn = copysign(0.5, d) * e * ir * ih;
}


template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < (NT / 32); ++w) s += red[w];   // fixed order
  return s;
}

struct OpRes {
  const double* U;
  const double* V;
  int r;
  double sc;
};

__device__ __forceinline__ OpRes resolve_op(const TOp& op, const TreeDev& T,
                                            int g, int beta, int side,
                                            int urow, int vrow) {
  const int* rb = rank_base(op.rank, g);
  int slot, r;
  if (op.sel == SEL_OWN) {
    slot = T.depth[beta];
    r = rb[beta * 2 + side];
  } else if (op.sel == SEL_ANC) {
    const int* an = T.anc + beta * (T.maxdepth + 1);
    int a = an[op.t];
    int ch = an[op.t - 1];
    slot = T.depth[a];
    r = rb[a * 2 + (ch == T.c0[a] ? 0 : 1)];
  } else {
    slot = T.depth[op.node];
    r = rb[op.node * 2 + op.fside];
    if (op.sel == SEL_FIXED && rb[op.node * 2 + 1 - op.fside] == 0) r = 0;
  }
  OpRes o;
  o.r = r;
  o.sc = op.scale;
  o.U = o.V = nullptr;
  if (r > 0) {
    o.U = src_col(op.U, T.n, g, slot, 0) + urow;
    o.V = src_col(op.V, T.n, g, slot, 0) + vrow;
  }
  return o;
}

// Half-CTA thread group with its own named barrier (ids 1, 2), so the QR of
// U and of V (and later the two Q applications) run concurrently.
struct Grp {
  int id, nt, t, nw, w, lane;
  double* red;
  double* bc;
};

__device__ __forceinline__ void gbar(const Grp& g) {
  asm volatile("bar.sync %0, %1;" ::"r"(g.id), "r"(g.nt) : "memory");
}

__device__ __forceinline__ double gsum(double v, const Grp& g) {
  v = warp_sum(v);
  gbar(g);
  if (g.lane == 0) g.red[g.w] = v;
  gbar(g);
  double s = 0.0;
  for (int w = 0; w < g.nw; ++w) s += g.red[w];   // fixed order
  return s;
}

__device__ void group_qr(double* W, int mr, int R, double* tau, const Grp& g) {
  const int p = mr < R ? mr : R;
  for (int j = 0; j < p; ++j) {
    double* cj = W + (long long)j * mr;
    double ss = 0.0;
    for (int i = j + 1 + g.t; i < mr; i += g.nt) ss += cj[i] * cj[i];
    ss = gsum(ss, g);
    const double alpha = cj[j];
    double tj = 0.0, scal = 0.0, beta = alpha;
    if (ss != 0.0) {
      householder(alpha, ss, beta, scal, tj);
    }
    gbar(g);                                  // everyone has read cj[j]
    if (tj != 0.0) {
      for (int i = j + 1 + g.t; i < mr; i += g.nt) cj[i] *= scal;
      if (g.t == 0) cj[j] = beta;
    }
    if (g.t == 0) tau[j] = tj;
    gbar(g);
    if (tj != 0.0) {
      for (int c = j + 1 + g.w; c < R; c += g.nw) {
        double* cc = W + (long long)c * mr;
        double w = 0.0;
        for (int i = j + 1 + g.lane; i < mr; i += 32) w += cj[i] * cc[i];
        w = (warp_sum(w) + cc[j]) * tj;
        for (int i = j + 1 + g.lane; i < mr; i += 32) cc[i] -= w * cj[i];
        if (g.lane == 0) cc[j] -= w;
      }
      gbar(g);
    }
  }
}

// Householder QR with look-ahead (same reflectors as group_qr up to the
// summation order of the tail norms): warp 0 of the group owns the next
// column -- it applies reflector j to column j + 1, then forms reflector
// j + 1 from it (norm, dlarfg, scaling) -- while the other warps apply
// reflector j to columns j + 2 .. R - 1.  One group barrier per reflector
// instead of four; the critical path per step is warp 0's single-column
// update plus two warp reductions.
__device__ __forceinline__ void la_update(double* W, int mr, int j, int c, double tj, int lane) {
  const double* v = W + (long long)j * mr;
  double* cc = W + (long long)c * mr;
  double w = 0.0;
  for (int i = j + 1 + lane; i < mr; i += 32) w += v[i] * cc[i];
  w = (warp_sum(w) + cc[j]) * tj;
  for (int i = j + 1 + lane; i < mr; i += 32) cc[i] -= w * v[i];
  __syncwarp();
  if (lane == 0) cc[j] -= w;
  __syncwarp();
}

__device__ __forceinline__ void la_prep(double* W, int mr, int j, double* tau, int lane) {
  double* cj = W + (long long)j * mr;
  double ss = 0.0;
  for (int i = j + 1 + lane; i < mr; i += 32) ss += cj[i] * cj[i];
  ss = warp_sum(ss);
  const double alpha = cj[j];
  double tj = 0.0, scal = 0.0, beta = alpha;
  if (ss != 0.0) householder(alpha, ss, beta, scal, tj);
  __syncwarp();
  if (tj != 0.0) {
    for (int i = j + 1 + lane; i < mr; i += 32) cj[i] *= scal;
    if (lane == 0) cj[j] = beta;
  }
  if (lane == 0) tau[j] = tj;
  __syncwarp();
}

__device__ void group_qr_la(double* W, int mr, int R, double* tau, const Grp& g) {
  const int p = mr < R ? mr : R;
  if (p <= 0) return;
  if (g.w == 0) la_prep(W, mr, 0, tau, g.lane);
  gbar(g);
  const int nwo = g.nw - 1;                  // warps on the trailing columns (groups have >= 2)
  for (int j = 0; j < p; ++j) {
    const double tj = tau[j];
    if (g.w == 0) {
      if (j + 1 < p) {
        if (tj != 0.0) la_update(W, mr, j, j + 1, tj, g.lane);
        la_prep(W, mr, j + 1, tau, g.lane);
      }
    } else if (tj != 0.0) {
      // columns j + 2 .. R - 1 (and j + 1 when it is past the last reflector)
      const int c0 = j + 1 < p ? j + 2 : j + 1;
      for (int c = c0 + (g.w - 1); c < R; c += nwo) la_update(W, mr, j, c, tj, g.lane);
    }
    gbar(g);
  }
}

__device__ void group_apply_q(const double* W, int mr, int p, const double* tau,
                              double* X, int nc, const Grp& g) {
  for (int j = p - 1; j >= 0; --j) {
    const double tj = tau[j];
    if (tj != 0.0) {
      const double* v = W + (long long)j * mr;
      for (int c = g.w; c < nc; c += g.nw) {
        double* xc = X + (long long)c * mr;
        double w = 0.0;
        for (int i = j + 1 + g.lane; i < mr; i += 32) w += v[i] * xc[i];
        w = (warp_sum(w) + xc[j]) * tj;
        for (int i = j + 1 + g.lane; i < mr; i += 32) xc[i] -= w * v[i];
        if (g.lane == 0) xc[j] -= w;
      }
      gbar(g);
    }
  }
}

// Explicit Q (mr x p) formed in place over the reflectors (LAPACK dorg2r
// order: last reflector first); the R factor in the upper triangle is
// overwritten, so the core product must be formed before.
__device__ void group_form_q(double* W, int mr, int p, const double* tau, const Grp& g) {
  for (int j = p - 1; j >= 0; --j) {
    const double tj = tau[j];
    const double* v = W + (long long)j * mr;
    if (tj != 0.0) {
      for (int c = j + 1 + g.w; c < p; c += g.nw) {
        double* xc = W + (long long)c * mr;
        double w = 0.0;
        for (int i = j + 1 + g.lane; i < mr; i += 32) w += v[i] * xc[i];
        w = (warp_sum(w) + xc[j]) * tj;
        for (int i = j + 1 + g.lane; i < mr; i += 32) xc[i] -= w * v[i];
        if (g.lane == 0) xc[j] -= w;
      }
    }
    gbar(g);
    double* cj = W + (long long)j * mr;
    for (int i = g.t; i < mr; i += g.nt)
      cj[i] = i > j ? -tj * cj[i] : (i == j ? 1.0 - tj : 0.0);
    gbar(g);
  }
}

__constant__ bool jacobi_skip_confirm = true;
__constant__ bool trunc_qsplit = true;    // ACR_NO_QSPLIT=1: large cores on the whole CTA
__constant__ bool qr_lookahead = true;
__constant__ int qr_la_max = 512;   // look-ahead QR for panels of at most this many rows (taller: every warp on the norm and the scaling)

__device__ __forceinline__ int rr_player(int step, int x, int np) {
  if (x == 0) return 0;
  int t = x - 1 + step;              // < 2 (np - 1): one conditional wrap
  if (t >= np - 1) t -= np - 1;
  return 1 + t;
}

// One-sided Jacobi on B (pr x pc, column-major ld pr) accumulating J (pc x pc).
// The disjoint pairs of one round-robin step are spread over lane groups of
// size gs (power of two) across the whole CTA.
template <int NT>
__device__ int block_jacobi(double* B, int pr, int pc, double* J, int* flag) {
  const int tid = threadIdx.x;
  const int lb = pr | 1, lj = pc | 1;      // odd column strides: no bank conflicts
  for (int i = tid; i < pc * pc; i += NT) {
    const int c = i / pc, r = i - c * pc;
    J[c * lj + r] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  if (pc < 2) return 0;
  const int np = pc + (pc & 1), npairs = np / 2;
  int gs = 32;
  while (gs > 1 && gs * npairs > NT) gs >>= 1;
  const int per = NT / gs;
  const int sub = tid & (gs - 1), grp = tid / gs;
  const double tol = sqrt((double)pr) * 2.220446049250313e-16;
  // columns below eps64 * |B|_F cannot move any singular value that a
  // relative threshold >= 1e-14 keeps: rotations involving them are skipped
  double nb = 0.0;
  for (int i = tid; i < pr * pc; i += NT) {
    const double x = B[(i / pr) * lb + i % pr];
    nb += x * x;
  }
  __shared__ double s_nb[(NT / 32)];
  nb = warp_sum(nb);
  if ((tid & 31) == 0) s_nb[tid >> 5] = nb;
  __syncthreads();
  nb = 0.0;
  for (int w = 0; w < (NT / 32); ++w) nb += s_nb[w];
  const double tiny = nb * 4.930380657631324e-32;   // (eps64 |B|_F)^2
  (void)flag;
  for (int sweep = 0; sweep < 40; ++sweep) {
    int rot = 0;
    for (int step = 0; step < np - 1; ++step) {
      for (int base = 0; base < npairs; base += per) {
        const int k = base + grp;
        int i = 0, j = 0;
        bool valid = k < npairs;
        if (valid) {
          i = rr_player(step, k, np);
          j = rr_player(step, np - 1 - k, np);
          valid = i < pc && j < pc;
        }
        double a = 0.0, b = 0.0, c = 0.0;
        double* bi = B + (long long)i * lb;
        double* bj = B + (long long)j * lb;
        if (valid)
          for (int r = sub; r < pr; r += gs) {
            double x = bi[r], y = bj[r];
            a += x * x;
            b += y * y;
            c += x * y;
          }
        for (int o = gs >> 1; o; o >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o);
          b += __shfl_xor_sync(0xffffffffu, b, o);
          c += __shfl_xor_sync(0xffffffffu, c, o);
        }
        if (valid && a > tiny && b > tiny && c != 0.0 &&
            c * c > tol * tol * a * b) {
          const double d = b - a, e = 2.0 * c;
          double cs, sn;
          jacobi_rot(d, e, cs, sn);
          for (int r = sub; r < pr; r += gs) {
            double x = bi[r], y = bj[r];
            bi[r] = cs * x - sn * y;
            bj[r] = sn * x + cs * y;
          }
          double* ji = J + (long long)i * lj;
          double* jj = J + (long long)j * lj;
          for (int r = sub; r < pc; r += gs) {
            double x = ji[r], y = jj[r];
            ji[r] = cs * x - sn * y;
            jj[r] = sn * x + cs * y;
          }
          rot = 1;
        }
        __syncthreads();
      }
    }
    if (!__syncthreads_or(rot)) return sweep + 1;
  }
  return 40;
}

// block_jacobi on a subset of the CTA: threads t = 0 .. JT-1 (whole warps),
// named barrier `bar`, so the other warps can form the explicit Q meanwhile
// (direct launches: a large core's Jacobi is the longest phase of the task).
// Same pairing, lane groups and arithmetic as block_jacobi for JT threads,
// plus warp_jacobi's rule that a sweep of sub-1e-9 rotations ends the
// iteration (the confirmation sweep would rotate nothing).
__device__ int group_jacobi(double* B, int pr, int pc, double* J, int t, int JT, int bar) {
  __shared__ double gj_nb[16];
  __shared__ int gj_flag[3][2];
  auto sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(JT) : "memory"); };
  const int lb = pr | 1, lj = pc | 1;
  for (int i = t; i < pc * pc; i += JT) {
    const int c = i / pc, r = i - c * pc;
    J[c * lj + r] = (r == c) ? 1.0 : 0.0;
  }
  if (t < 6) gj_flag[t >> 1][t & 1] = 0;
  sync();
  if (pc < 2) return 0;
  const int np = pc + (pc & 1), npairs = np / 2;
  int gs = 32;
  while (gs > 1 && gs * npairs > JT) gs >>= 1;
  const int per = JT / gs;
  const int sub = t & (gs - 1), grp = t / gs;
  const double tol = sqrt((double)pr) * 2.220446049250313e-16;
  double nb = 0.0;
  for (int i = t; i < pr * pc; i += JT) {
    const double x = B[(i / pr) * lb + i % pr];
    nb += x * x;
  }
  nb = warp_sum(nb);
  if ((t & 31) == 0) gj_nb[t >> 5] = nb;
  sync();
  nb = 0.0;
  for (int w = 0; w < JT / 32; ++w) nb += gj_nb[w];
  const double tiny = nb * 4.930380657631324e-32;   // (eps64 |B|_F)^2
  const bool skipc = jacobi_skip_confirm;
  for (int sweep = 0; sweep < 40; ++sweep) {
    bool rot = false, big = false;
    const int fp = sweep % 3;
    if (t < 2) gj_flag[(sweep + 1) % 3][t] = 0;   // last read two sweeps ago
    for (int step = 0; step < np - 1; ++step) {
      for (int base = 0; base < npairs; base += per) {
        const int k = base + grp;
        int i = 0, j = 0;
        bool valid = k < npairs;
        if (valid) {
          i = rr_player(step, k, np);
          j = rr_player(step, np - 1 - k, np);
          valid = i < pc && j < pc;
        }
        double a = 0.0, b = 0.0, c = 0.0;
        double* bi = B + (long long)i * lb;
        double* bj = B + (long long)j * lb;
        if (valid)
          for (int r = sub; r < pr; r += gs) {
            double x = bi[r], y = bj[r];
            a += x * x;
            b += y * y;
            c += x * y;
          }
        for (int o = gs >> 1; o; o >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o);
          b += __shfl_xor_sync(0xffffffffu, b, o);
          c += __shfl_xor_sync(0xffffffffu, c, o);
        }
        if (valid && a > tiny && b > tiny && c != 0.0 &&
            c * c > tol * tol * a * b) {
          const double d = b - a, e = 2.0 * c;
          double cs, sn;
          jacobi_rot(d, e, cs, sn);
          for (int r = sub; r < pr; r += gs) {
            double x = bi[r], y = bj[r];
            bi[r] = cs * x - sn * y;
            bj[r] = sn * x + cs * y;
          }
          double* ji = J + (long long)i * lj;
          double* jj = J + (long long)j * lj;
          for (int r = sub; r < pc; r += gs) {
            double x = ji[r], y = jj[r];
            ji[r] = cs * x - sn * y;
            jj[r] = sn * x + cs * y;
          }
          rot = true;
          big |= c * c > 1e-18 * a * b;
        }
        sync();
      }
    }
    if (rot) gj_flag[fp][0] = 1;
    if (big) gj_flag[fp][1] = 1;
    sync();
    if (!gj_flag[fp][0]) return sweep + 1;
    if (skipc && !gj_flag[fp][1]) return sweep + 1;
  }
  return 40;
}

template <int NT>
__device__ void copy_factor(const OpRes& s, double* Uo, double* Vo, int um,
                            int vm, int n, int r) {
  if (s.U == Uo && s.V == Vo && s.sc == 1.0) return;
  for (int idx = threadIdx.x; idx < um * r; idx += NT) {
    int c = idx / um, i = idx - c * um;
    Uo[(long long)c * n + i] = s.sc * s.U[(long long)c * n + i];
  }
  for (int idx = threadIdx.x; idx < vm * r; idx += NT) {
    int c = idx / vm, i = idx - c * vm;
    Vo[(long long)c * n + i] = s.V[(long long)c * n + i];
  }
}

// ---------------------------------------------------------------------------
// task resolution shared by the warp and block paths
// ---------------------------------------------------------------------------
struct TaskCtx {
  OpRes a, b;
  int um, vm;
  double* Uo;
  double* Vo;
  int* ro;
  int Rout;
};

__device__ __forceinline__ TaskCtx resolve_task(const TruncArgs& A, int task, int g) {
  const TreeDev& T = A.T;
  const int n = T.n;
  const int beta = A.tasks[task * 3 + 1], side = A.tasks[task * 3 + 2];
  const int lo = T.lo[beta], hi = T.hi[beta], mid = T.mid[beta];
  const int urow = side ? mid : lo;
  const int vrow = side ? lo : mid;
  TaskCtx c;
  c.um = side ? hi - mid : mid - lo;
  c.vm = side ? mid - lo : hi - mid;
  c.a = resolve_op(A.a, T, g, beta, side, urow, vrow);
  c.b.r = 0;
  c.b.U = c.b.V = nullptr;
  c.b.sc = 1.0;
  if (A.mode != TM_TRUNCATE) c.b = resolve_op(A.b, T, g, beta, side, urow, vrow);
  if (A.mode == TM_COMBINE_SWAP1 && side == 1) {
    OpRes t = c.a;
    c.a = c.b;
    c.b = t;
  }
  const HB out = A.out[g];
  const long long oslot = (long long)T.depth[beta] * out.R * n;
  c.Uo = out.U + oslot + urow;
  c.Vo = out.V + oslot + vrow;
  c.ro = out.rk + beta * 2 + side;
  c.Rout = out.R;
  return c;
}

// 0: nothing to compute beyond a copy / zero (handled by the caller), 1: full
__device__ __forceinline__ bool task_is_full(const TruncArgs& A, const TaskCtx& c) {
  if (A.mode != TM_TRUNCATE) return c.a.r > 0 && c.b.r > 0;
  return c.a.r >= 2;
}

__host__ __device__ long long trunc_need_doubles(int um, int vm, int R) {
  return (long long)(um + vm) * R + 4LL * R * R + 6LL * R + 8;
}

// panels (um + vm) R, cores B and J R (R + 1) each (odd strides), tau_u, tau_v,
// sig R each, the rank order R ints, the output columns um + vm
__host__ __device__ long long warp_need_doubles(int um, int vm, int R) {
  return (long long)(um + vm) * R + 2LL * R * (R + 1) + 3LL * R + (R + 1) / 2 + um + vm;
}

__device__ int warp_jacobi(double* B, int pr, int pc, double* J, int lane);
__device__ int blk_jacobi(double* B, int pr, int pc, double* J, int lane);

// ---------------------------------------------------------------------------
// block path (one CTA per queued task; used for tasks too large for a warp)
// ---------------------------------------------------------------------------
template <int NT>
// score: when the work area is in global scratch, an optional shared-memory
// area for the Jacobi core and rotations (B, J) -- the Jacobi is most of a
// large task's time and should not run on global memory
__device__ __forceinline__ void trunc_block_full(const TruncArgs& A, const TaskCtx& tc, double* wk,
                                 double* red, int* iflag, double* score = nullptr) {
  const int tid = threadIdx.x, n = A.T.n;
  const OpRes& a = tc.a;
  const OpRes& b = tc.b;
  const int um = tc.um, vm = tc.vm;
  double* Uo = tc.Uo;
  double* Vo = tc.Vo;
  int* ro = tc.ro;
  const int R = a.r + b.r;
  const int pu = um < R ? um : R, pv = vm < R ? vm : R;
  double* Uw = wk;
  double* Vw = Uw + (long long)um * R;
  double* Bm = score ? score : Vw + (long long)vm * R;
  double* Jm = Bm + (long long)R * (R + 1);   // odd-strided cores (pr | 1, pc | 1)
  double* Cu = Vw + (long long)vm * R + 2LL * R * (R + 1);   // pu x keep coefficients
  double* Cv = Cu + (long long)R * R;          // pv x keep
  double* tauU = Cv + (long long)R * R;
  double* tauV = tauU + R;
  double* sig = tauV + R;
  int* ord = reinterpret_cast<int*>(sig + R);

  long long ph[6] = {0, 0, 0, 0, 0, 0};
  long long t_ph = clock64();
#define ACR_PH(i) do { if (A.ctr) { long long t_ = clock64(); ph[i] += t_ - t_ph; t_ph = t_; } } while (0)
  // operands by asynchronous copies (every element of a thread in flight at
  // once); the exact sign scales of the U columns applied after the wait.
  // Work areas in global scratch (tasks larger than shared memory) load
  // synchronously.
  if (!__isShared(Uw)) {
    for (int idx = tid; idx < um * R; idx += NT) {
      int c = idx / um, i = idx - c * um;
      Uw[idx] = c < a.r ? a.sc * a.U[(long long)c * n + i]
                        : b.sc * b.U[(long long)(c - a.r) * n + i];
    }
    for (int idx = tid; idx < vm * R; idx += NT) {
      int c = idx / vm, i = idx - c * vm;
      Vw[idx] = c < a.r ? a.V[(long long)c * n + i] : b.V[(long long)(c - a.r) * n + i];
    }
    __syncthreads();
  } else {
  for (int c = 0; c < R; ++c) {
    const double* su = c < a.r ? a.U + (long long)c * n : b.U + (long long)(c - a.r) * n;
    const double* sv = c < a.r ? a.V + (long long)c * n : b.V + (long long)(c - a.r) * n;
    for (int i = tid; i < um; i += NT) cp_async8(Uw + (long long)c * um + i, su + i, true);
    for (int i = tid; i < vm; i += NT) cp_async8(Vw + (long long)c * vm + i, sv + i, true);
  }
  cp_async_wait_all();
  __syncthreads();
  if (a.sc != 1.0 || b.sc != 1.0) {
    for (int idx = tid; idx < um * R; idx += NT)
      Uw[idx] *= idx < um * a.r ? a.sc : b.sc;
    __syncthreads();
  }
  }
  ACR_PH(0);
  {
    const int half = tid >= NT / 2 ? 1 : 0;
    const int t = tid - half * (NT / 2);
    Grp g{1 + half, NT / 2, t, (NT / 32) / 2, t >> 5, tid & 31, red + half * ((NT / 32) / 2),
          nullptr};
    if (qr_lookahead && (half ? vm : um) <= qr_la_max) {
      if (!half) group_qr_la(Uw, um, R, tauU, g);
      else group_qr_la(Vw, vm, R, tauV, g);
    } else {
      if (!half) group_qr(Uw, um, R, tauU, g);
      else group_qr(Vw, vm, R, tauV, g);
    }
  }
  __syncthreads();
  ACR_PH(1);

  // Frobenius norms of the triangular factors (hodlr.py:191-192)
  double nu2 = 0.0, nv2 = 0.0;
  for (int idx = tid; idx < pu * R; idx += NT) {
    int l = idx / pu, i = idx - l * pu;
    if (l >= i) { double x = Uw[(long long)l * um + i]; nu2 += x * x; }
  }
  for (int idx = tid; idx < pv * R; idx += NT) {
    int l = idx / pv, i = idx - l * pv;
    if (l >= i) { double x = Vw[(long long)l * vm + i]; nv2 += x * x; }
  }
  nu2 = block_sum<NT>(nu2, red);
  nv2 = block_sum<NT>(nv2, red);

  // core M = Ru Rv^T (pu x pv); B = M (pu >= pv) or M^T
  const bool tr = pu < pv;
  const int pr = tr ? pv : pu, pc = tr ? pu : pv;
  for (int idx = tid; idx < pu * pv; idx += NT) {
    int i = idx / pv, j = idx - i * pv;
    int l0 = i > j ? i : j;
    double s = 0.0;
    for (int l = l0; l < R; ++l)
      s += Uw[(long long)l * um + i] * Vw[(long long)l * vm + j];
    if (!tr) Bm[(long long)j * (pr | 1) + i] = s;
    else Bm[(long long)i * (pr | 1) + j] = s;
  }
  __syncthreads();
  ACR_PH(2);
  // small cores: one warp, warp-level syncs per rotation step (a CTA barrier
  // per step costs more than the step); large cores: the whole CTA
  int sweeps;
  const bool wj = pc <= 16 && pr <= 128;      // larger cores: every warp of the CTA
  // (cores of up to 40 columns: a larger core's Jacobi is bound by its work,
  // not by the chain of its steps, and wants all sixteen warps -- config 4,
  // ranks up to 101: 1.27 s with this limit, 1.90 s without)
  const bool qsplit = !wj && NT >= 512 && trunc_qsplit && pc <= 40;
  if (wj) {
    __shared__ int s_sw;
    if (tid < 32) {
      const int sw = blk_jacobi(Bm, pr, pc, Jm, tid);
      if (tid == 0) s_sw = sw;
    } else {
      // meanwhile the other warps form the explicit Q of both sides (it does
      // not depend on the SVD; the core has been formed from the R factors)
      const int t2 = tid - 32, nw2 = NT / 32 - 1, wu = nw2 / 2;
      const int half = (t2 >> 5) >= wu ? 1 : 0;
      const int nthr = (half ? nw2 - wu : wu) * 32;
      const int t = half ? t2 - wu * 32 : t2;
      Grp g{1 + half, nthr, t, nthr / 32, t >> 5, tid & 31, red + (half ? wu : 0), nullptr};
      if (!half) group_form_q(Uw, um, pu, tauU, g);
      else group_form_q(Vw, vm, pv, tauV, g);
    }
    __syncthreads();
    sweeps = s_sw;
  } else if (qsplit) {
    // large core, 512-thread CTA: the Jacobi on the first eight warps, the
    // explicit Q of both sides on the other eight (four per side) meanwhile
    __shared__ int s_sw2;
    if (tid < NT / 2) {
      const int sw = group_jacobi(Bm, pr, pc, Jm, tid, NT / 2, 3);
      if (tid == 0) s_sw2 = sw;
    } else {
      const int t2 = tid - NT / 2, nw2 = NT / 64, wu = nw2 / 2;
      const int half = (t2 >> 5) >= wu ? 1 : 0;
      const int nthr = (half ? nw2 - wu : wu) * 32;
      const int t = half ? t2 - wu * 32 : t2;
      Grp g{1 + half, nthr, t, nthr / 32, t >> 5, tid & 31, red + (half ? wu : 0), nullptr};
      if (!half) group_form_q(Uw, um, pu, tauU, g);
      else group_form_q(Vw, vm, pv, tauV, g);
    }
    __syncthreads();
    sweeps = s_sw2;
  } else {
    sweeps = block_jacobi<NT>(Bm, pr, pc, Jm, iflag);
  }
  ACR_PH(3);
  for (int j = tid; j < pc; j += NT) {
    double s = 0.0;
    const double* bj = Bm + (long long)j * (pr | 1);
    for (int r = 0; r < pr; ++r) s += bj[r] * bj[r];
    sig[j] = sqrt(s);
  }
  __syncthreads();
  for (int j = tid; j < pc; j += NT) {
    double sj = sig[j];
    int rnk = 0;
    for (int i = 0; i < pc; ++i) {
      double si = sig[i];
      rnk += (si > sj) || (si == sj && i < j);
    }
    ord[rnk] = j;
  }
  __syncthreads();
  const double s1 = sig[ord[0]];
  const double guard = (double)R * 2.220446049250313e-16 * sqrt(nu2) * sqrt(nv2);
  int keep = 0;
  if (s1 > guard) {
    const double thr = A.eps * s1;
    for (int i = 0; i < pc; ++i) keep += sig[i] >= thr;
    if (A.cap > 0 && keep > A.cap) keep = A.cap;
  }
  if (keep > tc.Rout) {
    if (tid == 0) atomicMax(A.overflow, keep);
    keep = 0;
  }
  ACR_PH(4);
  if (A.ctr && tid == 0) {   // census formulas of SURVEY.md Appendix C
    unsigned long long fl = 4ull * um * R * R + 4ull * vm * R * R + 24ull * R * R * R +
                            2ull * (um + vm) * R * keep;
    atomicAdd(A.ctr, fl);
    atomicAdd(A.ctr + 1, 8ull * ((unsigned long long)um * R + vm * R + um * keep + vm * keep));
    atomicAdd(A.ctr + 8, 1ull);
    atomicAdd(A.ctr + 10, (unsigned long long)sweeps);
  }
  if (keep == 0) {
    if (tid == 0) *ro = 0;
    if (A.ctr && tid == 0)
      for (int i = 0; i < 5; ++i) atomicAdd(A.ctr + 2 + i, (unsigned long long)ph[i]);
    return;
  }
  // coefficients of the kept singular pairs, then explicit Q (in place over
  // the reflectors, half-CTA per side) and U' = Q_u C_u, V' = Q_v C_v written
  // straight to the output columns
  for (int idx = tid; idx < pu * keep; idx += NT) {
    const int c = idx / pu, i = idx - c * pu;
    const int j = ord[c];
    Cu[idx] = tr ? sig[j] * Jm[(long long)j * (pc | 1) + i] : Bm[(long long)j * (pr | 1) + i];
  }
  for (int idx = tid; idx < pv * keep; idx += NT) {
    const int c = idx / pv, i = idx - c * pv;
    const int j = ord[c];
    Cv[idx] = tr ? Bm[(long long)j * (pr | 1) + i] / sig[j] : Jm[(long long)j * (pc | 1) + i];
  }
  if (!wj && !qsplit) {
    const int half = tid >= NT / 2 ? 1 : 0;
    const int t = tid - half * (NT / 2);
    Grp g{1 + half, NT / 2, t, (NT / 32) / 2, t >> 5, tid & 31, red + half * ((NT / 32) / 2),
          nullptr};
    if (!half) group_form_q(Uw, um, pu, tauU, g);
    else group_form_q(Vw, vm, pv, tauV, g);
  }
  __syncthreads();
  for (int idx = tid; idx < um * keep; idx += NT) {
    const int c = idx / um, i = idx - c * um;
    const double* cc = Cu + (long long)c * pu;
    double y = 0.0;
    for (int l = 0; l < pu; ++l) y += Uw[(long long)l * um + i] * cc[l];
    Uo[(long long)c * n + i] = y;
  }
  for (int idx = tid; idx < vm * keep; idx += NT) {
    const int c = idx / vm, i = idx - c * vm;
    const double* cc = Cv + (long long)c * pv;
    double y = 0.0;
    for (int l = 0; l < pv; ++l) y += Vw[(long long)l * vm + i] * cc[l];
    Vo[(long long)c * n + i] = y;
  }
  if (tid == 0) *ro = keep;
  ACR_PH(5);
  if (A.ctr && tid == 0 && A.direct_tag) {   // direct (latency-bound) launches apart
    atomicAdd(A.ctr + 160, 1ull);
    for (int i = 0; i < 6; ++i) atomicAdd(A.ctr + 161 + i, (unsigned long long)ph[i]);
    const int rb = R <= 8 ? 0 : R <= 16 ? 1 : R <= 32 ? 2 : R <= 64 ? 3 : 4;
    const int mm = um > vm ? um : vm;
    const int mb = mm <= 128 ? 0 : mm <= 256 ? 1 : mm <= 512 ? 2 : mm <= 1024 ? 3 : 4;
    long long tot = 0;
    for (int i = 0; i < 6; ++i) tot += ph[i];
    atomicAdd(A.ctr + 170 + rb * 5 + mb, 1ull);
    atomicAdd(A.ctr + 195 + rb * 5 + mb, (unsigned long long)tot);
    atomicAdd(A.ctr + 220 + rb * 5 + mb, (unsigned long long)ph[1]);
  }
  if (A.ctr && tid == 0) {
    for (int i = 0; i < 6; ++i) atomicAdd(A.ctr + 2 + i, (unsigned long long)ph[i]);
    // histogram: R bucket (<=8, <=16, <=32, <=64, >64) x m bucket (<=128, 256,
    // 512, 1024, >1024): count, total cycles, Jacobi cycles
    const int rb = R <= 8 ? 0 : R <= 16 ? 1 : R <= 32 ? 2 : R <= 64 ? 3 : 4;
    const int mm = um > vm ? um : vm;
    const int mb = mm <= 128 ? 0 : mm <= 256 ? 1 : mm <= 512 ? 2 : mm <= 1024 ? 3 : 4;
    long long tot = 0;
    for (int i = 0; i < 6; ++i) tot += ph[i];
    atomicAdd(A.ctr + 72 + rb * 5 + mb, 1ull);
    atomicAdd(A.ctr + 97 + rb * 5 + mb, (unsigned long long)tot);
    atomicAdd(A.ctr + 122 + rb * 5 + mb, (unsigned long long)ph[3]);
  }
}


// rank-0 / passthrough / rank-1 shortcut cases, whole CTA (uniform branch)
template <int NT>
__device__ bool block_trivial(const TruncArgs& A, const TaskCtx& c, double* red) {
  const int tid = threadIdx.x, n = A.T.n;
  if (A.mode != TM_TRUNCATE && (c.a.r == 0 || c.b.r == 0)) {   // algebra.py:93-96
    const OpRes& s = c.a.r ? c.a : c.b;
    int r = s.r;
    if (r > c.Rout) {
      if (tid == 0) atomicMax(A.overflow, r);
      r = c.Rout;
    }
    if (r) copy_factor<NT>(s, c.Uo, c.Vo, c.um, c.vm, n, r);
    if (tid == 0) {
      *c.ro = r;
      if (A.ctr && r && !(s.U == c.Uo && s.V == c.Vo && s.sc == 1.0))
        atomicAdd(A.ctr + 1, 16ull * (c.um + c.vm) * r);
    }
    return true;
  }
  if (A.mode == TM_TRUNCATE && c.a.r < 2) {
    int r = 0;
    if (c.a.r == 1) {                                           // hodlr.py:181-185
      double nzu = 0.0, nzv = 0.0;
      for (int i = tid; i < c.um; i += NT) nzu += (c.a.U[i] != 0.0) ? 1.0 : 0.0;
      for (int i = tid; i < c.vm; i += NT) nzv += (c.a.V[i] != 0.0) ? 1.0 : 0.0;
      nzu = block_sum<NT>(nzu, red);
      nzv = block_sum<NT>(nzv, red);
      r = (nzu > 0.0 && nzv > 0.0) ? 1 : 0;
      if (r > c.Rout) {
        if (tid == 0) atomicMax(A.overflow, r);
        r = 0;
      }
      if (r) copy_factor<NT>(c.a, c.Uo, c.Vo, c.um, c.vm, n, 1);
    }
    if (tid == 0) *c.ro = r;
    return true;
  }
  return false;
}

// q == nullptr: direct mode, one CTA per item (small launches, latency bound)
// otherwise: persistent CTAs over the queue of tasks the warp path rejected
template <int NT>
__global__ void __launch_bounds__(NT, 512 / NT) k_trunc_big(TruncArgs A, const int* q,
                                                  const int* qcount, int nitems) {
  ACR_PDL_ENTRY();
  extern __shared__ double sm[];
  __shared__ double red[(NT / 32) + 4];
  __shared__ int iflag[2];
  const int cnt = q ? *qcount : nitems;
  __shared__ int s_next;
  for (int i = blockIdx.x;; i += gridDim.x) {
    if (q) {
      // queue mode: the next queued task from a counter (qcount + 3; tasks
      // differ widely in size, static striding left CTAs idle at the tail)
      __syncthreads();
      if (threadIdx.x == 0) s_next = atomicAdd(const_cast<int*>(qcount) + 3, 1);
      __syncthreads();
      i = s_next;
    }
    if (i >= cnt) break;
    const int item = q ? q[i] : i;
    const int task = item % A.ntasks, g = item / A.ntasks;
    TaskCtx c = resolve_task(A, task, g);
    __syncthreads();
    if (!q && block_trivial<NT>(A, c, red)) {
      __syncthreads();
      continue;
    }
    const int R = c.a.r + c.b.r;
    const long long need = trunc_need_doubles(c.um, c.vm, R);
    if (need > A.smem_doubles) {
      if (A.gscr == nullptr || need > A.gscr_stride) {
        if (threadIdx.x == 0) atomicMax(A.overflow, 1 << 29);
        continue;
      }
      trunc_block_full<NT>(A, c, A.gscr + (long long)blockIdx.x * A.gscr_stride, red, iflag,
                           2LL * R * (R + 1) <= A.smem_doubles ? sm : nullptr);
    } else {
      // separate inlined copy on the shared-memory work area: LDS / STS
      // instead of generic loads and stores
      trunc_block_full<NT>(A, c, sm, red, iflag);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// CTA-pair path (thread-block cluster of 2) for latency-bound launches of
// large tasks: CTA 0 owns U, CTA 1 owns V, each with all TT threads and its
// panel in its own shared memory.  R_v and |R_v|_F reach CTA 0 through
// distributed shared memory; CTA 0 forms the core, runs the Jacobi SVD and
// the rank decision and writes the coefficients of both sides (C_v into CTA
// 1's shared memory); then each CTA forms its explicit Q in place and writes
// its output factor.  Same arithmetic as trunc_block_full.
// ---------------------------------------------------------------------------
__host__ __device__ long long pair_need_doubles(int m, int R) {
  return (long long)m * R + 4LL * R * R + 5LL * R + 8;
}

__device__ __forceinline__ bool task_trivial(const TruncArgs& A, const TaskCtx& c) {
  if (A.mode != TM_TRUNCATE) return c.a.r == 0 || c.b.r == 0;
  return c.a.r < 2;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TT, 1)
    k_trunc_pair(TruncArgs A, int nitems) {
  ACR_PDL_ENTRY();
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double sm[];
  __shared__ double red[NWB + 4];
  __shared__ int iflag[2];
  const int side = (int)cl.block_rank();
  const int tid = threadIdx.x, n = A.T.n;
  for (int item = blockIdx.x / 2; item < nitems; item += gridDim.x / 2) {
    const int task = item % A.ntasks, g = item / A.ntasks;
    TaskCtx c = resolve_task(A, task, g);
    __syncthreads();
    if (task_trivial(A, c)) {                 // both CTAs agree; CTA 0 writes
      if (side == 0) block_trivial<TT>(A, c, red);
      __syncthreads();
      continue;
    }
    const OpRes& a = c.a;
    const OpRes& b = c.b;
    const int R = a.r + b.r;
    const int m = side ? c.vm : c.um;
    const int p = m < R ? m : R;
    // small arrays first (offsets depend on R only: the same in both CTAs,
    // which address each other's through DSMEM), the panel after them -- or
    // in a per-CTA global area when it does not fit (rare: capacities size
    // the launch, actual ranks are usually far below them)
    double* Rs = sm;                          // own R factor, [l][i] = Rs[l * R + i]
    double* Bm = Rs + (long long)R * R;
    double* Jm = Bm + (long long)R * (R + 1);   // odd-strided cores (pr | 1, pc | 1)
    double* Cs = Jm + (long long)R * (R + 1);       // own coefficients p x keep
    double* tau = Cs + (long long)R * R;
    double* sig = tau + R;
    int* ord = reinterpret_cast<int*>(sig + R);
    double* misc = sig + 2 * R;               // [0] |R|_F^2, [1] keep
    const long long small = 4LL * R * R + 5LL * R + 8;   // through misc[0..1]
    const bool w_sm = small + (long long)m * R <= A.smem_doubles;
    double* W = w_sm ? sm + small : A.gscr + (long long)blockIdx.x * A.gscr_stride;
    long long ph[6] = {0, 0, 0, 0, 0, 0};
    long long t_ph = clock64();
    for (int cc = 0; cc < R; ++cc) {
      const double* src = side == 0
          ? (cc < a.r ? a.U + (long long)cc * n : b.U + (long long)(cc - a.r) * n)
          : (cc < a.r ? a.V + (long long)cc * n : b.V + (long long)(cc - a.r) * n);
      if (w_sm)
        for (int i = tid; i < m; i += TT) cp_async8(W + (long long)cc * m + i, src + i, true);
      else
        for (int i = tid; i < m; i += TT) W[(long long)cc * m + i] = src[i];
    }
    cp_async_wait_all();
    __syncthreads();
    if (side == 0 && (a.sc != 1.0 || b.sc != 1.0)) {
      for (int idx = tid; idx < m * R; idx += TT) W[idx] *= idx < m * a.r ? a.sc : b.sc;
      __syncthreads();
    }
    ACR_PH(0);
    const Grp gf{1, TT, tid, NWB, tid >> 5, tid & 31, red, nullptr};
    if (qr_lookahead && m <= qr_la_max) group_qr_la(W, m, R, tau, gf);
    else group_qr(W, m, R, tau, gf);
    __syncthreads();
    ACR_PH(1);
    double nr2 = 0.0;
    for (int idx = tid; idx < R * R; idx += TT) {
      const int l = idx / R, i = idx - l * R;
      const double x = (i < p && l >= i) ? W[(long long)l * m + i] : 0.0;
      Rs[idx] = x;
      nr2 += x * x;
    }
    nr2 = block_sum<TT>(nr2, red);
    if (tid == 0) misc[0] = nr2;
    cl.sync();                                 // both R factors published
    // the explicit Q of each side does not depend on the SVD: side 1 forms
    // its Q while side 0 runs the core and the Jacobi; side 0's other warps
    // form Q_u during a single-warp Jacobi
    bool qdone = false;
    if (side == 1) {
      group_form_q(W, m, p, tau, gf);
      qdone = true;
    }
    if (side == 0) {
      const double* Rv = cl.map_shared_rank(Rs, 1);
      const double* mv = cl.map_shared_rank(misc, 1);
      double* Cv = cl.map_shared_rank(Cs, 1);
      double* mv_w = cl.map_shared_rank(misc, 1);
      const double nu2 = nr2, nv2 = mv[0];
      const int pu = p, pv = c.vm < R ? c.vm : R;
      const bool tr = pu < pv;
      const int pr = tr ? pv : pu, pc = tr ? pu : pv;
      for (int idx = tid; idx < pu * pv; idx += TT) {
        const int i = idx / pv, j = idx - i * pv;
        const int l0 = i > j ? i : j;
        double sacc = 0.0;
        for (int l = l0; l < R; ++l) sacc += Rs[l * R + i] * Rv[l * R + j];
        if (!tr) Bm[(long long)j * (pr | 1) + i] = sacc;
        else Bm[(long long)i * (pr | 1) + j] = sacc;
      }
      __syncthreads();
      ACR_PH(2);
      int sweeps;
      if (pc <= 16 && pr <= 128) {   // larger cores: every warp of the CTA
        __shared__ int s_sw;
        if (tid < 32) {
          const int sw = blk_jacobi(Bm, pr, pc, Jm, tid);
          if (tid == 0) s_sw = sw;
        } else {
          const Grp gq{1, TT - 32, tid - 32, NWB - 1, (tid - 32) >> 5, tid & 31, red, nullptr};
          group_form_q(W, m, p, tau, gq);
        }
        __syncthreads();
        sweeps = s_sw;
        qdone = true;
      } else {
        sweeps = block_jacobi<TT>(Bm, pr, pc, Jm, iflag);
      }
      ACR_PH(3);
      for (int j = tid; j < pc; j += TT) {
        double sacc = 0.0;
        const double* bj = Bm + (long long)j * (pr | 1);
        for (int r = 0; r < pr; ++r) sacc += bj[r] * bj[r];
        sig[j] = sqrt(sacc);
      }
      __syncthreads();
      for (int j = tid; j < pc; j += TT) {
        const double sj = sig[j];
        int rnk = 0;
        for (int i = 0; i < pc; ++i) {
          const double si = sig[i];
          rnk += (si > sj) || (si == sj && i < j);
        }
        ord[rnk] = j;
      }
      __syncthreads();
      const double s1 = sig[ord[0]];
      const double guard = (double)R * 2.220446049250313e-16 * sqrt(nu2) * sqrt(nv2);
      int keep = 0;
      if (s1 > guard) {
        const double thr = A.eps * s1;
        for (int i = 0; i < pc; ++i) keep += sig[i] >= thr;
        if (A.cap > 0 && keep > A.cap) keep = A.cap;
      }
      if (keep > c.Rout) {
        if (tid == 0) atomicMax(A.overflow, keep);
        keep = 0;
      }
      for (int idx = tid; idx < pu * keep; idx += TT) {
        const int cc = idx / pu, i = idx - cc * pu;
        const int j = ord[cc];
        Cs[idx] = tr ? sig[j] * Jm[(long long)j * (pc | 1) + i] : Bm[(long long)j * (pr | 1) + i];
      }
      for (int idx = tid; idx < pv * keep; idx += TT) {
        const int cc = idx / pv, i = idx - cc * pv;
        const int j = ord[cc];
        Cv[idx] = tr ? Bm[(long long)j * (pr | 1) + i] / sig[j] : Jm[(long long)j * (pc | 1) + i];
      }
      if (tid == 0) {
        misc[1] = keep;
        mv_w[1] = keep;
      }
      ACR_PH(4);
      if (A.ctr && tid == 0) {   // census formulas of SURVEY.md Appendix C
        const unsigned long long um = c.um, vm = c.vm;
        unsigned long long fl = 4ull * um * R * R + 4ull * vm * R * R + 24ull * R * R * R +
                                2ull * (um + vm) * R * keep;
        atomicAdd(A.ctr, fl);
        atomicAdd(A.ctr + 1, 8ull * (um * R + vm * R + um * keep + vm * keep));
        atomicAdd(A.ctr + 8, 1ull);
        atomicAdd(A.ctr + 10, (unsigned long long)sweeps);
      }
    }
    cl.sync();                                 // coefficients and keep published
    const int keep = (int)misc[1];
    if (keep > 0) {
      if (!qdone) group_form_q(W, m, p, tau, gf);
      __syncthreads();
      double* O = side ? c.Vo : c.Uo;
      for (int idx = tid; idx < m * keep; idx += TT) {
        const int cc = idx / m, i = idx - cc * m;
        const double* co = Cs + (long long)cc * p;
        double y = 0.0;
        for (int l = 0; l < p; ++l) y += W[(long long)l * m + i] * co[l];
        O[(long long)cc * n + i] = y;
      }
    }
    if (side == 0 && tid == 0) *c.ro = keep;
    ACR_PH(5);
    if (A.ctr && side == 0 && tid == 0) {
      for (int i = 0; i < 6; ++i) atomicAdd(A.ctr + 2 + i, (unsigned long long)ph[i]);
      const int rb = R <= 8 ? 0 : R <= 16 ? 1 : R <= 32 ? 2 : R <= 64 ? 3 : 4;
      const int mm = c.um > c.vm ? c.um : c.vm;
      const int mb = mm <= 128 ? 0 : mm <= 256 ? 1 : mm <= 512 ? 2 : mm <= 1024 ? 3 : 4;
      long long tot = 0;
      for (int i = 0; i < 6; ++i) tot += ph[i];
      atomicAdd(A.ctr + 72 + rb * 5 + mb, 1ull);
      atomicAdd(A.ctr + 97 + rb * 5 + mb, (unsigned long long)tot);
      atomicAdd(A.ctr + 122 + rb * 5 + mb, (unsigned long long)ph[3]);
    }
    __syncthreads();
  }
}

void trunc_init_flags();

cudaError_t launch_trunc_pair(const TruncArgs& a, int nelem, long long smem_doubles,
                              cudaStream_t st) {
  if (a.ntasks == 0 || nelem == 0) return cudaSuccess;
  trunc_init_flags();
  const size_t bytes = (size_t)smem_doubles * 8 + 64;
  static size_t attr = 0;
  if (bytes > attr) {
    cudaError_t e = cudaFuncSetAttribute(k_trunc_pair,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)bytes);
    if (e != cudaSuccess) return e;
    attr = bytes;
  }
  const int nitems = a.ntasks * nelem;
  CK_PDL(launch_pdl(k_trunc_pair, dim3(2 * nitems), dim3(TT), bytes, st, a, nitems));
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// warp path: one warp per task, work area carved from a per-CTA smem pool
// ---------------------------------------------------------------------------
static constexpr int TW = 20;          // warps per CTA (96 registers, no spills)
static constexpr int SLOT = 448;       // doubles per slot (3.5 KB)
static constexpr int NSLOT = 64;       // 224 KB pool, one 64-bit occupancy mask
static constexpr unsigned FULL = 0xffffffffu;
static constexpr int QHALF = 112 * 1024;   // queue CTAs: two per SM below this work area
static constexpr int QHALF_D = (QHALF - 64) / 8;

// Reserve ns contiguous slots of the per-CTA pool.  The whole warp runs the
// loop (lane 0 does the atomics, the outcome is broadcast every iteration),
// so no lane ever waits in a shuffle while lane 0 spins alone.
__device__ __forceinline__ int acquire_slots(unsigned long long* mask, int ns, int lane) {
  const unsigned long long want = ns >= 64 ? ~0ull : ((1ull << ns) - 1ull);
  while (true) {
    int s = -1;
    if (lane == 0) {
      const unsigned long long m = atomicAdd(mask, 0ull);
      // bit k of run: slots k .. k+ns-1 all free (the shifts bring in zeros =
      // used), by doubling: O(log ns) steps for the warps that spin here
      unsigned long long run = ~m;
      for (int have = 1; have < ns;) {
        const int step = have < ns - have ? have : ns - have;
        run &= run >> step;
        have += step;
      }
      if (run) {
        s = __ffsll((long long)run) - 1;
        if (atomicCAS(mask, m, m | (want << s)) != m) s = -2;
      }
    }
    s = __shfl_sync(FULL, s, 0);
    if (s >= 0) return s;
    if (s == -1) __nanosleep(128);
  }
}

__device__ __forceinline__ void warp_copy_factor(const OpRes& s, double* Uo, double* Vo,
                                                 int um, int vm, int n, int r, int lane) {
  if (s.U == Uo && s.V == Vo && s.sc == 1.0) return;
  for (int c = 0; c < r; ++c) {
    const double* su = s.U + (long long)c * n;
    double* du = Uo + (long long)c * n;
    for (int i = lane; i < um; i += 32) du[i] = s.sc * su[i];
    const double* sv = s.V + (long long)c * n;
    double* dv = Vo + (long long)c * n;
    for (int i = lane; i < vm; i += 32) dv[i] = sv[i];
  }
}

// Householder QR of U (mu x R) and V (mv x R) by one warp, interleaved: the
// two factorisations are independent, so their reduction chains overlap.
template <int MR>
__device__ __forceinline__ void warp_reflector(double* cj, int j, int mr, double ss,
                                               double& tj, int lane) {
  const double alpha = cj[j];
  double scal = 0.0, beta = alpha;
  tj = 0.0;
  if (ss != 0.0) {
    householder(alpha, ss, beta, scal, tj);
  }
  __syncwarp();
  if (tj != 0.0) {
    if constexpr (MR > 0) {
#pragma unroll
      for (int h = 0; h < MR; ++h)
        if (lane + 32 * h > j) cj[lane + 32 * h] *= scal;
    } else {
      for (int i = j + 1 + lane; i < mr; i += 32) cj[i] *= scal;
    }
    if (lane == 0) cj[j] = beta;
  }
}

// MR > 0: both panels have exactly 32 MR rows (lane owns rows lane + 32 h);
// the same operations in the same per-lane order as the generic MR = 0 path.
template <int MR>
__device__ void warp_qr2(double* Wu, int mu, double* tu, double* Wv, int mv, double* tv,
                         int R, int lane) {
  const int pu = mu < R ? mu : R, pv = mv < R ? mv : R;
  const int p = pu > pv ? pu : pv;
  for (int j = 0; j < p; ++j) {
    const bool du = j < pu, dv = j < pv;
    double* cu = Wu + (long long)j * mu;
    double* cv = Wv + (long long)j * mv;
    double su = 0.0, sv = 0.0;
    if constexpr (MR > 0) {
#pragma unroll
      for (int h = 0; h < MR; ++h) {
        const int i = lane + 32 * h;
        if (i > j) {
          if (du) su += cu[i] * cu[i];
          if (dv) sv += cv[i] * cv[i];
        }
      }
    } else {
      if (du) for (int i = j + 1 + lane; i < mu; i += 32) su += cu[i] * cu[i];
      if (dv) for (int i = j + 1 + lane; i < mv; i += 32) sv += cv[i] * cv[i];
    }
    warp_sum2(su, sv, lane);
    double tju = 0.0, tjv = 0.0;
    if (du) warp_reflector<MR>(cu, j, mu, su, tju, lane);
    if (dv) warp_reflector<MR>(cv, j, mv, sv, tjv, lane);
    if (lane == 0) {
      if (du) tu[j] = tju;
      if (dv) tv[j] = tjv;
    }
    __syncwarp();
    const bool au = du && tju != 0.0, av = dv && tjv != 0.0;
    if (!au && !av) continue;
    int cfirst = j + 1;
    if constexpr (MR > 0) {
      // four trailing columns per pass: the reflector is read once for the
      // four, their eight sums are reduced together (warp_sum_multi), the
      // updates follow; per column the same operations in the same order
      for (; cfirst + 3 < R; cfirst += 4) {
        double w[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) w[q] = 0.0;
        double ru[MR], rv[MR];
#pragma unroll
        for (int h = 0; h < MR; ++h) {
          const int i = lane + 32 * h;
          ru[h] = (au && i > j) ? cu[i] : 0.0;
          rv[h] = (av && i > j) ? cv[i] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double* ccu = Wu + (long long)(cfirst + q) * mu;
          const double* ccv = Wv + (long long)(cfirst + q) * mv;
#pragma unroll
          for (int h = 0; h < MR; ++h) {
            const int i = lane + 32 * h;
            if (i > j) {
              if (au) w[q] += ru[h] * ccu[i];
              if (av) w[4 + q] += rv[h] * ccv[i];
            }
          }
        }
        warp_sum_multi<8>(w, lane);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double* ccu = Wu + (long long)(cfirst + q) * mu;
          double* ccv = Wv + (long long)(cfirst + q) * mv;
          if (au) {
            const double wu = (w[q] + ccu[j]) * tju;
#pragma unroll
            for (int h = 0; h < MR; ++h)
              if (lane + 32 * h > j) ccu[lane + 32 * h] -= wu * ru[h];
            if (lane == 0) ccu[j] -= wu;
          }
          if (av) {
            const double wv = (w[4 + q] + ccv[j]) * tjv;
#pragma unroll
            for (int h = 0; h < MR; ++h)
              if (lane + 32 * h > j) ccv[lane + 32 * h] -= wv * rv[h];
            if (lane == 0) ccv[j] -= wv;
          }
        }
      }
    }
    for (int c = cfirst; c < R; ++c) {
      double* ccu = Wu + (long long)c * mu;
      double* ccv = Wv + (long long)c * mv;
      double wu = 0.0, wv = 0.0;
      if constexpr (MR > 0) {
#pragma unroll
        for (int h = 0; h < MR; ++h) {
          const int i = lane + 32 * h;
          if (i > j) {
            if (au) wu += cu[i] * ccu[i];
            if (av) wv += cv[i] * ccv[i];
          }
        }
      } else {
        if (au) for (int i = j + 1 + lane; i < mu; i += 32) wu += cu[i] * ccu[i];
        if (av) for (int i = j + 1 + lane; i < mv; i += 32) wv += cv[i] * ccv[i];
      }
      warp_sum2(wu, wv, lane);
      if (au) {
        wu = (wu + ccu[j]) * tju;
        if constexpr (MR > 0) {
#pragma unroll
          for (int h = 0; h < MR; ++h)
            if (lane + 32 * h > j) ccu[lane + 32 * h] -= wu * cu[lane + 32 * h];
        } else {
          for (int i = j + 1 + lane; i < mu; i += 32) ccu[i] -= wu * cu[i];
        }
        if (lane == 0) ccu[j] -= wu;
      }
      if (av) {
        wv = (wv + ccv[j]) * tjv;
        if constexpr (MR > 0) {
#pragma unroll
          for (int h = 0; h < MR; ++h)
            if (lane + 32 * h > j) ccv[lane + 32 * h] -= wv * cv[lane + 32 * h];
        } else {
          for (int i = j + 1 + lane; i < mv; i += 32) ccv[i] -= wv * cv[i];
        }
        if (lane == 0) ccv[j] -= wv;
      }
    }
    __syncwarp();
  }
}

// xu := Qu xu and xv := Qv xv, interleaved
template <int MR>
__device__ void warp_apply_q2(const double* Wu, int mu, int pu, const double* tu,
                              double* xu, const double* Wv, int mv, int pv,
                              const double* tv, double* xv, int lane) {
  const int p = pu > pv ? pu : pv;
  for (int j = p - 1; j >= 0; --j) {
    const double tju = j < pu ? tu[j] : 0.0;
    const double tjv = j < pv ? tv[j] : 0.0;
    if (tju == 0.0 && tjv == 0.0) continue;
    const double* vu = Wu + (long long)j * mu;
    const double* vv = Wv + (long long)j * mv;
    double wu = 0.0, wv = 0.0;
    if constexpr (MR > 0) {
#pragma unroll
      for (int h = 0; h < MR; ++h) {
        const int i = lane + 32 * h;
        if (i > j) {
          if (tju != 0.0) wu += vu[i] * xu[i];
          if (tjv != 0.0) wv += vv[i] * xv[i];
        }
      }
    } else {
      if (tju != 0.0) for (int i = j + 1 + lane; i < mu; i += 32) wu += vu[i] * xu[i];
      if (tjv != 0.0) for (int i = j + 1 + lane; i < mv; i += 32) wv += vv[i] * xv[i];
    }
    warp_sum2(wu, wv, lane);
    if (tju != 0.0) {
      wu = (wu + xu[j]) * tju;
      if constexpr (MR > 0) {
#pragma unroll
        for (int h = 0; h < MR; ++h)
          if (lane + 32 * h > j) xu[lane + 32 * h] -= wu * vu[lane + 32 * h];
      } else {
        for (int i = j + 1 + lane; i < mu; i += 32) xu[i] -= wu * vu[i];
      }
    }
    if (tjv != 0.0) {
      wv = (wv + xv[j]) * tjv;
      if constexpr (MR > 0) {
#pragma unroll
        for (int h = 0; h < MR; ++h)
          if (lane + 32 * h > j) xv[lane + 32 * h] -= wv * vv[lane + 32 * h];
      } else {
        for (int i = j + 1 + lane; i < mv; i += 32) xv[i] -= wv * vv[i];
      }
    }
    __syncwarp();
    if (lane == 0) {
      if (tju != 0.0) xu[j] -= wu;
      if (tjv != 0.0) xv[j] -= wv;
    }
    __syncwarp();
  }
}



// Output factors for panels of MR * 32 rows per side (um == vm): KC kept
// columns at a time live in registers (rows lane + 32 h), every reflector is
// applied to all of them with one pass over its smem entries and independent
// warp reductions, and the head element is folded into the reduction
// (v_j[j] = 1), so there is no per-column shared-memory round trip or lane-0
// step.  x := Q_u x (and Q_v on the other side), written straight to HBM.
template <int MR, int KC>
__device__ __forceinline__ void warp_out_reg(const double* Wu, const double* Wv, int m,
                                             int pu, int pv, const double* tu,
                                             const double* tv, const double* Bm,
                                             const double* Jm, const double* sig,
                                             const int* ord, int pr, int pc, bool tr,
                                             int c0, int kk, double* Uo, double* Vo,
                                             int n, int lane) {
  double xu[KC][MR], xv[KC][MR];
#pragma unroll
  for (int c = 0; c < KC; ++c) {
    const int j = ord[c0 + (c < kk ? c : 0)];
    const double sj = sig[j];
#pragma unroll
    for (int h = 0; h < MR; ++h) {
      const int i = lane + 32 * h;
      double u = 0.0, v = 0.0;
      if (c < kk) {
        if (i < pu) u = tr ? sj * Jm[(long long)j * (pc | 1) + i] : Bm[(long long)j * (pr | 1) + i];
        if (i < pv) v = tr ? Bm[(long long)j * (pr | 1) + i] / sj : Jm[(long long)j * (pc | 1) + i];
      }
      xu[c][h] = u;
      xv[c][h] = v;
    }
  }
  const int p = pu > pv ? pu : pv;
  for (int j = p - 1; j >= 0; --j) {
    const double tju = j < pu ? tu[j] : 0.0;
    const double tjv = j < pv ? tv[j] : 0.0;
    const double* vu = Wu + (long long)j * m;
    const double* vv = Wv + (long long)j * m;
    double au[MR], av[MR];
#pragma unroll
    for (int h = 0; h < MR; ++h) {
      const int i = lane + 32 * h;
      au[h] = i > j ? vu[i] : (i == j ? 1.0 : 0.0);
      av[h] = i > j ? vv[i] : (i == j ? 1.0 : 0.0);
    }
    double w[2 * KC];                             // [c]: U side, [KC + c]: V side
#pragma unroll
    for (int c = 0; c < KC; ++c) {
      w[c] = 0.0;
      w[KC + c] = 0.0;
#pragma unroll
      for (int h = 0; h < MR; ++h) {
        w[c] = fma(au[h], xu[c][h], w[c]);
        w[KC + c] = fma(av[h], xv[c][h], w[KC + c]);
      }
    }
    warp_sum_multi<2 * KC>(w, lane);
#pragma unroll
    for (int c = 0; c < KC; ++c) {
      const double gu = w[c] * tju, gv = w[KC + c] * tjv;
#pragma unroll
      for (int h = 0; h < MR; ++h) {
        xu[c][h] = fma(-gu, au[h], xu[c][h]);
        xv[c][h] = fma(-gv, av[h], xv[c][h]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < KC; ++c)
    if (c < kk) {
      double* du = Uo + (long long)(c0 + c) * n;
      double* dv = Vo + (long long)(c0 + c) * n;
#pragma unroll
      for (int h = 0; h < MR; ++h) {
        du[lane + 32 * h] = xu[c][h];
        dv[lane + 32 * h] = xv[c][h];
      }
    }
}

template <int MR>
__device__ __forceinline__ void warp_out_regs(const double* Wu, const double* Wv, int m,
                                              int pu, int pv, const double* tu,
                                              const double* tv, const double* Bm,
                                              const double* Jm, const double* sig,
                                              const int* ord, int pr, int pc, bool tr,
                                              int keep, double* Uo, double* Vo, int n,
                                              int lane) {
  constexpr int KM = MR >= 4 ? 1 : 4;   // register budget: KM x MR doubles per side
  for (int c0 = 0; c0 < keep; c0 += KM) {
    const int kk = keep - c0 < KM ? keep - c0 : KM;
    if constexpr (KM == 1) {
      warp_out_reg<MR, 1>(Wu, Wv, m, pu, pv, tu, tv, Bm, Jm, sig, ord, pr, pc, tr, c0, kk, Uo,
                          Vo, n, lane);
    } else {
      if (kk > 2)
        warp_out_reg<MR, 4>(Wu, Wv, m, pu, pv, tu, tv, Bm, Jm, sig, ord, pr, pc, tr, c0, kk,
                            Uo, Vo, n, lane);
      else
        warp_out_reg<MR, 2>(Wu, Wv, m, pu, pv, tu, tv, Bm, Jm, sig, ord, pr, pc, tr, c0, kk,
                            Uo, Vo, n, lane);
    }
  }
}

// 128-row panels: out of line (keeps the caller's register allocation)
__device__ __noinline__ void warp_out_regs4(const double* Wu, const double* Wv, int m, int pu,
                                            int pv, const double* tu, const double* tv,
                                            const double* Bm, const double* Jm,
                                            const double* sig, const int* ord, int pr, int pc,
                                            bool tr, int keep, double* Uo, double* Vo, int n,
                                            int lane) {
  warp_out_regs<4>(Wu, Wv, m, pu, pv, tu, tv, Bm, Jm, sig, ord, pr, pc, tr, keep, Uo, Vo, n,
                   lane);
}

// Single-warp Jacobi of the block and CTA-pair paths (one warp on the task's
// critical path, 128 registers available): same pairing, lane groups,
// arithmetic and order as warp_jacobi, with the row loops unrolled to RPL rows
// per lane and each lane's elements kept in registers between the norms and
// the rotation, so the loads of a step issue together instead of one
// dependent shared-memory round trip per row.
template <int RPL>
__device__ int blk_jacobi_t(double* B, int pr, int pc, double* J, int lane, int gs) {
  const int lb = pr | 1, lj = pc | 1;
  const int np = pc + (pc & 1), npairs = np / 2;
  const int per = 32 / gs;
  const double tol = sqrt((double)pr) * 2.220446049250313e-16;
  const int sub = lane & (gs - 1), grp = lane / gs;
  double nb = 0.0;
  for (int i = lane; i < pr * pc; i += 32) {
    const double x = B[(i / pr) * lb + i % pr];
    nb += x * x;
  }
  const double tiny = warp_sum(nb) * 4.930380657631324e-32;   // (eps64 |B|_F)^2
  // a sweep whose rotations were all below 1e-9 (|c| / sqrt(ab)) leaves
  // off-diagonals O(1e-18) << tol: the confirmation sweep that would follow
  // rotates nothing and is skipped (ACR_JACOBI_CONFIRM=1 keeps it)
  const bool skipc = jacobi_skip_confirm;
  for (int sweep = 0; sweep < 40; ++sweep) {
    bool rot = false, big = false;
    for (int step = 0; step < np - 1; ++step) {
      for (int base = 0; base < npairs; base += per) {
        const int k = base + grp;
        int i = 0, j = 0;
        bool valid = k < npairs;
        if (valid) {
          i = rr_player(step, k, np);
          j = rr_player(step, np - 1 - k, np);
          valid = i < pc && j < pc;
        }
        double* bi = B + (long long)i * lb;
        double* bj = B + (long long)j * lb;
        double xr[RPL], yr[RPL];
#pragma unroll
        for (int h = 0; h < RPL; ++h) {
          const int r = sub + gs * h;
          const bool in = valid && r < pr;
          xr[h] = in ? bi[r] : 0.0;
          yr[h] = in ? bj[r] : 0.0;
        }
        double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
        for (int h = 0; h < RPL; ++h) {
          if (sub + gs * h < pr) {
            a += xr[h] * xr[h];
            b += yr[h] * yr[h];
            c += xr[h] * yr[h];
          }
        }
        for (int o = gs >> 1; o; o >>= 1) {
          a += __shfl_xor_sync(FULL, a, o);
          b += __shfl_xor_sync(FULL, b, o);
          c += __shfl_xor_sync(FULL, c, o);
        }
        if (valid && a > tiny && b > tiny && c != 0.0 &&
            c * c > tol * tol * a * b) {
          const double d = b - a, e = 2.0 * c;
          double cs, sn;
          jacobi_rot(d, e, cs, sn);
          double* ji = J + (long long)i * lj;
          double* jj = J + (long long)j * lj;
          double xj[RPL], yj[RPL];
#pragma unroll
          for (int h = 0; h < RPL; ++h) {
            const int r = sub + gs * h;
            xj[h] = r < pc ? ji[r] : 0.0;
            yj[h] = r < pc ? jj[r] : 0.0;
          }
#pragma unroll
          for (int h = 0; h < RPL; ++h) {
            const int r = sub + gs * h;
            if (r < pr) {
              bi[r] = cs * xr[h] - sn * yr[h];
              bj[r] = sn * xr[h] + cs * yr[h];
            }
            if (r < pc) {
              ji[r] = cs * xj[h] - sn * yj[h];
              jj[r] = sn * xj[h] + cs * yj[h];
            }
          }
          rot = true;
          big |= c * c > 1e-18 * a * b;
        }
        __syncwarp();
      }
    }
    if (!__any_sync(FULL, rot)) return sweep + 1;
    if (skipc && !__any_sync(FULL, big)) return sweep + 1;
  }
  return 40;
}

__device__ int warp_jacobi(double* B, int pr, int pc, double* J, int lane);

__device__ int blk_jacobi(double* B, int pr, int pc, double* J, int lane) {
  if (pc < 2 || pr > 4 * 32) return warp_jacobi(B, pr, pc, J, lane);
  const int lj = pc | 1;
  for (int i = lane; i < pc * pc; i += 32) {
    const int c = i / pc, r = i - c * pc;
    J[c * lj + r] = (r == c) ? 1.0 : 0.0;
  }
  __syncwarp();
  const int npairs = (pc + (pc & 1)) / 2;
  int gs = 32;
  while (gs > 1 && gs * npairs > 32) gs >>= 1;
  const int rpl = (pr + gs - 1) / gs;
  if (rpl <= 1) return blk_jacobi_t<1>(B, pr, pc, J, lane, gs);
  if (rpl <= 2) return blk_jacobi_t<2>(B, pr, pc, J, lane, gs);
  if (rpl <= 4) return blk_jacobi_t<4>(B, pr, pc, J, lane, gs);
  return warp_jacobi(B, pr, pc, J, lane);
}

// one-sided Jacobi on B (pr x pc col-major), J (pc x pc); pairs of a
// round-robin step are spread over lane groups of size gs
__device__ int warp_jacobi(double* B, int pr, int pc, double* J, int lane) {
  const int lb = pr | 1, lj = pc | 1;      // odd column strides: no bank conflicts
  for (int i = lane; i < pc * pc; i += 32) {
    const int c = i / pc, r = i - c * pc;
    J[c * lj + r] = (r == c) ? 1.0 : 0.0;
  }
  __syncwarp();
  if (pc < 2) return 0;
  const int np = pc + (pc & 1), npairs = np / 2;
  int gs = 32;
  while (gs > 1 && gs * npairs > 32) gs >>= 1;
  const int per = 32 / gs;                 // pairs per pass
  const double tol = sqrt((double)pr) * 2.220446049250313e-16;
  const int sub = lane & (gs - 1), grp = lane / gs;
  double nb = 0.0;
  for (int i = lane; i < pr * pc; i += 32) {
    const double x = B[(i / pr) * lb + i % pr];
    nb += x * x;
  }
  const double tiny = warp_sum(nb) * 4.930380657631324e-32;   // (eps64 |B|_F)^2
  // a sweep whose rotations were all below 1e-9 (|c| / sqrt(ab)) leaves
  // off-diagonals O(1e-18) << tol: the confirmation sweep that would follow
  // rotates nothing and is skipped (ACR_JACOBI_CONFIRM=1 keeps it)
  const bool skipc = jacobi_skip_confirm;
  for (int sweep = 0; sweep < 40; ++sweep) {
    bool rot = false, big = false;
    for (int step = 0; step < np - 1; ++step) {
      for (int base = 0; base < npairs; base += per) {
        const int k = base + grp;
        int i = 0, j = 0;
        bool valid = k < npairs;
        if (valid) {
          i = rr_player(step, k, np);
          j = rr_player(step, np - 1 - k, np);
          valid = i < pc && j < pc;
        }
        double a = 0.0, b = 0.0, c = 0.0;
        double* bi = B + (long long)i * lb;
        double* bj = B + (long long)j * lb;
        if (valid)
          for (int r = sub; r < pr; r += gs) {
            double x = bi[r], y = bj[r];
            a += x * x;
            b += y * y;
            c += x * y;
          }
        for (int o = gs >> 1; o; o >>= 1) {
          a += __shfl_xor_sync(FULL, a, o);
          b += __shfl_xor_sync(FULL, b, o);
          c += __shfl_xor_sync(FULL, c, o);
        }
        if (valid && a > tiny && b > tiny && c != 0.0 &&
            c * c > tol * tol * a * b) {
          const double d = b - a, e = 2.0 * c;
          double cs, sn;
          jacobi_rot(d, e, cs, sn);
          for (int r = sub; r < pr; r += gs) {
            double x = bi[r], y = bj[r];
            bi[r] = cs * x - sn * y;
            bj[r] = sn * x + cs * y;
          }
          double* ji = J + (long long)i * lj;
          double* jj = J + (long long)j * lj;
          for (int r = sub; r < pc; r += gs) {
            double x = ji[r], y = jj[r];
            ji[r] = cs * x - sn * y;
            jj[r] = sn * x + cs * y;
          }
          rot = true;
          big |= c * c > 1e-18 * a * b;
        }
        __syncwarp();
      }
    }
    if (!__any_sync(FULL, rot)) return sweep + 1;
    if (skipc && !__any_sync(FULL, big)) return sweep + 1;
  }
  return 40;
}


// W[c*m + i] = [A | B] columns, every element an asynchronous 8-byte copy (all
// of a lane's loads in flight at once); the exact sign scales are applied
// after the wait (warp_scale_cols)
__device__ __forceinline__ void warp_issue_cols(double* __restrict__ W, int m,
                                                const double* __restrict__ A, int ra,
                                                const double* __restrict__ B, int rb, int n,
                                                int lane) {
  for (int c = 0; c < ra; ++c)
    for (int i = lane; i < m; i += 32) cp_async8(W + (long long)c * m + i, A + (long long)c * n + i, true);
  for (int c = 0; c < rb; ++c)
    for (int i = lane; i < m; i += 32)
      cp_async8(W + (long long)(ra + c) * m + i, B + (long long)c * n + i, true);
}

__device__ __forceinline__ void warp_scale_cols(double* W, int m, int ra, double sa, int rb,
                                                double sb, int lane) {
  if (sa != 1.0)
    for (int idx = lane; idx < ra * m; idx += 32) W[idx] *= sa;
  if (sb != 1.0)
    for (int idx = lane; idx < rb * m; idx += 32) W[ra * m + idx] *= sb;
}

__device__ void trunc_warp_full(const TruncArgs& A, const TaskCtx& tc, double* wk,
                                int lane) {
  const int n = A.T.n;
  const OpRes& a = tc.a;
  const OpRes& b = tc.b;
  const int um = tc.um, vm = tc.vm;
  const int R = a.r + b.r;
  const int pu = um < R ? um : R, pv = vm < R ? vm : R;
  double* Uw = wk;
  double* Vw = Uw + (long long)um * R;
  double* Bm = Vw + (long long)vm * R;
  double* Jm = Bm + (long long)R * (R + 1);   // odd-strided cores (pr | 1, pc | 1)
  double* tauU = Jm + (long long)R * (R + 1);
  double* tauV = tauU + R;
  double* sig = tauV + R;
  int* ord = reinterpret_cast<int*>(sig + R);
  // operand load: all global reads of a lane issued before its smem stores
  long long ph[6] = {0, 0, 0, 0, 0, 0};
  long long t_ph = clock64();
  warp_issue_cols(Uw, um, a.U, a.r, b.U, b.r, n, lane);
  warp_issue_cols(Vw, vm, a.V, a.r, b.V, b.r, n, lane);
  cp_async_wait_all();
  __syncwarp();
  if (a.sc != 1.0 || b.sc != 1.0) {
    warp_scale_cols(Uw, um, a.r, a.sc, b.r, b.sc, lane);
    __syncwarp();
  }
  ACR_PH(0);
  const int mrl = (um == vm && (um & 31) == 0) ? um >> 5 : 0;   // rows per lane
  if (mrl == 2) warp_qr2<2>(Uw, um, tauU, Vw, vm, tauV, R, lane);
  else if (mrl == 4) warp_qr2<4>(Uw, um, tauU, Vw, vm, tauV, R, lane);
  else if (mrl == 1) warp_qr2<1>(Uw, um, tauU, Vw, vm, tauV, R, lane);
  else warp_qr2<0>(Uw, um, tauU, Vw, vm, tauV, R, lane);
  ACR_PH(1);
  double nu2 = 0.0, nv2 = 0.0;
  for (int idx = lane; idx < pu * R; idx += 32) {
    int l = idx / pu, i = idx - l * pu;
    if (l >= i) { double x = Uw[(long long)l * um + i]; nu2 += x * x; }
  }
  for (int idx = lane; idx < pv * R; idx += 32) {
    int l = idx / pv, i = idx - l * pv;
    if (l >= i) { double x = Vw[(long long)l * vm + i]; nv2 += x * x; }
  }
  nu2 = warp_sum(nu2);
  nv2 = warp_sum(nv2);
  const bool tr = pu < pv;
  const int pr = tr ? pv : pu, pc = tr ? pu : pv;
  for (int idx = lane; idx < pu * pv; idx += 32) {
    int i = idx / pv, j = idx - i * pv;
    int l0 = i > j ? i : j;
    double s = 0.0;
    for (int l = l0; l < R; ++l) s += Uw[(long long)l * um + i] * Vw[(long long)l * vm + j];
    if (!tr) Bm[(long long)j * (pr | 1) + i] = s;
    else Bm[(long long)i * (pr | 1) + j] = s;
  }
  __syncwarp();
  ACR_PH(2);
  const int sweeps = warp_jacobi(Bm, pr, pc, Jm, lane);
  ACR_PH(3);
  for (int j = lane; j < pc; j += 32) {
    double s = 0.0;
    const double* bj = Bm + (long long)j * (pr | 1);
    for (int r = 0; r < pr; ++r) s += bj[r] * bj[r];
    sig[j] = sqrt(s);
  }
  __syncwarp();
  for (int j = lane; j < pc; j += 32) {
    double sj = sig[j];
    int rnk = 0;
    for (int i = 0; i < pc; ++i) {
      double si = sig[i];
      rnk += (si > sj) || (si == sj && i < j);
    }
    ord[rnk] = j;
  }
  __syncwarp();
  const double s1 = sig[ord[0]];
  const double guard = (double)R * 2.220446049250313e-16 * sqrt(nu2) * sqrt(nv2);
  int keep = 0;
  if (s1 > guard) {
    const double thr = A.eps * s1;
    for (int i = 0; i < pc; ++i) keep += sig[i] >= thr;
    if (A.cap > 0 && keep > A.cap) keep = A.cap;
  }
  if (keep > tc.Rout) {
    if (lane == 0) atomicMax(A.overflow, keep);
    keep = 0;
  }
  ACR_PH(4);
  if (A.ctr && lane == 0) {   // census formulas of SURVEY.md Appendix C
    unsigned long long fl = 4ull * um * R * R + 4ull * vm * R * R + 24ull * R * R * R +
                            2ull * (um + vm) * R * keep;
    atomicAdd(A.ctr, fl);
    atomicAdd(A.ctr + 1, 8ull * ((unsigned long long)um * R + vm * R + um * keep + vm * keep));
    atomicAdd(A.ctr + 9, 1ull);
    atomicAdd(A.ctr + 11, (unsigned long long)sweeps);
  }
  double* ob = sig + R + (R + 1) / 2; // after the R ints of ord: one output column per side
  double* ob2 = ob + um;
  if (mrl == 2)
    warp_out_regs<2>(Uw, Vw, um, pu, pv, tauU, tauV, Bm, Jm, sig, ord, pr, pc, tr, keep, tc.Uo,
                     tc.Vo, n, lane);
  else if (mrl == 4)
    warp_out_regs4(Uw, Vw, um, pu, pv, tauU, tauV, Bm, Jm, sig, ord, pr, pc, tr, keep, tc.Uo,
                   tc.Vo, n, lane);
  else if (mrl == 1)
    warp_out_regs<1>(Uw, Vw, um, pu, pv, tauU, tauV, Bm, Jm, sig, ord, pr, pc, tr, keep, tc.Uo,
                     tc.Vo, n, lane);
  else
  for (int c = 0; c < keep; ++c) {
    const int j = ord[c];
    for (int i = lane; i < um; i += 32) {
      double v = 0.0;
      if (i < pu) v = tr ? sig[j] * Jm[(long long)j * (pc | 1) + i] : Bm[(long long)j * (pr | 1) + i];
      ob[i] = v;
    }
    for (int i = lane; i < vm; i += 32) {
      double v = 0.0;
      if (i < pv) v = tr ? Bm[(long long)j * (pr | 1) + i] / sig[j] : Jm[(long long)j * (pc | 1) + i];
      ob2[i] = v;
    }
    __syncwarp();
    warp_apply_q2<0>(Uw, um, pu, tauU, ob, Vw, vm, pv, tauV, ob2, lane);
    double* du = tc.Uo + (long long)c * n;
    for (int i = lane; i < um; i += 32) du[i] = ob[i];
    double* dv = tc.Vo + (long long)c * n;
    for (int i = lane; i < vm; i += 32) dv[i] = ob2[i];
    __syncwarp();
  }
  if (lane == 0) *tc.ro = keep;
  ACR_PH(5);
  if (A.ctr && lane == 0) {
    for (int i = 0; i < 6; ++i) atomicAdd(A.ctr + (i < 4 ? 12 + i : 62 + i), (unsigned long long)ph[i]);
    // histogram: R bucket (<=4, <=8, <=16, <=32, >32) x m bucket (<=32, 64, 128, 256, >256)
    const int rb = R <= 4 ? 0 : R <= 8 ? 1 : R <= 16 ? 2 : R <= 32 ? 3 : 4;
    const int mm = um > vm ? um : vm;
    const int mb = mm <= 32 ? 0 : mm <= 64 ? 1 : mm <= 128 ? 2 : mm <= 256 ? 3 : 4;
    long long tot = 0;
    for (int i = 0; i < 6; ++i) tot += ph[i];
    atomicAdd(A.ctr + 16 + rb * 5 + mb, 1ull);
    atomicAdd(A.ctr + 41 + rb * 5 + mb, (unsigned long long)tot);
  }
}

// Classification pass of a launch whose tasks may exceed the warp path (the
// ranks, and so the work areas, are only known on the device): one thread per
// item; large work areas, and cores above warp_rmax columns (a single warp's
// Jacobi would walk whole column pairs per lane) go to the block-path queues
// -- queue 0: work area fits a half-SM CTA (two 256-thread CTAs per SM),
// queue 1 (stored from bigq + nitems): one 512-thread CTA per SM -- and are
// flagged in cls so the warp kernel skips them.  The three kernels then run
// concurrently on their own streams.
__global__ void __launch_bounds__(256) k_trunc_classify(TruncArgs A, int nitems, int* bigq,
                                                        int* bigcount, unsigned char* cls) {
  ACR_PDL_ENTRY();
  const int em = blockIdx.x * 256 + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int which = -1;
  if (em < nitems) {
    const int task = em % A.ntasks, g = em / A.ntasks;
    const TaskCtx tc = resolve_task(A, task, g);
    if (task_is_full(A, tc)) {
      const int R = tc.a.r + tc.b.r;
      const long long need = warp_need_doubles(tc.um, tc.vm, R);
      if (need > (long long)NSLOT * SLOT / 8 || R > A.warp_rmax || need > A.warp_maxneed)
        which = trunc_need_doubles(tc.um, tc.vm, R) <= QHALF_D ? 0 : 1;
    }
    cls[em] = which >= 0 ? 1 : 0;
  }
  // warp-aggregated appends
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const unsigned m = __ballot_sync(FULL, which == k);
    if (m == 0u) continue;
    int base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(bigcount + k, __popc(m));
    base = __shfl_sync(FULL, base, __ffs(m) - 1);
    if (which == k) bigq[(long long)k * nitems + base + __popc(m & ((1u << lane) - 1u))] = em;
  }
}

__global__ void __launch_bounds__(TW * 32, 1) k_trunc_warp(TruncArgs A, int nitems,
                                                          const unsigned char* cls) {
  ACR_PDL_ENTRY();
  extern __shared__ double pool[];
  __shared__ unsigned long long mask;
  if (threadIdx.x == 0) mask = 0ull;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = A.T.n;
  const int nelem = nitems / A.ntasks;
  for (int it = blockIdx.x * TW + warp;; it += gridDim.x * TW) {
    // dynamic: the next item from a global counter (tasks differ in size by
    // orders of magnitude; static striding left warps idle at the tail)
    int item = it;
    if (A.wq) {
      int v = 0;
      if (lane == 0) v = atomicAdd(A.wq, 1);
      item = __shfl_sync(FULL, v, 0);
    }
    if (item >= nitems) break;
    const int task = A.task_major ? item / nelem : item % A.ntasks;
    const int g = A.task_major ? item - task * nelem : item / A.ntasks;
    // tasks the classification pass sent to the block-path queues
    if (cls != nullptr && cls[(long long)g * A.ntasks + task]) continue;
    TaskCtx tc = resolve_task(A, task, g);
    __syncwarp();
    const OpRes& a = tc.a;
    const OpRes& b = tc.b;
    if (A.mode != TM_TRUNCATE && (a.r == 0 || b.r == 0)) {   // algebra.py:93-96
      const OpRes& s = a.r ? a : b;
      int r = s.r;
      if (r > tc.Rout) {
        if (lane == 0) atomicMax(A.overflow, r);
        r = tc.Rout;
      }
      if (r) warp_copy_factor(s, tc.Uo, tc.Vo, tc.um, tc.vm, n, r, lane);
      if (lane == 0) {
        *tc.ro = r;
        if (A.ctr && r && !(s.U == tc.Uo && s.V == tc.Vo && s.sc == 1.0))
          atomicAdd(A.ctr + 1, 16ull * (tc.um + tc.vm) * r);
      }
      continue;
    }
    if (A.mode == TM_TRUNCATE && a.r < 2) {
      int r = 0;
      if (a.r == 1) {                                           // hodlr.py:181-185
        bool nzu = false, nzv = false;
        for (int i = lane; i < tc.um; i += 32) nzu |= a.U[i] != 0.0;
        for (int i = lane; i < tc.vm; i += 32) nzv |= a.V[i] != 0.0;
        nzu = __any_sync(FULL, nzu);
        nzv = __any_sync(FULL, nzv);
        r = (nzu && nzv) ? 1 : 0;
        if (r > tc.Rout) {
          if (lane == 0) atomicMax(A.overflow, r);
          r = 0;
        }
        if (r) warp_copy_factor(a, tc.Uo, tc.Vo, tc.um, tc.vm, n, 1, lane);
      }
      if (lane == 0) *tc.ro = r;
      continue;
    }
    const int R = a.r + b.r;
    const long long need = warp_need_doubles(tc.um, tc.vm, R);
    if (need > (long long)NSLOT * SLOT / 8) {   // cannot happen: sized by the host or classified
      if (lane == 0) atomicMax(A.overflow, 1 << 29);
      continue;
    }
    const int ns = (int)((need + SLOT - 1) / SLOT);
    const long long t_acq = A.ctr ? clock64() : 0;
    const int s0 = acquire_slots(&mask, ns, lane);
    if (A.ctr && lane == 0) atomicAdd(A.ctr + 68, (unsigned long long)(clock64() - t_acq));
    // order this warp's accesses to the slots after the previous owner's
    // (without this fence the hand-over raced once the tasks got shorter)
    __syncwarp();
    __threadfence_block();
    trunc_warp_full(A, tc, pool + (long long)s0 * SLOT, lane);
    __syncwarp();
    __threadfence_block();
    if (lane == 0) {
      const unsigned long long want = ns >= 64 ? ~0ull : ((1ull << ns) - 1ull);
      atomicAnd(&mask, ~(want << s0));
    }
  }
}

int trunc_warp_pool_doubles() { return NSLOT * SLOT / 8; }

// development aid: ACR_JACOBI_CONFIRM=1 keeps the confirmation sweep
void trunc_init_flags() {
  static bool done = false;
  if (done) return;
  done = true;
  if (getenv("ACR_JACOBI_CONFIRM")) {
    const bool v = false;
    cudaMemcpyToSymbol(jacobi_skip_confirm, &v, sizeof(v));
  }
  if (getenv("ACR_NO_QSPLIT")) {
    const bool v = false;
    cudaMemcpyToSymbol(trunc_qsplit, &v, sizeof(v));
  }
  if (getenv("ACR_QR_LAMAX")) {               // development aid
    const int v = atoi(getenv("ACR_QR_LAMAX"));
    cudaMemcpyToSymbol(qr_la_max, &v, sizeof(v));
  }
  if (getenv("ACR_QR_NOLA")) {                // development aid: plain group QR
    const bool v = false;
    cudaMemcpyToSymbol(qr_lookahead, &v, sizeof(v));
  }
}

cudaError_t launch_trunc(const TruncArgs& a, int nelem, bool direct, bool may_big,
                         int* bigq, int* bigcount, cudaStream_t st, const TruncAux* aux) {
  if (a.ntasks == 0 || nelem == 0) return cudaSuccess;
  static bool attr = false;
  static int nsm = 148;
  if (!attr) {
    cudaFuncSetAttribute(k_trunc_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         NSLOT * SLOT * 8);
    cudaFuncSetAttribute(k_trunc_big<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         28416 * 8 + 64);   // engine caps smem_doubles at 28416
    cudaFuncSetAttribute(k_trunc_big<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         QHALF);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    attr = true;
  }
  trunc_init_flags();
  const int nitems = a.ntasks * nelem;
  const size_t bsm = (size_t)a.smem_doubles * 8 + 64;
  if (direct) {
    TruncArgs ad = a;
    ad.direct_tag = 1;
    // more tasks than SMs: 256-thread CTAs, two per SM, when the work areas fit
    if (nitems > nsm && bsm <= QHALF)
      CK_PDL(launch_pdl(k_trunc_big<256>, dim3(nitems), dim3(256), bsm, st, ad, nullptr, nullptr, nitems));
    else
      CK_PDL(launch_pdl(k_trunc_big<512>, dim3(nitems), dim3(512), bsm, st, ad, nullptr, nullptr, nitems));
    return cudaGetLastError();
  }
  if (may_big || a.wq) {
    // [0], [1] queue lengths, [2] warp-path item counter, [3], [4] queue
    // fetch counters
    cudaError_t e = cudaMemsetAsync(bigcount, 0, 5 * sizeof(int), st);
    if (e != cudaSuccess) return e;
  }
  int blocks = (nitems + TW - 1) / TW;
  if (blocks > nsm) blocks = nsm;
  if (!may_big) {
    CK_PDL(launch_pdl(k_trunc_warp, dim3(blocks), dim3(TW * 32), NSLOT * SLOT * 8, st, a, nitems,
                      (const unsigned char*)nullptr));
    return cudaGetLastError();
  }
  // Queued launch: classify, then the two block-path queue kernels and the
  // warp kernel side by side (aux streams; without them, in turn on st).  The
  // queue kernels go first: they hold the longest tasks, and the many short
  // warp-path tasks fill the SMs their CTAs leave.  Queue 0: two 256-thread
  // CTAs per SM for work areas within half an SM's shared memory; queue 1: one
  // 512-thread CTA per SM for the rest.
  CK_PDL(launch_pdl(k_trunc_classify, dim3((nitems + 255) / 256), dim3(256), 0, st, a, nitems,
                    bigq, bigcount, aux ? aux->cls : nullptr));
  const bool conc = aux != nullptr && aux->q0 != nullptr && aux->q0 != st;
  cudaStream_t s0 = conc ? aux->q0 : st, s1 = conc ? aux->q1 : st;
  const bool full = bsm > QHALF;
  if (conc) {
    cudaError_t e = cudaEventRecord(aux->ef, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s0, aux->ef, 0);
    if (e == cudaSuccess && full) e = cudaStreamWaitEvent(s1, aux->ef, 0);
    if (e != cudaSuccess) return e;
  }
  if (full) {
    const int bb = nitems < nsm ? nitems : nsm;
    CK_PDL(launch_pdl(k_trunc_big<512>, dim3(bb), dim3(512), bsm, s1, a, bigq + nitems, bigcount + 1, nitems));
  }
  {
    TruncArgs ah = a;
    ah.smem_doubles = QHALF_D;
    const int bb = nitems < 2 * nsm ? nitems : 2 * nsm;
    CK_PDL(launch_pdl(k_trunc_big<256>, dim3(bb), dim3(256), QHALF, s0, ah, bigq, bigcount, nitems));
  }
  CK_PDL(launch_pdl(k_trunc_warp, dim3(blocks), dim3(TW * 32), NSLOT * SLOT * 8, st, a, nitems,
                    (const unsigned char*)(aux ? aux->cls : nullptr)));
  if (conc) {
    cudaError_t e = cudaEventRecord(aux->ej0, s0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, aux->ej0, 0);
    if (e == cudaSuccess && full) e = cudaEventRecord(aux->ej1, s1);
    if (e == cudaSuccess && full) e = cudaStreamWaitEvent(st, aux->ej1, 0);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

int trunc_direct_max() { return 4 * 148; }


}  // namespace acr
