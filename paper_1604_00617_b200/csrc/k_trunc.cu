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
#include "acr_types.cuh"
#include "acr_launch.h"

namespace acr {

static constexpr int TT = 128;   // threads per truncation CTA

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  return red[0] + red[1] + red[2] + red[3];
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
    if (rb[op.node * 2 + 1 - op.fside] == 0) r = 0;
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

// Householder QR of W (mr x R, column-major, ld = mr), in place.  On exit
// the upper trapezoid holds R, below-diagonal the reflector tails, tau[j].
__device__ void block_qr(double* W, int mr, int R, double* tau, double* red,
                         double* bc) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int p = mr < R ? mr : R;
  for (int j = 0; j < p; ++j) {
    double* cj = W + (long long)j * mr;
    double ss = 0.0;
    for (int i = j + 1 + tid; i < mr; i += TT) ss += cj[i] * cj[i];
    ss = block_sum(ss, red);
    if (tid == 0) {
      double alpha = cj[j];
      double tj = 0.0, scal = 0.0;
      if (ss != 0.0) {
        double xnorm = sqrt(ss);
        double beta = -copysign(hypot(alpha, xnorm), alpha);
        tj = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
        cj[j] = beta;
      }
      tau[j] = tj;
      bc[0] = scal;
    }
    __syncthreads();
    const double tj = tau[j];
    if (tj != 0.0) {
      const double scal = bc[0];
      for (int i = j + 1 + tid; i < mr; i += TT) cj[i] *= scal;
      __syncthreads();
      for (int c = j + 1 + warp; c < R; c += TT / 32) {
        double* cc = W + (long long)c * mr;
        double w = 0.0;
        for (int i = j + 1 + lane; i < mr; i += 32) w += cj[i] * cc[i];
        w = warp_sum(w) + cc[j];
        w *= tj;
        if (lane == 0) cc[j] -= w;
        for (int i = j + 1 + lane; i < mr; i += 32) cc[i] -= w * cj[i];
      }
    }
    __syncthreads();
  }
}

// X (mr x nc, ld mr) := Q X where Q = H_0 ... H_{p-1} from block_qr.
__device__ void block_apply_q(const double* W, int mr, int p, const double* tau,
                              double* X, int nc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = p - 1; j >= 0; --j) {
    const double tj = tau[j];
    if (tj != 0.0) {
      const double* v = W + (long long)j * mr;
      for (int c = warp; c < nc; c += TT / 32) {
        double* xc = X + (long long)c * mr;
        double w = 0.0;
        for (int i = j + 1 + lane; i < mr; i += 32) w += v[i] * xc[i];
        w = (warp_sum(w) + xc[j]) * tj;
        if (lane == 0) xc[j] -= w;
        for (int i = j + 1 + lane; i < mr; i += 32) xc[i] -= w * v[i];
      }
    }
    __syncthreads();
  }
}

// Round-robin (circle method) pairing of np players (np even).
__device__ __forceinline__ int rr_player(int step, int x, int np) {
  return x == 0 ? 0 : 1 + ((x - 1 + step) % (np - 1));
}

// One-sided Jacobi on B (pr x pc, column-major ld pr) accumulating J (pc x pc).
__device__ void block_jacobi(double* B, int pr, int pc, double* J, int* flag) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < pc * pc; i += TT) J[i] = (i / pc == i % pc) ? 1.0 : 0.0;
  const int np = pc + (pc & 1);
  const double tol = sqrt((double)pr) * 2.220446049250313e-16;
  __syncthreads();
  if (pc < 2) return;
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (tid == 0) *flag = 0;
    __syncthreads();
    for (int step = 0; step < np - 1; ++step) {
      for (int k = warp; k < np / 2; k += TT / 32) {
        int i = rr_player(step, k, np), j = rr_player(step, np - 1 - k, np);
        if (i >= pc || j >= pc) continue;
        double* bi = B + (long long)i * pr;
        double* bj = B + (long long)j * pr;
        double a = 0.0, b = 0.0, c = 0.0;
        for (int r = lane; r < pr; r += 32) {
          double x = bi[r], y = bj[r];
          a += x * x;
          b += y * y;
          c += x * y;
        }
        a = warp_sum(a);
        b = warp_sum(b);
        c = warp_sum(c);
        if (a == 0.0 || b == 0.0 || c == 0.0) continue;
        if (fabs(c) <= tol * sqrt(a) * sqrt(b)) continue;
        double zeta = (b - a) / (2.0 * c);
        double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double cs = 1.0 / sqrt(1.0 + t * t);
        double sn = cs * t;
        for (int r = lane; r < pr; r += 32) {
          double x = bi[r], y = bj[r];
          bi[r] = cs * x - sn * y;
          bj[r] = sn * x + cs * y;
        }
        double* ji = J + (long long)i * pc;
        double* jj = J + (long long)j * pc;
        for (int r = lane; r < pc; r += 32) {
          double x = ji[r], y = jj[r];
          ji[r] = cs * x - sn * y;
          jj[r] = sn * x + cs * y;
        }
        if (lane == 0) *flag = 1;
      }
      __syncthreads();
    }
    int f = *flag;
    __syncthreads();
    if (!f) break;
  }
}

__device__ void copy_factor(const OpRes& s, double* Uo, double* Vo, int um,
                            int vm, int n, int r) {
  if (s.U == Uo && s.V == Vo && s.sc == 1.0) return;
  for (int idx = threadIdx.x; idx < um * r; idx += TT) {
    int c = idx / um, i = idx - c * um;
    Uo[(long long)c * n + i] = s.sc * s.U[(long long)c * n + i];
  }
  for (int idx = threadIdx.x; idx < vm * r; idx += TT) {
    int c = idx / vm, i = idx - c * vm;
    Vo[(long long)c * n + i] = s.V[(long long)c * n + i];
  }
}

__global__ void __launch_bounds__(TT) k_trunc(TruncArgs A) {
  extern __shared__ double sm[];
  __shared__ double red[8];
  __shared__ int iflag[2];
  const int task = blockIdx.x, g = blockIdx.y, tid = threadIdx.x;
  const TreeDev& T = A.T;
  const int n = T.n;
  const int beta = A.tasks[task * 3 + 1], side = A.tasks[task * 3 + 2];
  const int lo = T.lo[beta], hi = T.hi[beta], mid = T.mid[beta];
  const int urow = side ? mid : lo, um = side ? hi - mid : mid - lo;
  const int vrow = side ? lo : mid, vm = side ? mid - lo : hi - mid;
  OpRes a = resolve_op(A.a, T, g, beta, side, urow, vrow);
  OpRes b;
  b.r = 0;
  b.U = b.V = nullptr;
  b.sc = 1.0;
  if (A.mode != TM_TRUNCATE) b = resolve_op(A.b, T, g, beta, side, urow, vrow);
  if (A.mode == TM_COMBINE_SWAP1 && side == 1) {
    OpRes t = a;
    a = b;
    b = t;
  }
  const HB out = A.out[g];
  const long long oslot = (long long)T.depth[beta] * out.R * n;
  double* Uo = out.U + oslot + urow;
  double* Vo = out.V + oslot + vrow;
  int* ro = out.rk + beta * 2 + side;
  __syncthreads();   // every thread has read the ranks before any write

  if (A.mode != TM_TRUNCATE) {
    if (a.r == 0 || b.r == 0) {                      // algebra.py:93-96
      const OpRes& s = a.r ? a : b;
      int r = s.r;
      if (r > out.R) {
        if (tid == 0) atomicMax(A.overflow, r);
        r = out.R;
      }
      if (r) copy_factor(s, Uo, Vo, um, vm, n, r);
      if (tid == 0) {
        *ro = r;
        if (A.ctr && r && !(s.U == Uo && s.V == Vo && s.sc == 1.0))
          atomicAdd(A.ctr + 1, 16ull * (um + vm) * r);
      }
      return;
    }
  } else {
    if (a.r == 0) {
      if (tid == 0) *ro = 0;
      return;
    }
    if (a.r == 1) {                                   // hodlr.py:181-185
      double nzu = 0.0, nzv = 0.0;
      for (int i = tid; i < um; i += TT) nzu += (a.U[i] != 0.0) ? 1.0 : 0.0;
      for (int i = tid; i < vm; i += TT) nzv += (a.V[i] != 0.0) ? 1.0 : 0.0;
      nzu = block_sum(nzu, red);
      nzv = block_sum(nzv, red);
      int r = (nzu > 0.0 && nzv > 0.0) ? 1 : 0;
      if (r > out.R) {
        if (tid == 0) atomicMax(A.overflow, r);
        r = 0;
      }
      if (r) copy_factor(a, Uo, Vo, um, vm, n, 1);
      if (tid == 0) *ro = r;
      return;
    }
  }

  // ---- full truncation of [a | b] -------------------------------------
  const int R = a.r + b.r;
  const int pu = um < R ? um : R, pv = vm < R ? vm : R;
  const long long need = 2LL * (um + vm) * R + 2LL * R * R + 4LL * R + 8;
  double* wk = sm;
  if (need > A.smem_doubles) {
    if (task >= A.gscr_ntasks || A.gscr == nullptr) {
      if (tid == 0) atomicMax(A.overflow, 1 << 29);
      return;
    }
    wk = A.gscr + ((long long)g * A.gscr_ntasks + task) * A.gscr_stride;
  }
  double* Uw = wk;
  double* Vw = Uw + (long long)um * R;
  double* Ou = Vw + (long long)vm * R;
  double* Ov = Ou + (long long)um * R;
  double* Bm = Ov + (long long)vm * R;
  double* Jm = Bm + (long long)R * R;
  double* tauU = Jm + (long long)R * R;
  double* tauV = tauU + R;
  double* sig = tauV + R;
  int* ord = reinterpret_cast<int*>(sig + R);

  for (int idx = tid; idx < um * R; idx += TT) {
    int c = idx / um, i = idx - c * um;
    Uw[idx] = c < a.r ? a.sc * a.U[(long long)c * n + i]
                      : b.sc * b.U[(long long)(c - a.r) * n + i];
  }
  for (int idx = tid; idx < vm * R; idx += TT) {
    int c = idx / vm, i = idx - c * vm;
    Vw[idx] = c < a.r ? a.V[(long long)c * n + i] : b.V[(long long)(c - a.r) * n + i];
  }
  __syncthreads();
  block_qr(Uw, um, R, tauU, red, red + 4);
  block_qr(Vw, vm, R, tauV, red, red + 4);

  // Frobenius norms of the triangular factors (hodlr.py:191-192)
  double nu2 = 0.0, nv2 = 0.0;
  for (int idx = tid; idx < pu * R; idx += TT) {
    int l = idx / pu, i = idx - l * pu;
    if (l >= i) { double x = Uw[(long long)l * um + i]; nu2 += x * x; }
  }
  for (int idx = tid; idx < pv * R; idx += TT) {
    int l = idx / pv, i = idx - l * pv;
    if (l >= i) { double x = Vw[(long long)l * vm + i]; nv2 += x * x; }
  }
  nu2 = block_sum(nu2, red);
  nv2 = block_sum(nv2, red);

  // core M = Ru Rv^T (pu x pv); B = M (pu >= pv) or M^T
  const bool tr = pu < pv;
  const int pr = tr ? pv : pu, pc = tr ? pu : pv;
  for (int idx = tid; idx < pu * pv; idx += TT) {
    int i = idx / pv, j = idx - i * pv;
    int l0 = i > j ? i : j;
    double s = 0.0;
    for (int l = l0; l < R; ++l)
      s += Uw[(long long)l * um + i] * Vw[(long long)l * vm + j];
    if (!tr) Bm[(long long)j * pr + i] = s;
    else Bm[(long long)i * pr + j] = s;
  }
  __syncthreads();
  block_jacobi(Bm, pr, pc, Jm, iflag);
  for (int j = tid; j < pc; j += TT) {
    double s = 0.0;
    const double* bj = Bm + (long long)j * pr;
    for (int r = 0; r < pr; ++r) s += bj[r] * bj[r];
    sig[j] = sqrt(s);
  }
  __syncthreads();
  for (int j = tid; j < pc; j += TT) {
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
  if (keep > out.R) {
    if (tid == 0) atomicMax(A.overflow, keep);
    keep = 0;
  }
  if (A.ctr && tid == 0) {   // census formulas of SURVEY.md Appendix C
    unsigned long long fl = 4ull * um * R * R + 4ull * vm * R * R + 24ull * R * R * R +
                            2ull * (um + vm) * R * keep;
    atomicAdd(A.ctr, fl);
    atomicAdd(A.ctr + 1, 8ull * ((unsigned long long)um * R + vm * R + um * keep + vm * keep));
  }
  if (keep == 0) {
    if (tid == 0) *ro = 0;
    return;
  }
  // left/right factors padded with zeros, then Q applied
  for (int idx = tid; idx < um * keep; idx += TT) {
    int c = idx / um, i = idx - c * um;
    int j = ord[c];
    double v = 0.0;
    if (i < pu) v = tr ? sig[j] * Jm[(long long)j * pc + i] : Bm[(long long)j * pr + i];
    Ou[idx] = v;
  }
  for (int idx = tid; idx < vm * keep; idx += TT) {
    int c = idx / vm, i = idx - c * vm;
    int j = ord[c];
    double v = 0.0;
    if (i < pv) v = tr ? Bm[(long long)j * pr + i] / sig[j] : Jm[(long long)j * pc + i];
    Ov[idx] = v;
  }
  __syncthreads();
  block_apply_q(Uw, um, pu, tauU, Ou, keep);
  block_apply_q(Vw, vm, pv, tauV, Ov, keep);
  for (int idx = tid; idx < um * keep; idx += TT) {
    int c = idx / um, i = idx - c * um;
    Uo[(long long)c * n + i] = Ou[idx];
  }
  for (int idx = tid; idx < vm * keep; idx += TT) {
    int c = idx / vm, i = idx - c * vm;
    Vo[(long long)c * n + i] = Ov[idx];
  }
  if (tid == 0) *ro = keep;
}

long long trunc_need_doubles(int um, int vm, int R) {
  return 2LL * (um + vm) * R + 2LL * R * R + 4LL * R + 8;
}

cudaError_t launch_trunc(const TruncArgs& a, int nelem, size_t smem_bytes,
                         cudaStream_t st) {
  if (a.ntasks == 0 || nelem == 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_trunc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  dim3 grid(a.ntasks, nelem);
  k_trunc<<<grid, TT, smem_bytes, st>>>(a);
  return cudaGetLastError();
}

}  // namespace acr
