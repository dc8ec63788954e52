// Dense cutoff solve and I/O kernels.
//   k_todense        HBlockTridiag.to_dense (reference reduction.py:66-75,
//                    hodlr.py:146-155) for the cutoff assembly / export
//   lu_factor/solve  dense LU with partial pivoting (reference oracles.py:20-31,
//                    scipy getrf/getrs semantics: first max pivot, singular if
//                    a U diagonal entry is exactly 0)
//   k_residual       ||A u - f|| / ||f|| from the bands (oracles.py:34-49)
#include <cooperative_groups.h>
#include <cstdlib>

#include "acr_types.cuh"
#include "acr_launch.h"
#include "acr_pdl.cuh"

namespace acr {

// one CTA per (dense block, row chunk); A row-major with leading dim ld
__global__ void k_todense(TreeDev T, const HB* blk, const int* rowblk,
                          const int* colblk, double* A, int ld) {
  ACR_PDL_ENTRY();
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
  CK_PDL(launch_pdl(k_todense, dim3(dim3(bx, nblk)), dim3(256), 0, st, T, blk, rowblk, colblk, A, ld));
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
      for (; i + 7 * ST < N; i += 8 * ST) {      // 8 independent rows in flight
        double l[8], a[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          l[u] = A[(long long)(i + u * ST) * N + j];
          a[u] = A[(long long)(i + u * ST) * N + c];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) A[(long long)(i + u * ST) * N + c] = a[u] - l[u] * ajc;
      }
      for (; i < N; i += ST) A[(long long)i * N + c] -= A[(long long)i * N + j] * ajc;
    }
    __syncthreads();
  }
}

// A12 := L11^{-1} A12 (unit lower), one thread per column, L11 in smem
__global__ void k_lu_trsm(double* A, int N, int j0, int jb) {
  ACR_PDL_ENTRY();
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
  ACR_PDL_ENTRY();
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

// Panel j0 (rows j0..N-1, jb columns) factored in sub-panels of LU_SB columns
// held in shared memory (column-major, ld = rows), right-looking inside the
// panel: getf2 on the sub-panel (pivot = first index of the largest |a|,
// whole panel row swapped, scale by 1/pivot, rank-1 updates), then the
// sub-panel's U row block (unit-lower solve) and the rank-LU_SB update of the
// panel columns to its right.  piv is absolute; columns outside the panel
// are swapped afterwards by k_lu_laswp.
static constexpr int LU_SB = 8;

__device__ __forceinline__ void lu_argmax(double best, int bidx, double* bv, int* bi, int* out,
                                          int tid) {
  const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (ov > best || (ov == best && oi < bidx)) { best = ov; bidx = oi; }
  }
  if (lane == 0) { bv[warp] = best; bi[warp] = bidx; }
  __syncthreads();
  if (warp == 0) {
    best = lane < LU_PT / 32 ? bv[lane] : -2.0;
    bidx = lane < LU_PT / 32 ? bi[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (ov > best || (ov == best && oi < bidx)) { best = ov; bidx = oi; }
    }
    if (lane == 0) *out = bidx;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(LU_PT) k_lu_panel_blk(double* A, int N, int j0, int jb,
                                                       int* piv, int* info) {
  extern __shared__ double S[];                 // LU_SB x Ms, column-major
  __shared__ double bv[LU_PT / 32];
  __shared__ int bi[LU_PT / 32];
  __shared__ int sp;
  const int tid = threadIdx.x;
  for (int s0 = 0; s0 < jb; s0 += LU_SB) {
    const int sb = jb - s0 < LU_SB ? jb - s0 : LU_SB;
    const int js = j0 + s0, Ms = N - js;
    for (int idx = tid; idx < Ms * sb; idx += LU_PT) {
      const int r = idx / sb, c = idx - r * sb;
      S[c * Ms + r] = A[(long long)(js + r) * N + js + c];
    }
    __syncthreads();
    for (int jj = 0; jj < sb; ++jj) {
      const double* cj = S + jj * Ms;
      double best = -1.0;
      int bidx = jj;
      for (int i = jj + tid; i < Ms; i += LU_PT) {
        const double v = fabs(cj[i]);
        if (v > best) { best = v; bidx = i; }
      }
      lu_argmax(best, bidx, bv, bi, &sp, tid);
      const int p = sp;
      const double pv = cj[p];
      if (tid == 0) {
        piv[js + jj] = js + p;
        if (pv == 0.0 && *info == 0) *info = js + jj + 1;
      }
      __syncthreads();                            // everyone has read the pivot
      if (p != jj && tid < sb) {                  // sub-panel rows in smem
        double* cc = S + tid * Ms;
        const double t = cc[jj];
        cc[jj] = cc[p];
        cc[p] = t;
      }
      __syncthreads();
      // scale and rank-1 update fused per row (the row's own multiplier)
      const double rinv = pv != 0.0 ? 1.0 / pv : 0.0;
      for (int i = jj + 1 + tid; i < Ms; i += LU_PT) {
        double* cw = S + jj * Ms;
        const double l = pv != 0.0 ? cw[i] * rinv : cw[i];
        cw[i] = l;
        for (int c = jj + 1; c < sb; ++c) {
          double* cc = S + c * Ms;
          cc[i] = cc[i] - l * cc[jj];
        }
      }
      __syncthreads();
    }
    // the sub-panel's row interchanges on the other panel columns: touched
    // rows (<= 2 LU_SB) staged in shared memory, swaps replayed, written back
    {
      __shared__ int rws[2 * LU_SB], sa[LU_SB], sbb[LU_SB], nrw;
      __shared__ double tile[2 * LU_SB][LU_NB];
      // slots 0..sb-1: the sub-panel rows; pivot rows below it get one extra
      // slot each (duplicates share their first occurrence's slot): built by
      // one warp with match/ballot instead of a serial scan by one thread
      if (tid < 32) {
        const bool act = tid < sb;
        const int pr = act ? piv[js + tid] : -1;
        const bool ext = act && pr >= js + sb;
        const unsigned extm = __ballot_sync(0xffffffffu, ext);
        const unsigned same = __match_any_sync(0xffffffffu, ext ? pr : -1 - tid);
        const int leader = __ffs(same & extm) - 1;
        const unsigned firsts = __ballot_sync(0xffffffffu, ext && leader == tid);
        if (act) {
          rws[tid] = js + tid;
          sa[tid] = tid;
          if (ext) {
            const int slot = sb + __popc(firsts & ((1u << leader) - 1u));
            sbb[tid] = slot;
            if (leader == tid) rws[slot] = pr;
          } else {
            sbb[tid] = pr - js;
          }
        }
        if (tid == 0) nrw = sb + __popc(firsts);
      }
      __syncthreads();
      const int ncol = jb - sb;                   // panel columns outside the sub-panel
      for (int idx = tid; idx < nrw * ncol; idx += LU_PT) {
        const int q = idx / ncol, k = idx - q * ncol;
        const int c = j0 + (k < s0 ? k : k + sb);
        tile[q][k] = A[(long long)rws[q] * N + c];
      }
      __syncthreads();
      if (tid < ncol)
        for (int k = 0; k < sb; ++k) {
          const double t = tile[sa[k]][tid];
          tile[sa[k]][tid] = tile[sbb[k]][tid];
          tile[sbb[k]][tid] = t;
        }
      __syncthreads();
      for (int idx = tid; idx < nrw * ncol; idx += LU_PT) {
        const int q = idx / ncol, k = idx - q * ncol;
        const int c = j0 + (k < s0 ? k : k + sb);
        A[(long long)rws[q] * N + c] = tile[q][k];
      }
    }
    for (int idx = tid; idx < Ms * sb; idx += LU_PT) {
      const int r = idx / sb, c = idx - r * sb;
      A[(long long)(js + r) * N + js + c] = S[c * Ms + r];
    }
    const int c0 = js + sb, nr = j0 + jb - c0;   // panel columns to the right
    if (nr > 0) {
      // U12 = L11^{-1} A12 (unit lower), one thread per column; also kept in
      // shared memory for the update below (read once per element otherwise)
      __shared__ double u12[LU_SB][LU_NB];
      if (tid < nr) {
        const int c = c0 + tid;
        double x[LU_SB];
#pragma unroll
        for (int k = 0; k < LU_SB; ++k) {
          if (k < sb) {
            double v = A[(long long)(js + k) * N + c];
            for (int q = 0; q < k; ++q) v -= S[q * Ms + k] * x[q];
            x[k] = v;
            A[(long long)(js + k) * N + c] = v;
            u12[k][tid] = v;
          }
        }
      }
      __syncthreads();
      // A22 -= L21 U12 for the panel columns to the right
      for (int idx = tid; idx < (Ms - sb) * nr; idx += LU_PT) {
        const int r = sb + idx / nr, cc = idx % nr, c = c0 + cc;
        double v = A[(long long)(js + r) * N + c];
        for (int k = 0; k < sb; ++k) v -= S[k * Ms + r] * u12[k][cc];
        A[(long long)(js + r) * N + c] = v;
      }
    }
    __syncthreads();
  }
}

// Panel factorisation on a thread-block cluster of LUC CTAs (distributed
// shared memory): the whole jb-column panel stays on chip, split by rows
// over the CTAs (a single SM streamed every sub-panel and its in-panel
// update through L2, ~120 us per panel).  Row interchanges are implicit --
// rows never move inside the panel; every CTA keeps the same position ->
// physical-row map and each thread its own row's position -- and the panel
// is written back in its final (swapped) order.  Per column: the CTAs' local
// pivot candidates (largest |a|, first position on ties: getrf's rule),
// one cluster barrier, the winner and the pivot row read through DSMEM, the
// rank-1 update of the remaining panel columns (scale by the reciprocal of
// the pivot, as dgetf2).  piv / info as the other panel kernels.
static constexpr int LUC = 4;
static constexpr int LUCT = 512;

__global__ void __cluster_dims__(LUC, 1, 1) __launch_bounds__(LUCT, 1)
    k_lu_panel_cl(double* A, int N, int j0, int jb, int* piv, int* info) {
  ACR_PDL_ENTRY();
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double sm[];
  constexpr int NW = LUCT / 32;
  const int crank = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int Ms = N - j0;
  const int RB = (Ms + LUC - 1) / LUC;
  const int r0 = crank * RB;
  const int nr = Ms - r0 < RB ? (Ms - r0 > 0 ? Ms - r0 : 0) : RB;
  double* P = sm;                                        // [c][i], column c of own rows
  int* p2r = reinterpret_cast<int*>(P + (size_t)jb * RB);  // position -> physical row
  // per-warp pivot candidates, double-buffered by column parity (read by
  // every CTA of the cluster through DSMEM after the cluster barrier)
  __shared__ double wv[2][NW];
  __shared__ int wpos[2][NW], wrow[2][NW];
  __shared__ double prow[LU_NB];
  __shared__ int s_pos, s_row, s_a;
  for (int idx = tid; idx < nr * jb; idx += LUCT) {
    const int i = idx / jb, c = idx - i * jb;
    P[c * RB + i] = A[(long long)(j0 + r0 + i) * N + j0 + c];
  }
  for (int q = tid; q < Ms; q += LUCT) p2r[q] = q;
  int my_pos = tid < nr ? r0 + tid : 0x7fffffff;
  __syncthreads();
  for (int jj = 0; jj < jb; ++jj) {
    const int par = jj & 1;
    // warp candidate: rows not yet pivoted (position >= jj)
    double best = -1.0;
    int bpos = 0x7fffffff, brow = -1;
    if (tid < nr && my_pos >= jj) {
      best = fabs(P[jj * RB + tid]);
      bpos = my_pos;
      brow = r0 + tid;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int op = __shfl_xor_sync(0xffffffffu, bpos, o);
      const int orr = __shfl_xor_sync(0xffffffffu, brow, o);
      if (ov > best || (ov == best && op < bpos)) { best = ov; bpos = op; brow = orr; }
    }
    if (lane == 0) { wv[par][warp] = best; wpos[par][warp] = bpos; wrow[par][warp] = brow; }
    cl.sync();                                  // all candidates and rows of step jj ready
    if (warp == 0) {
      // the winner among the LUC x NW warp candidates (lane t reads CTA
      // t / (32 / NW)'s... every CTA's NW slots, LUC * NW <= 64: two per lane)
      best = -1.0;
      bpos = 0x7fffffff;
      brow = -1;
#pragma unroll
      for (int h = 0; h < (LUC * NW + 31) / 32; ++h) {
        const int t = lane + 32 * h;
        if (t < LUC * NW) {
          const int cr = t / NW, w = t - cr * NW;
          const double v = cl.map_shared_rank(&wv[par][0], cr)[w];
          const int pp = cl.map_shared_rank(&wpos[par][0], cr)[w];
          const int rr = cl.map_shared_rank(&wrow[par][0], cr)[w];
          if (v > best || (v == best && pp < bpos)) { best = v; bpos = pp; brow = rr; }
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int op = __shfl_xor_sync(0xffffffffu, bpos, o);
        const int orr = __shfl_xor_sync(0xffffffffu, brow, o);
        if (ov > best || (ov == best && op < bpos)) { best = ov; bpos = op; brow = orr; }
      }
      const int owner = brow / RB, li = brow - owner * RB;
      const double* opn = cl.map_shared_rank(P, owner);
      if (lane >= jj && lane < jb) prow[lane] = opn[lane * RB + li];
      if (lane == 0) {
        const int a = p2r[jj];                  // physical row now at position jj
        s_pos = bpos;
        s_row = brow;
        s_a = a;
        p2r[jj] = brow;
        p2r[bpos] = a;
      }
    }
    __syncthreads();
    const int ppos = s_pos, prw = s_row, a = s_a;
    if (tid < nr) {
      if (r0 + tid == a) my_pos = ppos;
      if (r0 + tid == prw) my_pos = jj;
    }
    const double pv = prow[jj];
    if (crank == 0 && tid == 0) {
      piv[j0 + jj] = j0 + ppos;
      if (pv == 0.0 && *info == 0) *info = j0 + jj + 1;
    }
    if (tid < nr && my_pos > jj) {
      const double rinv = pv != 0.0 ? 1.0 / pv : 0.0;
      const double l = pv != 0.0 ? P[jj * RB + tid] * rinv : P[jj * RB + tid];
      P[jj * RB + tid] = l;
      for (int c = jj + 1; c < jb; ++c) P[c * RB + tid] = P[c * RB + tid] - l * prow[c];
    }
    // prow is rewritten by warp 0 only after the next cluster barrier, which
    // every thread of this CTA reaches after its update
  }
  cl.sync();                                    // remote reads of this CTA's rows done
  __shared__ int fpos[LUCT];                    // each row's final position
  fpos[tid] = tid < nr ? my_pos : 0;
  __syncthreads();
  for (int idx = tid; idx < nr * jb; idx += LUCT) {
    const int i = idx / jb, c = idx - i * jb;
    A[(long long)(j0 + fpos[i]) * N + j0 + c] = P[c * RB + i];
  }
}

// Register-resident variant of the cluster panel (jb <= 32): every thread
// keeps its row of the panel in registers, so the rank-1 update of a column
// step is 31 FMAs on registers (the shared-memory panel paid a load and a
// store per element), and a step costs one DSMEM round trip instead of two:
// every CTA first reduces its warps' candidates to one and stages that row,
// and after the cluster barrier warp 0 reads the four CTA candidates and the
// four staged rows together.  Same pivot rule, implicit interchanges and
// write-back order as k_lu_panel_cl.
__global__ void __cluster_dims__(LUC, 1, 1) __launch_bounds__(LUCT, 1)
    k_lu_panel_reg(double* A, int N, int j0, int jb, int* piv, int* info) {
  ACR_PDL_ENTRY();
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double sm[];
  constexpr int NW = LUCT / 32;
  constexpr int NB = LU_NB;
  const int crank = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int Ms = N - j0;
  const int RB = (Ms + LUC - 1) / LUC;
  const int r0 = crank * RB;
  const int nr = Ms - r0 < RB ? (Ms - r0 > 0 ? Ms - r0 : 0) : RB;
  double* tile = sm + (size_t)warp * 32 * 33;              // per-warp 32 x 33 transpose tile
  int* p2r = reinterpret_cast<int*>(sm + (size_t)NW * 32 * 33);   // position -> physical row
  __shared__ double wv[NW], wrowbuf[NW][NB];
  __shared__ int wpos[NW], wrow[NW];
  __shared__ double cta_v[2], cta_row[2][NB];     // double-buffered by column parity
  __shared__ int cta_pos[2], cta_rw[2];
  __shared__ double prow[NB];
  __shared__ int s_pos, s_row, s_a;
  // rows of this warp, coalesced through the tile
  double row[NB];
  {
    const int wr0 = r0 + warp * 32;                        // first row of this warp
    for (int r = 0; r < 32; ++r) {
      const int rr = warp * 32 + r;
      tile[r * 33 + lane] = (rr < nr && lane < jb) ? A[(long long)(j0 + wr0 + r) * N + j0 + lane] : 0.0;
    }
    __syncwarp();
#pragma unroll
    for (int c = 0; c < NB; ++c) row[c] = tile[lane * 33 + c];
    __syncwarp();
  }
  for (int q = tid; q < Ms; q += LUCT) p2r[q] = q;
  int my_pos = tid < nr ? r0 + tid : 0x7fffffff;
  __syncthreads();
#pragma unroll
  for (int jj = 0; jj < NB; ++jj) {
    if (jj >= jb) break;
    const int par = jj & 1;
    // warp candidate: rows not yet pivoted (position >= jj)
    double best = -1.0;
    int bpos = 0x7fffffff, brow = -1;
    if (tid < nr && my_pos >= jj) {
      best = fabs(row[jj]);
      bpos = my_pos;
      brow = r0 + tid;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int op = __shfl_xor_sync(0xffffffffu, bpos, o);
      const int orr = __shfl_xor_sync(0xffffffffu, brow, o);
      if (ov > best || (ov == best && op < bpos)) { best = ov; bpos = op; brow = orr; }
    }
    if (lane == 0) { wv[warp] = best; wpos[warp] = bpos; wrow[warp] = brow; }
    if (brow >= 0 && r0 + tid == brow) {
#pragma unroll
      for (int c = 0; c < NB; ++c)
        if (c >= jj) wrowbuf[warp][c] = row[c];
    }
    __syncthreads();
    if (warp == 0) {                            // this CTA's candidate and its row
      best = lane < NW ? wv[lane] : -1.0;
      bpos = lane < NW ? wpos[lane] : 0x7fffffff;
      int bw = lane;
#pragma unroll
      for (int o = NW / 2; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int op = __shfl_xor_sync(0xffffffffu, bpos, o);
        const int ow = __shfl_xor_sync(0xffffffffu, bw, o);
        if (ov > best || (ov == best && op < bpos)) { best = ov; bpos = op; bw = ow; }
      }
      bw = __shfl_sync(0xffffffffu, bw, 0);
      best = __shfl_sync(0xffffffffu, best, 0);
      bpos = __shfl_sync(0xffffffffu, bpos, 0);
      cta_row[par][lane] = (best >= 0.0 && lane >= jj) ? wrowbuf[bw][lane] : 0.0;
      if (lane == 0) { cta_v[par] = best; cta_pos[par] = bpos; cta_rw[par] = best >= 0.0 ? wrow[bw] : -1; }
    }
    cl.sync();                                  // every CTA's candidate and row staged
    if (warp == 0) {
      double rv[LUC];
#pragma unroll
      for (int k = 0; k < LUC; ++k) rv[k] = cl.map_shared_rank(&cta_row[par][0], k)[lane];
      best = -1.0;
      bpos = 0x7fffffff;
      brow = -1;
      int bk = lane;
      if (lane < LUC) {
        best = *cl.map_shared_rank(&cta_v[par], lane);
        bpos = *cl.map_shared_rank(&cta_pos[par], lane);
        brow = *cl.map_shared_rank(&cta_rw[par], lane);
      }
#pragma unroll
      for (int o = LUC / 2; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int op = __shfl_xor_sync(0xffffffffu, bpos, o);
        const int orr = __shfl_xor_sync(0xffffffffu, brow, o);
        const int ok = __shfl_xor_sync(0xffffffffu, bk, o);
        if (ov > best || (ov == best && op < bpos)) { best = ov; bpos = op; brow = orr; bk = ok; }
      }
      bk = __shfl_sync(0xffffffffu, bk, 0);
      bpos = __shfl_sync(0xffffffffu, bpos, 0);
      brow = __shfl_sync(0xffffffffu, brow, 0);
      double pr = rv[0];
#pragma unroll
      for (int k = 1; k < LUC; ++k)
        if (bk == k) pr = rv[k];
      prow[lane] = pr;
      if (lane == 0) {
        const int a = p2r[jj];                  // physical row now at position jj
        s_pos = bpos;
        s_row = brow;
        s_a = a;
        p2r[jj] = brow;
        p2r[bpos] = a;
      }
    }
    __syncthreads();
    const int ppos = s_pos, prw = s_row, a = s_a;
    if (tid < nr) {
      if (r0 + tid == a) my_pos = ppos;
      if (r0 + tid == prw) my_pos = jj;
    }
    const double pv = prow[jj];
    if (crank == 0 && tid == 0) {
      piv[j0 + jj] = j0 + ppos;
      if (pv == 0.0 && *info == 0) *info = j0 + jj + 1;
    }
    if (tid < nr && my_pos > jj) {
      const double rinv = pv != 0.0 ? 1.0 / pv : 0.0;
      const double l = pv != 0.0 ? row[jj] * rinv : row[jj];
      row[jj] = l;
#pragma unroll
      for (int c = 0; c < NB; ++c)
        if (c > jj) row[c] = row[c] - l * prow[c];
    }
    // prow, the warp slots and the staged rows of this parity are rewritten
    // only after barriers every reader reaches after its reads
  }
  cl.sync();                                    // remote reads of this CTA's staged rows done
  // write back in final (swapped) order, coalesced through the tile
  {
#pragma unroll
    for (int c = 0; c < NB; ++c) tile[lane * 33 + c] = row[c];
    __syncwarp();
    for (int r = 0; r < 32; ++r) {
      const int pos = __shfl_sync(0xffffffffu, my_pos, r);
      if (warp * 32 + r < nr && lane < jb)
        A[(long long)(j0 + pos) * N + j0 + lane] = tile[r * 33 + lane];
    }
  }
}

// Row interchanges of panel j0 applied to every column outside it (laswp):
// a CTA stages the <= 2 jb touched rows of its 32 columns in shared memory,
// replays the swaps there (thread per column) and writes the rows back.
__global__ void k_lu_laswp(double* A, int N, int j0, int jb, const int* piv) {
  ACR_PDL_ENTRY();
  __shared__ double t[2 * LU_NB][33];
  __shared__ int rows[2 * LU_NB], sa[LU_NB], sb[LU_NB], nrows;
  // slots 0..jb-1: rows j0..j0+jb-1; pivot rows below the panel get extra
  // slots in first-occurrence order (parallel over k)
  __shared__ int extra[LU_NB];
  const int tl = threadIdx.y * 32 + threadIdx.x;
  if (tl < jb) {
    const int pr = piv[j0 + tl];
    int first = 1;
    if (pr >= j0 + jb)
      for (int q = 0; q < tl; ++q)
        if (piv[j0 + q] == pr) { first = 0; break; }
    extra[tl] = (pr >= j0 + jb && first) ? 1 : 0;
    rows[tl] = j0 + tl;
  }
  __syncthreads();
  if (tl < jb) {
    const int pr = piv[j0 + tl];
    sa[tl] = tl;
    if (pr < j0 + jb) {
      sb[tl] = pr - j0;
    } else {
      int q0 = tl;                                // first occurrence of pr
      for (int q = 0; q < tl; ++q)
        if (piv[j0 + q] == pr) { q0 = q; break; }
      int pos = jb;
      for (int q = 0; q < q0; ++q) pos += extra[q];
      sb[tl] = pos;
      if (q0 == tl) rows[pos] = pr;
    }
  }
  if (tl == 0) {
    int cnt = jb;
    for (int q = 0; q < jb; ++q) cnt += extra[q];
    nrows = cnt;
  }
  __syncthreads();
  // columns of this CTA: [0, j0) and [j0 + jb, N) enumerated contiguously
  int c = blockIdx.x * 32 + threadIdx.x;
  if (c >= j0) c += jb;
  const bool okc = c < N;
  for (int q = threadIdx.y; q < nrows; q += blockDim.y)
    t[q][threadIdx.x] = okc ? A[(long long)rows[q] * N + c] : 0.0;
  __syncthreads();
  if (threadIdx.y == 0 && okc)
    for (int k = 0; k < jb; ++k) {
      const double x = t[sa[k]][threadIdx.x];
      t[sa[k]][threadIdx.x] = t[sb[k]][threadIdx.x];
      t[sb[k]][threadIdx.x] = x;
    }
  __syncthreads();
  for (int q = threadIdx.y; q < nrows; q += blockDim.y)
    if (okc) A[(long long)rows[q] * N + c] = t[q][threadIdx.x];
}

cudaError_t lu_factor(double* A, int N, int* piv, int* info, double* work,
                      cudaStream_t st) {
  (void)work;
  cudaMemsetAsync(info, 0, sizeof(int), st);
  for (int j0 = 0; j0 < N; j0 += LU_NB) {
    int jb = N - j0 < LU_NB ? N - j0 : LU_NB;
    const size_t sbytes = (size_t)LU_SB * (N - j0) * sizeof(double);
    const int Ms = N - j0, RB = (Ms + LUC - 1) / LUC;
    const size_t cbytes = (size_t)jb * RB * sizeof(double) + (size_t)Ms * sizeof(int);
    static const bool nocl = getenv("ACR_LU_NOCLUSTER") != nullptr;   // A/B aid
    if (!nocl && RB <= LUCT && cbytes <= 200 * 1024) {   // whole panel on a CTA cluster
      static bool attr_c = false;
      if (!attr_c) {
        cudaFuncSetAttribute(k_lu_panel_cl, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
        attr_c = true;
      }
      static const bool noreg = getenv("ACR_LU_NOREG") != nullptr;   // A/B aid
      const size_t rbytes = (size_t)(LUCT / 32) * 32 * 33 * sizeof(double) + (size_t)Ms * sizeof(int);
      if (!noreg && rbytes <= 200 * 1024) {
        static bool attr_r = false;
        if (!attr_r) {
          cudaFuncSetAttribute(k_lu_panel_reg, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               200 * 1024);
          attr_r = true;
        }
        CK_PDL(launch_pdl(k_lu_panel_reg, dim3(LUC), dim3(LUCT), rbytes, st, A, N, j0, jb, piv, info));
      } else {
        CK_PDL(launch_pdl(k_lu_panel_cl, dim3(LUC), dim3(LUCT), cbytes, st, A, N, j0, jb, piv, info));
      }
      if (N - jb > 0) CK_PDL(launch_pdl(k_lu_laswp, dim3((N - jb + 31) / 32), dim3(dim3(32, 8)), 0, st, A, N, j0, jb, piv));
    } else if (sbytes <= 200 * 1024) {   // sub-panels in shared memory
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(k_lu_panel_blk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
        attr = true;
      }
      k_lu_panel_blk<<<1, LU_PT, sbytes, st>>>(A, N, j0, jb, piv, info);
      if (N - jb > 0) CK_PDL(launch_pdl(k_lu_laswp, dim3((N - jb + 31) / 32), dim3(dim3(32, 8)), 0, st, A, N, j0, jb, piv));
    } else {
      k_lu_panel<<<1, LU_PT, 0, st>>>(A, N, j0, jb, piv, info);
    }
    int rest = N - j0 - jb;
    if (rest > 0) {
      CK_PDL(launch_pdl(k_lu_trsm, dim3((rest + 63) / 64), dim3(64), 0, st, A, N, j0, jb));
      dim3 g((rest + 63) / 64, (rest + 63) / 64);
      CK_PDL(launch_pdl(k_lu_gemm, dim3(g), dim3(256), 0, st, A, N, j0, jb));
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

// Blocked substitution for one right-hand side per CTA, the column in shared
// memory: row interchanges replayed in shared memory, then 32-row blocks --
// warp 0 solves the diagonal block from a staged tile, all threads apply the
// block to the remaining rows.  Every row subtracts its terms in the same
// order as k_lu_solve (ascending j forward, descending j backward), so the
// result is identical.
static constexpr int LS_T = 1024;

// At: the LU factors transposed (column-major), so that the block updates'
// reads A[i][b0 + k] = At[(b0 + k) N + i] are coalesced over the rows i
__global__ void k_transpose(const double* A, int N, double* At) {
  __shared__ double t[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int i = by + r, j = bx + threadIdx.x;
    if (i < N && j < N) t[r][threadIdx.x] = A[(long long)i * N + j];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int j = bx + r, i = by + threadIdx.x;
    if (i < N && j < N) At[(long long)j * N + i] = t[threadIdx.x][r];
  }
}

// row order after the factorisation's interchanges (perm[i] = original row
// that ends up in position i): computed once per factorisation, so a solve
// gathers its right-hand side instead of replaying N dependent swaps
__global__ void k_lu_perm(const int* piv, int N, int* perm) {
  extern __shared__ int pm[];
  for (int i = threadIdx.x; i < N; i += blockDim.x) pm[i] = i;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int j = 0; j < N; ++j) {
      const int p = piv[j];
      if (p != j) { const int t = pm[j]; pm[j] = pm[p]; pm[p] = t; }
    }
  __syncthreads();
  for (int i = threadIdx.x; i < N; i += blockDim.x) perm[i] = pm[i];
}

// One CTA per right-hand-side column, y in shared memory.  Per 32-row block:
// the diagonal block (prefetched into the other buffer during the previous
// step) is solved by one warp, then every remaining row takes its update with
// 16 loads in flight (At = A^T: coalesced across the rows).
__global__ void __launch_bounds__(LS_T, 1) k_lu_solve_blk(const double* A, const double* At,
                                                      int N, const int* piv, const int* perm,
                                                      double* B) {
  extern __shared__ double y[];                 // N doubles, then N ints
  int* pv = reinterpret_cast<int*>(y + N);
  __shared__ double Tb[2][32][33];
  double* b = B + (long long)blockIdx.x * N;
  const int tid = threadIdx.x, lane = tid & 31;
  if (perm) {
    for (int i = tid; i < N; i += LS_T) y[i] = b[perm[i]];
  } else {
    for (int i = tid; i < N; i += LS_T) { y[i] = b[i]; pv[i] = piv[i]; }
    __syncthreads();
    if (tid == 0)
      for (int j = 0; j < N; ++j) {
        const int p = pv[j];
        if (p != j) { const double t = y[j]; y[j] = y[p]; y[p] = t; }
      }
  }
  const int tr = tid >> 5, tc = tid & 31;       // this thread's element of a diagonal block
  auto diag_elem = [&](int b0) {
    const int r = b0 + tr, c = b0 + tc;
    return (b0 >= 0 && b0 < N && r < N && c < N) ? A[(long long)r * N + c] : 0.0;
  };
  int cur = 0;
  Tb[0][tr][tc] = diag_elem(0);
  __syncthreads();
  // forward: unit lower L
  for (int b0 = 0; b0 < N; b0 += 32) {
    const int bs = N - b0 < 32 ? N - b0 : 32;
    const double tn = diag_elem(b0 + 32);        // next block, in flight during this step
    if (tid < 32) {
      double v = lane < bs ? y[b0 + lane] : 0.0;
      for (int k = 0; k < bs; ++k) {
        const double yk = __shfl_sync(0xffffffffu, v, k);
        if (lane > k && lane < bs) v -= Tb[cur][lane][k] * yk;
      }
      if (lane < bs) y[b0 + lane] = v;
    }
    __syncthreads();
    for (int i = b0 + bs + tid; i < N; i += LS_T) {
      const double* ar = At + (long long)b0 * N + i;   // A[i][b0 + k] = ar[k N]
      double v = y[i];
      for (int kb = 0; kb < bs; kb += 16) {      // 16 loads in flight, order kept
        double a[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) a[u] = kb + u < bs ? ar[(long long)(kb + u) * N] : 0.0;
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (kb + u < bs) v -= a[u] * y[b0 + kb + u];
      }
      y[i] = v;
    }
    Tb[cur ^ 1][tr][tc] = tn;
    cur ^= 1;
    __syncthreads();
  }
  // backward: upper U (non-unit diagonal), blocks from the bottom
  const int blast = ((N - 1) / 32) * 32;
  Tb[cur][tr][tc] = diag_elem(blast);
  __syncthreads();
  for (int b0 = blast; b0 >= 0; b0 -= 32) {
    const int bs = N - b0 < 32 ? N - b0 : 32;
    const double tn = diag_elem(b0 - 32);
    if (tid < 32) {
      double v = lane < bs ? y[b0 + lane] : 0.0;
      for (int k = bs - 1; k >= 0; --k) {
        if (lane == k) v = v / Tb[cur][k][k];
        const double yk = __shfl_sync(0xffffffffu, v, k);
        if (lane < k) v -= Tb[cur][lane][k] * yk;
      }
      if (lane < bs) y[b0 + lane] = v;
    }
    __syncthreads();
    for (int i = tid; i < b0; i += LS_T) {
      const double* ar = At + (long long)b0 * N + i;   // A[i][b0 + k] = ar[k N]
      double v = y[i];
      for (int kb = bs - 1; kb >= 0; kb -= 16) {  // descending, 16 loads in flight
        double a[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) a[u] = kb - u >= 0 ? ar[(long long)(kb - u) * N] : 0.0;
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (kb - u >= 0) v -= a[u] * y[b0 + kb - u];
      }
      y[i] = v;
    }
    Tb[cur ^ 1][tr][tc] = tn;
    cur ^= 1;
    __syncthreads();
  }
  for (int i = tid; i < N; i += LS_T) b[i] = y[i];
}

cudaError_t lu_perm(const int* piv, int N, int* perm, cudaStream_t st) {
  const size_t smem = (size_t)N * sizeof(int);
  if (smem > 160 * 1024) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_lu_perm, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    attr = true;
  }
  k_lu_perm<<<1, 1024, smem, st>>>(piv, N, perm);
  return cudaGetLastError();
}

cudaError_t lu_transpose(const double* A, int N, double* At, cudaStream_t st) {
  dim3 g((N + 31) / 32, (N + 31) / 32), b(32, 8);
  k_transpose<<<g, b, 0, st>>>(A, N, At);
  return cudaGetLastError();
}

cudaError_t lu_solve(const double* A, const double* At, int N, const int* piv, double* B,
                     int nrhs, cudaStream_t st, const int* perm) {
  if (!nrhs) return cudaSuccess;
  const size_t smem = (size_t)N * (sizeof(double) + sizeof(int));
  if (smem <= 160 * 1024 && At) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_lu_solve_blk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           160 * 1024);
      attr = true;
    }
    k_lu_solve_blk<<<nrhs, LS_T, smem, st>>>(A, At, N, piv, perm, B);
  } else {
    k_lu_solve<<<nrhs, 1024, 0, st>>>(A, N, piv, B);
  }
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
