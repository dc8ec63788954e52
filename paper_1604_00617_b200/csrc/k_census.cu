// Algorithmic FLOP / byte census of the low-rank and panel kernels, for the
// instrumented factor only (plan option 2).  Each census kernel runs right
// after the kernel it describes, outside that kernel's timing events, reads
// the same device-resident ranks and adds SURVEY.md Appendix C's per-call
// formulas to the plan's counters:
//   HODLR x panel (k_hmatA/B): per subtree root mu with c panel columns,
//     every leaf (b rows):           leaf_matmat  2 b^2 c FLOP, 8 (b^2 + 2 b c) B
//     every branch side of rank r:   lr_apply     2 (m + k) r c FLOP,
//                                                 8 ((m + k) r + (m + k) c) B
//   small panel products (k_gp): K = X^T Y over l1 rows, Z = W K over l2 rows
//     2 (l1 + l2) rx ry FLOP, 8 (l1 (rx + ry) + l2 (rx + ry) + rx ry) B
//   low-rank leaf update (k_leaflr): per leaf (s rows) of rank r
//     leaf_add_uvT  2 s^2 r + s^2 FLOP, 8 (2 s^2 + 2 s r) B
// Counter slots: [150]/[151] hmat FLOP/B, [152]/[153] gp, [154]/[155] leaflr.
#include <algorithm>

#include "acr_types.cuh"
#include "acr_launch.h"

namespace acr {

__device__ __forceinline__ bool in_sub(const TreeDev& T, int v, int mu) {
  const int k = T.depth[v] - T.depth[mu];
  return k >= 0 && T.anc[v * (T.maxdepth + 1) + k] == mu;
}

struct CensusJobs {
  MMJob j[2];
};

__global__ void k_census_hmat(TreeDev T, CensusJobs JJ, int njobs, int nelem,
                              unsigned long long* ctr) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int span0 = JJ.j[0].mu1 - JJ.j[0].mu0;
  const int span1 = njobs > 1 ? JJ.j[1].mu1 - JJ.j[1].mu0 : 0;
  const int per = span0 + span1;
  if (t >= per * nelem) return;
  const int g = t / per;
  int q = t - g * per;
  const int jb = q < span0 ? 0 : 1;
  const MMJob& J = JJ.j[jb];
  const int mu = J.mu0 + (jb ? q - span0 : q);
  int c;
  if (J.cols_fixed >= 0) {
    c = J.cols_fixed;
  } else {
    if (mu == 0) return;
    const int p = T.parent[mu];
    const int ci = mu == T.c0[p] ? 0 : 1;
    c = rank_base(J.cols, g)[p * 2 + (ci ^ J.swap)];
  }
  if (!c) return;
  const int* rk = J.H[g].rk;
  unsigned long long fl = 0, by = 0;
  for (int v = 0; v < T.nnodes; ++v) {
    if (!in_sub(T, v, mu)) continue;
    const unsigned long long sz = T.hi[v] - T.lo[v];
    if (T.isleaf[v]) {
      fl += 2ull * sz * sz * c;
      by += 8ull * (sz * sz + 2ull * sz * c);
    } else {
      for (int s = 0; s < 2; ++s) {
        const unsigned long long r = rk[v * 2 + s];
        if (!r) continue;
        fl += 2ull * sz * r * c;
        by += 8ull * (sz * r + sz * c);
      }
    }
  }
  atomicAdd(ctr + 150, fl);
  atomicAdd(ctr + 151, by);
}

cudaError_t launch_census_hmat(const TreeDev& T, const MMJob* jobs, int njobs, int nelem,
                               unsigned long long* ctr, cudaStream_t st) {
  if (!ctr || !nelem || !njobs) return cudaSuccess;
  CensusJobs JJ;
  JJ.j[0] = jobs[0];
  JJ.j[1] = njobs > 1 ? jobs[1] : jobs[0];
  const int per = (jobs[0].mu1 - jobs[0].mu0) + (njobs > 1 ? jobs[1].mu1 - jobs[1].mu0 : 0);
  const long long tot = (long long)per * nelem;
  if (tot <= 0) return cudaSuccess;
  k_census_hmat<<<(unsigned)((tot + 127) / 128), 128, 0, st>>>(T, JJ, njobs, nelem, ctr);
  return cudaGetLastError();
}

struct CensusGP {
  GPJob j[2];
};

__global__ void k_census_gp(TreeDev T, CensusGP JJ, int njobs, const int* nodes, int nnodes,
                            int nelem, unsigned long long* ctr) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nnodes * nelem * njobs) return;
  const int jb = t / (nnodes * nelem);
  const int rem = t - jb * nnodes * nelem;
  const int g = rem / nnodes, nu = nodes[rem - g * nnodes];
  const GPJob& J = JJ.j[jb];
  const unsigned long long rx = rank_base(J.rx, g)[nu * 2 + J.sx];
  const unsigned long long ry = rank_base(J.ry, g)[nu * 2 + J.sy];
  if (!rx || !ry) return;
  const int lo = T.lo[nu], hi = T.hi[nu], mid = T.mid[nu];
  const unsigned long long l1 = J.hx ? hi - mid : mid - lo, l2 = J.hw ? hi - mid : mid - lo;
  atomicAdd(ctr + 152, 2ull * (l1 + l2) * rx * ry);
  atomicAdd(ctr + 153, 8ull * (l1 * (rx + ry) + l2 * (rx + ry) + rx * ry));
}

cudaError_t launch_census_gp(const TreeDev& T, const GPJob* jobs, int njobs, const int* nodes,
                             int nnodes, int nelem, unsigned long long* ctr, cudaStream_t st) {
  if (!ctr || !nelem || !njobs || !nnodes) return cudaSuccess;
  CensusGP JJ;
  JJ.j[0] = jobs[0];
  JJ.j[1] = njobs > 1 ? jobs[1] : jobs[0];
  const long long tot = (long long)nnodes * nelem * njobs;
  k_census_gp<<<(unsigned)((tot + 127) / 128), 128, 0, st>>>(T, JJ, njobs, nodes, nnodes,
                                                            nelem, ctr);
  return cudaGetLastError();
}

__global__ void k_census_leaflr(TreeDev T, RankRef rr, int node, int fside, int mu, int nelem,
                                unsigned long long* ctr) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nelem) return;
  const int* rb = rank_base(rr, g);
  unsigned long long r = rb[node * 2 + fside];
  if (rb[node * 2 + 1 - fside] == 0) r = 0;
  if (!r) return;
  unsigned long long fl = 0, by = 0;
  for (int v = 0; v < T.nnodes; ++v) {
    if (!T.isleaf[v] || !in_sub(T, v, mu)) continue;
    const unsigned long long s = T.hi[v] - T.lo[v];
    fl += 2ull * s * s * r + s * s;
    by += 8ull * (2ull * s * s + 2ull * s * r);
  }
  atomicAdd(ctr + 154, fl);
  atomicAdd(ctr + 155, by);
}

cudaError_t launch_census_leaflr(const TreeDev& T, RankRef rr, int node, int fside, int mu,
                                 int nelem, unsigned long long* ctr, cudaStream_t st) {
  if (!ctr || !nelem) return cudaSuccess;
  k_census_leaflr<<<(nelem + 127) / 128, 128, 0, st>>>(T, rr, node, fside, mu, nelem, ctr);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Rank statistics of one level (the host's profile_level / max_rank_of,
// reference algebra.py:272-291, computed where the rank tables live so the
// per-level host round trip moves nd numbers instead of three m x nnodes
// tables).  Blocks of D (all), E (i >= 1) and F (i <= m-2) are profiled,
// both sides of every branch node, bucketed by depth; the capacity maximum
// runs over every block and side.  out (zeroed by the caller):
//   u32 [0, nd) max, [nd, 2 nd) count, [2 nd] capacity max, [2 nd + 1] pad,
//   u64 sums at u32 offset 2 nd + 2.
// ---------------------------------------------------------------------------
__global__ void k_rank_stats(const int* rD, const int* rE, const int* rF, long long sr, int mm,
                             const int* branches, int nbr, const int* depth, int nd,
                             unsigned* out) {
  __shared__ unsigned smax[64], scnt[64];
  __shared__ unsigned long long ssum[64];
  __shared__ unsigned sg;
  for (int d = threadIdx.x; d < nd; d += blockDim.x) {
    smax[d] = 0;
    scnt[d] = 0;
    ssum[d] = 0;
  }
  if (threadIdx.x == 0) sg = 0;
  __syncthreads();
  const long long per = (long long)mm * nbr, tot = 3 * per;
  unsigned gmax = 0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
       t += (long long)gridDim.x * blockDim.x) {
    const int tb = (int)(t / per);
    const long long rem = t - tb * per;
    const int i = (int)(rem / nbr), v = branches[rem - (long long)i * nbr];
    const int* rk = (tb == 0 ? rD : tb == 1 ? rE : rF) + (long long)i * sr + 2 * v;
    const unsigned r0 = (unsigned)rk[0], r1 = (unsigned)rk[1];
    gmax = max(gmax, max(r0, r1));
    if (tb == 0 || (tb == 1 && i >= 1) || (tb == 2 && i + 1 < mm)) {
      const int d = depth[v];
      atomicMax(&smax[d], max(r0, r1));
      atomicAdd(&scnt[d], 2u);
      atomicAdd(&ssum[d], (unsigned long long)(r0 + r1));
    }
  }
  atomicMax(&sg, gmax);
  __syncthreads();
  unsigned long long* osum = reinterpret_cast<unsigned long long*>(out + 2 * nd + 2);
  for (int d = threadIdx.x; d < nd; d += blockDim.x) {
    if (!scnt[d]) continue;
    atomicMax(out + d, smax[d]);
    atomicAdd(out + nd + d, scnt[d]);
    atomicAdd(osum + d, ssum[d]);
  }
  if (threadIdx.x == 0) atomicMax(out + 2 * nd, sg);
}

cudaError_t launch_rank_stats(const int* rD, const int* rE, const int* rF, long long sr, int mm,
                              const int* branches, int nbr, const int* depth, int nd,
                              unsigned* out, cudaStream_t st) {
  if (nd > 64) return cudaErrorInvalidValue;
  const long long tot = 3LL * mm * nbr;
  if (tot <= 0) return cudaSuccess;
  const int grid = (int)std::min<long long>((tot + 255) / 256, 148);
  k_rank_stats<<<grid, 256, 0, st>>>(rD, rE, rF, sr, mm, branches, nbr, depth, nd, out);
  return cudaGetLastError();
}

}  // namespace acr
