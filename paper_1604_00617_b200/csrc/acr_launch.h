// Host-side launchers of the ACR kernels (internal; the public C ABI is
// include/acr_b200.h).
#pragma once
#include <cuda_runtime.h>
#include "acr_types.cuh"

namespace acr {

long long trunc_need_doubles(int um, int vm, int R);
int trunc_warp_pool_doubles();
// warp-per-task recompression; tasks too large for the warp pool are queued
// to bigq and processed by a persistent block-level kernel (may_big)
// direct: one 512-thread CTA per (task, element) -- small, latency-bound
// launches; otherwise warp kernel, with oversized tasks queued to bigq
// aux (required with may_big): cls = nitems bytes of device scratch for the
// classification flags; q0 / q1 = streams for the two queue kernels, which
// then run beside the warp kernel (events ef, ej0, ej1 order them around st);
// null streams run the three kernels in turn on st
struct TruncAux {
  unsigned char* cls;
  cudaStream_t q0, q1;
  cudaEvent_t ef, ej0, ej1;
};
cudaError_t launch_trunc(const TruncArgs& a, int nelem, bool direct, bool may_big,
                         int* bigq, int* bigcount, cudaStream_t st,
                         const TruncAux* aux = nullptr);
int trunc_direct_max();
long long warp_need_doubles(int um, int vm, int R);
// CTA-pair (cluster of 2) recompression for direct launches of large tasks
cudaError_t launch_trunc_pair(const TruncArgs& a, int nelem, long long smem_doubles,
                              cudaStream_t st);
long long pair_need_doubles(int m, int R);

// leaf kernels (k_leaf.cu)
cudaError_t launch_leafinv(const TreeDev& T, const HB* H, int nelem, int leaf,
                           int* sing, cudaStream_t st);
// tridiagonal leaves (lifted level); a nonzero off the band raises *fail |= 1 << 28
cudaError_t launch_leafinv_tri(const TreeDev& T, const HB* H, int nelem, int leaf, int* sing,
                               int* fail, cudaStream_t st);
// diag: 0 general (DMMA), 1 A diagonal, 2 B diagonal (exact fast path)
cudaError_t launch_leafgemm(const TreeDev& T, const HB* A, const HB* B,
                            const HB* C, int nelem, Src PX, RankRef xr, int diag,
                            cudaStream_t st);
cudaError_t launch_leaflr_n(const TreeDev& T, const HB* H, int nelem, int mu,
                            int nleaf, Src U, Src V, RankRef rr, int node,
                            int fside, cudaStream_t st);
// fused Schur step at a branch node with two leaf children (k_leaf.cu)
size_t schur_leaf_smem(int bw, int R);
cudaError_t launch_schur_leaf(const TreeDev& T, const HB* H, int nelem, int nu, int half,
                              Src P1, Src P2, int R, cudaStream_t st);
cudaError_t launch_leafadd(const TreeDev& T, const HB* A, const HB* B,
                           const HB* C, double sb, int nelem, cudaStream_t st);
// int copy (e.g. device -> mapped pinned host memory, bypassing the copy
// engines) and fill
cudaError_t launch_copy_i32(int* dst, const int* src, long long n, cudaStream_t st);
cudaError_t launch_fill_i32(int* dst, int v, long long n, cudaStream_t st);
cudaError_t launch_negate(const TreeDev& T, const HB* H, int nelem,
                          cudaStream_t st);
cudaError_t launch_copyhb(const TreeDev& T, const HB* S, const HB* D, int nelem,
                          int* overflow, cudaStream_t st);
cudaError_t launch_zerohb(const TreeDev& T, const HB* D, int nelem,
                          cudaStream_t st);
cudaError_t launch_lift(const TreeDev& T, const double* sub, const double* diag,
                        const double* sup, const HB* D, int nelem,
                        cudaStream_t st);
cudaError_t launch_liftdiag(const TreeDev& T, const double* d, const HB* D,
                            int nelem, cudaStream_t st);
cudaError_t launch_build_tab(HB* tab, HB base, long long sl, long long sf,
                             long long sr, int first, int step, int count,
                             cudaStream_t st);

// HODLR x panel (k_hmat.cu)
cudaError_t launch_hmat(const TreeDev& T, const MMJob* jobs, int njobs,
                        int nelem, cudaStream_t st, int zskip = 0);
// HODLR x panel for a diagonal HODLR operand (row scaling; level 0)
cudaError_t launch_hmat_diag(const TreeDev& T, const MMJob& job, int nelem, cudaStream_t st);
cudaError_t launch_gp(const TreeDev& T, const GPJob* jobs, int njobs,
                      const int* nodes, int nnodes, int nelem, int kcap,
                      cudaStream_t st, int rxcap = 0, int rycap = 0);
cudaError_t launch_rhs_combine(const double* f, long long fs, const double* a,
                               long long as, const double* b, long long bs,
                               double* out, long long os, int count, int len,
                               cudaStream_t st);

// census of the low-rank / panel kernels for the instrumented factor
// (k_census.cu; counter slots 150..155)
cudaError_t launch_census_hmat(const TreeDev& T, const MMJob* jobs, int njobs, int nelem,
                               unsigned long long* ctr, cudaStream_t st);
cudaError_t launch_census_gp(const TreeDev& T, const GPJob* jobs, int njobs, const int* nodes,
                             int nnodes, int nelem, unsigned long long* ctr, cudaStream_t st);
cudaError_t launch_rank_stats(const int* rD, const int* rE, const int* rF, long long sr, int mm,
                              const int* branches, int nbr, const int* depth, int nd,
                              unsigned* out, cudaStream_t st);
cudaError_t launch_census_leaflr(const TreeDev& T, RankRef rr, int node, int fside, int mu,
                                 int nelem, unsigned long long* ctr, cudaStream_t st);

// dense kernels (k_dense.cu)
cudaError_t launch_todense(const TreeDev& T, const HB* blk, int nblk,
                           const int* rowblk, const int* colblk, double* A,
                           int ld, cudaStream_t st);
// work: unused (reserved), pass null
cudaError_t lu_factor(double* A, int N, int* piv, int* info, double* work, cudaStream_t st);
cudaError_t lu_transpose(const double* A, int N, double* At, cudaStream_t st);
// perm (optional): row order after the interchanges, from lu_perm
cudaError_t lu_solve(const double* A, const double* At, int N, const int* piv, double* B,
                     int nrhs, cudaStream_t st, const int* perm = nullptr);
cudaError_t lu_perm(const int* piv, int N, int* perm, cudaStream_t st);
cudaError_t launch_rhs_in(const double* rhs, int N, int k, int n, double* P,
                          cudaStream_t st);
cudaError_t launch_u_out(const double* P, int N, int k, int n, double* u,
                         cudaStream_t st);
cudaError_t launch_residual(int m, int n, int k, const double* sub,
                            const double* diag, const double* sup,
                            const double* E, const double* F, const double* u,
                            const double* f, double* partial, int nparts,
                            cudaStream_t st);

// problem generators (k_gen.cu)
struct GenField {
  double c[8];
  long long p[8], q[8];
  double phi[8];
};
cudaError_t launch_gen_const(int m, int n, const double* v, double* D_sub, double* D_diag,
                             double* D_sup, double* E, double* F, cudaStream_t st);
cudaError_t launch_gen_varcoef(int n, const GenField& P, double* work, double* D_sub,
                               double* D_diag, double* D_sup, double* E, double* F,
                               cudaStream_t st);
cudaError_t launch_gen_uniform(const unsigned long long* state, long long N, int k,
                               double low, double high, double* out, cudaStream_t st);

}  // namespace acr
