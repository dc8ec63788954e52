/* acr_b200 -- C ABI of the B200-native ACR factor/solve hot path.
 *
 * Replaces the reference's only solve entry point,
 *   acrsolve.reduction.acr_solve(sys, tol, cutoff_blocks=1, leaf_size=32,
 *                                inversion_order="forward")
 *   (/root/reference/pkg/src/acrsolve/reduction.py:273-326, re-exported at
 *   __init__.py:20-22),
 * split into plan / factor / solve so that several right-hand sides reuse one
 * factorisation.  The reference has no FFI; its "plugin API" is that Python
 * function, which paper_1604_00617_b200.acr_solve mirrors on top of this ABI.
 *
 * All array arguments are fp64 DEVICE pointers owned by the caller (torch
 * tensors in the Python shim); the library borrows them for the call.  The
 * library owns its HODLR storage (stream-ordered cudaMallocAsync).  `stream`
 * is a cudaStream_t (NULL = legacy default stream).
 *
 * Streams and threads: acr_factor, acr_solve and acr_block_to_dense are
 * ordered on the stream they are given; acr_solve returns without waiting
 * for the GPU (u is complete when the stream reaches the call).  Successive
 * calls on one plan may name different streams: each call's stream first
 * waits for everything the plan queued before, and the plan's buffers are
 * recycled only on work ordered after their last use.  One plan must not be
 * used from two host threads at once; independent plans may run on any
 * number of threads concurrently (reference SPEC.md:213) -- the library has
 * no unsynchronised global state (error text of plan-less calls is
 * per thread).
 *
 * Status codes: 0 ok, 1 bad argument (Python: ValueError), 2 singular pivot
 * (SingularBlockError / LinAlgError), 3 CUDA error, 4 internal limit.
 */
#ifndef ACR_B200_H
#define ACR_B200_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct acr_plan acr_plan_t;

enum { ACR_OK = 0, ACR_EARG = 1, ACR_ESINGULAR = 2, ACR_ECUDA = 3,
       ACR_EINTERNAL = 4 };

/* m block rows of dimension n; H parameters as reference Tolerance
 * (hodlr.py:29-44: eps > 0, max_rank_cap >= 1 or 0 for none), leaf_size
 * (cluster.py:54-71), cutoff_blocks >= 1 (reduction.py:284-285). */
int acr_plan_create(int m, int n, int leaf_size, double eps, int max_rank_cap,
                    int cutoff_blocks, acr_plan_t** out);
void acr_plan_destroy(acr_plan_t* p);

/* Sharded plan: rank `rank` of `nranks` owns global block
 * rows [bnd0[rank], bnd0[rank+1]) (bnd0: nranks+1 host ints, bnd0[0] = 0,
 * bnd0[nranks] = m, even starts).  Per level a rank sends its first even
 * block's {Dinv, E, F} to rank-1 over NCCL; the top levels are gathered on
 * rank 0.  nccl_id: 128 bytes from acr_nccl_unique_id() on rank 0,
 * broadcast by the caller.  acr_factor / acr_solve then take the GLOBAL band,
 * rhs and u arrays (each rank writes its own rows of u). */
int acr_nccl_unique_id(void* out128);
int acr_plan_create_dist(int m, int n, int leaf_size, double eps, int max_rank_cap,
                         int cutoff_blocks, int rank, int nranks, const int* bnd0,
                         const void* nccl_id, acr_plan_t** out);
/* The same sharded factor + solve with `nranks` virtual ranks as threads of
 * this process on the current GPU (loopback transport; tests the sharded
 * path on one GPU).  factor_ms: max over ranks. */
int acr_loopback_solve(int nranks, const int* bnd0, int m, int n, int leaf_size,
                       double eps, int max_rank_cap, int cutoff_blocks,
                       const double* D_sub, const double* D_diag, const double* D_sup,
                       const double* E, const double* F, const double* rhs, int nrhs,
                       double* u, double* factor_ms);

/* option 1: keep every level's D blocks for export (tests); value 0/1
 * option 2: per-kernel-class instrumentation (CUDA events around every
 *           launch of a class + algorithmic FLOP/byte counters); 0/1
 * option 3: route every latency-bound (direct) recompression launch that
 *           fits through the CTA-pair cluster kernel (tests); 0/1 */
int acr_plan_set_option(acr_plan_t* p, int option, long long value);

/* Factor phase (reference lift_system reduction.py:156-166 + reduce_level
 * loop :294-302 + the cutoff LU oracles.py:20-31), no right-hand side.
 * Bands: D_sub (m,n-1), D_diag (m,n), D_sup (m,n-1), E (m-1,n), F (m-1,n),
 * row-major (problems.py:97-104).  inversion_order 0 forward, 1 reversed
 * (only changes which singular block is reported first). */
int acr_factor(acr_plan_t* p, const double* D_sub, const double* D_diag,
               const double* D_sup, const double* E, const double* F,
               int inversion_order, void* stream);

/* Solve phase: forward RHS sweep (reduction.py:204-216), cutoff solve
 * (:305-310), back-substitution (:235-256).  rhs and u are (m*n, nrhs)
 * row-major; u may alias rhs. */
int acr_solve(acr_plan_t* p, const double* rhs, int nrhs, double* u,
              void* stream);

/* Factor with the forward sweep of a right-hand side fused in (the
 * reference fuses its single RHS into the reduction, reduction.py:204-216):
 * each level's RHS update runs on a side stream right after the level's
 * record is complete, overlapping the next levels' factorisation.  rhs
 * (m*n, nrhs) row-major, read during the call's stream work; single-GPU
 * plans.  acr_solve_back then runs the cutoff solve and back-substitution
 * into u (m*n, nrhs), once per fused factorisation.  The side stream has the
 * device's lowest priority; the plan's other helper streams take the priority
 * of `stream`, so a caller that passes a high-priority stream keeps the sweep
 * out of the way of the factorisation's dependent chain. */
int acr_factor_rhs(acr_plan_t* p, const double* D_sub, const double* D_diag,
                   const double* D_sup, const double* E, const double* F,
                   int inversion_order, const double* rhs, int nrhs, void* stream);
int acr_solve_back(acr_plan_t* p, double* u, void* stream);

/* Report (SolveReport fields, reduction.py:124-153). */
int acr_levels(const acr_plan_t* p);
int acr_cutoff_blocks(const acr_plan_t* p);
int acr_tree_depths(const acr_plan_t* p);
/* per-level rank profile, level in [0, levels]; arrays of tree_depths */
int acr_rank_profile(const acr_plan_t* p, int level, int* max_by_depth,
                     double* mean_by_depth);
/* reference-accounted storage bytes (hodlr.py:157-163, reduction.py:80-110)
 * for an nrhs-column right-hand side */
long long acr_storage_bytes(const acr_plan_t* p, int nrhs);
long long acr_device_bytes(const acr_plan_t* p);
double acr_factor_ms(const acr_plan_t* p);
double acr_solve_ms(const acr_plan_t* p);
long long acr_kernel_launches(const acr_plan_t* p);
/* Instrumented factor only (option 2): per kernel class, launches, summed
 * CUDA-event time and algorithmic counters (SURVEY.md Appendix C formulas
 * over the run's actual shapes and ranks).  Classes: 0 recompression
 * (k_trunc), 1 leaf inverse, 2 dense leaf GEMM (DMMA), 3 HODLR x panel
 * (k_hmat: leaf_matmat + lr_apply), 4 level-0 exact diagonal leaf products,
 * 5 small panel products (k_gp), 6 low-rank leaf updates (k_leaflr:
 * leaf_add_uvT), 7 elementwise block ops (leaf add, negate, copy), 8 cutoff
 * LU.  counters[16]: [0] algorithmic FLOPs, [1] algorithmic bytes (class 4:
 * [0] holds its bytes).  Class 0 also: [2..7] block-path clock64 cycles per
 * phase (load, QR, core, Jacobi, select, output), [8] block-path full tasks,
 * [9] warp-path full tasks, [10]/[11] Jacobi sweeps (block / warp), [12..15]
 * warp-path cycles (load, QR, core, Jacobi).  cls 100: the raw 160 device
 * counters ([16..65] warp-path histogram, [66]/[67] warp-path select /
 * output cycles, [72..146] block-path histogram: counts, cycles, Jacobi
 * cycles by rank x rows bucket, [150..155] census of classes 3, 5, 6). */
int acr_kernel_stats(const acr_plan_t* p, int cls, long long* launches,
                     double* ms, unsigned long long* counters);
int acr_last_error(const acr_plan_t* p, char* buf, int len);
/* error of the calling thread's last plan-less call (acr_plan_create,
 * acr_residual, generators, kernel-level entry points) */
int acr_global_error(char* buf, int len);

/* Dense export of one block for tests: which 0 = D, 1 = E, 2 = F of the
 * level-`level` system (requires option 1 for level < levels), 3 = Dinv of
 * even block `block` from the level's elimination record.  out: n x n
 * row-major device buffer. */
int acr_block_to_dense(acr_plan_t* p, int level, int which, int block,
                       double* out, void* stream);

/* Raw storage of one block of the factorisation (same level / which / block
 * addressing as acr_block_to_dense), for the host HODLR objects of
 * paper_1604_00617_b200.hodlr (reference HodlrMatrix / LowRankFactor,
 * hodlr.py:47-173).  Layout: leaf n x bw (row i of
 * the leaf holding i, column j - lo), U and V nd x R x n (depth slot k, column
 * c, row i: node [lo,mid,hi) at depth k has off12 = U[k][:r12, lo:mid]^T
 * V[k][:r12, mid:hi] and off21 = U[k][:r21, mid:hi]^T V[k][:r21, lo:mid]),
 * ranks 2 x nnodes (off12, off21 of each node).  Device buffers; pass all
 * four as NULL to only receive R (column capacity) and the block count. */
int acr_block_export(acr_plan_t* p, int level, int which, int block, double* leaf,
                     double* U, double* V, int* ranks, int* R_out, int* count_out,
                     void* stream);

/* Stepwise API: the reference's lower-level surface (reduction.py:156-256),
 * used by its own tests (test_reduction.py:46-151), on device-resident levels
 * and elimination-record entries named by integer handles owned by the plan.
 *   acr_step_lift    lift_system (reduction.py:156-166) of the plan's (m, n,
 *                    leaf) system -> level handle (level 0)
 *   acr_step_reduce  reduce_level (reduction.py:173-232) of a level with the
 *                    given eps / cap; inversion_order: NULL or a permutation
 *                    of the even-block indices (only changes which singular
 *                    pivot is reported first) -> new level + record handles.
 *                    The input level is not modified.
 *   acr_step_rhs     the level's forward RHS update (reduction.py:204-216):
 *                    f (m_l n, k) -> f' (floor(m_l/2) n, k), row-major
 *   acr_step_backsub one back-substitution level (reduction.py:235-256): the
 *                    level's f and the odd blocks' u -> u of every block
 *   acr_step_info    block count / column capacity of which 0 D, 1 E, 2 F of a
 *                    level handle, 3 Dinv, 4 E, 5 F of a record handle; the
 *                    level index and its block count
 *   acr_step_export  raw storage of one block as acr_block_export
 *   acr_step_free    release a handle */
int acr_step_lift(acr_plan_t* p, const double* D_sub, const double* D_diag,
                  const double* D_sup, const double* E, const double* F, int* level_out,
                  void* stream);
int acr_step_reduce(acr_plan_t* p, int level, double eps, int max_rank_cap,
                    const int* inversion_order, int* level_out, int* record_out,
                    void* stream);
int acr_step_rhs(acr_plan_t* p, int record, const double* f, int nrhs, double* f_out,
                 void* stream);
int acr_step_backsub(acr_plan_t* p, int record, const double* f, const double* u_odd,
                     int nrhs, double* u, void* stream);
int acr_step_info(acr_plan_t* p, int handle, int which, int* count, int* R, int* level,
                  int* m_level);
int acr_step_export(acr_plan_t* p, int handle, int which, int block, double* leaf,
                    double* U, double* V, int* ranks, void* stream);
int acr_step_free(acr_plan_t* p, int handle);

/* ||A u - f||_2 per column and ||f||_2 per column straight from the bands
 * (oracles.py:34-49); u, f (m*n, k) row-major; out_r, out_f host arrays[k]. */
int acr_residual(int m, int n, int k, const double* D_sub, const double* D_diag,
                 const double* D_sup, const double* E, const double* F,
                 const double* u, const double* f, double* out_r,
                 double* out_f, void* stream);

/* Problem generators on the device (formulas of 8(d),
 * the reference's BlockTridiagSystem layout, problems.py:88-133).
 * acr_gen_constant: every band constant; values5 = {sub, diag, sup, E, F}
 *   (configs 1, 3, 4).
 * acr_gen_varcoef: configs 2 and 5, a = exp(sum_k c_k cos(2 pi (p_k x +
 *   q_k y) + phi_k)) on the (n+2)^2 nodes (work: (n+2)^2 doubles),
 *   harmonic-mean faces; parameters drawn on the host (numpy draw order).
 * acr_gen_uniform: N x k row-major Uniform[low, high) = the transposed
 *   (k, N) sample of numpy's default_rng continuing from the PCG64 state
 *   pcg_state4 = {state_hi, state_lo, inc_hi, inc_lo}; bitwise numpy's. */
int acr_gen_constant(int m, int n, const double* values5, double* D_sub, double* D_diag,
                     double* D_sup, double* E, double* F, void* stream);
int acr_gen_varcoef(int n, const double* c8, const long long* p8, const long long* q8,
                    const double* phi8, double* work, double* D_sub, double* D_diag,
                    double* D_sup, double* E, double* F, void* stream);
int acr_gen_uniform(const unsigned long long* pcg_state4, long long N, int k, double low,
                    double high, double* out, void* stream);

/* Kernel-level entry points (parity tests against hodlr.py:176-200 and
 * algebra.py:199-207 on captured operands).  U (m x R) and V (k x R) are
 * column-major; Uo (m x R), Vo (k x R) receive the truncated factor. */
int acr_truncate_factor(int m, int k, int R, const double* U, const double* V,
                        double eps, int max_rank_cap, double* Uo, double* Vo,
                        int* rank_out, void* stream);
/* Test hook: recompression path used by acr_truncate_factor (0 = one CTA per
 * task (default), 1 = warp-per-task kernel, 2 = CTA pair).  Per calling
 * thread. */
int acr_set_truncate_path(int path);
/* A: s x s row-major; X: inverse; *singular set to 1 on a zero pivot or a
 * non-finite result. */
int acr_leaf_inverse(int s, const double* A, double* X, int* singular,
                     void* stream);

#ifdef __cplusplus
}
#endif
#endif
