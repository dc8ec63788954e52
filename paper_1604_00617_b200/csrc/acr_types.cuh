// Device-side data layout of the ACR engine.
//
// One HODLR block of dimension n (reference hodlr.py:102-173) is stored as
//   leaf : double[n][bw]            row i of the leaf [lo,hi) containing i,
//                                   column j-lo at leaf[i*bw + (j-lo)]
//   U, V : double[nd][R][n]         per branch depth k, column-major n-row
//                                   panels; node nu at depth k keeps
//                                   off12 = U[k][:, lo:mid] V[k][:, mid:hi]^T
//                                   off21 = U[k][:, mid:hi] V[k][:, lo:mid]^T
//   rk   : int[nnodes][2]           rank of off12 (side 0) / off21 (side 1)
// Every factor is therefore addressed by *global row range*: the U rows of
// (nu, side) are [lo,mid) for side 0 and [mid,hi) for side 1, the V rows the
// other half.  Scratch panels use the same [slot][C][n] layout so a cross
// term of an ancestor restricts to a descendant by plain row indexing.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace acr {

struct HB {                 // one HODLR block
  double* leaf;
  double* U;
  double* V;
  int* rk;
  int R;                    // column capacity of U/V per depth slot
  int pad_;
};

struct TreeDev {            // node table (tree.py), breadth-first ids
  int n, bw, nd, nnodes, maxdepth, nleaves;
  const int* lo;
  const int* hi;
  const int* mid;           // split point (lo+hi)/2 for the bisection tree
  const int* depth;
  const int* parent;
  const int* c0;
  const int* c1;
  const int* isleaf;
  const int* anc;           // [nnodes][maxdepth+1]; anc[v*(maxdepth+1)+t]
  const int* posA;          // [nnodes][nnodes]: BFS position of branch b in subtree(mu) or -1
  const int* startA;        // [nnodes+1]: entries (mu, beta, side) of listA
  const int* listA;         // [totalA][3]
  const int* startB;        // [nnodes+1]
  const int* listB;         // [totalB][2]: (mu, leaf)
};

// A source of n-row panel columns for element g:
//   kind 0: strided panel   p + g*s + (slot*C + c)*n + row
//   kind 1: table panel     tab[g] + (slot*C + c)*n + row
//   kind 2: HB U            hb[g].U + (slot*hb[g].R + c)*n + row
//   kind 3: HB V
struct Src {
  int kind;
  int C;
  double* p;
  long long s;
  double* const* tab;
  const HB* hb;
};

__device__ __forceinline__ double* src_col(const Src& S, int n, int g, int slot,
                                           int c) {
  switch (S.kind) {
    case 0: return S.p + g * S.s + ((long long)slot * S.C + c) * n;
    case 1: return S.tab[g] + ((long long)slot * S.C + c) * n;
    case 2: { const HB& h = S.hb[g]; return h.U + ((long long)slot * h.R + c) * n; }
    default: { const HB& h = S.hb[g]; return h.V + ((long long)slot * h.R + c) * n; }
  }
}

// Where a rank comes from: hb ? hb[g].rk : arr + g*s, then [node*2+side].
struct RankRef {
  const HB* hb;
  const int* arr;
  long long s;
};

__device__ __forceinline__ const int* rank_base(const RankRef& r, int g) {
  return r.hb ? r.hb[g].rk : r.arr + g * r.s;
}

// Slot / rank selection rules for truncation operands.
enum { SEL_OWN = 0, SEL_ANC = 1, SEL_FIXED = 2, SEL_NODE = 3 };

struct TOp {
  Src U, V;
  RankRef rank;
  int sel;        // SEL_OWN: slot depth(beta), rank (beta, side)
                  // SEL_ANC: alpha = anc(beta, t): slot depth(alpha), rank [alpha][child of alpha holding beta]
                  // SEL_FIXED: slot depth(node), rank (node, fside) if (node, 1-fside) != 0 else 0
                  // SEL_NODE: slot depth(node), rank (node, fside) as stored (a snapshot that
                  //           already carries the SEL_FIXED rule)
  int t;
  int node;
  int fside;
  double scale;   // applied to U columns (exact sign flips only)
};

enum { TM_COMBINE = 0, TM_COMBINE_SWAP1 = 1, TM_TRUNCATE = 2 };

struct TruncArgs {
  TreeDev T;
  TOp a, b;
  int mode;
  const HB* out;            // output block per element
  const int* tasks;         // listA slice: (mu, beta, side) triples
  int ntasks;
  double eps;
  int cap;                  // max_rank_cap or 0
  int* overflow;            // atomicMax of ranks that did not fit
  double* gscr;             // global work areas for tasks that exceed smem
  long long gscr_stride;    // doubles per (g, task)
  int gscr_ntasks;          // tasks [0, gscr_ntasks) of the slice own a global area
  int smem_doubles;         // dynamic smem capacity in doubles
  unsigned long long* ctr;  // optional [flops, bytes] algorithmic counters
  int* wq;                  // warp path: dynamic work counter (null: static striding)
  int task_major;           // warp path item order: 0 element-major, 1 task-major
  int direct_tag;           // instrumentation: direct (one CTA per item) launch
  int warp_rmax;            // warp path takes tasks of at most this many columns
  long long warp_maxneed;   // ... and work areas of at most this many doubles
};

// HODLR x panel product over subtrees (reference algebra.py:52-83):
//   Y[rows(mu)] = alpha * H_mu X[rows(mu)]     (trans: H_mu^T X)
// for every subtree root mu in [mu0, mu1); slot = depth(parent(mu)) (0 at root);
// column count = fixed if >= 0 else rank(parent(mu), childidx(mu) ^ swap).
struct MMJob {
  const HB* H;
  Src X, Y;
  int trans;
  RankRef cols;
  int cols_fixed;
  int swap;
  double alpha;
  int mu0, mu1;
  double* tbuf;             // [g][entryA - startA[mu0]][RT][CT]
  int RT, CT;
  int nA;                   // startA[mu1] - startA[mu0]
  int nB;                   // startB[mu1] - startB[mu0]
};

// Z[rows hw of nu] = alpha * W[rows hw] (X[rows hx]^T Y[rows hx])
// X/W columns: rank(nu, sx) from rx; Y columns: rank(nu, sy) from ry.
// If either rank is zero nothing is written and out rank (if any) is 0.
struct GPJob {
  Src X, Y, W, Z;
  int hx, hw;
  RankRef rx, ry;
  int sx, sy;
  int* orank;
  long long ors;
  int oside;
  double alpha;
};

// 8-byte asynchronous global -> shared copy; valid = false zero-fills
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src),
               "r"(valid ? 8 : 0));
}
// 16-byte asynchronous global -> shared copy (both addresses 16-byte aligned)
__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
}

}  // namespace acr
