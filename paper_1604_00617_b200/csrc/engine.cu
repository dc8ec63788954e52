// ACR engine: plan, level loop, batched invert / multiply / add schedules,
// solve sweep, report, and the C ABI of include/acr_b200.h.
//
// Every HODLR operation of the reference (algebra.py) is executed for ALL
// blocks of a level at once: the host walks the reference's recursion
// structure once (it is identical for every block because one cluster tree
// serves all blocks, reduction.py:159) and launches one batched kernel per
// step; data-dependent branches (zero ranks, passthroughs, rank-1 shortcuts)
// are decided per block on the device from device-resident ranks.  The
// truncation schedule is the reference's.
#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <string>
#include <vector>

#include "acr_launch.h"
#include "acr_types.cuh"
#include "dist.h"
#include "../../include/acr_b200.h"

namespace acr {

struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& s) : std::runtime_error(s) {}
};
struct ArgError : std::runtime_error {
  explicit ArgError(const std::string& s) : std::runtime_error(s) {}
};
struct SingularError : std::runtime_error {
  explicit SingularError(const std::string& s) : std::runtime_error(s) {}
};
struct InternalError : std::runtime_error {
  explicit InternalError(const std::string& s) : std::runtime_error(s) {}
};

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess)                                                 \
      throw acr::CudaError(std::string(cudaGetErrorString(e_)) + " at " +       \
                      __FILE__ + ":" + std::to_string(__LINE__));          \
  } while (0)

// ---------------------------------------------------------------------------
// stream-ordered device memory
// ---------------------------------------------------------------------------
// bytes held through Dev (all plans of the process; plans may run on several
// host threads at once)
static std::atomic<long long> g_live{0}, g_peak{0};
static void note_alloc(long long b) {
  const long long now = g_live.fetch_add(b) + b;
  long long pk = g_peak.load();
  while (now > pk && !g_peak.compare_exchange_weak(pk, now)) {
  }
}

// Size-class caching allocator.  A factor requests the same sizes in the
// same order every time, so after the first factor every request is served
// from the cache (no new device mappings inside a timed factor).  Free blocks
// are keyed by the stream they were last used on and only handed to requests
// on that stream, so reuse is stream-ordered.  Blocks go back to the driver
// (after a device synchronisation: they may have been used on any stream)
// when an allocation fails or the last plan dies.
struct DevCache {
  std::mutex mu;
  std::multimap<std::pair<size_t, cudaStream_t>, void*> free_;
  std::vector<void*> all;
  std::atomic<int> plans{0};
  static size_t cls(size_t b) {
    if (b <= 4096) return (b + 255) & ~size_t(255);
    int lg = 63 - __builtin_clzll(b);
    size_t step = size_t(1) << (lg > 3 ? lg - 3 : 0);   // 8 classes per octave
    return (b + step - 1) & ~(step - 1);
  }
  void* get(size_t bytes, size_t* cap, cudaStream_t s) {
    size_t c = cls(bytes);
    {
      std::lock_guard<std::mutex> g(mu);
      auto it = free_.find({c, s});
      if (it != free_.end()) {
        void* p = it->second;
        free_.erase(it);
        *cap = c;
        return p;
      }
    }
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, c, s);
    if (e != cudaSuccess) {
      cudaGetLastError();
      trim(s);                       // give cached blocks back, retry once
      CK(cudaMallocAsync(&p, c, s));
    }
    std::lock_guard<std::mutex> g(mu);
    all.push_back(p);
    *cap = c;
    return p;
  }
  void put(void* p, size_t cap, cudaStream_t s) {
    std::lock_guard<std::mutex> g(mu);
    free_.emplace(std::make_pair(cap, s), p);
  }
  void trim(cudaStream_t s) {
    std::lock_guard<std::mutex> g(mu);
    if (free_.empty()) return;
    // a cached block's last use may be pending on another stream
    cudaDeviceSynchronize();
    for (auto& kv : free_) {
      cudaFreeAsync(kv.second, s);
      all.erase(std::find(all.begin(), all.end(), kv.second));
    }
    free_.clear();
  }
};
static DevCache g_cache;

struct Dev {
  void* p = nullptr;
  size_t n = 0;
  size_t cap = 0;
  cudaStream_t st = 0;
  Dev() {}
  Dev(size_t bytes, cudaStream_t s) { alloc(bytes, s); }
  void alloc(size_t bytes, cudaStream_t s) {
    release();
    st = s;
    n = bytes;
    if (bytes) {
      p = g_cache.get(bytes, &cap, s);
      note_alloc((long long)cap);
    }
  }
  void release() {
    if (p) {
      g_cache.put(p, cap, st);
      g_live -= (long long)cap;
    }
    p = nullptr;
    n = 0;
    cap = 0;
  }
  ~Dev() { release(); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  Dev(Dev&& o) noexcept : p(o.p), n(o.n), cap(o.cap), st(o.st) {
    o.p = nullptr;
    o.n = 0;
    o.cap = 0;
  }
  Dev& operator=(Dev&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      cap = o.cap;
      st = o.st;
      o.p = nullptr;
      o.n = 0;
      o.cap = 0;
    }
    return *this;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

// ---------------------------------------------------------------------------
// node table (mirrors paper_1604_00617_b200/tree.py, reference cluster.py)
// ---------------------------------------------------------------------------
struct HostTree {
  int n = 0, leaf = 0, bw = 0, nd = 0, nnodes = 0, maxdepth = 0, nleaves = 0;
  std::vector<int> lo, hi, mid, depth, parent, c0, c1, isleaf, anc, posA,
      startA, listA, startB, listB, branches, iota;

  bool in_subtree(int b, int mu) const {
    int k = depth[b] - depth[mu];
    return k >= 0 && anc[b * (maxdepth + 1) + k] == mu;
  }

  void build(int n_, int leaf_) {
    n = n_;
    leaf = leaf_;
    lo = {0};
    hi = {n};
    depth = {0};
    parent = {-1};
    for (size_t i = 0; i < lo.size(); ++i) {
      int a = lo[i], b = hi[i];
      if (b - a <= leaf) {
        c0.push_back(-1);
        c1.push_back(-1);
      } else {
        int m = (a + b) / 2;
        int c = (int)lo.size();
        lo.push_back(a); hi.push_back(m);
        lo.push_back(m); hi.push_back(b);
        depth.push_back(depth[i] + 1); depth.push_back(depth[i] + 1);
        parent.push_back((int)i); parent.push_back((int)i);
        c0.push_back(c);
        c1.push_back(c + 1);
      }
    }
    nnodes = (int)lo.size();
    mid.resize(nnodes);
    isleaf.resize(nnodes);
    bw = 0;
    nd = 0;
    maxdepth = 0;
    nleaves = 0;
    for (int v = 0; v < nnodes; ++v) {
      mid[v] = (lo[v] + hi[v]) / 2;
      isleaf[v] = c0[v] < 0;
      maxdepth = std::max(maxdepth, depth[v]);
      if (isleaf[v]) {
        bw = std::max(bw, hi[v] - lo[v]);
        ++nleaves;
      } else {
        nd = std::max(nd, depth[v] + 1);
        branches.push_back(v);
      }
      iota.push_back(v);
    }
    bw = (bw + 1) & ~1;   // leaf panel width even: 16-byte vector access to every block
    const int D1 = maxdepth + 1;
    anc.assign((size_t)nnodes * D1, -1);
    for (int v = 0; v < nnodes; ++v) {
      int a = v;
      for (int t = 0; t <= depth[v]; ++t) {
        anc[(size_t)v * D1 + t] = a;
        a = parent[a];
      }
    }
    posA.assign((size_t)nnodes * nnodes, -1);
    startA.assign(nnodes + 1, 0);
    startB.assign(nnodes + 1, 0);
    listA.clear();
    listB.clear();
    for (int mu = 0; mu < nnodes; ++mu) {
      startA[mu] = (int)listA.size() / 3;
      int cnt = 0;
      for (int b = 0; b < nnodes; ++b) {
        if (isleaf[b] || !in_subtree(b, mu)) continue;
        posA[(size_t)mu * nnodes + b] = cnt++;
        for (int s = 0; s < 2; ++s) {
          listA.push_back(mu);
          listA.push_back(b);
          listA.push_back(s);
        }
      }
      startB[mu] = (int)listB.size() / 2;
      std::vector<int> lv;
      for (int b = 0; b < nnodes; ++b)
        if (isleaf[b] && in_subtree(b, mu)) lv.push_back(b);
      std::sort(lv.begin(), lv.end(), [&](int x, int y) { return lo[x] < lo[y]; });
      for (int b : lv) {
        listB.push_back(mu);
        listB.push_back(b);
      }
    }
    startA[nnodes] = (int)listA.size() / 3;
    startB[nnodes] = (int)listB.size() / 2;
  }

  int nleaves_under(int mu) const { return startB[mu + 1] - startB[mu]; }
  int nA(int mu0, int mu1) const { return startA[mu1] - startA[mu0]; }
};

struct DeviceTree {
  Dev buf;
  TreeDev T;
  const int* d_listA = nullptr;
  const int* d_branches = nullptr;
  const int* d_iota = nullptr;

  void upload(const HostTree& h, cudaStream_t st) {
    std::vector<const std::vector<int>*> parts = {
        &h.lo, &h.hi, &h.mid, &h.depth, &h.parent, &h.c0, &h.c1, &h.isleaf,
        &h.anc, &h.posA, &h.startA, &h.listA, &h.startB, &h.listB,
        &h.branches, &h.iota};
    size_t tot = 0;
    for (auto* p : parts) tot += p->size() + 1;
    std::vector<int> host(tot, 0);
    std::vector<size_t> off;
    size_t o = 0;
    for (auto* p : parts) {
      off.push_back(o);
      std::copy(p->begin(), p->end(), host.begin() + o);
      o += p->size() + 1;
    }
    buf.alloc(tot * sizeof(int), st);
    CK(cudaMemcpyAsync(buf.p, host.data(), tot * sizeof(int),
                       cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    const int* b = buf.as<int>();
    T.n = h.n;
    T.bw = h.bw;
    T.nd = h.nd;
    T.nnodes = h.nnodes;
    T.maxdepth = h.maxdepth;
    T.nleaves = h.nleaves;
    T.lo = b + off[0];
    T.hi = b + off[1];
    T.mid = b + off[2];
    T.depth = b + off[3];
    T.parent = b + off[4];
    T.c0 = b + off[5];
    T.c1 = b + off[6];
    T.isleaf = b + off[7];
    T.anc = b + off[8];
    T.posA = b + off[9];
    T.startA = b + off[10];
    T.listA = b + off[11];
    T.startB = b + off[12];
    T.listB = b + off[13];
    d_listA = T.listA;
    d_branches = b + off[14];
    d_iota = b + off[15];
  }
};

// ---------------------------------------------------------------------------
// a contiguous set of HODLR blocks with one column capacity
// ---------------------------------------------------------------------------
struct Batch {
  int cnt = 0, R = 0;
  Dev leaf, U, V, rk;
  long long sl = 0, sf = 0, sr = 0;
  void alloc(const HostTree& t, int cnt_, int R_, cudaStream_t st) {
    cnt = cnt_;
    R = std::max(R_, 1);
    sl = (long long)t.n * t.bw;
    sf = (long long)std::max(t.nd, 1) * R * t.n;
    sr = 2LL * t.nnodes;
    leaf.alloc(sizeof(double) * sl * std::max(cnt, 1), st);
    U.alloc(sizeof(double) * sf * std::max(cnt, 1), st);
    V.alloc(sizeof(double) * sf * std::max(cnt, 1), st);
    rk.alloc(sizeof(int) * sr * std::max(cnt, 1), st);
    CK(cudaMemsetAsync(rk.p, 0, rk.n, st));
  }
  HB base() const {
    HB h;
    h.leaf = leaf.as<double>();
    h.U = U.as<double>();
    h.V = V.as<double>();
    h.rk = rk.as<int>();
    h.R = R;
    h.pad_ = 0;
    return h;
  }
  long long bytes() const {
    return (long long)(leaf.n + U.n + V.n + rk.n);
  }
};

struct Seg {
  const Batch* b;
  int first, step, count;
};

// A level is a window [first, first+m) of a global level of mg blocks (one
// GPU: first = 0, m = mg).  E of global block 0 and F of global block mg-1
// are unused (rank 0).
struct Level {
  int m = 0, first = 0, mg = 0;
  int R = 1;
  int lvl = 0;                      // reduction level index (0 = lifted system)
  Batch D, E, F;
};

struct Record {
  int m = 0, first = 0, mg = 0;
  bool right = false;               // a right neighbour (other rank) exists
  bool diagEF = false;              // E, F are the lifted level's diagonals (rank 0, diagonal leaves)
  Batch Dinv, E, F;
  std::vector<int> hDinv, hE, hF;   // host ranks (storage accounting)
};

struct Profile {
  std::vector<int> mx;
  std::vector<double> mean;
};

static Src s_pan(double* p, long long s, int C) {
  Src x;
  memset(&x, 0, sizeof(x));
  x.kind = 0;
  x.p = p;
  x.s = s;
  x.C = C;
  return x;
}
static Src s_hbU(const HB* t) {
  Src x;
  memset(&x, 0, sizeof(x));
  x.kind = 2;
  x.hb = t;
  return x;
}
static Src s_hbV(const HB* t) {
  Src x = s_hbU(t);
  x.kind = 3;
  return x;
}
static RankRef r_hb(const HB* t) {
  RankRef r;
  r.hb = t;
  r.arr = nullptr;
  r.s = 0;
  return r;
}
static RankRef r_arr(const int* a, long long s) {
  RankRef r;
  r.hb = nullptr;
  r.arr = a;
  r.s = s;
  return r;
}
static TOp op_own(Src U, Src V, RankRef r, double sc = 1.0) {
  TOp o;
  memset(&o, 0, sizeof(o));
  o.U = U;
  o.V = V;
  o.rank = r;
  o.sel = SEL_OWN;
  o.scale = sc;
  return o;
}

static bool dbg() {
  static int v = -1;
  if (v < 0) v = getenv("ACR_DEBUG") ? 1 : 0;
  return v == 1;
}

static const long long SMEM_MAX_BYTES = 196 * 1024;
static const long long GSCR_BUDGET_BYTES = 2LL << 30;

// ---------------------------------------------------------------------------
// the plan
// ---------------------------------------------------------------------------
struct Plan {
  int m, n, leaf, cutoff, cap;
  double eps;
  bool keep_levels = false;
  bool no_side = false;       // option 4: every launch on the plan's stream
  bool force_pair = false;    // option 3: CTA-pair recompression for every direct launch that fits
  int warp_small = 0;         // option 6: launches of at most this many items use the warp kernel
  int direct_max = -1;        // option 5: largest launch (items) run one CTA per task; -1 default
  int warp_sched = 2;         // option 8: warp-path items 0 static, 1 dynamic, 2 dynamic task-major
  int warp_rmax = 16;         // option 9: widest core (columns) the warp path takes
  long long warp_maxneed = 0; // option 10: largest warp-path work area (doubles); 0 = the pool
  HostTree ht;
  DeviceTree dt;
  cudaStream_t st = 0;
  std::vector<Record> recs;
  std::vector<Level> kept;
  Level last;
  Dev lu, piv, info;
  Dev lut;                    // LU factors transposed for the cutoff solve (per factor)
  bool lut_ok = false;
  int Nc = 0;
  std::vector<Profile> prof;
  std::vector<std::vector<int>> lastR;   // host ranks of the final level D, E, F
  double fms = 0, sms = 0;
  bool sms_pending = false;
  long long launches = 0;
  bool factored = false;
  long long reserved = 0;
  std::string err;
  // sharding: level-0 block boundaries of every rank
  Transport* tp = nullptr;
  bool own_tp = false;
  std::vector<int> bnd0;
  int first0 = 0, mloc0 = 0;  // this rank's level-0 window
  // per-kernel-class instrumentation (option 2)
  bool prof_on = false;
  // classes: 0 recompression, 1 leaf inverse, 2 leaf GEMM (DMMA), 3 HODLR x
  // panel, 4 level-0 diagonal leaf products, 5 small panel products (k_gp),
  // 6 low-rank leaf updates (k_leaflr), 7 elementwise block ops (leaf add,
  // negate, copy, zero), 8 cutoff LU
  enum { NCLS = 10 };
  std::vector<cudaEvent_t> evpool;
  size_t evused = 0;
  std::vector<std::pair<int, size_t>> evmarks;   // (class, index of start event)
  double kms[NCLS] = {0};
  long long kcnt[NCLS] = {0};
  unsigned long long kctr[256] = {0};
  double hflops[NCLS] = {0};   // host-side FLOP counts (leaf classes), per factor
  double hbytes[NCLS] = {0};   // host-side algorithmic byte counts
  Dev dctr;
  // scratch pool
  std::vector<Dev> scr;
  Dev ovf, sing;
  // Per-level flags and rank tables reach the host through mapped pinned
  // memory written by a copy kernel, not through the copy engines: an
  // application's bulk transfers on other streams (the next step's bands, the
  // previous step's solution) would otherwise queue these small reads behind
  // hundreds of MB and stall the factorisation at every level.
  int* hmap = nullptr;       // host view
  int* hmap_d = nullptr;     // device alias
  size_t hmap_cap = 0, hmap_used = 0;
  struct Pend {
    std::vector<int>* out;
    size_t off, n;
  };
  std::vector<Pend> pend;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t sev0 = nullptr, sev1 = nullptr;   // solve timing (read lazily)

  Plan(int m_, int n_, int leaf_, double eps_, int cap_, int cutoff_)
      : m(m_), n(n_), leaf(leaf_), cutoff(cutoff_), cap(cap_), eps(eps_) {
    ht.build(n, leaf);
    scr.resize(72);
  }
  ~Plan() {
    if (hmap) cudaFreeHost(hmap);
    if (evsw) cudaEventDestroy(evsw);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (sev0) cudaEventDestroy(sev0);
    if (sev1) cudaEventDestroy(sev1);
    for (auto e : evpool) cudaEventDestroy(e);
    drop_chain_streams();
    if (stf) {
      cudaStreamSynchronize(stf);
      cudaStreamDestroy(stf);
      cudaEventDestroy(evfl);
      cudaEventDestroy(evfj);
    }
    if (stc) {
      cudaStreamSynchronize(stc);
      cudaStreamDestroy(stc);
      cudaEventDestroy(evcf);
      cudaEventDestroy(evcj);
    }
    if (own_tp) delete tp;
  }

  // streams of the recompression queue kernels (run beside the warp kernel),
  // one set per launching stream (main / side)
  struct QStreams {
    cudaStream_t q0 = nullptr, q1 = nullptr;
    cudaEvent_t ef = nullptr, ej0 = nullptr, ej1 = nullptr;
  };
  QStreams qstr[3 + 8];
  bool no_qstreams = getenv("ACR_NO_QSTREAMS") != nullptr;   // development aid
  bool no_fuse_leaf = getenv("ACR_NO_FUSE_LEAF") != nullptr; // development aid

  // The factor's helper streams carry parts of its dependent chain: they take
  // the priority of the caller's stream, the fused forward right-hand-side
  // sweep runs on a stream of the lowest priority.  A caller that passes a
  // high-priority stream thus gets a sweep that only fills the SMs the chain
  // leaves idle; with a default stream everything is at one priority, as
  // before.  (ACR_NO_PRIO=1 creates every stream at the default.)
  int chain_prio = 0;   // priority of the caller's stream when the helper streams were made
  void make_stream(cudaStream_t* s, bool chain) {
    static const bool off = getenv("ACR_NO_PRIO") != nullptr;
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(s, cudaStreamNonBlocking, (off || !chain) ? lo : chain_prio));
  }
  // the helper streams that carry parts of the chain (side, deferred, per-depth
  // and queue streams) are dropped when the caller's stream changes priority;
  // they are made again, at the new priority, on first use
  void drop_chain_streams() {
    for (int i = 0; i < NDS; ++i)
      if (dstr[i]) {
        cudaStreamSynchronize(dstr[i]);
        cudaStreamDestroy(dstr[i]);
        cudaEventDestroy(evds[i]);
        dstr[i] = nullptr;
      }
    if (st3) {
      cudaStreamSynchronize(st3);
      cudaStreamDestroy(st3);
      for (auto& e : evdef) cudaEventDestroy(e);
      st3 = nullptr;
    }
    if (st2) {
      cudaStreamSynchronize(st2);
      cudaStreamDestroy(st2);
      cudaEventDestroy(evf);
      cudaEventDestroy(evj);
      st2 = nullptr;
    }
    for (auto& qs : qstr)
      if (qs.q0) {
        cudaStreamSynchronize(qs.q0);
        cudaStreamSynchronize(qs.q1);
        cudaStreamDestroy(qs.q0);
        cudaStreamDestroy(qs.q1);
        cudaEventDestroy(qs.ef);
        cudaEventDestroy(qs.ej0);
        cudaEventDestroy(qs.ej1);
        qs.q0 = qs.q1 = nullptr;
      }
  }
  // second stream for independent launches at latency-bound levels (disabled
  // while instrumenting so per-class event timings stay on one stream)
  cudaStream_t st2 = nullptr;
  cudaEvent_t evf = nullptr, evj = nullptr;
  cudaStream_t side() {
    if (prof_on || no_side) return st;
    if (!st2) {
      make_stream(&st2, true);
      CK(cudaEventCreateWithFlags(&evf, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&evj, cudaEventDisableTiming));
    }
    return st2;
  }
  // streams of multiply's per-depth recompression chains
  static constexpr int NDS = 8;
  cudaStream_t dstr[NDS] = {};
  cudaEvent_t evds[NDS] = {};
  bool no_dsplit = getenv("ACR_NO_DSPLIT") != nullptr;   // development aid
  cudaStream_t depth_stream(int i) {
    if (!dstr[i]) {
      make_stream(&dstr[i], true);
      CK(cudaEventCreateWithFlags(&evds[i], cudaEventDisableTiming));
    }
    return dstr[i];
  }

  // third stream: recompressions of a Schur complement's upper tree levels,
  // deferred until the inversion reaches the nodes they update
  cudaStream_t st3 = nullptr;
  cudaEvent_t evdef[32] = {};
  bool no_defer = getenv("ACR_NO_DEFER") != nullptr;   // development aid
  cudaStream_t deferred() {
    if (prof_on || no_side || no_defer) return st;
    if (!st3) {
      make_stream(&st3, true);
      for (auto& e : evdef) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    return st3;
  }
  void fork(cudaStream_t s) {
    if (s == st) return;
    CK(cudaEventRecord(evf, st));
    CK(cudaStreamWaitEvent(s, evf, 0));
  }
  void join(cudaStream_t s) {
    if (s == st) return;
    CK(cudaEventRecord(evj, s));
    CK(cudaStreamWaitEvent(st, evj, 0));
  }

  // Every ABI call names its stream.  When it differs from the previous
  // call's, the new stream waits for everything the plan queued so far, and
  // every buffer the plan holds is re-tagged to the new stream so that, when
  // released, the caching allocator only hands it to work ordered after its
  // last use (solve is asynchronous on its stream).
  bool st_set = false;
  cudaEvent_t evsw = nullptr;
  void retag(Dev& d, cudaStream_t s) { d.st = s; }
  void retag(Batch& b, cudaStream_t s) {
    retag(b.leaf, s); retag(b.U, s); retag(b.V, s); retag(b.rk, s);
  }
  // (factor only: a solve on a stream of another priority -- say a
  // back-substitution pushed behind the next factorisation -- keeps them)
  void match_priority(cudaStream_t s) {
    int pr = 0;
    CK(cudaStreamGetPriority(s, &pr));
    if (pr != chain_prio) {
      drop_chain_streams();
      chain_prio = pr;
    }
  }
  void use_stream(cudaStream_t s) {
    if (st_set && s == st) return;
    if (st_set) {
      if (!evsw) CK(cudaEventCreateWithFlags(&evsw, cudaEventDisableTiming));
      CK(cudaEventRecord(evsw, st));
      CK(cudaStreamWaitEvent(s, evsw, 0));
    }
    {
      for (auto& r : recs) { retag(r.Dinv, s); retag(r.E, s); retag(r.F, s); }
      for (auto& l : kept) { retag(l.D, s); retag(l.E, s); retag(l.F, s); }
      retag(last.D, s); retag(last.E, s); retag(last.F, s);
      for (Dev* d : {&lu, &piv, &info, &lut, &ovf, &sing, &dctr, &dt.buf}) retag(*d, s);
      for (auto& d : scr) retag(d, s);
      for (auto& d : ffs) retag(d, s);
    }
    st = s;
    st_set = true;
  }

  // comm stream for halo transfers that overlap compute (sharded plans)
  cudaStream_t stc = nullptr;
  cudaEvent_t evcf = nullptr, evcj = nullptr;
  bool ef_pending = false;
  int nb_left = -1, nb_right = -1;   // active neighbours at the current level
  cudaStream_t comm_stream() {
    if (!stc) {
      CK(cudaStreamCreateWithFlags(&stc, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&evcf, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&evcj, cudaEventDisableTiming));
    }
    return stc;
  }
  void comm_fork() {
    cudaStream_t c = comm_stream();
    CK(cudaEventRecord(evcf, st));
    CK(cudaStreamWaitEvent(c, evcf, 0));
  }
  void comm_join() {
    CK(cudaEventRecord(evcj, stc));
    CK(cudaStreamWaitEvent(st, evcj, 0));
  }

  int nranks() const { return tp ? tp->size() : 1; }
  int me() const { return tp ? tp->rank() : 0; }

  // ---- sharding schedule; host-only and identical on
  //      every rank (mirrored by paper_1604_00617_b200/dist.py schedule) ----
  // wins[l]: block boundaries of every rank at level l after that level's
  // merges (b[P] = global block count; a retired rank has an empty window).
  // Before reducing level l the active windows must each start even, hold
  // >= 2 blocks and (except the last) have even length; while they do not,
  // active ranks merge pairwise (the 2i+1-th active rank hands its window
  // to the 2i-th), so the upper levels consolidate onto P/2, P/4, ... GPUs
  // as the block count halves.  At the cutoff everything merges onto rank 0.
  struct MergeStep {
    int lvl;
    std::vector<int> before, after;
  };
  std::vector<std::vector<int>> wins;
  std::vector<MergeStep> msteps;
  int Lsched = 0;

  static std::vector<int> active_of(const std::vector<int>& b) {
    std::vector<int> a;
    for (size_t r = 0; r + 1 < b.size(); ++r)
      if (b[r + 1] > b[r]) a.push_back((int)r);
    return a;
  }
  static bool win_ok(const std::vector<int>& b) {
    std::vector<int> a = active_of(b);
    for (size_t i = 0; i < a.size(); ++i) {
      const int r = a[i], c = b[r + 1] - b[r];
      if ((b[r] & 1) || c < 2) return false;
      if (i + 1 < a.size() && (c & 1)) return false;
    }
    return true;
  }
  static std::vector<int> merge_pairs(const std::vector<int>& b) {
    std::vector<int> a = active_of(b), nb = b;
    for (size_t i = 0; 2 * i + 1 < a.size(); ++i) {
      const int dst = a[2 * i], src = a[2 * i + 1];
      for (int x = dst + 1; x <= src; ++x) nb[x] = b[src + 1];
    }
    return nb;
  }
  void schedule() {
    wins.clear();
    msteps.clear();
    const int P = nranks();
    std::vector<int> cur = P > 1 ? bnd0 : std::vector<int>{0, m};
    int mg = m, l = 0;
    while (true) {
      const bool last = mg <= cutoff;
      while (active_of(cur).size() > 1 && (last || !win_ok(cur))) {
        std::vector<int> nb = merge_pairs(cur);
        msteps.push_back({l, cur, nb});
        cur = nb;
      }
      wins.push_back(cur);
      if (last) break;
      mg /= 2;
      ++l;
      for (int r = 0; r < P; ++r) cur[r] >>= 1;
      cur[P] = mg;
    }
    Lsched = l;
  }
  int nactive(int l) const { return (int)active_of(wins[l]).size(); }
  bool active_at(int l) const { return wins[l][me() + 1] > wins[l][me()]; }
  // previous / next active rank at level l (-1 if none)
  int left_nb(int l) const {
    for (int r = me() - 1; r >= 0; --r)
      if (wins[l][r + 1] > wins[l][r]) return r;
    return -1;
  }
  int right_nb(int l) const {
    for (int r = me() + 1; r + 1 < (int)wins[l].size(); ++r)
      if (wins[l][r + 1] > wins[l][r]) return r;
    return -1;
  }
  // active rank whose window (boundaries b) holds block position pos
  static int owner(const std::vector<int>& b, int pos) {
    for (size_t r = 0; r + 1 < b.size(); ++r)
      if (b[r] <= pos && pos < b[r + 1]) return (int)r;
    return -1;
  }

  void block_msgs(std::vector<Msg>& msgs, const Batch& b, int e, int peer, bool send) {
    msgs.push_back({peer, b.leaf.as<double>() + e * b.sl, sizeof(double) * b.sl, send});
    msgs.push_back({peer, b.U.as<double>() + e * b.sf, sizeof(double) * b.sf, send});
    msgs.push_back({peer, b.V.as<double>() + e * b.sf, sizeof(double) * b.sf, send});
    msgs.push_back({peer, b.rk.as<int>() + e * b.sr, sizeof(int) * b.sr, send});
  }
  void range_msgs(std::vector<Msg>& msgs, const Batch& b, int e0, int cnt, int peer,
                  bool send) {
    if (cnt <= 0) return;
    msgs.push_back({peer, b.leaf.as<double>() + e0 * b.sl, sizeof(double) * b.sl * cnt, send});
    msgs.push_back({peer, b.U.as<double>() + e0 * b.sf, sizeof(double) * b.sf * cnt, send});
    msgs.push_back({peer, b.V.as<double>() + e0 * b.sf, sizeof(double) * b.sf * cnt, send});
    msgs.push_back({peer, b.rk.as<int>() + e0 * b.sr, sizeof(int) * b.sr * cnt, send});
  }

  cudaEvent_t next_event() {
    if (evused == evpool.size()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      evpool.push_back(e);
    }
    return evpool[evused++];
  }
  // bracket a launch of class `cls` with events when profiling
  void kbegin(int cls) {
    if (!prof_on) return;
    evmarks.push_back({cls, evused});
    CK(cudaEventRecord(next_event(), st));
  }
  void kend() {
    if (!prof_on) return;
    CK(cudaEventRecord(next_event(), st));
  }
  unsigned long long* ctrp() { return prof_on ? dctr.as<unsigned long long>() : nullptr; }
  // instrumented launch wrappers: class events around the kernel, census
  // kernel (algorithmic FLOP / bytes from the device ranks) after it
  void hmat(const MMJob* J, int nj, int G, cudaStream_t s, bool zskip = false) {
    kbegin(3);
    CK(launch_hmat(dt.T, J, nj, G, s, zskip ? 1 : 0));
    kend();
    launches += 2;
    if (prof_on) CK(launch_census_hmat(dt.T, J, nj, G, ctrp(), s));
  }
  void gp(const GPJob* J, int nj, const int* nodes, int nnodes, int G, int rxcap, int rycap,
          cudaStream_t s) {
    kbegin(5);
    CK(launch_gp(dt.T, J, nj, nodes, nnodes, G, rxcap * rycap, s, rxcap, rycap));
    kend();
    ++launches;
    if (prof_on) CK(launch_census_gp(dt.T, J, nj, nodes, nnodes, G, ctrp(), s));
  }
  void leaflr(const HB* H, int G, int mu, Src U, Src V, RankRef rr, int node, int fside,
              cudaStream_t s) {
    kbegin(6);
    CK(launch_leaflr_n(dt.T, H, G, mu, ht.nleaves_under(mu), U, V, rr, node, fside, s));
    kend();
    ++launches;
    if (prof_on) CK(launch_census_leaflr(dt.T, rr, node, fside, mu, G, ctrp(), s));
  }
  // elementwise block ops: bytes = blocks x words touched (leaf panel n x bw
  // plus factor panels where the op reads / writes them)
  void elem_bytes(int G, double words_per_block) {
    if (prof_on) hbytes[7] += 8.0 * G * words_per_block;
  }

  void prof_reset() {
    evused = 0;
    evmarks.clear();
    for (int i = 0; i < NCLS; ++i) { kms[i] = 0; kcnt[i] = 0; hflops[i] = 0; hbytes[i] = 0; }
    for (auto& c : kctr) c = 0;
    if (prof_on) {
      if (!dctr.p) dctr.alloc(256 * sizeof(unsigned long long), st);
      CK(cudaMemsetAsync(dctr.p, 0, 256 * sizeof(unsigned long long), st));
    }
  }
  void prof_collect() {   // after a stream sync
    if (!prof_on) return;
    for (auto& mk : evmarks) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, evpool[mk.second], evpool[mk.second + 1]));
      kms[mk.first] += ms;
      kcnt[mk.first] += 1;
    }
    CK(cudaMemcpy(kctr, dctr.p, sizeof(kctr), cudaMemcpyDeviceToHost));
  }

  template <class T> T* scratch(int slot, size_t count) {
    size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    if (scr[slot].n < bytes) scr[slot].alloc(bytes + bytes / 4, st);
    return scr[slot].as<T>();
  }

  Dev make_tab(std::initializer_list<Seg> segs) {
    int tot = 0;
    for (auto& s : segs) tot += std::max(s.count, 0);
    Dev t(sizeof(HB) * std::max(tot, 1), st);
    int o = 0;
    for (auto& s : segs) {
      if (s.count <= 0) continue;
      CK(launch_build_tab(t.as<HB>() + o, s.b->base(), s.b->sl, s.b->sf, s.b->sr,
                          s.first, s.step, s.count, st));
      ++launches;
      o += s.count;
    }
    return t;
  }

  // ---- truncation launcher: warp kernel + persistent block kernel for
  //      tasks that exceed the per-CTA smem pool ----
  void run_trunc(TruncArgs a, int t0, int t1, const HB* out, int nelem, int Ra,
                 int Rb, cudaStream_t s = nullptr) {
    if (t1 <= t0 || nelem <= 0) return;
    if (!s) s = st;
    // own scratch slots (and queue streams) per launching stream: main,
    // side, deferred
    int bank = s == st ? 0 : (st3 != nullptr && s == st3 ? 2 : 1);
    for (int i = 0; i < NDS; ++i)
      if (dstr[i] != nullptr && s == dstr[i]) bank = 3 + i;
    const int SL_G[3] = {10, 15, 21}, SL_Q[3] = {13, 16, 22}, SL_C[3] = {14, 17, 23},
              SL_F[3] = {19, 20, 24};
    auto slot_of = [&](const int* base3, int k) { return bank < 3 ? base3[bank] : 32 + 4 * (bank - 3) + k; };
    a.T = dt.T;
    a.out = out;
    a.eps = eps;
    a.cap = cap;
    a.overflow = ovf.as<int>();
    a.tasks = dt.d_listA + 3 * t0;
    a.ntasks = t1 - t0;
    a.ctr = prof_on ? dctr.as<unsigned long long>() : nullptr;
    const int Rw = (a.mode == TM_TRUNCATE) ? Ra : Ra + Rb;
    long long wworst = 0, bworst = 0, pworst = 0;
    for (int i = t0; i < t1; ++i) {
      int bb = ht.listA[i * 3 + 1];
      int um = ht.mid[bb] - ht.lo[bb], vm = ht.hi[bb] - ht.mid[bb];
      wworst = std::max(wworst, warp_need_doubles(um, vm, Rw));
      bworst = std::max(bworst, trunc_need_doubles(um, vm, Rw));
      pworst = std::max(pworst, pair_need_doubles(std::max(um, vm), Rw));
    }
    const int nitems = a.ntasks * nelem;
    const bool direct = nitems <= (direct_max >= 0 ? direct_max : trunc_direct_max()) &&
                        nitems > warp_small;
    static const bool trace = getenv("ACR_TRACE_TRUNC") != nullptr;
    if (trace) {
      int mmax = 0;
      for (int i = t0; i < t1; ++i) {
        int bb = ht.listA[i * 3 + 1];
        mmax = std::max(mmax, std::max(ht.mid[bb] - ht.lo[bb], ht.hi[bb] - ht.mid[bb]));
      }
      fprintf(stderr, "TRUNC mode %d tasks %d nelem %d mmax %d Rw %d direct %d\n", a.mode,
              t1 - t0, nelem, mmax, Rw, (int)direct);
    }
    const long long SMD = 28416;                 // 222 KB of doubles
    // latency-bound launches whose panels do not fit one CTA's shared memory:
    // one CTA per side (cluster pair) instead of the global-memory scratch.
    // The sizes here come from capacities (Ra + Rb columns); a task whose
    // actual panel still exceeds one CTA's shared memory keeps it in a
    // per-CTA global area (rare)
    const long long pair_small = 4LL * Rw * Rw + 5LL * Rw + 8;   // the pair kernel's non-panel arrays
    if (direct && (bworst > SMD || force_pair) && pair_small <= SMD) {
      a.smem_doubles = (int)std::min(pworst, SMD);
      a.gscr = nullptr;
      a.gscr_stride = 0;
      if (pworst > SMD) {
        a.gscr = scratch<double>(slot_of(SL_G, 0), (size_t)2 * nitems * pworst);
        a.gscr_stride = pworst;
      }
      fork(s);
      kbegin(0);
      CK(launch_trunc_pair(a, nelem, a.smem_doubles, s));
      kend();
      launches += 1;
      return;
    }
    const long long wmax = warp_maxneed > 0 ? std::min<long long>(warp_maxneed, trunc_warp_pool_doubles())
                                            : trunc_warp_pool_doubles();
    const bool may_big = !direct && wworst > wmax;
    int* q = nullptr;
    int* qc = nullptr;
    a.wq = nullptr;
    a.task_major = warp_sched == 2 ? 1 : 0;
    a.warp_rmax = warp_rmax;
    a.warp_maxneed = wmax;
    if (!direct && warp_sched > 0) {
      qc = scratch<int>(slot_of(SL_C, 2), 8);
      a.wq = qc + 2;
    }
    a.smem_doubles = (int)std::min(bworst, SMD);
    a.gscr = nullptr;
    a.gscr_stride = 0;
    a.gscr_ntasks = 0;
    if (may_big) {
      q = scratch<int>(slot_of(SL_Q, 1), 2 * (size_t)nitems + 2);
      qc = scratch<int>(slot_of(SL_C, 2), 8);
    }
    if (!direct && warp_sched > 0) a.wq = qc + 2;
    if ((direct || may_big) && bworst > SMD) {
      const int nblk = direct ? nitems : std::min(nitems, 148);
      a.gscr = scratch<double>(slot_of(SL_G, 0), (size_t)nblk * bworst);
      a.gscr_stride = bworst;
    }
    fork(s);
    kbegin(0);
    TruncAux aux;
    memset(&aux, 0, sizeof(aux));
    if (may_big) {
      aux.cls = scratch<unsigned char>(slot_of(SL_F, 3), (size_t)nitems);
      if (!prof_on && !no_qstreams) {          // instrumented runs keep one stream
        QStreams& qs = qstr[bank];
        if (!qs.q0) {
          make_stream(&qs.q0, true);
          make_stream(&qs.q1, true);
          CK(cudaEventCreateWithFlags(&qs.ef, cudaEventDisableTiming));
          CK(cudaEventCreateWithFlags(&qs.ej0, cudaEventDisableTiming));
          CK(cudaEventCreateWithFlags(&qs.ej1, cudaEventDisableTiming));
        }
        aux.q0 = qs.q0; aux.q1 = qs.q1; aux.ef = qs.ef; aux.ej0 = qs.ej0; aux.ej1 = qs.ej1;
      }
    }
    CK(launch_trunc(a, nelem, direct, may_big, q, qc, s, &aux));
    kend();
    launches += may_big ? ((long long)a.smem_doubles * 8 + 64 > 112 * 1024 ? 3 : 2) : 1;
    if (getenv("ACR_TDUMP")) tdump(a, t0, t1, out, nelem, direct, may_big);
  }

  // development aid: per-launch checksum of the recompression outputs
  void tdump(const TruncArgs& a, int t0, int t1, const HB* out, int nelem, bool direct,
             bool may_big) {
    static long long idx = 0;
    CK(cudaDeviceSynchronize());
    std::vector<HB> hb(nelem);
    CK(cudaMemcpy(hb.data(), out, sizeof(HB) * nelem, cudaMemcpyDeviceToHost));
    long long rs = 0;
    double ss = 0.0;
    int maxR = 0;
    for (int g = 0; g < nelem; ++g) {
      const int nn = (int)ht.lo.size();
      std::vector<int> rk(2 * nn);
      CK(cudaMemcpy(rk.data(), hb[g].rk, sizeof(int) * 2 * nn, cudaMemcpyDeviceToHost));
      for (int i = t0; i < t1; ++i) {
        const int beta = ht.listA[i * 3 + 1], side = ht.listA[i * 3 + 2];
        const int r = rk[beta * 2 + side];
        rs += r;
        maxR = std::max(maxR, r);
        const int lo = ht.lo[beta], mid = ht.mid[beta], hi = ht.hi[beta];
        const int urow = side ? mid : lo, vrow = side ? lo : mid;
        const int um = side ? hi - mid : mid - lo, vm = side ? mid - lo : hi - mid;
        const long long slot = (long long)ht.depth[beta] * hb[g].R * n;
        std::vector<double> col(std::max(um, vm));
        std::vector<double> dense((size_t)um * vm, 0.0), uc((size_t)um * r), vc((size_t)vm * r);
        for (int c = 0; c < r; ++c) {
          CK(cudaMemcpy(col.data(), hb[g].U + slot + (long long)c * n + urow, 8 * um, cudaMemcpyDeviceToHost));
          for (int k = 0; k < um; ++k) { ss += col[k] * col[k]; uc[(size_t)c * um + k] = col[k]; }
          CK(cudaMemcpy(col.data(), hb[g].V + slot + (long long)c * n + vrow, 8 * vm, cudaMemcpyDeviceToHost));
          for (int k = 0; k < vm; ++k) { ss += col[k] * col[k] * 1.7; vc[(size_t)c * vm + k] = col[k]; }
        }
        static FILE* fdump = getenv("ACR_TDUMP_FILE") ? fopen(getenv("ACR_TDUMP_FILE"), "wb") : nullptr;
        if (fdump && idx == atoll(getenv("ACR_TDUMP_IDX") ? getenv("ACR_TDUMP_IDX") : "-1")) {
          for (int x = 0; x < um; ++x)
            for (int y = 0; y < vm; ++y) {
              double acc = 0.0;
              for (int c = 0; c < r; ++c) acc += uc[(size_t)c * um + x] * vc[(size_t)c * vm + y];
              dense[(size_t)x * vm + y] = acc;
            }
          int hdr[6] = {g, i, beta, side, r, um * 1000 + vm};
          fwrite(hdr, sizeof(int), 6, fdump);
          fwrite(dense.data(), 8, dense.size(), fdump);
          fflush(fdump);
        }
      }
    }
    fprintf(stderr, "TDUMP %lld mode %d tasks %d nelem %d direct %d big %d ranksum %lld maxr %d ss %.17g\n",
            idx++, a.mode, t1 - t0, nelem, (int)direct, (int)may_big, rs, maxR, ss);
  }

  static void offset_src(Src& s, int e0) {
    if (s.kind == 0) s.p = s.p ? s.p + e0 * s.s : nullptr;
    else if (s.kind == 1) s.tab = s.tab ? s.tab + e0 : nullptr;
    else s.hb = s.hb ? s.hb + e0 : nullptr;
  }
  static void offset_rank(RankRef& r, int e0) {
    if (r.hb) r.hb += e0;
    else if (r.arr) r.arr += e0 * r.s;
  }
  static void offset_op(TOp& o, int e0) {
    offset_src(o.U, e0);
    offset_src(o.V, e0);
    offset_rank(o.rank, e0);
  }

  // ---- multiply: C = A B for G elements (reference algebra.py:159-185) ----
  void multiply(const HB* A, const HB* B, const HB* C, int G, int RA, int RB,
                int RC, int diag = 0) {
    if (G <= 0) return;
    const int nd = std::max(ht.nd, 1), nn = ht.nnodes;
    const int nA1 = ht.nA(1, nn);
    long long per = (long long)nd * n * (2LL * RB + RA) * 8 + 2LL * nA1 * RA * RB * 8 +
                    (long long)nn * 8;
    int chunk = (int)std::max<long long>(1, (4LL << 30) / std::max<long long>(per, 1));
    for (int g0 = 0; g0 < G; g0 += chunk) {
      int cg = std::min(chunk, G - g0);
      multiply_chunk(A + g0, B + g0, C + g0, cg, RA, RB, RC, diag);
    }
  }

  void multiply_chunk(const HB* A, const HB* B, const HB* C, int G, int RA,
                      int RB, int RC, int diag) {
    const int nd = std::max(ht.nd, 1), nn = ht.nnodes;
    const long long ps = (long long)nd * n;
    double* PX = scratch<double>(0, (size_t)G * ps * RB);
    double* Yp = scratch<double>(1, (size_t)G * ps * RB);
    double* Zp = scratch<double>(2, (size_t)G * ps * RA);
    int* cr = scratch<int>(3, (size_t)G * nn * 2);
    const int nA1 = ht.nA(1, nn);
    double* tbY = scratch<double>(4, (size_t)G * std::max(nA1, 1) * RA * RB);
    double* tbZ = scratch<double>(5, (size_t)G * std::max(nA1, 1) * RA * RB);
    CK(cudaMemsetAsync(cr, 0, sizeof(int) * G * nn * 2, st));
    // cross terms X11 = (U_A12 (V_A12^T U_B21), V_B21), X22 likewise (none
    // when an operand is the level-0 diagonal: its factors have rank 0, the
    // cross-term ranks stay 0 from the memset)
    if (!ht.branches.empty() && !diag) {
      GPJob j[2];
      memset(j, 0, sizeof(j));
      for (int s = 0; s < 2; ++s) {
        j[s].X = s_hbV(A);
        j[s].Y = s_hbU(B);
        j[s].W = s_hbU(A);
        j[s].Z = s_pan(PX, ps * RB, RB);
        j[s].rx = r_hb(A);
        j[s].ry = r_hb(B);
        j[s].orank = cr;
        j[s].ors = nn * 2;
        j[s].oside = s;
        j[s].alpha = 1.0;
      }
      j[0].hx = 1; j[0].hw = 0; j[0].sx = 0; j[0].sy = 1;
      j[1].hx = 0; j[1].hw = 1; j[1].sx = 1; j[1].sy = 0;
      gp(j, 2, dt.d_branches, (int)ht.branches.size(), G, RA, RB, st);
    }
    const cudaStream_t s2 = side();
    fork(s2);
    // class 2: dense leaf products on DMMA, 2 s^3 FLOP each; class 4: the exact
    // diagonal path (level 0, E/F diagonal), HBM-bound: algorithmic bytes =
    // read the dense leaf and the diagonal, write the product, 8 (2 s^2 + s)
    kbegin(diag ? 4 : 2);
    if (prof_on)
      for (int v = 0; v < nn; ++v)
        if (ht.isleaf[v]) {
          const double sz = ht.hi[v] - ht.lo[v];
          if (diag) hflops[4] += (double)G * 8.0 * (2.0 * sz * sz + sz);
          else {
            hflops[2] += (double)G * 2.0 * sz * sz * sz;
            hbytes[2] += (double)G * 24.0 * sz * sz;      // leaf_gemm: A, B read, C written
          }
        }
    CK(launch_leafgemm(dt.T, A, B, C, G, s_pan(PX, ps * RB, RB), r_arr(cr, nn * 2), diag,
                       s2));
    kend();
    ++launches;
    struct Joiner {
      Plan* p;
      cudaStream_t s;
      ~Joiner() { p->join(s); }
    } jn{this, s2};
    if (ht.branches.empty()) return;
    MMJob J[2];
    memset(J, 0, sizeof(J));
    J[0].H = A;
    J[0].X = s_hbU(B);
    J[0].Y = s_pan(Yp, ps * RB, RB);
    J[0].trans = 0;
    J[0].cols = r_hb(B);
    J[0].cols_fixed = -1;
    J[0].swap = 0;
    J[0].tbuf = tbY;
    J[0].RT = RA;
    J[0].CT = RB;
    J[1].H = B;
    J[1].X = s_hbV(A);
    J[1].Y = s_pan(Zp, ps * RA, RA);
    J[1].trans = 1;
    J[1].cols = r_hb(A);
    J[1].cols_fixed = -1;
    J[1].swap = 1;
    J[1].tbuf = tbZ;
    J[1].RT = RB;
    J[1].CT = RA;
    for (auto& j : J) {
      j.alpha = 1.0;
      j.mu0 = 1;
      j.mu1 = nn;
      j.nA = nA1;
      j.nB = ht.startB[nn] - ht.startB[1];
    }
    if (diag) {
      // level 0: one operand is an exact diagonal with rank-0 factors.  The
      // job with the diagonal operand as H is a row scaling; the other one
      // has no columns (rank 0) and is skipped (M2 passes the other operand
      // through, algebra.py:93-96)
      kbegin(3);
      CK(launch_hmat_diag(dt.T, J[diag == 1 ? 0 : 1], G, st));
      kend();
      ++launches;
      if (prof_on) CK(launch_census_hmat(dt.T, &J[diag == 1 ? 0 : 1], 1, G, ctrp(), st));
    } else {
      hmat(J, 2, G, st);
    }
    // M2: off12 = combine(f1, f2), off21 = combine(g1, g2)
    TruncArgs a;
    memset(&a, 0, sizeof(a));
    a.mode = TM_COMBINE_SWAP1;
    a.a = op_own(s_pan(Yp, ps * RB, RB), s_hbV(B), r_hb(B));
    a.b = op_own(s_hbU(A), s_pan(Zp, ps * RA, RA), r_hb(A));
    // M3: ancestors' cross terms, parent first, root last (all rank 0 with a
    // diagonal operand: every combine would pass C through unchanged)
    auto m3 = [&](int t) {
      TruncArgs b;
      memset(&b, 0, sizeof(b));
      b.mode = TM_COMBINE;
      b.a = op_own(s_hbU(C), s_hbV(C), r_hb(C));
      b.b = op_own(s_pan(PX, ps * RB, RB), s_hbV(B), r_arr(cr, nn * 2));
      b.b.sel = SEL_ANC;
      b.b.t = t;
      return b;
    };
    const int t0 = ht.startA[0], t1 = ht.startA[1];
    static const long long dsplit_max = getenv("ACR_DSPLIT_MAX") ? atoll(getenv("ACR_DSPLIT_MAX")) : 1200;
    if (!prof_on && !no_side && !no_dsplit && !diag && ht.nd > 1 && ht.nd <= NDS + 1 &&
        (long long)(t1 - t0) * G <= dsplit_max) {
      // A node of depth d takes M2 and then the d rounds of M3 (one per
      // ancestor), independently of every other node.  Launched per round over
      // all nodes, each round lasts as long as its largest task (the root's in
      // M2, the depth-t nodes' in round t) and the rounds add up; launched per
      // depth, each depth's chain runs on its own stream and the step lasts as
      // long as the longest chain.  The tasks are listed by depth.
      std::vector<std::pair<int, int>> rng;   // [first, last) of every depth
      for (int e0 = t0; e0 < t1;) {
        const int d = ht.depth[ht.listA[e0 * 3 + 1]];
        int e1 = e0;
        while (e1 < t1 && ht.depth[ht.listA[e1 * 3 + 1]] == d) ++e1;
        if ((int)rng.size() != d) throw InternalError("task list not ordered by depth");
        rng.push_back({e0, e1});
        e0 = e1;
      }
      const int nd = (int)rng.size();
      for (int d = 0; d < nd; ++d) {          // the deepest level (most rounds) on the main stream, last
        const cudaStream_t sd = d == nd - 1 ? st : depth_stream(d);
        run_trunc(a, rng[d].first, rng[d].second, C, G, RB, RA, sd);
        for (int t = 1; t <= d; ++t) run_trunc(m3(t), rng[d].first, rng[d].second, C, G, RC, RB, sd);
        if (sd != st) CK(cudaEventRecord(evds[d], sd));
      }
      for (int d = 0; d + 1 < nd; ++d) CK(cudaStreamWaitEvent(st, evds[d], 0));
      return;
    }
    run_trunc(a, t0, t1, C, G, RB, RA);
    for (int t = 1; t < ht.nd && !diag; ++t) {
      int s0 = t0;
      while (s0 < t1 && ht.depth[ht.listA[s0 * 3 + 1]] < t) ++s0;
      if (s0 >= t1) break;
      run_trunc(m3(t), s0, t1, C, G, RC, RB);
    }
  }

  // ---- add: C = A + sb*B (reference algebra.py:100-112) ----
  void add(const HB* A, const HB* B, const HB* C, int G, double sb, int RA,
           int RB) {
    if (G <= 0) return;
    const cudaStream_t s2 = side();
    fork(s2);
    kbegin(7);
    CK(launch_leafadd(dt.T, A, B, C, sb, G, s2));
    kend();
    elem_bytes(G, 3.0 * n * ht.bw);          // read A, B leaves, write C
    ++launches;
    if (!ht.branches.empty()) {
      TruncArgs a;
      memset(&a, 0, sizeof(a));
      a.mode = TM_COMBINE;
      a.a = op_own(s_hbU(A), s_hbV(A), r_hb(A));
      a.b = op_own(s_hbU(B), s_hbV(B), r_hb(B), sb);
      run_trunc(a, ht.startA[0], ht.startA[1], C, G, RA, RB);
    }
    join(s2);
  }

  // ---- invert in place (reference algebra.py:192-240) ----
  struct InvCtx {
    const HB* H;
    int G, R;
    double *P1, *P2, *P3, *tb;
    long long ps;
    int* sing;
    int* rs = nullptr;   // rank snapshot [g][nnodes][2] (see inv_node: b11 beside b12 / b21)
    bool tri = false;    // leaves are tridiagonal (lifted level): banded leaf inverse
    bool pend = false;   // S's off-diagonal recompressions still running on the side stream
    bool defer[32] = {}; // tree depths whose recompressions run on the deferred stream
  };

  // the deferred recompressions of tree depth d must finish before anything
  // reads or writes the factors of a node at that depth
  void use_depth(InvCtx& c, int d) {
    if (c.defer[d]) {
      CK(cudaStreamWaitEvent(st, evdef[d], 0));
      c.defer[d] = false;
    }
  }

  // tri: every leaf the inversion meets is tridiagonal (the lifted level);
  // the banded leaf kernel checks it and raises TRI_FAIL in the overflow flag
  bool tri_ok = getenv("ACR_NO_TRI") == nullptr;
  bool tri_all = getenv("ACR_TRI_ALL") != nullptr;   // test aid: ask for it at every level (exercises the fallback)
  void invert(const HB* H, int G, int R, int* sing, bool tri = false) {
    if (G <= 0) return;
    InvCtx c;
    c.tri = (tri || tri_all) && tri_ok && ht.bw <= 64;
    c.H = H;
    c.G = G;
    c.R = R;
    c.ps = (long long)std::max(ht.nd, 1) * n;
    c.P1 = scratch<double>(6, (size_t)G * c.ps * R);
    c.P2 = scratch<double>(7, (size_t)G * c.ps * R);
    c.P3 = scratch<double>(8, (size_t)G * c.ps * R);
    int maxA = 1;
    for (int v = 0; v < ht.nnodes; ++v) maxA = std::max(maxA, ht.nA(v, v + 1));
    c.tb = scratch<double>(9, (size_t)G * maxA * R * R);
    c.rs = scratch<int>(25, (size_t)G * ht.nnodes * 2);
    c.sing = sing;
    inv_node(c, 0);
    settle(c);
    for (int d = 0; d < 32; ++d) use_depth(c, d);
  }

  // the side-stream recompressions of a Schur complement must finish before
  // anything reads its off-diagonal factors (only leaf inverses may overlap)
  void settle(InvCtx& c) {
    if (c.pend) {
      join(side());
      c.pend = false;
    }
  }

  void inv_hmat(InvCtx& c, int mu, bool second) {
    // first pass (mu = c0): T = x11 U12 -> P1, Hh = x11^T V21 -> P2
    // second pass (mu = c1): Z = sinv U21 -> P1, S2 = sinv^T V12 -> P2
    MMJob J[2];
    memset(J, 0, sizeof(J));
    for (int k = 0; k < 2; ++k) {
      J[k].H = c.H;
      J[k].cols = r_hb(c.H);
      J[k].cols_fixed = -1;
      J[k].alpha = 1.0;
      J[k].mu0 = mu;
      J[k].mu1 = mu + 1;
      J[k].tbuf = c.tb + (size_t)k * 0;
      J[k].RT = c.R;
      J[k].CT = c.R;
      J[k].nA = ht.nA(mu, mu + 1);
      J[k].nB = ht.nleaves_under(mu);
    }
    (void)second;
    J[0].X = s_hbU(c.H);
    J[0].Y = s_pan(c.P1, c.ps * c.R, c.R);
    J[0].trans = 0;
    J[0].swap = 0;
    J[1].X = s_hbV(c.H);
    J[1].Y = s_pan(c.P2, c.ps * c.R, c.R);
    J[1].trans = 1;
    J[1].swap = 1;
    // the two jobs need distinct t-buffers
    double* tb2 = scratch<double>(11, (size_t)c.G * std::max(J[0].nA, 1) * c.R * c.R);
    J[1].tbuf = tb2;
    hmat(J, 2, c.G, st, c.tri);   // lifted level: panels with one nonzero row
  }

  // add_lowrank(H_mu, (U, V)) with rank (nu, fside) if (nu, 1-fside) != 0:
  // factor recompressions on st, the leaves' dense update on s2 (disjoint
  // data); the caller joins s2
  void inv_lowrank(InvCtx& c, int nu, int mu, Src U, Src V, int fside, cudaStream_t s2,
                   const int* snap = nullptr) {
    fork(s2);
    leaflr(c.H, c.G, mu, U, V, r_hb(c.H), nu, fside, s2);
    int t0 = ht.startA[mu], t1 = ht.startA[mu + 1];
    if (t1 > t0) {
      TruncArgs a;
      memset(&a, 0, sizeof(a));
      a.mode = TM_COMBINE;
      a.a = op_own(s_hbU(c.H), s_hbV(c.H), r_hb(c.H));
      a.b = op_own(U, V, r_hb(c.H));
      a.b.sel = SEL_FIXED;
      a.b.node = nu;
      a.b.fside = fside;
      if (snap) {
        // ranks of nu from the snapshot (the caller overwrites them concurrently)
        a.b.rank = r_arr(snap, (long long)ht.nnodes * 2);
        a.b.sel = SEL_NODE;
      }
      run_trunc(a, t0, t1, c.H, c.G, c.R, c.R);
    }
  }

  void inv_node(InvCtx& c, int nu) {
    if (ht.isleaf[nu]) {
      kbegin(1);
      if (prof_on) {   // Gauss-Jordan inverse: 2 s^3
        const double sz = ht.hi[nu] - ht.lo[nu];
        hflops[1] += (double)c.G * 2.0 * sz * sz * sz;
        hbytes[1] += (double)c.G * 16.0 * sz * sz;        // leaf_inv: read + write
      }
      if (c.tri) CK(launch_leafinv_tri(dt.T, c.H, c.G, nu, c.sing, ovf.as<int>(), st));
      else CK(launch_leafinv(dt.T, c.H, c.G, nu, c.sing, st));
      kend();
      ++launches;
      return;
    }
    const int a0 = ht.c0[nu], a1 = ht.c1[nu];
    const Src P1 = s_pan(c.P1, c.ps * c.R, c.R);
    const Src P2 = s_pan(c.P2, c.ps * c.R, c.R);
    const Src P3 = s_pan(c.P3, c.ps * c.R, c.R);
    if (ht.isleaf[a0] && ht.isleaf[a1] && !prof_on && !no_fuse_leaf &&
        schur_leaf_smem(ht.bw, c.R) <= 200 * 1024) {
      // both children are leaves: each half's HODLR x panel products, panel
      // product and leaf update in one launch (k_schur_leaf)
      inv_node(c, a0);                                 // x11
      settle(c);
      use_depth(c, ht.depth[nu]);
      CK(launch_schur_leaf(dt.T, c.H, c.G, nu, 0, P1, P2, c.R, st));   // T, Hh; S = H22 + W V12^T
      inv_node(c, a1);                                 // sinv
      CK(launch_schur_leaf(dt.T, c.H, c.G, nu, 1, P1, P2, c.R, st));   // Z, S2; b11 = x11 + G Hh^T
      launches += 2;
      TruncArgs a;                                     // b12, b21
      memset(&a, 0, sizeof(a));
      a.mode = TM_TRUNCATE;
      a.a = op_own(P1, P2, r_hb(c.H), -1.0);
      run_trunc(a, ht.startA[nu], ht.startA[nu] + 2, c.H, c.G, c.R, 0);
      return;
    }
    inv_node(c, a0);                                   // x11
    settle(c);
    use_depth(c, ht.depth[nu]);
    inv_hmat(c, a0, false);                            // T, Hh
    {
      GPJob j;                                          // W = -U21 (V21^T T)
      memset(&j, 0, sizeof(j));
      j.X = s_hbV(c.H); j.hx = 0; j.rx = r_hb(c.H); j.sx = 1;
      j.Y = P1; j.ry = r_hb(c.H); j.sy = 0;
      j.W = s_hbU(c.H); j.hw = 1;
      j.Z = P3;
      j.alpha = -1.0;
      gp(&j, 1, dt.d_iota + nu, 1, c.G, c.R, c.R, st);
    }
    const cudaStream_t s2 = side();
    {                                                  // S = H22 + W V12^T
      // leaves on the main stream, off-diagonal combines on the side stream:
      // the first leaf inverse of sinv below overlaps the recompressions
      leaflr(c.H, c.G, a1, P3, s_hbV(c.H), r_hb(c.H), nu, 0, st);
      const int t0 = ht.startA[a1], t1 = ht.startA[a1 + 1];
      if (t1 > t0) {
        TruncArgs a;
        memset(&a, 0, sizeof(a));
        a.mode = TM_COMBINE;
        a.a = op_own(s_hbU(c.H), s_hbV(c.H), r_hb(c.H));
        a.b = op_own(P3, s_hbV(c.H), r_hb(c.H));
        a.b.sel = SEL_FIXED;
        a.b.node = nu;
        a.b.fside = 0;
        const cudaStream_t s3 = deferred();
        // the subtree's tasks are listed by depth; the deepest level is needed
        // first (right after the first leaf inverse) and goes to the side
        // stream; a node of depth d above it is first touched once its left
        // child has been inverted, so those levels -- the largest tasks -- run
        // on the deferred stream meanwhile (a depth always maps to the same
        // stream, which orders nested updates of the same nodes)
        int td = t1;
        if (s3 != st && s2 != st) {
          const int dmax = ht.depth[ht.listA[(t1 - 1) * 3 + 1]];
          while (td > t0 && ht.depth[ht.listA[(td - 1) * 3 + 1]] == dmax) --td;
        } else {
          td = t0;
        }
        fork(s2);
        run_trunc(a, td, t1, c.H, c.G, c.R, c.R, s2);
        c.pend = s2 != st;
        for (int e1 = td; e1 > t0;) {              // remaining depths, deepest first
          const int d = ht.depth[ht.listA[(e1 - 1) * 3 + 1]];
          int e0 = e1;
          while (e0 > t0 && ht.depth[ht.listA[(e0 - 1) * 3 + 1]] == d) --e0;
          use_depth(c, d);                         // an earlier update of this depth still pending
          fork(s3);
          run_trunc(a, e0, e1, c.H, c.G, c.R, c.R, s3);
          CK(cudaEventRecord(evdef[d], s3));
          c.defer[d] = true;
          e1 = e0;
        }
      }
    }
    inv_node(c, a1);                                   // sinv
    settle(c);
    inv_hmat(c, a1, true);                             // Z, S2
    {
      GPJob j;                                          // G = T (V12^T Z)
      memset(&j, 0, sizeof(j));
      j.X = s_hbV(c.H); j.hx = 1; j.rx = r_hb(c.H); j.sx = 0;
      j.Y = P1; j.ry = r_hb(c.H); j.sy = 1;
      j.W = P1; j.hw = 0;
      j.Z = P3;
      j.alpha = 1.0;
      // the column count of G / Hh -- rank(nu, 1), or 0 when rank(nu, 0) is --
      // is written to the snapshot: b11's recompressions below run beside the
      // b12 / b21 truncation, which overwrites the ranks of nu
      j.orank = c.rs;
      j.ors = (long long)ht.nnodes * 2;
      j.oside = 1;
      gp(&j, 1, dt.d_iota + nu, 1, c.G, c.R, c.R, st);
    }
    inv_lowrank(c, nu, a0, P3, P2, 1, s2, c.rs);       // b11 = x11 + G Hh^T
    TruncArgs a;                                       // b12, b21 (independent of b11)
    memset(&a, 0, sizeof(a));
    a.mode = TM_TRUNCATE;
    a.a = op_own(P1, P2, r_hb(c.H), -1.0);
    run_trunc(a, ht.startA[nu], ht.startA[nu] + 2, c.H, c.G, c.R, 0, s2);
    join(s2);
  }

  // ---- helpers for reports ----
  // n ints of the mapped staging buffer (grown only when nothing is pending)
  size_t hmap_take(size_t n) {
    // (space is reclaimed at the syncs that drain it: a stats_launch region
    // stays valid until the stats_read after the next sync)
    if (hmap_used + n > hmap_cap) {
      if (!pend.empty()) sync_fetch();
      if (n > hmap_cap) {
        CK(cudaStreamSynchronize(st));
        if (hmap) CK(cudaFreeHost(hmap));
        hmap_cap = std::max<size_t>(n, (size_t)12 * std::max(m, 1) * ht.nnodes + 2 * (size_t)m + 64);
        CK(cudaHostAlloc(reinterpret_cast<void**>(&hmap), hmap_cap * sizeof(int),
                         cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hmap_d), hmap, 0));
      }
    }
    const size_t off = hmap_used;
    hmap_used += n;
    return off;
  }

  void fetch_ranks(const Batch& b, std::vector<int>& out) {
    out.resize((size_t)b.cnt * ht.nnodes * 2);
    if (!b.cnt) return;
    const size_t off = hmap_take(out.size());
    CK(launch_copy_i32(hmap_d + off, b.rk.as<int>(), (long long)out.size(), st));
    pend.push_back({&out, off, out.size()});
  }

  // stream sync, then the fetched rank tables move to their host vectors
  void sync_fetch() {
    CK(cudaStreamSynchronize(st));
    drain_fetch();
  }

  // the stream has been synchronised: fetched tables move to their vectors
  void drain_fetch() {
    for (const Pend& p : pend) memcpy(p.out->data(), hmap + p.off, p.n * sizeof(int));
    pend.clear();
    hmap_used = 0;
  }

  // rank statistics of a level computed on the device (k_rank_stats) and
  // copied into the mapped buffer; stats_read after the next stream sync.
  // The per-level host round trip then moves 4 nd + 2 words instead of the
  // three m x nnodes rank tables (whose host scan was the largest GPU idle
  // gap at the top levels)
  size_t stats_launch(const Level& L) {
    const int nd = std::max(ht.nd, 1);
    const size_t nw = 4 * (size_t)nd + 2;
    unsigned* d = scratch<unsigned>(18, nw);
    CK(cudaMemsetAsync(d, 0, nw * sizeof(unsigned), st));
    CK(launch_rank_stats(L.D.rk.as<int>(), L.E.rk.as<int>(), L.F.rk.as<int>(), L.D.sr, L.m,
                         dt.d_branches, (int)ht.branches.size(), dt.T.depth, nd, d, st));
    const size_t off = hmap_take(nw);
    CK(launch_copy_i32(hmap_d + off, reinterpret_cast<const int*>(d), (long long)nw, st));
    launches += 2;
    return off;
  }

  // profile (profile_level's semantics) and capacity max of stats_launch's output
  int stats_read(size_t off, bool prof_it) {
    const int nd = std::max(ht.nd, 1);
    const unsigned* w = reinterpret_cast<const unsigned*>(hmap + off);
    if (prof_it) {
      Profile p;
      p.mx.assign(ht.nd, 0);
      p.mean.assign(ht.nd, 0.0);
      for (int d = 0; d < ht.nd; ++d) {
        unsigned long long sum;
        memcpy(&sum, w + 2 * nd + 2 + 2 * d, sizeof(sum));
        p.mx[d] = (int)w[d];
        p.mean[d] = w[nd + d] ? (double)(long long)sum / (double)(long long)w[nd + d] : 0.0;
      }
      prof.push_back(p);
    }
    return std::max((int)w[2 * nd], 1);
  }

  long long hb_bytes(const int* rk) const {
    long long s = 0;
    for (int v = 0; v < ht.nnodes; ++v) {
      int sz = ht.hi[v] - ht.lo[v];
      if (ht.isleaf[v]) s += (long long)sz * sz;
      else s += (long long)sz * (rk[v * 2] + rk[v * 2 + 1]);
    }
    return 8 * s;
  }

  int max_rank_of(const std::vector<int>& r) const {
    int mx = 0;
    const size_t per = (size_t)ht.nnodes * 2;
    for (size_t b = 0; b + per <= r.size(); b += per)
      for (int v : ht.branches) mx = std::max({mx, r[b + v * 2], r[b + v * 2 + 1]});
    return mx;
  }

  Batch clone(const Batch& b) {
    Batch c;
    c.alloc(ht, b.cnt, b.R, st);
    const size_t cnt = (size_t)std::max(b.cnt, 1);
    CK(cudaMemcpyAsync(c.leaf.p, b.leaf.p, sizeof(double) * b.sl * cnt, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(c.U.p, b.U.p, sizeof(double) * b.sf * cnt, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(c.V.p, b.V.p, sizeof(double) * b.sf * cnt, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(c.rk.p, b.rk.p, sizeof(int) * b.sr * cnt, cudaMemcpyDeviceToDevice, st));
    return c;
  }

  // column capacity of a level's output from the input's max rank (a
  // truncation that would exceed it flags overflow and the level is redone)
  int rout_for(int maxr, int LR) const {
    int Rout = std::max(4, (3 * maxr + 1) / 2 + 4);
    if (cap > 0) Rout = std::min(Rout, std::max(cap, 1));
    return std::max(Rout, LR);
  }

  // ---- lift (reference lift_system reduction.py:156-166, from_tridiagonal
  //      hodlr.py:242-291, from_diagonal :294-314) of the global blocks
  //      [first, first + mloc) ----
  void lift(Level& L, int first, int mloc, const double* sub, const double* diag,
            const double* sup, const double* E, const double* F) {
    L.m = mloc;
    L.first = first;
    L.mg = m;
    L.R = 1;
    L.lvl = 0;
    L.D.alloc(ht, L.m, 1, st);
    L.E.alloc(ht, L.m, 1, st);
    L.F.alloc(ht, L.m, 1, st);
    const int e0 = first == 0 ? 1 : 0;                        // E exists for g >= 1
    const int ne_ = L.m - e0;
    const int nf_ = std::min(L.m, m - 1 - first);             // F exists for g <= m-2
    Dev tD = make_tab({{&L.D, 0, 1, L.m}});
    CK(launch_lift(dt.T, sub + (long long)first * (n - 1), diag + (long long)first * n,
                   sup + (long long)first * (n - 1), tD.as<HB>(), L.m, st));
    Dev tE = make_tab({{&L.E, e0, 1, ne_}});
    CK(launch_liftdiag(dt.T, E + (long long)(first + e0 - 1) * n, tE.as<HB>(), ne_, st));
    Dev tF = make_tab({{&L.F, 0, 1, nf_}});
    CK(launch_liftdiag(dt.T, F + (long long)first * n, tF.as<HB>(), nf_, st));
    Dev tZ = make_tab({{&L.E, 0, 1, e0}, {&L.F, nf_, 1, L.m - nf_}});
    CK(launch_zerohb(dt.T, tZ.as<HB>(), e0 + L.m - nf_, st));
    launches += 4;
  }

  // ---- one reduction level (reference reduction.py:173-232) ----
  // Local window [first, first+m) of a global level of mg blocks; the last
  // local odd block takes {Dinv, E, F} of the right neighbour's first block.
  bool reduce(Level& L, int Rout, int lvl, int order, Level& nx, Record& rec,
              int& need, bool dlev, const int* perm = nullptr, bool keep_input = false,
              size_t* stats_off = nullptr) {
    const int mm = L.m, first = L.first, mg = L.mg, ne = (mm + 1) / 2, no = mm / 2;
    const bool right = first + mm < mg;
    int nq = 0, nq_loc = 0, nq_h = 0, nf = 0, nf_loc = 0, nf_h = 0;
    for (int j = 1; j < mm; j += 2) {
      const int jg = first + j;
      if (jg + 1 <= mg - 1) { ++nq; if (j + 1 < mm) ++nq_loc; else ++nq_h; }
      if (jg + 2 <= mg - 1) { ++nf; if (j + 1 < mm) ++nf_loc; else ++nf_h; }
    }
    const int i0 = first >= 2 ? 0 : 1;        // first new block with an E' (jg >= 2)
    const int nep = std::max(no - i0, 0);
    CK(cudaMemsetAsync(ovf.p, 0, sizeof(int), st));
    int* sg = sing.as<int>();
    CK(launch_fill_i32(sg, INT_MAX, (long long)ne, st));
    // 0. halo E, F of the right neighbour's first even block (level inputs):
    //    on the comm stream, overlapped with the invert below
    Batch hE, hF;
    if (dlev) {
      std::vector<Msg> msgs;
      if (first > 0) {
        block_msgs(msgs, L.E, 0, nb_left, true);
        block_msgs(msgs, L.F, 0, nb_left, true);
      }
      if (right) {
        hE.alloc(ht, 1, L.R, st);
        hF.alloc(ht, 1, L.R, st);
        block_msgs(msgs, hE, 0, nb_right, false);
        block_msgs(msgs, hF, 0, nb_right, false);
      }
      comm_fork();
      tp->exchange(msgs, comm_stream());
      ef_pending = true;
    }
    // 1. Dinv of the even blocks
    rec.m = mm;
    rec.first = first;
    rec.mg = mg;
    rec.diagEF = lvl == 0;
    rec.right = right;
    rec.Dinv.alloc(ht, ne, Rout, st);
    {
      Dev tDe = make_tab({{&L.D, 0, 2, ne}});
      Dev tDi = make_tab({{&rec.Dinv, 0, 1, ne}});
      kbegin(7);
      CK(launch_copyhb(dt.T, tDe.as<HB>(), tDi.as<HB>(), ne, ovf.as<int>(), st));
      kend();
      elem_bytes(ne, 2.0 * n * ht.bw);       // leaves copied (+ factors below the rank)
      ++launches;
      invert(tDi.as<HB>(), ne, rec.Dinv.R, sg, lvl == 0);
    }
    // 1b. halo: our first even block to the left, the right neighbour's to us
    Batch hDi;
    if (dlev) {
      // Dinv of the first even block leaves once the invert is done; its E
      // and F (level inputs) already went out on the comm stream before the
      // invert (reduce step 0), so only a third of the halo is exposed
      std::vector<Msg> msgs;
      if (first > 0) block_msgs(msgs, rec.Dinv, 0, nb_left, true);
      if (right) {
        hDi.alloc(ht, 1, Rout, st);
        block_msgs(msgs, hDi, 0, nb_right, false);
      }
      comm_fork();
      tp->exchange(msgs, comm_stream());
      comm_join();
      ef_pending = false;
    }
    // 2. P_j = E_j Dinv_{j-1}, Q_j = F_j Dinv_{j+1}
    Batch PQ;
    PQ.alloc(ht, no + nq, Rout, st);
    {
      Dev tA = make_tab({{&L.E, 1, 2, no}, {&L.F, 1, 2, nq}});
      Dev tB = make_tab({{&rec.Dinv, 0, 1, no}, {&rec.Dinv, 1, 1, nq_loc}, {&hDi, 0, 1, nq_h}});
      Dev tC = make_tab({{&PQ, 0, 1, no + nq}});
      multiply(tA.as<HB>(), tB.as<HB>(), tC.as<HB>(), no + nq, L.R, rec.Dinv.R, PQ.R,
               lvl == 0 ? 1 : 0);
    }
    // 3. X = P F_{j-1}, Y = Q E_{j+1}, E' = -P E_{j-1}, F' = -Q F_{j+1}
    if (ef_pending) {
      comm_join();
      ef_pending = false;
    }
    nx.m = no;
    nx.first = first / 2;
    nx.mg = mg / 2;
    nx.R = Rout;
    nx.D.alloc(ht, no, Rout, st);
    nx.E.alloc(ht, no, Rout, st);
    nx.F.alloc(ht, no, Rout, st);
    Batch XY;
    XY.alloc(ht, no + nq, Rout, st);
    {
      Dev tA = make_tab({{&PQ, 0, 1, no}, {&PQ, no, 1, nq}, {&PQ, i0, 1, nep},
                         {&PQ, no, 1, nf}});
      Dev tB = make_tab({{&L.F, 0, 2, no}, {&L.E, 2, 2, nq_loc}, {&hE, 0, 1, nq_h},
                         {&L.E, 2 * i0, 2, nep}, {&L.F, 2, 2, nf_loc}, {&hF, 0, 1, nf_h}});
      Dev tC = make_tab({{&XY, 0, 1, no + nq}, {&nx.E, i0, 1, nep}, {&nx.F, 0, 1, nf}});
      int G = no + nq + nep + nf;
      multiply(tA.as<HB>(), tB.as<HB>(), tC.as<HB>(), G, PQ.R, L.R, Rout,
               lvl == 0 ? 2 : 0);
      Dev tE = make_tab({{&nx.E, i0, 1, nep}, {&nx.F, 0, 1, nf}});
      kbegin(7);
      CK(launch_negate(dt.T, tE.as<HB>(), nep + nf, st));
      kend();
      elem_bytes(nep + nf, 2.0 * n * ht.bw);
      ++launches;
      const int nz_e = std::min(i0, no);
      Dev tZ = make_tab({{&nx.E, 0, 1, nz_e}, {&nx.F, nf, 1, no - nf}});
      CK(launch_zerohb(dt.T, tZ.as<HB>(), nz_e + std::max(no - nf, 0), st));
      ++launches;
    }
    // 4. D' = add(add(D_j, -X), -Y)
    {
      Dev tA = make_tab({{&L.D, 1, 2, no}});
      Dev tB = make_tab({{&XY, 0, 1, no}});
      Dev tC = make_tab({{&nx.D, 0, 1, no}});
      add(tA.as<HB>(), tB.as<HB>(), tC.as<HB>(), no, -1.0, L.R, XY.R);
      Dev tB2 = make_tab({{&XY, no, 1, nq}});
      add(tC.as<HB>(), tB2.as<HB>(), tC.as<HB>(), nq, -1.0, nx.R, XY.R);
    }
    // overflow / singular checks (one sync per level)
    int h_ovf = 0;
    std::vector<int> hs(std::max(ne, 1));
    {
      if (stats_off) *stats_off = stats_launch(nx);
      const size_t off = hmap_take((size_t)ne + 1);
      CK(launch_copy_i32(hmap_d + off, ovf.as<int>(), 1, st));
      CK(launch_copy_i32(hmap_d + off + 1, sg, (long long)ne, st));
      CK(cudaStreamSynchronize(st));
      h_ovf = hmap[off];
      memcpy(hs.data(), hmap + off + 1, sizeof(int) * ne);
      for (const Pend& p : pend) memcpy(p.out->data(), hmap + p.off, p.n * sizeof(int));
      pend.clear();
      hmap_used = 0;
    }
    CK(cudaGetLastError());
    // singular leaves: report the first block in inversion order
    int bad = -1;
    for (int k = 0; k < ne; ++k) {
      int e = perm ? perm[k] : order ? ne - 1 - k : k;
      if (hs[e] != INT_MAX) { bad = e; break; }
    }
    if (dlev) {
      // every rank learns of a singular pivot anywhere; capacities agree
      const long long any = tp->allreduce_max(bad >= 0 ? 1 : 0, st);
      if (any && bad < 0) throw SingularError("singular dense leaf on another rank");
      h_ovf = (int)tp->allreduce_max(h_ovf, st);
    }
    if (bad >= 0) {
      int pos = hs[bad];
      std::vector<int> lv;
      for (int v = 0; v < ht.nnodes; ++v)
        if (ht.isleaf[v]) lv.push_back(v);
      std::sort(lv.begin(), lv.end(), [&](int x, int y) { return ht.lo[x] < ht.lo[y]; });
      int v = lv[pos];
      char buf[256];
      snprintf(buf, sizeof(buf),
               "singular dense leaf on index range [%d,%d): level %d, pivot block %d",
               ht.lo[v], ht.hi[v], lvl, first + 2 * bad);
      throw SingularError(buf);
    }
    if (dbg()) {
      static auto t_prev = std::chrono::steady_clock::now();
      auto now = std::chrono::steady_clock::now();
      fprintf(stderr, "[acr r%d] level %d m=%d/%d Rout=%d overflow=%d host_ms=%.2f\n", me(), lvl,
              mm, mg, Rout, h_ovf,
              std::chrono::duration<double, std::milli>(now - t_prev).count());
      t_prev = now;
    }
    if (h_ovf >= (1 << 28) && h_ovf < (1 << 29)) {
      // a leaf of the lifted level was not tridiagonal after all: redo the
      // level with the dense leaf inverse (never seen; the check is the guard)
      tri_ok = false;
      need = -1;
      return false;
    }
    if (h_ovf) {
      if (h_ovf >= (1 << 29)) throw InternalError("truncation work area too small");
      if (h_ovf > 4 * n + 64) throw InternalError("implausible rank " + std::to_string(h_ovf));
      need = h_ovf;
      return false;
    }
    // keep the level's couplings for the solve sweep (copies when the input
    // level must stay intact: the stepwise API is pure like the reference)
    if (keep_input) {
      rec.E = clone(L.E);
      rec.F = clone(L.F);
    } else {
      rec.E = std::move(L.E);
      rec.F = std::move(L.F);
    }
    return true;
  }

  // merges scheduled before reducing level l (progressive consolidation):
  // a retiring rank sends its whole window (D, E, F) to the active rank that
  // takes it over and returns false; a growing rank receives and
  // concatenates.  Windows are contiguous, so the merged level is the two
  // windows back to back.
  bool apply_merges(Level& L, int l) {
    const int r = me();
    for (const MergeStep& ms : msteps) {
      if (ms.lvl != l) continue;
      const bool was = ms.before[r + 1] > ms.before[r];
      if (!was) continue;
      const bool now = ms.after[r + 1] > ms.after[r];
      std::vector<Msg> msgs;
      if (!now) {
        const int dst = owner(ms.after, ms.before[r]);
        range_msgs(msgs, L.D, 0, L.m, dst, true);
        range_msgs(msgs, L.E, 0, L.m, dst, true);
        range_msgs(msgs, L.F, 0, L.m, dst, true);
        tp->exchange(msgs, st);
        CK(cudaStreamSynchronize(st));
        L = Level();
        return false;
      }
      if (ms.after[r + 1] == ms.before[r + 1]) continue;   // not involved
      Level G;
      G.m = ms.after[r + 1] - ms.after[r];
      G.first = L.first;
      G.mg = L.mg;
      G.R = L.R;
      G.lvl = L.lvl;
      for (Batch* d : {&G.D, &G.E, &G.F}) d->alloc(ht, G.m, G.R, st);
      auto cp = [&](Batch& dst, const Batch& src, int cnt) {
        CK(cudaMemcpyAsync(dst.leaf.p, src.leaf.p, sizeof(double) * src.sl * cnt,
                           cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(dst.U.p, src.U.p, sizeof(double) * src.sf * cnt,
                           cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(dst.V.p, src.V.p, sizeof(double) * src.sf * cnt,
                           cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(dst.rk.p, src.rk.p, sizeof(int) * src.sr * cnt,
                           cudaMemcpyDeviceToDevice, st));
      };
      cp(G.D, L.D, L.m);
      cp(G.E, L.E, L.m);
      cp(G.F, L.F, L.m);
      for (int q = r + 1; q + 1 < (int)ms.before.size(); ++q) {
        const int c = ms.before[q + 1] - ms.before[q];
        if (c <= 0) continue;
        if (ms.before[q] >= ms.after[r + 1]) break;
        const int off = ms.before[q] - ms.after[r];
        range_msgs(msgs, G.D, off, c, q, false);
        range_msgs(msgs, G.E, off, c, q, false);
        range_msgs(msgs, G.F, off, c, q, false);
      }
      tp->exchange(msgs, st);
      L = std::move(G);
    }
    return true;
  }

  // a rank that retired before level l still takes part in the level's
  // collectives (capacity and singular / overflow agreement), contributing
  // neutral values, so the active ranks' all-reduces complete
  void shadow_level(int l) {
    if (nactive(l) <= 1) return;
    tp->allreduce_max(0, st);                                 // Rout
    while (true) {
      if (tp->allreduce_max(0, st)) throw SingularError("singular dense leaf on another rank");
      const long long ov = tp->allreduce_max(0, st);
      if (!ov) break;
      if (ov >= (1 << 29) || ov > 4 * n + 64) throw InternalError("truncation overflow on another rank");
    }
  }

  // ---- factor ----
  void factor(const double* sub, const double* diag, const double* sup,
              const double* E, const double* F, int order) {
    // a previous factor that threw between fetch_ranks and sync_fetch left
    // entries pointing into its (gone) host vectors
    pend.clear();
    hmap_used = 0;
    recs.clear();
    kept.clear();
    prof.clear();
    launches = 0;
    prof_reset();
    factored = false;
    ff_ready = false;
    const bool fused = frhs != nullptr && nranks() == 1 && !prof_on;
    if (!ovf.p) ovf.alloc(sizeof(int), st);
    sing.alloc(sizeof(int) * std::max(m, 1), st);
    if (!ev0) {
      CK(cudaEventCreate(&ev0));
      CK(cudaEventCreate(&ev1));
    }
    CK(cudaEventRecord(ev0, st));
    const int P = nranks();
    schedule();
    first0 = P > 1 ? bnd0[me()] : 0;
    mloc0 = P > 1 ? bnd0[me() + 1] - bnd0[me()] : m;
    Level L;
    lift(L, first0, mloc0, sub, diag, sup, E, F);
    if (fused) fwd_begin();
    std::vector<int> dR, eR, fR;
    int maxr = 1;
    int lvl = 0;
    bool alive = true;
    auto ranks_of = [&](bool prof_it) {
      const size_t off = stats_launch(L);
      sync_fetch();
      maxr = stats_read(off, prof_it);
    };
    ranks_of(true);
    while (true) {
      if (P > 1 && !msteps.empty()) {
        const int m_before = L.m;
        if (!apply_merges(L, lvl)) {
          alive = false;
          break;
        }
        if (L.m != m_before) ranks_of(false);
      }
      if (L.mg <= cutoff) break;
      const bool dlev = P > 1 && nactive(lvl) > 1;
      if (dlev) {
        nb_left = left_nb(lvl);
        nb_right = right_nb(lvl);
      }
      int Rout = rout_for(maxr, L.R);
      if (dlev) Rout = (int)tp->allreduce_max(Rout, st);
      Record rec;
      Level nx;
      int need = 0;
      int tries = 0;
      size_t soff = 0;
      while (!reduce(L, Rout, lvl, order, nx, rec, need, dlev, nullptr, false, &soff)) {
        if (need >= 0) Rout = std::max(need, 2 * Rout);
        rec = Record();
        nx = Level();
        if (++tries > 8) throw InternalError("rank capacity retries exhausted");
      }
      // the record's host rank tables (storage accounting) are fetched
      // lazily by storage_bytes; the next level's statistics came back with
      // reduce's one sync
      maxr = stats_read(soff, true);
      if (keep_levels) kept.push_back(std::move(L));
      L = std::move(nx);
      ++lvl;
      L.lvl = lvl;
      recs.push_back(std::move(rec));
      // the forward sweep starts FWD_LAG levels behind: the first levels are
      // throughput-bound and a concurrent sweep would only compete for the
      // SMs; from level FWD_LAG on, the factorisation is a latency chain that
      // leaves most of the GPU idle
      if (fused)
        while (fwd_next + fwd_lag <= lvl - 1) fwd_level(fwd_next++);
    }
    if (fused)
      while (fwd_next < (int)recs.size()) fwd_level(fwd_next++);
    if (!alive) {
      // retired at level lvl: shadow the collectives of the levels still
      // reduced by several ranks, then this rank's part is done
      for (int l = lvl; l < Lsched; ++l) shadow_level(l);
      CK(cudaEventRecord(ev1, st));
      CK(cudaStreamSynchronize(st));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, ev0, ev1));
      fms = ms;
      prof_collect();
      lastR = {{}, {}, {}};
      last = Level();
      factored = true;
      return;
    }
    // the final level's full rank tables (storage accounting), drained at
    // the end-of-factor sync
    fetch_ranks(L.D, dR);
    fetch_ranks(L.E, eR);
    fetch_ranks(L.F, fR);
    // cutoff: dense LU of the remaining system
    const int mc = L.m;
    Nc = mc * n;
    lu.alloc(sizeof(double) * (size_t)Nc * Nc, st);
    piv.alloc(sizeof(int) * Nc, st);
    if (!info.p) info.alloc(sizeof(int), st);
    {
      std::vector<int> rb, cb;
      int cntb = 0;
      for (int i = 0; i < mc; ++i) { rb.push_back(i); cb.push_back(i); ++cntb; }
      for (int i = 1; i < mc; ++i) { rb.push_back(i); cb.push_back(i - 1); ++cntb; }
      for (int i = 0; i + 1 < mc; ++i) { rb.push_back(i); cb.push_back(i + 1); ++cntb; }
      Dev tab = make_tab({{&L.D, 0, 1, mc}, {&L.E, 1, 1, mc - 1}, {&L.F, 0, 1, mc - 1}});
      Dev drc(sizeof(int) * 2 * cntb, st);
      std::vector<int> h(rb);
      h.insert(h.end(), cb.begin(), cb.end());
      CK(cudaMemcpyAsync(drc.p, h.data(), sizeof(int) * h.size(), cudaMemcpyHostToDevice, st));
      CK(cudaMemsetAsync(lu.p, 0, sizeof(double) * (size_t)Nc * Nc, st));
      CK(launch_todense(dt.T, tab.as<HB>(), cntb, drc.as<int>(), drc.as<int>() + cntb,
                        lu.as<double>(), Nc, st));
      kbegin(8);
      CK(lu_factor(lu.as<double>(), Nc, piv.as<int>(), info.as<int>(), nullptr, st));
      kend();
      if (prof_on) {   // 2/3 N^3 FLOP; the N x N factor read and written once per panel sweep
        hflops[8] += 2.0 / 3.0 * (double)Nc * Nc * Nc;
        hbytes[8] += 16.0 * (double)Nc * Nc;
      }
      lut_ok = false;
      launches += 1 + 4 * ((Nc + 31) / 32);
      int hinfo = 0;
      CK(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      if (fused) fwd_end();
      CK(cudaEventRecord(ev1, st));
      CK(cudaStreamSynchronize(st));
      drain_fetch();
      lastR = {dR, eR, fR};
      if (hinfo) throw SingularError("matrix is singular to working precision");
    }
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, ev0, ev1));
    fms = ms;
    prof_collect();
    last = std::move(L);
    factored = true;
  }

  // ---- solve (reference reduction.py:204-216, 305-311, 235-256) ----
  // tbuf: the phase-A buffer (nullptr: plan scratch slot 12); s: stream
  void hmat_full(const HB* H, int G, int R, Src X, Src Y, int k, double* tbuf = nullptr,
                 cudaStream_t s = nullptr) {
    if (G <= 0) return;
    MMJob J;
    memset(&J, 0, sizeof(J));
    J.H = H;
    J.X = X;
    J.Y = Y;
    J.trans = 0;
    J.cols_fixed = k;
    J.alpha = 1.0;
    J.mu0 = 0;
    J.mu1 = 1;
    J.nA = ht.nA(0, 1);
    J.nB = ht.nleaves_under(0);
    J.RT = R;
    J.CT = k;
    J.tbuf = tbuf ? tbuf : scratch<double>(12, (size_t)G * std::max(J.nA, 1) * R * k);
    hmat(&J, 1, G, s ? s : st);
  }

  // E / F of the lifted level are diagonal (from_diagonal, hodlr.py:294-314):
  // their products with a right-hand-side panel are row scalings (bitwise the
  // dense leaf products), reading n values per block instead of n x bw
  void hmat_full_d(bool diag, const HB* H, int G, int R, Src X, Src Y, int k,
                   double* tbuf = nullptr, cudaStream_t s = nullptr) {
    static const bool off = getenv("ACR_NO_SOLVE_DIAG") != nullptr;   // A/B aid
    if (!diag || off) return hmat_full(H, G, R, X, Y, k, tbuf, s);
    if (G <= 0) return;
    MMJob J;
    memset(&J, 0, sizeof(J));
    J.H = H;
    J.X = X;
    J.Y = Y;
    J.cols_fixed = k;
    J.alpha = 1.0;
    J.mu0 = 0;
    J.mu1 = 1;
    kbegin(3);
    CK(launch_hmat_diag(dt.T, J, G, s ? s : st));
    kend();
    ++launches;
  }

  // ---- forward sweep fused into factor() (single GPU): right after level
  //      l's record is complete, its RHS update (reduction.py:204-216) runs
  //      on a side stream, overlapping the factorisation of the next levels
  //      (the upper levels leave the GPU mostly idle).  Every buffer is
  //      allocated on the plan's stream before the event the side stream
  //      waits for, and kept alive until the join at the end of factor(). ----
  const double* frhs = nullptr;   // right-hand side of the next factor (acr_factor_rhs)
  int fk = 0;
  std::vector<Dev> ffs;           // f of every level, internal layout
  bool ff_ready = false;
  int ff_k = 0;
  cudaStream_t stf = nullptr;
  cudaEvent_t evfl = nullptr, evfj = nullptr;
  std::vector<Dev> fkeep;         // tables / temporaries of the fused levels
  int fwd_next = 0;               // next level whose forward sweep is issued
  int fwd_lag = 5;                // levels the sweep trails the factorisation (ACR_FWD_LAG; measured 0..5: 5 best)

  void fwd_begin() {
    if (!stf) {
      make_stream(&stf, false);
      CK(cudaEventCreateWithFlags(&evfl, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&evfj, cudaEventDisableTiming));
    }
    // an earlier fused factor that failed may have left work on the side
    // stream that reads these buffers: order their release after it
    CK(cudaEventRecord(evfj, stf));
    CK(cudaStreamWaitEvent(st, evfj, 0));
    ffs.clear();
    fkeep.clear();
    ff_ready = false;
    fwd_next = 0;
    if (const char* e = getenv("ACR_FWD_LAG")) fwd_lag = atoi(e);
    int L = 0;
    for (int mg = m; mg > cutoff; mg /= 2) ++L;
    ffs.resize(L + 1);
    const long long kn = (long long)fk * n;
    ffs[0].alloc(sizeof(double) * kn * std::max(m, 1), st);
    CK(launch_rhs_in(frhs, m * n, fk, n, ffs[0].as<double>(), st));
    ++launches;
  }

  void fwd_level(int l) {
    Record& r = recs[l];
    const int k = fk;
    const long long kn = (long long)k * n;
    const int mm = r.m, ne = (mm + 1) / 2, no = mm / 2;
    int nq = 0;
    for (int j = 1; j < mm; j += 2)
      if (r.first + j + 1 <= r.mg - 1) ++nq;
    Dev z(sizeof(double) * kn * (std::max(ne, 1) + 1), st);
    Dev a(sizeof(double) * kn * std::max(no, 1), st);
    Dev bb(sizeof(double) * kn * std::max(nq, 1), st);
    ffs[l + 1].alloc(sizeof(double) * kn * std::max(no, 1), st);
    const long long nA = std::max(ht.nA(0, 1), 1);
    Dev t1(sizeof(double) * (size_t)std::max(ne, 1) * nA * r.Dinv.R * k, st);
    Dev t2(sizeof(double) * (size_t)std::max(no, 1) * nA * r.E.R * k, st);
    Dev t3(sizeof(double) * (size_t)std::max(nq, 1) * nA * r.F.R * k, st);
    Dev tDi = make_tab({{&r.Dinv, 0, 1, ne}});
    Dev tE = make_tab({{&r.E, 1, 2, no}});
    Dev tF = make_tab({{&r.F, 1, 2, nq}});
    CK(cudaEventRecord(evfl, st));
    CK(cudaStreamWaitEvent(stf, evfl, 0));
    double* fl = ffs[l].as<double>();
    hmat_full(tDi.as<HB>(), ne, r.Dinv.R, s_pan(fl, 2 * kn, k), s_pan(z.as<double>(), kn, k), k,
              t1.as<double>(), stf);
    hmat_full_d(r.diagEF, tE.as<HB>(), no, r.E.R, s_pan(z.as<double>(), kn, k), s_pan(a.as<double>(), kn, k),
              k, t2.as<double>(), stf);
    hmat_full_d(r.diagEF, tF.as<HB>(), nq, r.F.R, s_pan(z.as<double>() + kn, kn, k),
              s_pan(bb.as<double>(), kn, k), k, t3.as<double>(), stf);
    double* fn = ffs[l + 1].as<double>();
    CK(launch_rhs_combine(fl + kn, 2 * kn, a.as<double>(), kn, bb.as<double>(), kn, fn, kn, nq,
                          (int)kn, stf));
    CK(launch_rhs_combine(fl + kn + 2 * kn * nq, 2 * kn, a.as<double>() + kn * nq, kn, nullptr, 0,
                          fn + kn * nq, kn, no - nq, (int)kn, stf));
    launches += 2;
    for (Dev* d : {&z, &a, &bb, &t1, &t2, &t3, &tDi, &tE, &tF}) fkeep.push_back(std::move(*d));
  }

  void fwd_end() {
    CK(cudaEventRecord(evfj, stf));
    CK(cudaStreamWaitEvent(st, evfj, 0));
    fkeep.clear();                 // released on st, ordered after the side stream's work
    ff_ready = true;
    ff_k = fk;
  }

  // rhs == nullptr: back-substitution after a factorisation that ran the
  // forward sweep of its right-hand side (acr_factor_rhs / acr_solve_back)
  void solve(const double* rhs, int k, double* u) {
    if (!factored) throw ArgError("acr_solve called before a successful acr_factor");
    const bool fused = rhs == nullptr;
    if (fused) {
      if (!ff_ready) throw ArgError("acr_solve_back needs a preceding acr_factor_rhs");
      k = ff_k;
    }
    if (!sev0) {
      CK(cudaEventCreate(&sev0));
      CK(cudaEventCreate(&sev1));
    }
    CK(cudaEventRecord(sev0, st));
    const long long kn = (long long)k * n;
    const int P = nranks();
    const int Lt = P > 1 ? Lsched : (int)recs.size();   // level of the cutoff system
    const bool root = me() == 0;
    std::vector<Dev> f(Lt + 1);
    if (fused) {
      f = std::move(ffs);            // consumed: one back-substitution per fused factor
      ff_ready = false;
    } else {
      f[0].alloc(sizeof(double) * kn * std::max(mloc0, 1), st);
      CK(launch_rhs_in(rhs + (long long)first0 * n * k, mloc0 * n, k, n, f[0].as<double>(), st));
      ++launches;
    }
    // windows (block counts) this rank holds at level l before / after merges
    auto wcount = [&](const std::vector<int>& b) { return b[me() + 1] - b[me()]; };
    int lret = Lt;                     // level at which this rank retired (Lt: never)
    // forward sweep (reduction.py:204-216) with the factor's merges replayed
    for (int l = 0; l <= Lt && !fused; ++l) {
      if (P > 1) {
        bool out = false;
        for (const MergeStep& ms : msteps) {
          if (ms.lvl != l || wcount(ms.before) <= 0) continue;
          std::vector<Msg> msgs;
          if (wcount(ms.after) <= 0) {
            msgs.push_back({owner(ms.after, ms.before[me()]), f[l].p,
                            sizeof(double) * kn * wcount(ms.before), true});
            tp->exchange(msgs, st);
            out = true;
            break;
          }
          if (ms.after[me() + 1] == ms.before[me() + 1]) continue;
          Dev g(sizeof(double) * kn * wcount(ms.after), st);
          CK(cudaMemcpyAsync(g.p, f[l].p, sizeof(double) * kn * wcount(ms.before),
                             cudaMemcpyDeviceToDevice, st));
          for (int q = me() + 1; q + 1 < (int)ms.before.size(); ++q) {
            const int c = ms.before[q + 1] - ms.before[q];
            if (c <= 0) continue;
            if (ms.before[q] >= ms.after[me() + 1]) break;
            msgs.push_back({q, g.as<double>() + kn * (ms.before[q] - ms.after[me()]),
                            sizeof(double) * kn * c, false});
          }
          tp->exchange(msgs, st);
          f[l] = std::move(g);
        }
        if (out) {
          lret = l;
          break;
        }
      }
      if (l == Lt) break;
      Record& r = recs[l];
      const bool dlev = P > 1 && nactive(l) > 1;
      const int mm = r.m, ne = (mm + 1) / 2, no = mm / 2;
      int nq = 0;
      for (int j = 1; j < mm; j += 2)
        if (r.first + j + 1 <= r.mg - 1) ++nq;
      double* fl = f[l].as<double>();
      Dev z(sizeof(double) * kn * (std::max(ne, 1) + 1), st);   // + halo slot
      Dev a(sizeof(double) * kn * std::max(no, 1), st);
      Dev bb(sizeof(double) * kn * std::max(nq, 1), st);
      Dev tDi = make_tab({{&r.Dinv, 0, 1, ne}});
      hmat_full(tDi.as<HB>(), ne, r.Dinv.R, s_pan(fl, 2 * kn, k), s_pan(z.as<double>(), kn, k), k);
      if (dlev) {
        std::vector<Msg> msgs;
        if (r.first > 0) msgs.push_back({left_nb(l), z.p, sizeof(double) * kn, true});
        if (r.right) msgs.push_back({right_nb(l), z.as<double>() + kn * ne, sizeof(double) * kn, false});
        tp->exchange(msgs, st);
      }
      Dev tE = make_tab({{&r.E, 1, 2, no}});
      hmat_full_d(r.diagEF, tE.as<HB>(), no, r.E.R, s_pan(z.as<double>(), kn, k), s_pan(a.as<double>(), kn, k), k);
      // F_j z_{j+1}: z index i+1 (the halo slot ne for the right neighbour's block)
      Dev tF = make_tab({{&r.F, 1, 2, nq}});
      hmat_full_d(r.diagEF, tF.as<HB>(), nq, r.F.R, s_pan(z.as<double>() + kn, kn, k), s_pan(bb.as<double>(), kn, k), k);
      f[l + 1].alloc(sizeof(double) * kn * std::max(no, 1), st);
      double* fn = f[l + 1].as<double>();
      CK(launch_rhs_combine(fl + kn, 2 * kn, a.as<double>(), kn, bb.as<double>(), kn, fn, kn, nq, (int)kn, st));
      CK(launch_rhs_combine(fl + kn + 2 * kn * nq, 2 * kn, a.as<double>() + kn * nq, kn, nullptr, 0,
                            fn + kn * nq, kn, no - nq, (int)kn, st));
      launches += 2;
    }
    std::vector<Dev> uu(Lt + 1);
    if (root) {
      // cutoff solve (reduction.py:305-310)
      const int mc = last.m;
      uu[Lt].alloc(sizeof(double) * kn * std::max(mc, 1), st);
      Dev B(sizeof(double) * (size_t)Nc * k, st);
      for (int i = 0; i < mc; ++i)
        CK(cudaMemcpy2DAsync(B.as<double>() + (size_t)i * n, sizeof(double) * Nc,
                             f[Lt].as<double>() + i * kn, sizeof(double) * n,
                             sizeof(double) * n, k, cudaMemcpyDeviceToDevice, st));
      // transposed LU and the row order after the interchanges: once per factor
      const size_t lut_bytes = sizeof(double) * (size_t)Nc * Nc + sizeof(int) * (size_t)Nc;
      const bool use_perm = (size_t)Nc * sizeof(int) <= 160 * 1024;
      if (!lut_ok) {
        if (lut.n < lut_bytes) lut.alloc(lut_bytes, st);
        CK(lu_transpose(lu.as<double>(), Nc, lut.as<double>(), st));
        ++launches;
        if (use_perm) {
          CK(lu_perm(piv.as<int>(), Nc, reinterpret_cast<int*>(lut.as<double>() + (size_t)Nc * Nc), st));
          ++launches;
        }
        lut_ok = true;
      }
      CK(lu_solve(lu.as<double>(), lut.as<double>(), Nc, piv.as<int>(), B.as<double>(), k, st,
                  use_perm ? reinterpret_cast<const int*>(lut.as<double>() + (size_t)Nc * Nc) : nullptr));
      ++launches;
      for (int i = 0; i < mc; ++i)
        CK(cudaMemcpy2DAsync(uu[Lt].as<double>() + i * kn, sizeof(double) * n,
                             B.as<double>() + (size_t)i * n, sizeof(double) * Nc,
                             sizeof(double) * n, k, cudaMemcpyDeviceToDevice, st));
    }
    // back-substitution (reduction.py:235-256): undo level l's merges (the
    // solution goes back to the ranks that held those blocks), then level l-1
    for (int l = lret; l >= 0; --l) {
      if (P > 1) {
        for (auto it = msteps.rbegin(); it != msteps.rend(); ++it) {
          const MergeStep& ms = *it;
          if (ms.lvl != l || wcount(ms.before) <= 0) continue;
          std::vector<Msg> msgs;
          if (wcount(ms.after) <= 0) {             // this rank retired here: receive
            uu[l].alloc(sizeof(double) * kn * wcount(ms.before), st);
            msgs.push_back({owner(ms.after, ms.before[me()]), uu[l].p,
                            sizeof(double) * kn * wcount(ms.before), false});
            tp->exchange(msgs, st);
            continue;
          }
          if (ms.after[me() + 1] == ms.before[me() + 1]) continue;
          for (int q = me() + 1; q + 1 < (int)ms.before.size(); ++q) {
            const int c = ms.before[q + 1] - ms.before[q];
            if (c <= 0) continue;
            if (ms.before[q] >= ms.after[me() + 1]) break;
            msgs.push_back({q, uu[l].as<double>() + kn * (ms.before[q] - ms.after[me()]),
                            sizeof(double) * kn * c, true});
          }
          tp->exchange(msgs, st);
          Dev mine(sizeof(double) * kn * std::max(wcount(ms.before), 1), st);
          CK(cudaMemcpyAsync(mine.p, uu[l].p, sizeof(double) * kn * wcount(ms.before),
                             cudaMemcpyDeviceToDevice, st));
          CK(cudaStreamSynchronize(st));
          uu[l] = std::move(mine);
        }
      }
      if (l == 0) break;
      const int lv = l - 1;
      Record& r = recs[lv];
      const bool dlev = P > 1 && nactive(lv) > 1;
      const int mm = r.m, ne = (mm + 1) / 2, no = mm / 2;
      uu[lv].alloc(sizeof(double) * kn * mm, st);
      double* ul = uu[lv].as<double>();
      if (no)
        CK(cudaMemcpy2DAsync(ul + kn, sizeof(double) * 2 * kn, uu[l].as<double>(),
                             sizeof(double) * kn, sizeof(double) * kn, no,
                             cudaMemcpyDeviceToDevice, st));
      Dev uleft(sizeof(double) * kn, st);
      if (dlev) {
        // the left neighbour's last odd block feeds our first even block
        std::vector<Msg> msgs;
        if (r.right) msgs.push_back({right_nb(lv), ul + kn * (mm - 1), sizeof(double) * kn, true});
        if (r.first > 0) msgs.push_back({left_nb(lv), uleft.p, sizeof(double) * kn, false});
        tp->exchange(msgs, st);
      }
      int nb = 0;
      for (int i = 0; i <= mm - 1; i += 2)
        if (r.first + i <= r.mg - 2) ++nb;
      Dev a(sizeof(double) * kn * ne, st);
      Dev b(sizeof(double) * kn * ne, st);
      CK(cudaMemsetAsync(a.p, 0, sizeof(double) * kn * ne, st));
      CK(cudaMemsetAsync(b.p, 0, sizeof(double) * kn * ne, st));
      Dev tE = make_tab({{&r.E, 2, 2, ne - 1}});
      hmat_full_d(r.diagEF, tE.as<HB>(), ne - 1, r.E.R, s_pan(ul + kn, 2 * kn, k), s_pan(a.as<double>() + kn, kn, k), k);
      if (r.first > 0) {
        Dev tE0 = make_tab({{&r.E, 0, 1, 1}});
        hmat_full_d(r.diagEF, tE0.as<HB>(), 1, r.E.R, s_pan(uleft.as<double>(), kn, k),
                  s_pan(a.as<double>(), kn, k), k);
      }
      Dev tF = make_tab({{&r.F, 0, 2, nb}});
      hmat_full_d(r.diagEF, tF.as<HB>(), nb, r.F.R, s_pan(ul + kn, 2 * kn, k), s_pan(b.as<double>(), kn, k), k);
      Dev rr(sizeof(double) * kn * ne, st);
      CK(launch_rhs_combine(f[lv].as<double>(), 2 * kn, a.as<double>(), kn, b.as<double>(), kn,
                            rr.as<double>(), kn, ne, (int)kn, st));
      ++launches;
      Dev tDi = make_tab({{&r.Dinv, 0, 1, ne}});
      hmat_full(tDi.as<HB>(), ne, r.Dinv.R, s_pan(rr.as<double>(), kn, k), s_pan(ul, 2 * kn, k), k);
      uu[l].release();
    }
    CK(launch_u_out(uu[0].as<double>(), mloc0 * n, k, n, u + (long long)first0 * n * k, st));
    ++launches;
    CK(cudaEventRecord(sev1, st));
    // asynchronous on the caller's stream: the elapsed time is read when
    // asked for (solve_ms), not by blocking the host here
    sms_pending = true;
  }

  double solve_ms() {
    if (sms_pending) {
      CK(cudaEventSynchronize(sev1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, sev0, sev1));
      sms = ms;
      sms_pending = false;
    }
    return sms;
  }

  // ---- stepwise API: the reference's lower-level surface (lift_system,
  //      reduce_level, forward RHS update, backsubstitute; reduction.py:156-256)
  //      on device-resident levels and records held by handle ----
  std::map<int, Level> slev;
  std::map<int, Record> srec;
  int snext = 1;

  void step_prep() {
    if (!ovf.p) ovf.alloc(sizeof(int), st);
    if (sing.n < sizeof(int) * (size_t)std::max(m, 1)) sing.alloc(sizeof(int) * std::max(m, 1), st);
  }

  int step_lift(const double* sub, const double* diag, const double* sup, const double* E,
                const double* F) {
    step_prep();
    Level L;
    lift(L, 0, m, sub, diag, sup, E, F);
    const int id = snext++;
    slev[id] = std::move(L);
    return id;
  }

  Level& step_level(int id) {
    auto it = slev.find(id);
    if (it == slev.end()) throw ArgError("unknown level handle " + std::to_string(id));
    return it->second;
  }
  Record& step_record(int id) {
    auto it = srec.find(id);
    if (it == srec.end()) throw ArgError("unknown record handle " + std::to_string(id));
    return it->second;
  }

  // one level of reduce_level(level, tol, inversion_order) with the given
  // tolerance; the input level is left intact
  void step_reduce(int lid, double eps_, int cap_, const int* perm, int* nid, int* rid) {
    Level& L = step_level(lid);
    if (L.m < 2) throw ArgError("need at least 2 blocks to reduce, got " + std::to_string(L.m));
    const int ne = (L.m + 1) / 2;
    if (perm) {
      std::vector<int> q(perm, perm + ne);
      std::sort(q.begin(), q.end());
      for (int i = 0; i < ne; ++i)
        if (q[i] != i) throw ArgError("inversion_order must permute the even-block indices");
    }
    step_prep();
    const double eps0 = eps;
    const int cap0 = cap;
    eps = eps_;
    cap = cap_;
    struct Restore {
      Plan* p;
      double e;
      int c;
      ~Restore() { p->eps = e; p->cap = c; }
    } restore{this, eps0, cap0};
    std::vector<int> dR, eR, fR;
    fetch_ranks(L.D, dR);
    fetch_ranks(L.E, eR);
    fetch_ranks(L.F, fR);
    sync_fetch();
    const int maxr = std::max({max_rank_of(dR), max_rank_of(eR), max_rank_of(fR), 1});
    int Rout = rout_for(maxr, L.R);
    Record rec;
    Level nx;
    int need = 0, tries = 0;
    while (!reduce(L, Rout, L.lvl, 0, nx, rec, need, false, perm, true)) {
      if (need >= 0) Rout = std::max(need, 2 * Rout);
      rec = Record();
      nx = Level();
      if (++tries > 8) throw InternalError("rank capacity retries exhausted");
    }
    nx.lvl = L.lvl + 1;
    fetch_ranks(rec.Dinv, rec.hDinv);
    fetch_ranks(rec.E, rec.hE);
    fetch_ranks(rec.F, rec.hF);
    sync_fetch();
    *nid = snext++;
    slev[*nid] = std::move(nx);
    *rid = snext++;
    srec[*rid] = std::move(rec);
  }

  // forward RHS update of one level (reduction.py:204-216): f (mm*n, k) of the
  // level -> fo (no*n, k) of the reduced level, row-major like acr_solve
  void step_rhs(int rid, const double* f, int k, double* fo) {
    Record& r = step_record(rid);
    const long long kn = (long long)k * n;
    const int mm = r.m, ne = (mm + 1) / 2, no = mm / 2;
    int nq = 0;
    for (int j = 1; j < mm; j += 2)
      if (j + 1 <= mm - 1) ++nq;
    Dev fl(sizeof(double) * kn * mm, st);
    CK(launch_rhs_in(f, mm * n, k, n, fl.as<double>(), st));
    Dev z(sizeof(double) * kn * (ne + 1), st), a(sizeof(double) * kn * std::max(no, 1), st),
        bb(sizeof(double) * kn * std::max(nq, 1), st);
    Dev tDi = make_tab({{&r.Dinv, 0, 1, ne}});
    hmat_full(tDi.as<HB>(), ne, r.Dinv.R, s_pan(fl.as<double>(), 2 * kn, k),
              s_pan(z.as<double>(), kn, k), k);
    Dev tE = make_tab({{&r.E, 1, 2, no}});
    hmat_full_d(r.diagEF, tE.as<HB>(), no, r.E.R, s_pan(z.as<double>(), kn, k), s_pan(a.as<double>(), kn, k), k);
    Dev tF = make_tab({{&r.F, 1, 2, nq}});
    hmat_full_d(r.diagEF, tF.as<HB>(), nq, r.F.R, s_pan(z.as<double>() + kn, kn, k),
              s_pan(bb.as<double>(), kn, k), k);
    Dev fn(sizeof(double) * kn * std::max(no, 1), st);
    const double* f1 = fl.as<double>() + kn;
    CK(launch_rhs_combine(f1, 2 * kn, a.as<double>(), kn, bb.as<double>(), kn, fn.as<double>(),
                          kn, nq, (int)kn, st));
    CK(launch_rhs_combine(f1 + 2 * kn * nq, 2 * kn, a.as<double>() + kn * nq, kn, nullptr, 0,
                          fn.as<double>() + kn * nq, kn, no - nq, (int)kn, st));
    if (no) CK(launch_u_out(fn.as<double>(), no * n, k, n, fo, st));
    CK(cudaStreamSynchronize(st));
  }

  // one back-substitution level (reduction.py:235-256): u of the odd blocks
  // (no*n, k) and the level's f (mm*n, k) -> u (mm*n, k)
  void step_backsub(int rid, const double* f, const double* uodd, int k, double* u) {
    Record& r = step_record(rid);
    const long long kn = (long long)k * n;
    const int mm = r.m, ne = (mm + 1) / 2, no = mm / 2;
    Dev fl(sizeof(double) * kn * mm, st), ul(sizeof(double) * kn * mm, st);
    CK(launch_rhs_in(f, mm * n, k, n, fl.as<double>(), st));
    Dev uo(sizeof(double) * kn * std::max(no, 1), st);
    if (no) {
      CK(launch_rhs_in(uodd, no * n, k, n, uo.as<double>(), st));
      CK(cudaMemcpy2DAsync(ul.as<double>() + kn, sizeof(double) * 2 * kn, uo.as<double>(),
                           sizeof(double) * kn, sizeof(double) * kn, no,
                           cudaMemcpyDeviceToDevice, st));
    }
    int nb = 0;
    for (int i = 0; i <= mm - 1; i += 2)
      if (i <= mm - 2) ++nb;
    Dev a(sizeof(double) * kn * ne, st), b(sizeof(double) * kn * ne, st), rr(sizeof(double) * kn * ne, st);
    CK(cudaMemsetAsync(a.p, 0, sizeof(double) * kn * ne, st));
    CK(cudaMemsetAsync(b.p, 0, sizeof(double) * kn * ne, st));
    double* up = ul.as<double>();
    Dev tE = make_tab({{&r.E, 2, 2, ne - 1}});
    hmat_full_d(r.diagEF, tE.as<HB>(), ne - 1, r.E.R, s_pan(up + kn, 2 * kn, k), s_pan(a.as<double>() + kn, kn, k), k);
    Dev tF = make_tab({{&r.F, 0, 2, nb}});
    hmat_full_d(r.diagEF, tF.as<HB>(), nb, r.F.R, s_pan(up + kn, 2 * kn, k), s_pan(b.as<double>(), kn, k), k);
    CK(launch_rhs_combine(fl.as<double>(), 2 * kn, a.as<double>(), kn, b.as<double>(), kn,
                          rr.as<double>(), kn, ne, (int)kn, st));
    Dev tDi = make_tab({{&r.Dinv, 0, 1, ne}});
    hmat_full(tDi.as<HB>(), ne, r.Dinv.R, s_pan(rr.as<double>(), kn, k), s_pan(up, 2 * kn, k), k);
    CK(launch_u_out(up, mm * n, k, n, u, st));
    CK(cudaStreamSynchronize(st));
  }

  // storage of one block for export: which 0 D, 1 E, 2 F of a level handle;
  // 3 Dinv, 4 E, 5 F of a record handle
  const Batch* step_batch(int handle, int which) {
    if (which <= 2) {
      Level& L = step_level(handle);
      return which == 0 ? &L.D : which == 1 ? &L.E : &L.F;
    }
    Record& r = step_record(handle);
    return which == 3 ? &r.Dinv : which == 4 ? &r.E : &r.F;
  }

  // raw storage of one block (leaf n x bw, U/V nd x R x n column panels,
  // ranks 2 x nnodes) into caller device buffers; null buffers: sizes only
  void export_block(const Batch* b, int block, double* leaf, double* U, double* V, int* rk,
                    int* R_out, int* cnt_out) {
    if (R_out) *R_out = b->R;
    if (cnt_out) *cnt_out = b->cnt;
    if (!leaf && !U && !V && !rk) return;
    if (block < 0 || block >= b->cnt) throw ArgError("block out of range");
    if (leaf) CK(cudaMemcpyAsync(leaf, b->leaf.as<double>() + block * b->sl, sizeof(double) * b->sl,
                                 cudaMemcpyDeviceToDevice, st));
    if (U) CK(cudaMemcpyAsync(U, b->U.as<double>() + block * b->sf, sizeof(double) * b->sf,
                              cudaMemcpyDeviceToDevice, st));
    if (V) CK(cudaMemcpyAsync(V, b->V.as<double>() + block * b->sf, sizeof(double) * b->sf,
                              cudaMemcpyDeviceToDevice, st));
    if (rk) CK(cudaMemcpyAsync(rk, b->rk.as<int>() + block * b->sr, sizeof(int) * b->sr,
                               cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
  }

  // factor()'s storage: which 0 D, 1 E, 2 F of level `level`, 3 Dinv
  const Batch* factor_batch(int level, int which) {
    const int L = (int)recs.size();
    if (which == 3) {
      if (level < 0 || level >= L) throw ArgError("level out of range");
      return &recs[level].Dinv;
    }
    if (which < 0 || which > 3) throw ArgError("which must be 0..3");
    if (level == L) return which == 0 ? &last.D : which == 1 ? &last.E : &last.F;
    if (level >= 0 && level < (int)kept.size())
      return which == 0 ? &kept[level].D : which == 1 ? &recs[level].E : &recs[level].F;
    if (level >= 0 && level < L && which != 0) return which == 1 ? &recs[level].E : &recs[level].F;
    throw ArgError("level not retained (set option 1 before acr_factor)");
  }

  // the records' host rank tables, fetched on first use (the factor no
  // longer copies them out level by level)
  void ensure_rec_ranks() {
    bool any = false;
    for (auto& r : recs) {
      const std::pair<const Batch*, std::vector<int>*> t[3] = {
          {&r.Dinv, &r.hDinv}, {&r.E, &r.hE}, {&r.F, &r.hF}};
      for (auto& x : t) {
        if (!x.second->empty() || x.first->cnt <= 0) continue;
        x.second->resize((size_t)x.first->cnt * ht.nnodes * 2);
        CK(cudaMemcpyAsync(x.second->data(), x.first->rk.p, sizeof(int) * x.second->size(),
                           cudaMemcpyDeviceToHost, st));
        any = true;
      }
    }
    if (any) CK(cudaStreamSynchronize(st));
  }

  long long storage_bytes(int k) {
    ensure_rec_ranks();
    long long s = 0;
    const long long seg = 8LL * n * k;
    for (auto& r : recs) {
      const int mm = r.m, ne = (mm + 1) / 2;
      for (int e = 0; e < ne; ++e) {
        int i = 2 * e;
        s += hb_bytes(r.hDinv.data() + (size_t)e * ht.nnodes * 2);
        if (i >= 1) s += hb_bytes(r.hE.data() + (size_t)i * ht.nnodes * 2);
        if (i <= mm - 2) s += hb_bytes(r.hF.data() + (size_t)i * ht.nnodes * 2);
        s += seg;
      }
    }
    const int mc = last.m;
    for (int i = 0; i < mc; ++i) {
      s += hb_bytes(lastR[0].data() + (size_t)i * ht.nnodes * 2);
      if (i >= 1) s += hb_bytes(lastR[1].data() + (size_t)i * ht.nnodes * 2);
      if (i <= mc - 2) s += hb_bytes(lastR[2].data() + (size_t)i * ht.nnodes * 2);
      s += seg;
    }
    return s;
  }

  long long device_bytes() const {
    long long s = 0;
    for (auto& r : recs) s += r.Dinv.bytes() + r.E.bytes() + r.F.bytes();
    s += last.D.bytes() + last.E.bytes() + last.F.bytes();
    s += (long long)lu.n;
    return s;
  }
};

}  // namespace acr

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
using acr::Plan;

struct acr_plan {
  Plan* p;
};

// error text of the calling thread's last failed plan-less call (plans carry
// their own); thread-local so concurrent independent calls do
// not see each other's messages
static thread_local std::string g_err;

static int set_err(acr_plan_t* h, int code, const std::string& msg) {
  if (h && h->p) h->p->err = msg;
  g_err = msg;
  return code;
}

#define ACR_GUARD(h, ...)                                                   \
  try {                                                                     \
    __VA_ARGS__;                                                            \
  } catch (const acr::ArgError& e) {                                        \
    return set_err(h, ACR_EARG, e.what());                                  \
  } catch (const acr::SingularError& e) {                                   \
    return set_err(h, ACR_ESINGULAR, e.what());                             \
  } catch (const acr::CudaError& e) {                                       \
    return set_err(h, ACR_ECUDA, e.what());                                 \
  } catch (const std::exception& e) {                                       \
    return set_err(h, ACR_EINTERNAL, e.what());                             \
  }

extern "C" {

int acr_plan_create(int m, int n, int leaf_size, double eps, int max_rank_cap,
                    int cutoff_blocks, acr_plan_t** out) {
  if (!out) return set_err(nullptr, ACR_EARG, "null output handle");
  *out = nullptr;
  if (m < 1 || n < 2) return set_err(nullptr, ACR_EARG, "need m >= 1 and n >= 2");
  if (leaf_size < 1)
    return set_err(nullptr, ACR_EARG, "leaf_size must be >= 1, got " + std::to_string(leaf_size));
  if (!(eps > 0)) return set_err(nullptr, ACR_EARG, "eps must be > 0");
  if (max_rank_cap < 0) return set_err(nullptr, ACR_EARG, "max_rank_cap must be positive");
  if (cutoff_blocks < 1)
    return set_err(nullptr, ACR_EARG,
                   "cutoff_blocks must be >= 1, got " + std::to_string(cutoff_blocks));
  acr_plan_t* h = new acr_plan_t;
  h->p = nullptr;
  try {
    h->p = new Plan(m, n, leaf_size, eps, max_rank_cap, cutoff_blocks);
    if (h->p->ht.bw > 128) throw acr::ArgError("leaf blocks larger than 128 are not supported");
    cudaMemPool_t pool;
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      unsigned long long thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    h->p->dt.upload(h->p->ht, 0);
    acr::g_cache.plans++;
  } catch (const std::exception& e) {
    g_err = e.what();
    delete h->p;
    delete h;
    return ACR_ECUDA;
  }
  *out = h;
  return ACR_OK;
}

void acr_plan_destroy(acr_plan_t* h) {
  if (!h) return;
  if (h->p) {
    cudaStream_t st = h->p->st;
    cudaStreamSynchronize(st);
    delete h->p;
    if (--acr::g_cache.plans <= 0) {
      acr::g_cache.trim(st);
      cudaStreamSynchronize(st);
    }
  }
  delete h;
}

int acr_nccl_unique_id(void* out) {
  std::string e;
  if (acr::nccl_unique_id(out, &e)) return set_err(nullptr, ACR_ECUDA, e);
  return ACR_OK;
}

static int check_bounds(int m, int nranks, const int* bnd) {
  if (nranks < 1 || !bnd) return 0;
  if (bnd[0] != 0 || bnd[nranks] != m) return 0;
  for (int r = 0; r < nranks; ++r)
    if (bnd[r + 1] - bnd[r] < 1 || (bnd[r] & 1)) return 0;
  return 1;
}

int acr_plan_create_dist(int m, int n, int leaf_size, double eps, int max_rank_cap,
                         int cutoff_blocks, int rank, int nranks, const int* bnd0,
                         const void* nccl_id, acr_plan_t** out) {
  if (!check_bounds(m, nranks, bnd0) || rank < 0 || rank >= nranks)
    return set_err(nullptr, ACR_EARG, "bad rank partition");
  int rc = acr_plan_create(m, n, leaf_size, eps, max_rank_cap, cutoff_blocks, out);
  if (rc) return rc;
  Plan& P = *(*out)->p;
  P.bnd0.assign(bnd0, bnd0 + nranks + 1);
  if (nranks > 1) {
    std::string e;
    P.tp = acr::make_nccl(nccl_id, rank, nranks, &e);
    if (!P.tp) {
      acr_plan_destroy(*out);
      *out = nullptr;
      return set_err(nullptr, ACR_ECUDA, e);
    }
    P.own_tp = true;
  }
  return ACR_OK;
}

int acr_loopback_solve(int nranks, const int* bnd0, int m, int n, int leaf_size,
                       double eps, int max_rank_cap, int cutoff_blocks,
                       const double* D_sub, const double* D_diag, const double* D_sup,
                       const double* E, const double* F, const double* rhs, int nrhs,
                       double* u, double* factor_ms) {
  if (!check_bounds(m, nranks, bnd0)) return set_err(nullptr, ACR_EARG, "bad rank partition");
  acr::LoopbackHub hub(nranks);
  std::vector<int> rcs(nranks, 0);
  std::vector<std::string> errs(nranks);
  std::vector<double> fms(nranks, 0.0);
  int dev = 0;
  cudaGetDevice(&dev);
  std::vector<std::thread> th;
  for (int r = 0; r < nranks; ++r) {
    th.emplace_back([&, r] {
      cudaSetDevice(dev);
      cudaStream_t st;
      cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
      acr_plan_t* h = nullptr;
      int rc = acr_plan_create(m, n, leaf_size, eps, max_rank_cap, cutoff_blocks, &h);
      if (!rc) {
        Plan& P = *h->p;
        P.bnd0.assign(bnd0, bnd0 + nranks + 1);
        P.tp = acr::make_loopback(&hub, r);
        P.own_tp = true;
        rc = acr_factor(h, D_sub, D_diag, D_sup, E, F, 0, st);
        if (!rc) rc = acr_solve(h, rhs, nrhs, u, st);
        fms[r] = P.fms;
        if (rc) errs[r] = P.err;
      }
      rcs[r] = rc;
      acr_plan_destroy(h);
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    });
  }
  for (auto& t : th) t.join();
  double mx = 0;
  for (int r = 0; r < nranks; ++r) {
    mx = std::max(mx, fms[r]);
    if (rcs[r]) return set_err(nullptr, rcs[r], "rank " + std::to_string(r) + ": " + errs[r]);
  }
  if (factor_ms) *factor_ms = mx;
  return ACR_OK;
}

int acr_plan_set_option(acr_plan_t* h, int option, long long value) {
  if (!h || !h->p) return ACR_EARG;
  if (option == 1) {
    h->p->keep_levels = value != 0;
    return ACR_OK;
  }
  if (option == 2) {
    h->p->prof_on = value != 0;
    return ACR_OK;
  }
  if (option == 3) {
    h->p->force_pair = value != 0;
    return ACR_OK;
  }
  if (option == 4) {
    h->p->no_side = value != 0;
    return ACR_OK;
  }
  if (option == 5) {
    h->p->direct_max = (int)value;
    return ACR_OK;
  }
  if (option == 6) {
    h->p->warp_small = (int)value;
    return ACR_OK;
  }
  if (option == 8) {
    h->p->warp_sched = (int)value;
    return ACR_OK;
  }
  if (option == 9) {
    h->p->warp_rmax = (int)value;
    return ACR_OK;
  }
  if (option == 10) {
    h->p->warp_maxneed = value;
    return ACR_OK;
  }
  return set_err(h, ACR_EARG, "unknown option");
}

int acr_factor(acr_plan_t* h, const double* D_sub, const double* D_diag,
               const double* D_sup, const double* E, const double* F,
               int inversion_order, void* stream) {
  if (!h || !h->p) return set_err(h, ACR_EARG, "null plan");
  if (inversion_order != 0 && inversion_order != 1)
    return set_err(h, ACR_EARG, "unknown inversion_order");
  ACR_GUARD(h, {
    Plan& P = *h->p;
    P.match_priority((cudaStream_t)stream);
    P.use_stream((cudaStream_t)stream);
    P.factor(D_sub, D_diag, D_sup, E, F, inversion_order);
  });
  return ACR_OK;
}

int acr_solve(acr_plan_t* h, const double* rhs, int nrhs, double* u,
              void* stream) {
  if (!h || !h->p) return set_err(h, ACR_EARG, "null plan");
  if (nrhs < 1) return set_err(h, ACR_EARG, "nrhs must be >= 1");
  ACR_GUARD(h, {
    Plan& P = *h->p;
    P.use_stream((cudaStream_t)stream);
    P.solve(rhs, nrhs, u);
  });
  return ACR_OK;
}

int acr_factor_rhs(acr_plan_t* h, const double* D_sub, const double* D_diag,
                   const double* D_sup, const double* E, const double* F, int inversion_order,
                   const double* rhs, int nrhs, void* stream) {
  if (!h || !h->p) return set_err(h, ACR_EARG, "null plan");
  if (inversion_order != 0 && inversion_order != 1)
    return set_err(h, ACR_EARG, "unknown inversion_order");
  if (!rhs || nrhs < 1) return set_err(h, ACR_EARG, "need a right-hand side with nrhs >= 1");
  ACR_GUARD(h, {
    Plan& P = *h->p;
    if (P.nranks() > 1) throw acr::ArgError("acr_factor_rhs: single-GPU plans only");
    P.match_priority((cudaStream_t)stream);
    P.use_stream((cudaStream_t)stream);
    P.frhs = rhs;
    P.fk = nrhs;
    struct Clear {
      Plan& p;
      ~Clear() { p.frhs = nullptr; }
    } clear{P};
    P.factor(D_sub, D_diag, D_sup, E, F, inversion_order);
  });
  return ACR_OK;
}

int acr_solve_back(acr_plan_t* h, double* u, void* stream) {
  if (!h || !h->p) return set_err(h, ACR_EARG, "null plan");
  ACR_GUARD(h, {
    Plan& P = *h->p;
    P.use_stream((cudaStream_t)stream);
    P.solve(nullptr, 0, u);
  });
  return ACR_OK;
}

int acr_levels(const acr_plan_t* h) { return h && h->p ? (int)h->p->recs.size() : -1; }
int acr_cutoff_blocks(const acr_plan_t* h) { return h && h->p ? h->p->last.m : -1; }
int acr_tree_depths(const acr_plan_t* h) { return h && h->p ? h->p->ht.nd : -1; }

int acr_rank_profile(const acr_plan_t* h, int level, int* mx, double* mean) {
  if (!h || !h->p) return ACR_EARG;
  const Plan& P = *h->p;
  if (level < 0 || level >= (int)P.prof.size()) return ACR_EARG;
  for (int d = 0; d < P.ht.nd; ++d) {
    mx[d] = P.prof[level].mx[d];
    mean[d] = P.prof[level].mean[d];
  }
  return ACR_OK;
}

long long acr_storage_bytes(const acr_plan_t* h, int nrhs) {
  return h && h->p && h->p->factored ? h->p->storage_bytes(nrhs) : -1;
}
long long acr_device_bytes(const acr_plan_t* h) {
  return h && h->p ? h->p->device_bytes() : -1;
}
double acr_factor_ms(const acr_plan_t* h) { return h && h->p ? h->p->fms : -1.0; }
double acr_solve_ms(const acr_plan_t* h) {
  if (!h || !h->p) return -1.0;
  try {
    return h->p->solve_ms();
  } catch (...) {
    return -1.0;
  }
}
long long acr_kernel_launches(const acr_plan_t* h) { return h && h->p ? h->p->launches : -1; }

int acr_kernel_stats(const acr_plan_t* h, int cls, long long* launches,
                     double* ms, unsigned long long* counters) {
  if (!h || !h->p || cls < 0 || (cls >= Plan::NCLS && cls != 100)) return ACR_EARG;
  const Plan& P = *h->p;
  *launches = cls == 100 ? 0 : P.kcnt[cls];
  *ms = cls == 100 ? 0.0 : P.kms[cls];
  if (counters)
    for (int i = 0; i < 16; ++i) counters[i] = cls == 0 ? P.kctr[i] : 0;
  if (counters && cls > 0 && cls < Plan::NCLS) {
    counters[0] = (unsigned long long)P.hflops[cls];
    counters[1] = (unsigned long long)P.hbytes[cls];
    const int dev_slot = cls == 3 ? 150 : cls == 5 ? 152 : cls == 6 ? 154 : -1;
    if (dev_slot >= 0) {
      counters[0] = P.kctr[dev_slot];
      counters[1] = P.kctr[dev_slot + 1];
    }
  }
  if (counters && cls == 100)
    for (int i = 0; i < 256; ++i) counters[i] = P.kctr[i];
  return ACR_OK;
}

int acr_last_error(const acr_plan_t* h, char* buf, int len) {
  const std::string& s = (h && h->p) ? h->p->err : g_err;
  if (buf && len > 0) {
    strncpy(buf, s.c_str(), len - 1);
    buf[len - 1] = 0;
  }
  return (int)s.size();
}

int acr_global_error(char* buf, int len) {
  if (buf && len > 0) {
    strncpy(buf, g_err.c_str(), len - 1);
    buf[len - 1] = 0;
  }
  return (int)g_err.size();
}

int acr_block_to_dense(acr_plan_t* h, int level, int which, int block,
                       double* out, void* stream) {
  if (!h || !h->p) return ACR_EARG;
  ACR_GUARD(h, {
    Plan& P = *h->p;
    P.use_stream((cudaStream_t)stream);
    const acr::Batch* b = P.factor_batch(level, which);
    if (block < 0 || block >= b->cnt) throw acr::ArgError("block out of range");
    acr::Dev tab = P.make_tab({{b, block, 1, 1}});
    acr::Dev rc(sizeof(int) * 2, P.st);
    CK(cudaMemsetAsync(rc.p, 0, sizeof(int) * 2, P.st));
    CK(acr::launch_todense(P.dt.T, tab.as<acr::HB>(), 1, rc.as<int>(), rc.as<int>() + 1,
                           out, P.n, P.st));
    CK(cudaStreamSynchronize(P.st));
  });
  return ACR_OK;
}

int acr_residual(int m, int n, int k, const double* D_sub, const double* D_diag,
                 const double* D_sup, const double* E, const double* F,
                 const double* u, const double* f, double* out_r, double* out_f,
                 void* stream) {
  ACR_GUARD(nullptr, {
    cudaStream_t st = (cudaStream_t)stream;
    const int parts = 256;
    acr::Dev part(sizeof(double) * parts * k * 2, st);
    CK(acr::launch_residual(m, n, k, D_sub, D_diag, D_sup, E, F, u, f,
                            part.as<double>(), parts, st));
    std::vector<double> h((size_t)parts * k * 2);
    CK(cudaMemcpyAsync(h.data(), part.p, sizeof(double) * h.size(),
                       cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int c = 0; c < k; ++c) {
      double a = 0, b = 0;
      for (int p = 0; p < parts; ++p) {
        a += h[((size_t)p * k + c) * 2];
        b += h[((size_t)p * k + c) * 2 + 1];
      }
      out_r[c] = sqrt(a);
      out_f[c] = sqrt(b);
    }
  });
  return ACR_OK;
}

int acr_gen_constant(int m, int n, const double* values5, double* D_sub, double* D_diag,
                     double* D_sup, double* E, double* F, void* stream) {
  if (m < 1 || n < 1 || !values5) return set_err(nullptr, ACR_EARG, "bad shape");
  ACR_GUARD(nullptr, {
    CK(acr::launch_gen_const(m, n, values5, D_sub, D_diag, D_sup, E, F,
                             (cudaStream_t)stream));
  });
  return ACR_OK;
}

int acr_gen_varcoef(int n, const double* c8, const long long* p8, const long long* q8,
                    const double* phi8, double* work, double* D_sub, double* D_diag,
                    double* D_sup, double* E, double* F, void* stream) {
  if (n < 1 || !c8 || !p8 || !q8 || !phi8 || !work)
    return set_err(nullptr, ACR_EARG, "bad arguments");
  ACR_GUARD(nullptr, {
    acr::GenField P;
    for (int t = 0; t < 8; ++t) {
      P.c[t] = c8[t];
      P.p[t] = p8[t];
      P.q[t] = q8[t];
      P.phi[t] = phi8[t];
    }
    CK(acr::launch_gen_varcoef(n, P, work, D_sub, D_diag, D_sup, E, F, (cudaStream_t)stream));
  });
  return ACR_OK;
}

int acr_gen_uniform(const unsigned long long* pcg_state4, long long N, int k, double low,
                    double high, double* out, void* stream) {
  if (N < 0 || k < 1 || !pcg_state4) return set_err(nullptr, ACR_EARG, "bad arguments");
  ACR_GUARD(nullptr, {
    CK(acr::launch_gen_uniform(pcg_state4, N, k, low, high, out, (cudaStream_t)stream));
  });
  return ACR_OK;
}

static thread_local int g_trunc_path = 0;   // test hook, per calling thread

int acr_set_truncate_path(int path) {
  if (path < 0 || path > 2) return set_err(nullptr, ACR_EARG, "path must be 0, 1 or 2");
  g_trunc_path = path;
  return ACR_OK;
}

int acr_truncate_factor(int m, int k, int R, const double* U, const double* V,
                        double eps, int max_rank_cap, double* Uo, double* Vo,
                        int* rank_out, void* stream) {
  if (m < 1 || k < 1 || R < 0) return set_err(nullptr, ACR_EARG, "bad shape");
  ACR_GUARD(nullptr, {
    cudaStream_t st = (cudaStream_t)stream;
    // one branch node [0, m+k) split at m, two leaves
    int nn = m + k;
    std::vector<int> lo = {0, 0, m}, hi = {nn, m, nn}, mid = {m, m / 2, m + k / 2},
                     depth = {0, 1, 1}, parent = {-1, 0, 0}, c0 = {1, -1, -1},
                     c1 = {2, -1, -1}, isl = {0, 1, 1}, anc = {0, -1, 1, 0, 2, 0},
                     listA = {0, 0, 0, 0, 0, 1};
    std::vector<int> all;
    std::vector<size_t> off;
    for (auto* v : {&lo, &hi, &mid, &depth, &parent, &c0, &c1, &isl, &anc, &listA}) {
      off.push_back(all.size());
      all.insert(all.end(), v->begin(), v->end());
    }
    acr::Dev dtree(sizeof(int) * all.size(), st);
    CK(cudaMemcpyAsync(dtree.p, all.data(), sizeof(int) * all.size(), cudaMemcpyHostToDevice, st));
    const int* b = dtree.as<int>();
    acr::TreeDev T;
    memset(&T, 0, sizeof(T));
    T.n = nn;
    T.bw = std::max(m, k);
    T.nd = 1;
    T.nnodes = 3;
    T.maxdepth = 1;
    T.nleaves = 2;
    T.lo = b + off[0]; T.hi = b + off[1]; T.mid = b + off[2]; T.depth = b + off[3];
    T.parent = b + off[4]; T.c0 = b + off[5]; T.c1 = b + off[6]; T.isleaf = b + off[7];
    T.anc = b + off[8];
    int Rc = std::max(R, 1);
    acr::Dev Ub(sizeof(double) * (size_t)Rc * nn, st), Vb(sizeof(double) * (size_t)Rc * nn, st);
    acr::Dev rk(sizeof(int) * 6, st), ovf(sizeof(int), st);
    for (int c = 0; c < R; ++c) {
      CK(cudaMemcpyAsync(Ub.as<double>() + (size_t)c * nn, U + (size_t)c * m, sizeof(double) * m,
                         cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(Vb.as<double>() + (size_t)c * nn + m, V + (size_t)c * k,
                         sizeof(double) * k, cudaMemcpyDeviceToDevice, st));
    }
    int hr[6] = {R, 0, 0, 0, 0, 0};
    CK(cudaMemcpyAsync(rk.p, hr, sizeof(hr), cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(ovf.p, 0, sizeof(int), st));
    acr::HB hb;
    hb.leaf = nullptr;
    hb.U = Ub.as<double>();
    hb.V = Vb.as<double>();
    hb.rk = rk.as<int>();
    hb.R = Rc;
    hb.pad_ = 0;
    acr::Dev dhb(sizeof(acr::HB), st);
    CK(cudaMemcpyAsync(dhb.p, &hb, sizeof(hb), cudaMemcpyHostToDevice, st));
    acr::TruncArgs a;
    memset(&a, 0, sizeof(a));
    a.T = T;
    a.mode = acr::TM_TRUNCATE;
    a.a = acr::op_own(acr::s_hbU(dhb.as<acr::HB>()), acr::s_hbV(dhb.as<acr::HB>()),
                      acr::r_hb(dhb.as<acr::HB>()));
    a.out = dhb.as<acr::HB>();
    a.tasks = dtree.as<int>() + off[9];
    a.ntasks = 1;
    a.eps = eps;
    a.cap = max_rank_cap;
    a.overflow = ovf.as<int>();
    long long need = acr::trunc_need_doubles(m, k, Rc);
    acr::Dev g(sizeof(double) * std::max<long long>(need, 1) * 148, st);
    acr::Dev q(sizeof(int) * 4, st), qc(sizeof(int) * 4, st);
    a.smem_doubles = 24576;
    a.gscr = g.as<double>();
    a.gscr_stride = need;
    a.smem_doubles = (int)std::min<long long>(need, 24576);
    if (g_trunc_path == 2 && acr::pair_need_doubles(std::max(m, k), Rc) <= 28416)
      CK(acr::launch_trunc_pair(a, 1, acr::pair_need_doubles(std::max(m, k), Rc), st));
    else
    {
      acr::Dev cl(16, st);
      acr::TruncAux aux;
      memset(&aux, 0, sizeof(aux));
      aux.cls = cl.as<unsigned char>();
      CK(acr::launch_trunc(a, 1, g_trunc_path != 1, g_trunc_path == 1, q.as<int>(),
                           qc.as<int>(), st, &aux));
    }
    int hr2[6];
    CK(cudaMemcpyAsync(hr2, rk.p, sizeof(hr2), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    int r = hr2[0];
    *rank_out = r;
    for (int c = 0; c < r; ++c) {
      CK(cudaMemcpyAsync(Uo + (size_t)c * m, Ub.as<double>() + (size_t)c * nn,
                         sizeof(double) * m, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(Vo + (size_t)c * k, Vb.as<double>() + (size_t)c * nn + m,
                         sizeof(double) * k, cudaMemcpyDeviceToDevice, st));
    }
    CK(cudaStreamSynchronize(st));
  });
  return ACR_OK;
}

int acr_leaf_inverse(int s, const double* A, double* X, int* singular,
                     void* stream) {
  if (s < 1 || s > 128) return set_err(nullptr, ACR_EARG, "leaf size must be in [1,128]");
  ACR_GUARD(nullptr, {
    cudaStream_t st = (cudaStream_t)stream;
    std::vector<int> lo = {0}, hi = {s}, mid = {s / 2}, depth = {0}, parent = {-1},
                     c0 = {-1}, c1 = {-1}, isl = {1};
    std::vector<int> all;
    std::vector<size_t> off;
    for (auto* v : {&lo, &hi, &mid, &depth, &parent, &c0, &c1, &isl}) {
      off.push_back(all.size());
      all.insert(all.end(), v->begin(), v->end());
    }
    acr::Dev dtree(sizeof(int) * all.size(), st);
    CK(cudaMemcpyAsync(dtree.p, all.data(), sizeof(int) * all.size(), cudaMemcpyHostToDevice, st));
    const int* b = dtree.as<int>();
    acr::TreeDev T;
    memset(&T, 0, sizeof(T));
    T.n = s;
    T.bw = s;
    T.nnodes = 1;
    T.nleaves = 1;
    T.lo = b + off[0]; T.hi = b + off[1]; T.mid = b + off[2]; T.depth = b + off[3];
    T.parent = b + off[4]; T.c0 = b + off[5]; T.c1 = b + off[6]; T.isleaf = b + off[7];
    CK(cudaMemcpyAsync(X, A, sizeof(double) * s * s, cudaMemcpyDeviceToDevice, st));
    acr::HB hb;
    memset(&hb, 0, sizeof(hb));
    hb.leaf = X;
    hb.R = 1;
    acr::Dev dhb(sizeof(acr::HB), st), sg(sizeof(int), st);
    CK(cudaMemcpyAsync(dhb.p, &hb, sizeof(hb), cudaMemcpyHostToDevice, st));
    int big = INT_MAX;
    CK(cudaMemcpyAsync(sg.p, &big, sizeof(int), cudaMemcpyHostToDevice, st));
    CK(acr::launch_leafinv(T, dhb.as<acr::HB>(), 1, 0, sg.as<int>(), st));
    int hs = 0;
    CK(cudaMemcpyAsync(&hs, sg.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *singular = hs != INT_MAX ? 1 : 0;
  });
  return ACR_OK;
}

int acr_block_export(acr_plan_t* h, int level, int which, int block, double* leaf,
                     double* U, double* V, int* ranks, int* R_out, int* count_out,
                     void* stream) {
  if (!h || !h->p) return set_err(h, ACR_EARG, "null plan");
  ACR_GUARD(h, {
    Plan& P = *h->p;
    P.use_stream((cudaStream_t)stream);
    P.export_block(P.factor_batch(level, which), block, leaf, U, V, ranks, R_out, count_out);
  });
  return ACR_OK;
}

int acr_step_lift(acr_plan_t* h, const double* D_sub, const double* D_diag,
                  const double* D_sup, const double* E, const double* F, int* level_out,
                  void* stream) {
  if (!h || !h->p || !level_out) return set_err(h, ACR_EARG, "null plan or output");
  ACR_GUARD(h, {
    Plan& P = *h->p;
    P.use_stream((cudaStream_t)stream);
    *level_out = P.step_lift(D_sub, D_diag, D_sup, E, F);
    CK(cudaStreamSynchronize(P.st));
  });
  return ACR_OK;
}

int acr_step_reduce(acr_plan_t* h, int level, double eps, int max_rank_cap,
                    const int* inversion_order, int* level_out, int* record_out,
                    void* stream) {
  if (!h || !h->p || !level_out || !record_out) return set_err(h, ACR_EARG, "null plan or output");
  if (!(eps > 0)) return set_err(h, ACR_EARG, "eps must be > 0");
  if (max_rank_cap < 0) return set_err(h, ACR_EARG, "max_rank_cap must be positive");
  ACR_GUARD(h, {
    Plan& P = *h->p;
    P.use_stream((cudaStream_t)stream);
    P.step_reduce(level, eps, max_rank_cap, inversion_order, level_out, record_out);
  });
  return ACR_OK;
}

int acr_step_rhs(acr_plan_t* h, int record, const double* f, int nrhs, double* f_out,
                 void* stream) {
  if (!h || !h->p || nrhs < 1) return set_err(h, ACR_EARG, "null plan or nrhs < 1");
  ACR_GUARD(h, {
    Plan& P = *h->p;
    P.use_stream((cudaStream_t)stream);
    P.step_rhs(record, f, nrhs, f_out);
  });
  return ACR_OK;
}

int acr_step_backsub(acr_plan_t* h, int record, const double* f, const double* u_odd,
                     int nrhs, double* u, void* stream) {
  if (!h || !h->p || nrhs < 1) return set_err(h, ACR_EARG, "null plan or nrhs < 1");
  ACR_GUARD(h, {
    Plan& P = *h->p;
    P.use_stream((cudaStream_t)stream);
    P.step_backsub(record, f, u_odd, nrhs, u);
  });
  return ACR_OK;
}

int acr_step_info(acr_plan_t* h, int handle, int which, int* count, int* R, int* level,
                  int* m_level) {
  if (!h || !h->p) return set_err(h, ACR_EARG, "null plan");
  ACR_GUARD(h, {
    Plan& P = *h->p;
    const acr::Batch* b = P.step_batch(handle, which);
    if (count) *count = b->cnt;
    if (R) *R = b->R;
    if (which <= 2) {
      acr::Level& L = P.step_level(handle);
      if (level) *level = L.lvl;
      if (m_level) *m_level = L.m;
    } else {
      acr::Record& r = P.step_record(handle);
      if (level) *level = -1;
      if (m_level) *m_level = r.m;
    }
  });
  return ACR_OK;
}

int acr_step_export(acr_plan_t* h, int handle, int which, int block, double* leaf, double* U,
                    double* V, int* ranks, void* stream) {
  if (!h || !h->p) return set_err(h, ACR_EARG, "null plan");
  ACR_GUARD(h, {
    Plan& P = *h->p;
    P.use_stream((cudaStream_t)stream);
    P.export_block(P.step_batch(handle, which), block, leaf, U, V, ranks, nullptr, nullptr);
  });
  return ACR_OK;
}

int acr_step_free(acr_plan_t* h, int handle) {
  if (!h || !h->p) return set_err(h, ACR_EARG, "null plan");
  ACR_GUARD(h, {
    Plan& P = *h->p;
    if (!P.slev.erase(handle) && !P.srec.erase(handle))
      throw acr::ArgError("unknown handle " + std::to_string(handle));
  });
  return ACR_OK;
}

}  // extern "C"
