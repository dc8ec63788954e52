// Development harness: per-step latency of the leaf Gauss-Jordan (one CTA)
#include <cstdio>
#include <vector>
#include <cstdlib>
#include "../../paper_1604_00617_b200/csrc/k_leaf.cu"
namespace acr {
#include "li_ts.inc"
}
using namespace acr;
__global__ void clk(unsigned long long* o) {
  unsigned long long t0, t1; long long c0 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (clock64() - c0 < 20000000) {}
  long long c1 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  o[0] = c1 - c0; o[1] = t1 - t0;
}
int main() {
  const int S = 64;
  std::vector<double> h(S * S);
  srand(1);
  for (int i = 0; i < S * S; ++i) h[i] = (rand() / (double)RAND_MAX - 0.5) + ((i / S == i % S) ? 8.0 : 0.0);
  double* d; cudaMalloc(&d, 8 * S * S);
  int* sg; cudaMalloc(&sg, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int s : {1, 8, 16, 32, 48, 64}) {
    int tree[8] = {0, s, s / 2, 0, -1, -1, -1, 1};
    int* dt; cudaMalloc(&dt, sizeof(tree)); cudaMemcpy(dt, tree, sizeof(tree), cudaMemcpyHostToDevice);
    TreeDev T; memset(&T, 0, sizeof(T));
    T.n = S; T.bw = S; T.nnodes = 1; T.nleaves = 1;
    T.lo = dt; T.hi = dt + 1; T.mid = dt + 2; T.depth = dt + 3; T.parent = dt + 4; T.c0 = dt + 5; T.c1 = dt + 6; T.isleaf = dt + 7;
    HB hb; memset(&hb, 0, sizeof(hb)); hb.leaf = d; hb.R = 1;
    HB* dhb; cudaMalloc(&dhb, sizeof(HB)); cudaMemcpy(dhb, &hb, sizeof(HB), cudaMemcpyHostToDevice);
    cudaMemcpy(d, h.data(), 8 * S * S, cudaMemcpyHostToDevice);
    float best = 1e9, best10 = 1e9;
    for (int rep = 0; rep < 20; ++rep) {
      cudaEventRecord(e0);
      k_leafinv_v2<64, 4, 4, 3><<<1, 256>>>(T, dhb, 0, sg);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      cudaEventRecord(e0);
      for (int i = 0; i < 10; ++i) k_leafinv_v2<64, 4, 4, 3><<<1, 256>>>(T, dhb, 0, sg);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); if (ms / 10 < best10) best10 = ms / 10;
    }
    printf("s=%2d  single %.1f us  back-to-back %.1f us  (%s)\n", s, best * 1e3, best10 * 1e3, cudaGetErrorString(cudaGetLastError()));
  }
  {
    int s = 64;
    int tree[8] = {0, s, s / 2, 0, -1, -1, -1, 1};
    int* dt; cudaMalloc(&dt, sizeof(tree)); cudaMemcpy(dt, tree, sizeof(tree), cudaMemcpyHostToDevice);
    TreeDev T; memset(&T, 0, sizeof(T));
    T.n = S; T.bw = S; T.nnodes = 1; T.nleaves = 1;
    T.lo = dt; T.hi = dt + 1; T.mid = dt + 2; T.depth = dt + 3; T.parent = dt + 4; T.c0 = dt + 5; T.c1 = dt + 6; T.isleaf = dt + 7;
    HB hb; memset(&hb, 0, sizeof(hb)); hb.leaf = d; hb.R = 1;
    HB* dhb; cudaMalloc(&dhb, sizeof(HB)); cudaMemcpy(dhb, &hb, sizeof(HB), cudaMemcpyHostToDevice);
    long long* ts; cudaMalloc(&ts, 8 * 64 * 8); std::vector<long long> hts(64 * 8);
    for (int rep = 0; rep < 3; ++rep) li_ts<64, 4, 4, 3><<<1, 256>>>(T, dhb, 0, sg, ts);
    cudaMemcpy(hts.data(), ts, 8 * 64 * 8, cudaMemcpyDeviceToHost);
    for (int w = 0; w < 8; ++w) printf("warp %d per-step cycles: top-sync %lld  pv+rowP %lld  sync2 %lld  update %lld  pivsearch %lld  (of pv+rowP: piv/pv loads %lld)\n", w,
      hts[w*8]/64, hts[w*8+1]/64, hts[w*8+2]/64, hts[w*8+3]/64, hts[w*8+4]/64, hts[w*8+5]/64);
  }
  unsigned long long* o; cudaMalloc(&o, 16); unsigned long long ho[2];
  for (int i = 0; i < 3; ++i) { clk<<<1, 32>>>(o); cudaMemcpy(ho, o, 16, cudaMemcpyDeviceToHost); printf("single-CTA clock %.0f MHz\n", ho[0] * 1e3 / ho[1]); }
  return 0;
}
