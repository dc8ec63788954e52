// Dependent-chain latency micro-benchmark (cycles per operation) on one SM:
// DFMA, DMUL, double divide / sqrt / rsqrt, SHFL (64-bit value), LDS (64-bit,
// pointer chase), __syncthreads (256 threads), __syncwarp.
#include <cstdio>
#define N 4096
__global__ void k(double* out, long long* cyc, double x0, int* chase_init) {
  __shared__ int chase[1024];
  __shared__ double sd[1024];
  const int tid = threadIdx.x;
  for (int i = tid; i < 1024; i += blockDim.x) { chase[i] = (i * 97 + 13) & 1023; sd[i] = 1.0 + i * 1e-9; }
  __syncthreads();
  double x = x0 + tid * 1e-12;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = fma(x, 0.999999999, 1e-9);
  t1 = clock64(); if (tid == 0) cyc[0] = t1 - t0;
  // DMUL+DADD chain (2 ops)
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = x * 0.999999999 + 1e-9;
  t1 = clock64(); if (tid == 0) cyc[1] = t1 - t0;
  // divide chain
  t0 = clock64();
  for (int i = 0; i < N / 8; ++i) x = 1.0 / (x + 1.0);
  t1 = clock64(); if (tid == 0) cyc[2] = (t1 - t0) * 8;
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < N / 8; ++i) x = sqrt(x + 1.0);
  t1 = clock64(); if (tid == 0) cyc[3] = (t1 - t0) * 8;
  // rsqrt chain
  t0 = clock64();
  for (int i = 0; i < N / 8; ++i) x = rsqrt(x + 1.0);
  t1 = clock64(); if (tid == 0) cyc[4] = (t1 - t0) * 8;
  // shfl chain (64-bit)
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1);
  t1 = clock64(); if (tid == 0) cyc[5] = t1 - t0;
  // shfl + add chain (one butterfly round)
  t0 = clock64();
  for (int i = 0; i < N; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
  t1 = clock64(); if (tid == 0) cyc[6] = t1 - t0;
  // LDS pointer chase (32-bit)
  int p = tid & 1023;
  t0 = clock64();
  for (int i = 0; i < N; ++i) p = chase[p];
  t1 = clock64(); if (tid == 0) cyc[7] = t1 - t0;
  // LDS 64-bit dependent (address from value)
  t0 = clock64();
  for (int i = 0; i < N; ++i) { x = sd[p & 1023] + x * 1e-30; p = (int)x & 1; }
  t1 = clock64(); if (tid == 0) cyc[8] = t1 - t0;
  // __syncthreads
  t0 = clock64();
  for (int i = 0; i < N / 4; ++i) __syncthreads();
  t1 = clock64(); if (tid == 0) cyc[9] = (t1 - t0) * 4;
  // __syncwarp
  t0 = clock64();
  for (int i = 0; i < N; ++i) __syncwarp();
  t1 = clock64(); if (tid == 0) cyc[10] = t1 - t0;
  // STS + __syncwarp + LDS round trip (lane exchange through smem)
  t0 = clock64();
  for (int i = 0; i < N / 4; ++i) { sd[tid] = x; __syncwarp(); x = sd[tid ^ 1] * 1.0000001; __syncwarp(); }
  t1 = clock64(); if (tid == 0) cyc[11] = (t1 - t0) * 4;
  out[tid] = x + p;
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 4096 * 8); cudaMalloc(&c, 64 * 8);
  const char* names[] = {"DFMA", "DMUL+DADD", "DDIV", "DSQRT", "DRSQRT", "SHFL64", "SHFL64+DADD", "LDS32 chase", "LDS64 dep", "syncthreads(256)", "syncwarp", "STS+syncwarp+LDS x2"};
  for (int nt : {32, 256}) {
    k<<<1, nt>>>(d, c, 1.5, nullptr);
    cudaDeviceSynchronize();
    k<<<1, nt>>>(d, c, 1.5, nullptr);
    long long h[12]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threads %d (%s)\n", nt, cudaGetErrorString(cudaGetLastError()));
    for (int i = 0; i < 12; ++i) printf("  %-22s %7.1f cycles/op\n", names[i], h[i] / (double)N);
  }
  return 0;
}
