// Development harness: cycles of one warp_jacobi call (one warp alone on an
// SM) on random pc x pc cores; sweeps and cycles per step.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_1604_00617_b200/csrc/k_trunc.cu"

__global__ void k_jac(const double* in, int pr, int pc, long long* cyc, int* sweeps, double* out, int var) {
  __shared__ double B[32 * 33], J[32 * 33];
  const int lane = threadIdx.x;
  for (int i = lane; i < pr * pc; i += 32) B[i] = in[i];
  __syncwarp();
  long long t0 = clock64();
  int sw = acr::warp_jacobi(B, pr, pc, J, lane);   // B, J: odd column strides (pr | 1, pc | 1)
  __syncwarp();
  long long t1 = clock64();
  if (lane == 0) { *cyc = t1 - t0; *sweeps = sw; }
  for (int i = lane; i < pr * pc; i += 32) out[i] = B[i];
}

int main() {
  for (int pc : {4, 8, 12, 16, 20, 24, 32}) {
    const int pr = pc;
    std::vector<double> h(pr * pc);
    srand(pc);
    // graded singular values like a recompression core: random orthogonal-ish mix
    for (int i = 0; i < pr * pc; ++i) h[i] = ((rand() / (double)RAND_MAX) - 0.5) * pow(10.0, -(double)((i % pc) % 12));
    double *din, *dout; long long* dc; int* ds;
    cudaMalloc(&din, 8 * pr * pc); cudaMalloc(&dout, 8 * pr * pc); cudaMalloc(&dc, 8); cudaMalloc(&ds, 4);
    cudaMemcpy(din, h.data(), 8 * pr * pc, cudaMemcpyHostToDevice);
    for (int var = 0; var < 1; ++var) {
    long long c = 0; int s = 0;
    for (int rep = 0; rep < 3; ++rep) {
      k_jac<<<1, 32>>>(din, pr, pc, dc, ds, dout, var);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&s, ds, 4, cudaMemcpyDeviceToHost);
    const int np = pc + (pc & 1);
    const char* nm[] = {"base", "fastrot", "noJ", "constrot"};
    printf("pc=%2d %-8s sweeps=%2d cycles=%8lld  per step=%.0f  (%s)\n", pc, nm[var], s, c, c / (double)(s * (np - 1)), cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
