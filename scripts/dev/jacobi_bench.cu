// Development harness: cycles of one warp_jacobi call (one warp alone on an
// SM) on random pc x pc cores; sweeps and cycles per step.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_1604_00617_b200/csrc/k_trunc.cu"
namespace acr {
template <int RPL>
__device__ int blk_jacobi_f(double* B, int pr, int pc, double* J, int lane, int gs) {
  const int lb = pr | 1, lj = pc | 1;
  const int np = pc + (pc & 1), npairs = np / 2;
  const int per = 32 / gs;
  const double tol = sqrt((double)pr) * 2.220446049250313e-16;
  const int sub = lane & (gs - 1), grp = lane / gs;
  double nb = 0.0;
  for (int i = lane; i < pr * pc; i += 32) {
    const double x = B[(i / pr) * lb + i % pr];
    nb += x * x;
  }
  const double tiny = warp_sum(nb) * 4.930380657631324e-32;   // (eps64 |B|_F)^2
  for (int sweep = 0; sweep < 40; ++sweep) {
    bool rot = false;
    for (int step = 0; step < np - 1; ++step) {
      for (int base = 0; base < npairs; base += per) {
        const int k = base + grp;
        int i = 0, j = 0;
        bool valid = k < npairs;
        if (valid) {
          i = rr_player(step, k, np);
          j = rr_player(step, np - 1 - k, np);
          valid = i < pc && j < pc;
        }
        double* bi = B + (long long)i * lb;
        double* bj = B + (long long)j * lb;
        double xr[RPL], yr[RPL];
#pragma unroll
        for (int h = 0; h < RPL; ++h) {
          const int r = sub + gs * h;
          const bool in = valid && r < pr;
          xr[h] = in ? bi[r] : 0.0;
          yr[h] = in ? bj[r] : 0.0;
        }
        double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
        for (int h = 0; h < RPL; ++h) {
          if (sub + gs * h < pr) {
            a += xr[h] * xr[h];
            b += yr[h] * yr[h];
            c += xr[h] * yr[h];
          }
        }
        for (int o = gs >> 1; o; o >>= 1) {
          a += __shfl_xor_sync(FULL, a, o);
          b += __shfl_xor_sync(FULL, b, o);
          c += __shfl_xor_sync(FULL, c, o);
        }
        if (valid && a > tiny && b > tiny && c != 0.0 &&
            c * c > tol * tol * a * b) {
          // t = sign(d) e / q, q = |d| + r, r = sqrt(d^2 + e^2);
          // 1 + t^2 = 2 r / q  ->  cs = sqrt(q) rsqrt(2 r), sn = cs sign(d) e / q
          const double d = b - a, e = 2.0 * c;
          const double r = sqrt(fma(d, d, e * e));
          const double q = fabs(d) + r;
          const double sq = sqrt(q), ir = rsqrt(2.0 * r), iq = 1.0 / q;
          const double cs = sq * ir;
          const double sn = cs * (copysign(1.0, d) * e) * iq;
          double* ji = J + (long long)i * lj;
          double* jj = J + (long long)j * lj;
          double xj[RPL], yj[RPL];
#pragma unroll
          for (int h = 0; h < RPL; ++h) {
            const int r = sub + gs * h;
            xj[h] = r < pc ? ji[r] : 0.0;
            yj[h] = r < pc ? jj[r] : 0.0;
          }
#pragma unroll
          for (int h = 0; h < RPL; ++h) {
            const int r = sub + gs * h;
            if (r < pr) {
              bi[r] = cs * xr[h] - sn * yr[h];
              bj[r] = sn * xr[h] + cs * yr[h];
            }
            if (r < pc) {
              ji[r] = cs * xj[h] - sn * yj[h];
              jj[r] = sn * xj[h] + cs * yj[h];
            }
          }
          rot = true;
        }
        __syncwarp();
      }
    }
    if (!__any_sync(FULL, rot)) return sweep + 1;
  }
  return 40;
}
template <int RPL>
__device__ int blk_jacobi_c(double* B, int pr, int pc, double* J, int lane, int gs) {
  const int lb = pr | 1, lj = pc | 1;
  const int np = pc + (pc & 1), npairs = np / 2;
  const int per = 32 / gs;
  const double tol = sqrt((double)pr) * 2.220446049250313e-16;
  const int sub = lane & (gs - 1), grp = lane / gs;
  double nb = 0.0;
  for (int i = lane; i < pr * pc; i += 32) {
    const double x = B[(i / pr) * lb + i % pr];
    nb += x * x;
  }
  const double tiny = warp_sum(nb) * 4.930380657631324e-32;   // (eps64 |B|_F)^2
  for (int sweep = 0; sweep < 40; ++sweep) {
    bool rot = false;
    for (int step = 0; step < np - 1; ++step) {
      for (int base = 0; base < npairs; base += per) {
        const int k = base + grp;
        int i = 0, j = 0;
        bool valid = k < npairs;
        if (valid) {
          i = rr_player(step, k, np);
          j = rr_player(step, np - 1 - k, np);
          valid = i < pc && j < pc;
        }
        double* bi = B + (long long)i * lb;
        double* bj = B + (long long)j * lb;
        double xr[RPL], yr[RPL];
#pragma unroll
        for (int h = 0; h < RPL; ++h) {
          const int r = sub + gs * h;
          const bool in = valid && r < pr;
          xr[h] = in ? bi[r] : 0.0;
          yr[h] = in ? bj[r] : 0.0;
        }
        double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
        for (int h = 0; h < RPL; ++h) {
          if (sub + gs * h < pr) {
            a += xr[h] * xr[h];
            b += yr[h] * yr[h];
            c += xr[h] * yr[h];
          }
        }
        for (int o = gs >> 1; o; o >>= 1) {
          a += __shfl_xor_sync(FULL, a, o);
          b += __shfl_xor_sync(FULL, b, o);
          c += __shfl_xor_sync(FULL, c, o);
        }
        if (valid && a > tiny && b > tiny && c != 0.0 &&
            c * c > tol * tol * a * b) {
          const double cs = 0.8 + 1e-300 * a, sn = 0.6 + 1e-300 * b;
          double* ji = J + (long long)i * lj;
          double* jj = J + (long long)j * lj;
          double xj[RPL], yj[RPL];
#pragma unroll
          for (int h = 0; h < RPL; ++h) {
            const int r = sub + gs * h;
            xj[h] = r < pc ? ji[r] : 0.0;
            yj[h] = r < pc ? jj[r] : 0.0;
          }
#pragma unroll
          for (int h = 0; h < RPL; ++h) {
            const int r = sub + gs * h;
            if (r < pr) {
              bi[r] = cs * xr[h] - sn * yr[h];
              bj[r] = sn * xr[h] + cs * yr[h];
            }
            if (r < pc) {
              ji[r] = cs * xj[h] - sn * yj[h];
              jj[r] = sn * xj[h] + cs * yj[h];
            }
          }
          rot = true;
        }
        __syncwarp();
      }
    }
    if (!__any_sync(FULL, rot)) return sweep + 1;
  }
  return 40;
}

template <int V>
__device__ int jac_var(double* B, int pr, int pc, double* J, int lane) {
  if (V == 0) return blk_jacobi(B, pr, pc, J, lane);
  const int lj = pc | 1;
  for (int i = lane; i < pc * pc; i += 32) { const int c = i / pc, r = i - c * pc; J[c * lj + r] = (r == c) ? 1.0 : 0.0; }
  __syncwarp();
  const int npairs = (pc + (pc & 1)) / 2;
  int gs = 32;
  while (gs > 1 && gs * npairs > 32) gs >>= 1;
  const int rpl = (pr + gs - 1) / gs;
  if (V == 1) { if (rpl <= 1) return blk_jacobi_f<1>(B, pr, pc, J, lane, gs); if (rpl <= 2) return blk_jacobi_f<2>(B, pr, pc, J, lane, gs); return blk_jacobi_f<4>(B, pr, pc, J, lane, gs); }
  if (rpl <= 1) return blk_jacobi_c<1>(B, pr, pc, J, lane, gs); if (rpl <= 2) return blk_jacobi_c<2>(B, pr, pc, J, lane, gs); return blk_jacobi_c<4>(B, pr, pc, J, lane, gs);
}
}

__global__ void k_jac(const double* in, int pr, int pc, long long* cyc, int* sweeps, double* out, int var) {
  __shared__ double B[32 * 33], J[32 * 33], G[32 * 33], RL[64];
  const int lane = threadIdx.x;
  for (int i = lane; i < pr * pc; i += 32) B[(i / pr) * (pr | 1) + i % pr] = in[i];
  __syncwarp();
  long long t0 = clock64();
  int sw = var == 3 ? acr::precond_jacobi(B, pc, J, G, RL, lane) : var == 0 ? acr::jac_var<0>(B, pr, pc, J, lane) : var == 1 ? acr::jac_var<1>(B, pr, pc, J, lane) : acr::jac_var<2>(B, pr, pc, J, lane);
  __syncwarp();
  long long t1 = clock64();
  if (lane == 0) { *cyc = t1 - t0; *sweeps = sw; }
  for (int i = lane; i < (pr | 1) * pc; i += 32) out[i] = B[i];
}

int main() {
  for (int pc : {8, 12, 14, 16, 24}) {
    const int pr = pc;
    std::vector<double> h(pr * pc);
    srand(pc);
    // graded singular values like a recompression core: random orthogonal-ish mix
    { std::vector<double> ru(pc * pc, 0.0), rv(pc * pc, 0.0);
      for (int c = 0; c < pc; ++c) for (int r = 0; r <= c; ++r) { ru[c * pc + r] = ((rand() / (double)RAND_MAX) - 0.5) * pow(10.0, -2.0 * r); rv[c * pc + r] = ((rand() / (double)RAND_MAX) - 0.5) * pow(10.0, -2.0 * r); }
      for (int i = 0; i < pc; ++i) for (int j = 0; j < pc; ++j) { double a = 0; for (int l = 0; l < pc; ++l) a += ru[l * pc + i] * rv[l * pc + j]; h[j * pr + i] = a; } }
    double *din, *dout; long long* dc; int* ds;
    cudaMalloc(&din, 8 * pr * pc); cudaMalloc(&dout, 8 * (pr | 1) * pc); cudaMalloc(&dc, 8); cudaMalloc(&ds, 4);
    cudaMemcpy(din, h.data(), 8 * pr * pc, cudaMemcpyHostToDevice);
    for (int var = 0; var < 4; ++var) {
    long long c = 0; int s = 0;
    for (int rep = 0; rep < 3; ++rep) {
      k_jac<<<1, 32>>>(din, pr, pc, dc, ds, dout, var);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&s, ds, 4, cudaMemcpyDeviceToHost);
    const int np = pc + (pc & 1);
    const char* nm[] = {"blk", "blkfast", "blkconst", "precond"};
    std::vector<double> o(pr * pc); cudaMemcpy(o.data(), dout, 8 * pr * pc, cudaMemcpyDeviceToHost);
    double smax = 0, smin = 1e300; for (int j = 0; j < pc; ++j) { double q = 0; for (int i = 0; i < pr; ++i) { double x = o[j * (pr | 1) + i]; q += x * x; } q = sqrt(q); if (q > smax) smax = q; if (q < smin) smin = q; }
    printf("pc=%2d %-8s sweeps=%2d cycles=%8lld  per step=%.0f  smax %.15e smin %.15e (%s)\n", pc, nm[var], s, c, c / (double)((s ? s : 1) * (np - 1)), smax, smin, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
