// K3-like loop: C*S operand from shared memory (vector registers after LDS)
// vs from __constant__ memory with a warp-uniform index (uniform registers).
#include <cstdio>
#include <cuda_runtime.h>
__constant__ double2 c_sp[2048];
__global__ void k_smem(double *out, int iters, double c, const double2 *gsp) {
  __shared__ double2 sm[2048];
  for (int t = threadIdx.x; t < 2048; t += blockDim.x) sm[t] = gsp[t];
  __syncthreads();
  double ap[2], ac[2], g[2], h[2];
  for (int k = 0; k < 2; ++k) { ap[k] = 0.1 * k + threadIdx.x * 1e-9; ac[k] = 0.2; g[k] = 0; h[k] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const double2 s = sm[(i * 16 + m) & 2047];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const double anx = fma(c, ac[k], -ap[k]);
        ap[k] = ac[k]; ac[k] = anx;
        g[k] = fma(anx, s.y, fma(ap[k], s.x, g[k]));
        h[k] += g[k];
      }
    }
  }
  double t = 0;
  for (int k = 0; k < 2; ++k) t += g[k] + h[k];
  if (t == 1.2345) out[0] = t;
}
__global__ void k_const(double *out, int iters, double c) {
  double ap[2], ac[2], g[2], h[2];
  for (int k = 0; k < 2; ++k) { ap[k] = 0.1 * k + threadIdx.x * 1e-9; ac[k] = 0.2; g[k] = 0; h[k] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const double2 s = c_sp[(i * 16 + m) & 2047];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const double anx = fma(c, ac[k], -ap[k]);
        ap[k] = ac[k]; ac[k] = anx;
        g[k] = fma(anx, s.y, fma(ap[k], s.x, g[k]));
        h[k] += g[k];
      }
    }
  }
  double t = 0;
  for (int k = 0; k < 2; ++k) t += g[k] + h[k];
  if (t == 1.2345) out[0] = t;
}
int main() {
  double *d; double2 *gsp; cudaMalloc(&d, 64); cudaMalloc(&gsp, 2048 * 16);
  double2 hsp[2048]; for (int i = 0; i < 2048; ++i) hsp[i] = make_double2(0.1 + 1e-4 * i, 0.2 - 1e-5 * i);
  cudaMemcpy(gsp, hsp, sizeof hsp, cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(c_sp, hsp, sizeof hsp);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  for (int bpsm : {4, 8}) {
    dim3 g(148 * bpsm); int tpb = 128, it = 512;
    double instr = 5.0 * 2 * 16 * it * (double)tpb * g.x;
    k_smem<<<g, tpb>>>(d, it, 1.9, gsp); cudaEventRecord(e0); k_smem<<<g, tpb>>>(d, it, 1.9, gsp); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("smem  S' warps/SM %2d: %.2f Tinstr/s\n", bpsm * 4, instr / ms / 1e9);
    k_const<<<g, tpb>>>(d, it, 1.9); cudaEventRecord(e0); k_const<<<g, tpb>>>(d, it, 1.9); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("const S' warps/SM %2d: %.2f Tinstr/s\n", bpsm * 4, instr / ms / 1e9);
  }
  return 0;
}
