// Does DFMA throughput depend on how many operands come from registers?
// (a) x = fma(x, c1, c2): two constant-bank operands
// (b) x = fma(x, a, b):   a, b per-thread registers
// (c) K3-like: g = fma(an.x, s.y, fma(an.y, s.x, g)) with s from shared memory
#include <cstdio>
#include <cuda_runtime.h>
__global__ void kc(double *out, int iters, double c1, double c2) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], c1, c2);
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 1.2345) out[0] = s;
}
__global__ void kr(double *out, int iters, double c1, double c2) {
  double x[8], a[8], b[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { x[k] = threadIdx.x * 1e-9 + k; a[k] = c1 + threadIdx.x * 1e-12 * k; b[k] = c2 * (1 + 1e-9 * (threadIdx.x + k)); }
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a[k], b[k]);
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k] + a[k] + b[k];
  if (s == 1.2345) out[0] = s;
}
__global__ void ks(double *out, int iters, double c) {
  __shared__ double2 sm[64];
  if (threadIdx.x < 64) sm[threadIdx.x] = make_double2(0.1 + threadIdx.x * 1e-3, 0.2);
  __syncthreads();
  double ap[2], ac[2], g[2], h[2];
  for (int k = 0; k < 2; ++k) { ap[k] = 0.1 * k + threadIdx.x * 1e-9; ac[k] = 0.2; g[k] = 0; h[k] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const double2 s = sm[(i + m) & 63];
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
  double *d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int bpsm : {4, 8}) {
    dim3 g(148 * bpsm); int tpb = 128, it = 4096;
    kc<<<g, tpb>>>(d, it, 0.999999, 1e-7); cudaEventRecord(e0); kc<<<g, tpb>>>(d, it, 0.999999, 1e-7); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("const operands  warps/SM %2d: %.2f Tinstr/s\n", bpsm * 4, 8.0 * it * tpb * g.x / ms / 1e9);
    kr<<<g, tpb>>>(d, it, 0.999999, 1e-7); cudaEventRecord(e0); kr<<<g, tpb>>>(d, it, 0.999999, 1e-7); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("reg operands    warps/SM %2d: %.2f Tinstr/s\n", bpsm * 4, 8.0 * it * tpb * g.x / ms / 1e9);
    ks<<<g, tpb>>>(d, it / 16, 1.9); cudaEventRecord(e0); ks<<<g, tpb>>>(d, it / 16, 1.9); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("k3 smem operands warps/SM %2d: %.2f Tinstr/s\n", bpsm * 4, 4.0 * 2 * 16 * (it / 16) * tpb * g.x / ms / 1e9);
  }
  return 0;
}
