// FP64 dependent-chain latency (cycles per DFMA / DADD) and throughput of
// K3-like chains with 1, 2, 4 independent particles per warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double *out, long long *cyc, int n, double a, double b) {
  double x = threadIdx.x * 1e-9 + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  double y = x;
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) y = y + a;
  long long t3 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t3 - t2; }
  if (x + y == 1.2345) out[0] = x;
}
template <int NP>
__global__ void k3like(double *out, int iters, double c, double s0, double s1) {
  double ap[NP], ac[NP], g[NP], h[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) { ap[k] = 0.1 * k + threadIdx.x * 1e-9; ac[k] = 0.2; g[k] = 0; h[k] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const double an = fma(c, ac[k], -ap[k]);
      ap[k] = ac[k]; ac[k] = an;
      g[k] = fma(an, s0, fma(an, s1, g[k]));
      h[k] += g[k];
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < NP; ++k) s += g[k] + h[k];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double *d; long long *c; cudaMalloc(&d, 64); cudaMalloc(&c, 64);
  lat<<<1, 32>>>(d, c, 1 << 16, 0.9999999, 1e-9);
  long long h[2]; cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("dependent DFMA latency %.2f cycles, DADD %.2f cycles\n", h[0] / 65536.0, h[1] / 65536.0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int bpsm : {1, 2, 4}) {
    dim3 g(148 * bpsm); int tpb = 128, iters = 8192; float ms;
#define RUN(NP) k3like<NP><<<g, tpb>>>(d, iters, 1.9, 0.3, 0.2); cudaEventRecord(e0); k3like<NP><<<g, tpb>>>(d, iters, 1.9, 0.3, 0.2); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); printf("k3like NP=%d warps/SM=%d: %.2f Tinstr/s\n", NP, bpsm * 4, 4.0 * NP * iters * tpb * g.x / ms / 1e9);
    RUN(1) RUN(2) RUN(4)
  }
  return 0;
}
