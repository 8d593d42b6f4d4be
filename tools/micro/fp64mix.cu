// Microbenchmark: FP64 pipe throughput for (a) pure independent DFMA chains,
// (b) the K1 inner-loop mix (3-term recurrence 2 DFMA + accumulate 2 DADD per
// element, NCH independent chains), (c) same with DFMA-only accumulation.
#include <cstdio>
#include <cuda_runtime.h>
template <int NCH>
__global__ void k_mix(double *out, int iters, double c) {
  double p[NCH], q[NCH], a[NCH], b[NCH];
#pragma unroll
  for (int k = 0; k < NCH; ++k) { p[k] = 1e-3 * k + threadIdx.x * 1e-9; q[k] = 0.5 + k * 1e-3; a[k] = 0; b[k] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      const double nx = fma(c, q[k], -p[k]);   // recurrence x
      const double ny = fma(c, p[k], -q[k]);   // recurrence y (stand-in)
      a[k] += nx; b[k] += ny;                  // accumulate (DADD)
      p[k] = q[k]; q[k] = nx;
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < NCH; ++k) s += a[k] + b[k] + p[k];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_fma(double *out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double *d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = 148; int iters = 4096;
  for (int bpsm : {2, 4, 8}) {
    for (int tpb : {128, 256}) {
      dim3 g(sms * bpsm);
      float ms;
      k_fma<<<g, tpb>>>(d, iters, 0.999999, 1e-7);
      cudaEventRecord(e0); k_fma<<<g, tpb>>>(d, iters, 0.999999, 1e-7); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double instr = 8.0 * iters * tpb * g.x;
      printf("fma    bpsm %d tpb %d: %.2f Tinstr/s (%.1f TFLOP/s)\n", bpsm, tpb, instr / ms / 1e9, 2 * instr / ms / 1e9);
      k_mix<2><<<g, tpb>>>(d, iters, 1.9);
      cudaEventRecord(e0); k_mix<2><<<g, tpb>>>(d, iters, 1.9); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      instr = 4.0 * 2 * iters * tpb * g.x;
      printf("mix2   bpsm %d tpb %d: %.2f Tinstr/s\n", bpsm, tpb, instr / ms / 1e9);
      k_mix<4><<<g, tpb>>>(d, iters, 1.9);
      cudaEventRecord(e0); k_mix<4><<<g, tpb>>>(d, iters, 1.9); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      instr = 4.0 * 4 * iters * tpb * g.x;
      printf("mix4   bpsm %d tpb %d: %.2f Tinstr/s\n", bpsm, tpb, instr / ms / 1e9);
    }
  }
  return 0;
}
