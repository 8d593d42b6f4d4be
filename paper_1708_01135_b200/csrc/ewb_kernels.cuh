// ewb_kernels.cuh -- small kernels of the pipeline: per-particle preparation,
// deterministic sums, the velocity-Verlet integrator, self energy and the FP64
// roofline probe, Verlet-list helpers; it also includes the stage kernel
// headers.  Included by ewald_b200.cu inside its anonymous namespace;
// stage kernels: recip_fp64.cuh, rs_cells.cuh, rs_pairs.cuh,
// k1_tc.cuh and k3_tc.cuh.

// ---------------------------------------------------------------------------
// k_prep: per-particle derived data, O(N)
__global__ void k_prep(const double *__restrict__ pos, const double *__restrict__ q, int64_t n,
                       double L, double4 *__restrict__ frac, double2 *__restrict__ base,
                       double4 *__restrict__ xyzq, int *__restrict__ err) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = pos[3 * i], y = pos[3 * i + 1], z = pos[3 * i + 2], qi = q[i];
  if (!(x >= 0.0 && x < L && y >= 0.0 && y < L && z >= 0.0 && z < L)) atomicOr(err, ERR_UNWRAPPED);
  const double tx = x / L, ty = y / L, tz = z / L;
  frac[i] = make_double4(tx, ty, tz, qi);
  xyzq[i] = make_double4(x, y, z, qi);
  double s, c;
  sincospi(2.0 * tx, &s, &c);
  base[3 * i] = make_double2(c, -s);
  sincospi(2.0 * ty, &s, &c);
  base[3 * i + 1] = make_double2(c, -s);
  sincospi(2.0 * tz, &s, &c);
  base[3 * i + 2] = make_double2(c, -s);
}

#include "recip_fp64.cuh"

__global__ void __launch_bounds__(1024) k_sum(const double *__restrict__ v, int64_t n,
                                               double scale, double *__restrict__ out) {
  __shared__ double sh[32];
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 1024) a += v[i];
  const double r = block_sum<1024>(a, sh);
  if (threadIdx.x == 0) *out = scale * r;
}

#include "rs_cells.cuh"

#include "rs_pairs.cuh"

// Verlet-list reuse: positions in the build's cell order, each moved back by
// the box edge if it wrapped since the build (so the build's image shifts
// stay valid); particles that did not wrap keep their coordinates bit for bit
__global__ void k_verlet_gather(const double4 *__restrict__ xyzq, const int *__restrict__ order,
                                const double4 *__restrict__ xb, int64_t n, double L,
                                double4 *__restrict__ sorted, float4 *__restrict__ sorted_f,
                                int *__restrict__ err) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 p = xyzq[order[i]];
  // the binning's check (celllist.py:90-91): positions must be wrapped
  if (!(p.x >= 0.0 && p.x < L && p.y >= 0.0 && p.y < L && p.z >= 0.0 && p.z < L))
    atomicOr(err, ERR_UNWRAPPED);
  const double4 b = xb[i];
  const double il = 1.0 / L;
  const double x = __dadd_rn(p.x, L * rint((b.x - p.x) * il));
  const double y = __dadd_rn(p.y, L * rint((b.y - p.y) * il));
  const double z = __dadd_rn(p.z, L * rint((b.z - p.z) * il));
  sorted[i] = make_double4(x, y, z, p.w);
  sorted_f[i] = make_float4((float)x, (float)y, (float)z, 0.0f);
}

// largest squared minimum-image displacement since the build (bits of a
// non-negative double compare like the value)
__global__ void k_verlet_disp(const double *__restrict__ pos, const int *__restrict__ order,
                              const double4 *__restrict__ xb, int64_t n, double L,
                              unsigned long long *__restrict__ dmax) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double d2 = 0.0;
  if (i < n) {
    const int64_t o = order[i];
    const double4 b = xb[i];
    const double il = 1.0 / L;
    double dx = pos[3 * o] - b.x, dy = pos[3 * o + 1] - b.y, dz = pos[3 * o + 2] - b.z;
    dx -= L * rint(dx * il);
    dy -= L * rint(dy * il);
    dz -= L * rint(dz * il);
    d2 = dx * dx + dy * dy + dz * dz;
  }
  for (int o = 16; o > 0; o >>= 1) d2 = fmax(d2, __shfl_xor_sync(0xffffffffu, d2, o));
  if ((threadIdx.x & 31) == 0 && d2 > 0.0) atomicMax(dmax, (unsigned long long)__double_as_longlong(d2));
}

// ---------------------------------------------------------------------------
// Device-resident velocity Verlet (velocity_verlet_step, driver.py:134-153):
// v += 0.5 dt F/m; r += dt v; wrap into [0, L) (core.py:156-161); forces;
// v += 0.5 dt F/m.  Kinetic energy 0.5 sum m v.v (driver.py:129-131).
__global__ void k_md_kick_drift(double *__restrict__ pos, double *__restrict__ vel,
                                const double *__restrict__ force, const double *__restrict__ mass,
                                int64_t n, double dt, double L) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  // numpy's expression order, no contraction: v += ((0.5*dt)*F)*inv_m,
  // r += dt*v, w = r - L*floor(r/L), w >= L -> w - L
  const double inv_m = __ddiv_rn(1.0, mass[i]);
  const double hdt = __dmul_rn(0.5, dt);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double v = __dadd_rn(vel[3 * i + a], __dmul_rn(__dmul_rn(hdt, force[3 * i + a]), inv_m));
    vel[3 * i + a] = v;
    const double r = __dadd_rn(pos[3 * i + a], __dmul_rn(dt, v));
    double w = __dsub_rn(r, __dmul_rn(L, floor(__ddiv_rn(r, L))));
    if (w >= L) w = __dsub_rn(w, L);
    pos[3 * i + a] = w;
  }
}

__global__ void __launch_bounds__(RED_THREADS)
    k_md_kick(double *__restrict__ vel, const double *__restrict__ force,
              const double *__restrict__ mass, int64_t n, double dt, int kick,
              double *__restrict__ eblk) {
  __shared__ double sh[RED_THREADS / 32];
  const int64_t i = blockIdx.x * (int64_t)RED_THREADS + threadIdx.x;
  double ke = 0.0;
  if (i < n) {
    const double m = mass[i];
    const double inv_m = __ddiv_rn(1.0, m);
    const double hdt = __dmul_rn(0.5, dt);
    double vv = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double v = vel[3 * i + a];
      if (kick) {
        v = __dadd_rn(v, __dmul_rn(__dmul_rn(hdt, force[3 * i + a]), inv_m));
        vel[3 * i + a] = v;
      }
      vv = fma(v, v, vv);
    }
    ke = m * vv;
  }
  const double b = block_sum<RED_THREADS>(ke, sh);
  if (threadIdx.x == 0) eblk[blockIdx.x] = b;
}

// K7: sum q^2 (self energy) partials.
__global__ void __launch_bounds__(RED_THREADS) k7_sum_q2(const double4 *__restrict__ frac, int64_t n,
                                                         double *__restrict__ eblk) {
  __shared__ double sh[RED_THREADS / 32];
  double a = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)RED_THREADS + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * RED_THREADS) {
    const double q = frac[i].w;
    a = fma(q, q, a);
  }
  const double b = block_sum<RED_THREADS>(a, sh);
  if (threadIdx.x == 0) eblk[blockIdx.x] = b;
}

// FP64 peak probe: independent DFMA chains (2 flops each), for the roofline
// denominator (MEASURED_PEAKS.json carries no FP64 figure).
__global__ void __launch_bounds__(256) k_fp64_probe(double *__restrict__ out, int iters, double a,
                                                    double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 1.2345) out[0] = s;  // keep the chains alive
}

#include "k1_tc.cuh"
#include "k3_tc.cuh"

