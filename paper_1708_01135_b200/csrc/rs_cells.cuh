// rs_cells.cuh -- cell list of the real-space sum (celllist.py:75-108):
// binning, scans, deterministic in-cell order, gathers, force un-permute.  Included by ewald_b200.cu inside its anonymous
// namespace (shared helpers: cmul, warp_sum, block_sum, constants).

// ---------------------------------------------------------------------------
// Real space: counting-sort binning (celllist.py:75-108)
__global__ void k4_bin_count(const double4 *__restrict__ xyzq, int64_t n, double edge, int cpd,
                             int *__restrict__ cell_of, int *__restrict__ slot,
                             int *__restrict__ count) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 p = xyzq[i];
  int c = 0;
  if (cpd > 1) {
    const double v[3] = {p.x, p.y, p.z};
    int id[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double f = floor(v[a] / edge);
      int k = (f >= 0.0) ? (f < (double)cpd ? (int)f : cpd - 1) : 0;  // NaN -> 0
      id[a] = k;
    }
    c = id[0] + cpd * (id[1] + cpd * id[2]);
  }
  cell_of[i] = c;
  slot[i] = atomicAdd(count + c, 1);
}

// Single-block exclusive scans of cell counts (start) and K6_G-groups (gstart).
__global__ void __launch_bounds__(1024) k_scan_cells(const int *__restrict__ count, int n_cells,
                                                     int *__restrict__ start,
                                                     int *__restrict__ gstart) {
  __shared__ int wa[32], wb[32];
  __shared__ int carry_a, carry_b;
  if (threadIdx.x == 0) carry_a = carry_b = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int base = 0; base < n_cells; base += 1024) {
    const int c = base + threadIdx.x;
    const int a = c < n_cells ? count[c] : 0;
    const int b = (a + K6_G - 1) / K6_G;
    int ia = a, ib = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int ta = __shfl_up_sync(0xffffffffu, ia, o);
      const int tb = __shfl_up_sync(0xffffffffu, ib, o);
      if (lane >= o) {
        ia += ta;
        ib += tb;
      }
    }
    if (lane == 31) {
      wa[w] = ia;
      wb[w] = ib;
    }
    __syncthreads();
    if (w == 0) {
      int xa = wa[lane], xb = wb[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int ta = __shfl_up_sync(0xffffffffu, xa, o);
        const int tb = __shfl_up_sync(0xffffffffu, xb, o);
        if (lane >= o) {
          xa += ta;
          xb += tb;
        }
      }
      wa[lane] = xa;
      wb[lane] = xb;
    }
    __syncthreads();
    const int pa = (w ? wa[w - 1] : 0) + ia - a + carry_a;
    const int pb = (w ? wb[w - 1] : 0) + ib - b + carry_b;
    if (c < n_cells) {
      start[c] = pa;
      gstart[c] = pb;
    }
    __syncthreads();
    if (threadIdx.x == 1023) {
      carry_a = pa + a;
      carry_b = pb + b;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    start[n_cells] = carry_a;
    gstart[n_cells] = carry_b;
  }
}

__global__ void k5_scatter(const int *__restrict__ cell_of, const int *__restrict__ slot, int64_t n,
                           const int *__restrict__ start, int *__restrict__ order_tmp) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  order_tmp[start[cell_of[i]] + slot[i]] = (int)i;
}

// Restore a deterministic (ascending original index = stable) order in cells.
__global__ void __launch_bounds__(256) k5_cell_sort(const int *__restrict__ start,
                                                    const int *__restrict__ order_tmp,
                                                    int *__restrict__ order) {
  __shared__ int mem[SORT_CAP];
  const int c = blockIdx.x;
  const int s = start[c], e = start[c + 1], cnt = e - s;
  if (cnt > SORT_CAP) {
    for (int t = threadIdx.x; t < cnt; t += 256) order[s + t] = order_tmp[s + t];
    return;
  }
  for (int t = threadIdx.x; t < cnt; t += 256) mem[t] = order_tmp[s + t];
  __syncthreads();
  for (int t = threadIdx.x; t < cnt; t += 256) {
    const int v = mem[t];
    int r = 0;
    for (int u = 0; u < cnt; ++u) r += mem[u] < v;
    order[s + r] = v;
  }
}

// real-space forces, accumulated in cell-sorted order by k6 (partner atomics
// on neighbouring addresses, no order[] load per pair), added into the
// caller's order: force[order[p]] += fs[p]
__global__ void k_unpermute_add(const int *__restrict__ order, const double *__restrict__ fs,
                                int64_t n, double *__restrict__ force) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int64_t o = order[p];
  force[3 * o] += fs[3 * p];
  force[3 * o + 1] += fs[3 * p + 1];
  force[3 * o + 2] += fs[3 * p + 2];
}

// Scan-all (FOLD) binning in one pass: identity order, one cell, one row --
// replaces count / scans / iota / gather / row scan for small boxes.
__global__ void k_fold_prep(const double4 *__restrict__ xyzq, int64_t n, int units,
                            double4 *__restrict__ sorted, float4 *__restrict__ sorted_f,
                            int *__restrict__ sorted_cell, int *__restrict__ order,
                            int *__restrict__ start, int *__restrict__ row_ustart) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p == 0) {
    start[0] = 0;
    start[1] = (int)n;
    row_ustart[0] = 0;
    row_ustart[1] = units;
  }
  if (p >= n) return;
  const double4 v = xyzq[p];
  sorted[p] = v;
  sorted_f[p] = make_float4((float)v.x, (float)v.y, (float)v.z, 0.0f);
  sorted_cell[p] = 0;
  order[p] = (int)p;
}

__global__ void k5_gather(const int *__restrict__ order, const double4 *__restrict__ xyzq,
                          const int *__restrict__ cell_of, int64_t n,
                          double4 *__restrict__ sorted, float4 *__restrict__ sorted_f,
                          int *__restrict__ sorted_cell) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int o = order[p];
  const double4 v = xyzq[o];
  sorted[p] = v;
  sorted_f[p] = make_float4((float)v.x, (float)v.y, (float)v.z, 0.0f);
  sorted_cell[p] = cell_of[o];
}

