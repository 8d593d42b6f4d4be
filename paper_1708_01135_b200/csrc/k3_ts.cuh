// k3_ts.cuh -- the force GEMM of k3_tc.cuh with the A operand (the W slices)
// in TENSOR MEMORY ("TS" tcgen05.mma).  Included after k3_tc.cuh.
//
// Hypothesis tested here: with both operands in shared memory an M=128 int8
// MMA costs >= ~48 cycles whatever N (tools/i8_shapes.py); with A from TMEM
// the floor was expected at N/2 cycles.  Measured: the ~48-cycle floor holds
// in TS form too (N <= 48 identical; N=64 3175 vs 3035, N=80 3969 vs 3503,
// N=96 4553 vs 3904 TOP/s), so at the N = 64 the TMEM budget allows this
// kernel is slower than k3t_gemm at N = 80 (c5 120 vs 101 ms).  Kept as an
// option (T3_USE_TS) and for the record.  Four
// loader warps -- one per TMEM lane quarter, thread = A row -- read their
// row's slices of the next K step from global memory (L2-resident, row-major
// [M tile][K-block][row][slice][64 B]) and write them with tcgen05.st into a
// double-buffered TMEM A area; the MMA warp reads them from there.
//
// TMEM: 6 levels x 64 particles = 384 accumulator columns + 2 x 48 A columns
// (6 slices x 8 columns per 32-byte K step) = 480 of 512.

constexpr int TS_NP = 64;                      // particles per CTA (N)
constexpr int TS_PW = TS_NP / 8;               // producer warps
constexpr int TS_MMA_WARP = TS_PW;             // 8
constexpr int TS_LD_WARP0 = TS_PW + 1;         // 9..12: A loaders
constexpr int TS_THREADS = (TS_PW + 5) * 32;   // 416
constexpr int TS_BS = 3;                       // B ring depth
constexpr int TS_BSL = (TS_NP / 8) * TC_SBO;   // one B slice
constexpr int TS_ACC = T3_NL * TS_NP;          // accumulator columns
constexpr int TS_ACOL = 8 * T3_S;              // A columns per K step (all slices)
static_assert(TS_ACC + 2 * TS_ACOL <= 512, "TMEM budget");

__host__ __device__ constexpr int ts_smem_bytes(int A) {
  return (TS_BS * T3_S * TS_BSL) > (128 * (TS_NP + 1) * 8 + TS_NP * (A + 1) * 16)
             ? (TS_BS * T3_S * TS_BSL)
             : (128 * (TS_NP + 1) * 8 + TS_NP * (A + 1) * 16);
}


// W slices in the row-major layout of the TS kernel:
// wrow[(((mtile * nkb + kb) * 128 + r) * T3_S + s) * 64 + k]
__global__ void __launch_bounds__(256)
    k3s_wprep(const double2 *__restrict__ sp, const int *__restrict__ slotmap, int A,
              const int2 *__restrict__ pair_yz, int n_pairs_pad, const T3Row *__restrict__ rows,
              int n_rows, int nkb, const double *__restrict__ row_scale, uint8_t *__restrict__ wrow) {
  const int r = blockIdx.x;
  const int mtile = r / 128, rl = r % 128;
  const bool live = r < n_rows;
  const T3Row R = live ? rows[r] : T3Row{0, 0};
  const double mx = live ? row_scale[r] : 0.0;
  const double inv = mx > 0.0 ? 1.0 / mx : 0.0;
  for (int k4 = (blockIdx.y * blockDim.x + threadIdx.x) * 4; k4 < nkb * TC_KB;
       k4 += gridDim.y * blockDim.x * 4) {
    uint2 b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double v = live ? t3_value(sp, slotmap, A, pair_yz, n_pairs_pad, R, k4 + u) : 0.0;
      b[u] = t3_bits(fmin(1.0, fmax(-1.0, v * inv)));
    }
    uint32_t w[TC_S];
    tc_digits4(b[0], b[1], b[2], b[3], w);
    const int kb = k4 / TC_KB, kin = k4 % TC_KB;
    uint8_t *base = wrow + (((size_t)mtile * nkb + kb) * 128 + rl) * (size_t)(T3_S * 64);
#pragma unroll
    for (int s = 0; s < T3_S; ++s) *reinterpret_cast<uint32_t *>(base + s * 64 + kin) = w[s];
  }
}

__global__ void __launch_bounds__(TS_THREADS, 1)
    k3s_gemm(const double4 *__restrict__ frac, const double2 *__restrict__ base,
             const uint8_t *__restrict__ wrow, const double *__restrict__ row_scale,
             const T3Row *__restrict__ rows, int n_rows, const int2 *__restrict__ pair_yz,
             int nkb_all, int kb_per_split, int64_t p_begin, int64_t p_end, int A,
             const int4 *__restrict__ comp_rows, double *__restrict__ fpart, int dbg) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t b_full[TS_BS], b_empty[TS_BS], a_full[2], a_empty[2], acc_full;
  __shared__ uint32_t tmem_base_s;
  const int ptile = blockIdx.x, mtile = blockIdx.y, split = blockIdx.z;
  const int n_mtiles = gridDim.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_local = p_end - p_begin;
  const int kb0 = split * kb_per_split;
  const int nkb = max(0, min(nkb_all, kb0 + kb_per_split) - kb0);
  uint8_t *bbuf = smem;

  if (threadIdx.x == 0) {
    for (int i = 0; i < TS_BS; ++i) {
      mbar_init(smem_u32(&b_full[i]), TS_PW);
      mbar_init(smem_u32(&b_empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&a_full[i]), 4);
      mbar_init(smem_u32(&a_empty[i]), 1);
    }
    mbar_init(smem_u32(&acc_full), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&tmem_base_s))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;

  if (warp >= TS_LD_WARP0) {
    // ---- A loaders: thread = row; a warp may only touch the TMEM lanes of
    // quarter (warp id % 4), so warps 9, 10, 11, 12 own rows 32..63, 64..95,
    // 96..127, 0..31 ----
    const int q = warp & 3;
    const int r = 32 * q + lane;
    const uint32_t tlane = (uint32_t)(32 * q) << 16;
    for (int u = 0; u < 2 * nkb; ++u) {
      const int b = u & 1, it = u >> 1, ks = u & 1;
      if (u >= 2) mbar_wait(smem_u32(&a_empty[b]), ((u >> 1) - 1) & 1);
      const uint4 *src = reinterpret_cast<const uint4 *>(
          wrow + (((size_t)mtile * nkb_all + kb0 + it) * 128 + r) * (size_t)(T3_S * 64) + ks * 32);
#pragma unroll
      for (int s = 0; s < T3_S; ++s) {
        const uint4 lo = src[s * 4], hi = src[s * 4 + 1];  // 32 bytes of slice s
        const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
        tc_st8(tmem + tlane + (uint32_t)(TS_ACC + b * TS_ACOL + s * 8), w);
      }
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&a_full[b]));
    }
  } else if (warp == TS_MMA_WARP) {
    // ---- MMA issuer ----
    const uint32_t idesc =
        (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TS_NP >> 3) << 17) | (8u << 24);
    for (int it = 0; it < nkb; ++it) {
      const int bs = it % TS_BS;
      mbar_wait(smem_u32(&b_full[bs]), (it / TS_BS) & 1);
      const uint64_t bd = tc_desc(smem_u32(bbuf + bs * T3_S * TS_BSL));
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int u = 2 * it + ks, b = u & 1;
        mbar_wait(smem_u32(&a_full[b]), (u >> 1) & 1);
        tc_fence_after();
        __syncwarp();
        if (!(dbg & 2) && elect_one()) {
          const uint32_t acc0 = (it > 0 || ks > 0) ? 1u : 0u;
          const uint32_t abase = tmem + (uint32_t)(TS_ACC + b * TS_ACOL);
#pragma unroll
          for (int l = 0; l < T3_NL; ++l) {
            const int w = T3_W0 + l;
            const int s_lo = w - (T3_S - 1) > 0 ? w - (T3_S - 1) : 0;
#pragma unroll
            for (int s = 0; s < T3_S; ++s) {
              const int t = w - s;
              if (t < 0 || t >= T3_S) continue;
              tc_mma_ts(tmem + (uint32_t)(l * TS_NP), abase + (uint32_t)(s * 8),
                        bd + (uint64_t)((t * TS_BSL + ks * 256) >> 4), idesc,
                        s > s_lo ? 1u : acc0);
            }
          }
          tc_commit(smem_u32(&a_empty[b]));
          if (ks == 1) tc_commit(smem_u32(&b_empty[bs]));
        } else if ((dbg & 2) && lane == 0) {
          mbar_arrive(smem_u32(&a_empty[b]));
          if (ks == 1) mbar_arrive(smem_u32(&b_empty[bs]));
        }
        __syncwarp();
      }
    }
    if (lane == 0) {
      if (!(dbg & 2) && nkb > 0)
        tc_commit(smem_u32(&acc_full));
      else
        mbar_arrive(smem_u32(&acc_full));
    }
  } else {
    // ---- B producers: particle pn, run g of the K-block (8 pairs = 16 k) ----
    const int pn = warp * 8 + (lane & 7);
    const int g = lane >> 3;
    const int64_t jg = p_begin + (int64_t)ptile * TS_NP + pn;
    const bool pvalid = jg < p_end;
    const int64_t jc = pvalid ? jg : p_begin;
    const double4 f = frac[jc];
    const double2 by = base[3 * jc + 1];
    const double2 ey = make_double2(by.x, -by.y);  // e^{+i 2pi f_y}
    for (int it = 0; it < nkb; ++it) {
      const int bs = it % TS_BS;
      uint8_t *sb = bbuf + bs * T3_S * TS_BSL;
      if (it >= TS_BS) mbar_wait(smem_u32(&b_empty[bs]), ((it / TS_BS) - 1) & 1);
      if (!(dbg & 1)) {
        const int p0 = (kb0 + it) * (TC_KB / 2) + 8 * g;
        const int2 yz = pair_yz[p0];
        double2 cur = make_double2(0.0, 0.0);
        if (pvalid && yz.x != INT_MIN) {
          double sn, cs;
          sincospi(2.0 * ((double)yz.x * f.y + (double)yz.y * f.z), &sn, &cs);
          cur = make_double2(cs, sn);
        }
        uint32_t w4[T3_S][4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const double2 v0 = cur;
          cur = cmul(cur, ey);
          const double2 v1 = cur;
          cur = cmul(cur, ey);
          uint32_t w[TC_S];
          tc_digits4(t3_bits(v0.x), t3_bits(v0.y), t3_bits(v1.x), t3_bits(v1.y), w);
#pragma unroll
          for (int s = 0; s < T3_S; ++s) w4[s][q4] = w[s];
        }
        const int off = tc_off(pn, 16 * g);
#pragma unroll
        for (int s = 0; s < T3_S; ++s)
          *reinterpret_cast<uint4 *>(sb + s * TS_BSL + off) =
              make_uint4(w4[s][0], w4[s][1], w4[s][2], w4[s][3]);
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&b_full[bs]));
    }
  }

  // ---- epilogue (as k3t_gemm) ----
  mbar_wait(smem_u32(&acc_full), 0);
  tc_fence_after();
  __syncthreads();
  constexpr int ES = TS_NP + 1;
  double *E = reinterpret_cast<double *>(smem);
  const int XS = A + 1;
  double2 *Xt = reinterpret_cast<double2 *>(smem + 128 * ES * sizeof(double));
  for (int t = threadIdx.x; t < TS_NP * ((XS + 7) / 8); t += TS_THREADS) {
    const int n = t % TS_NP, a0 = 8 * (t / TS_NP);
    const int64_t jg = p_begin + (int64_t)ptile * TS_NP + n;
    const double fx = jg < p_end ? frac[jg].x : 0.0;
    double sn, cs;
    sincospi(2.0 * fx, &sn, &cs);
    const double2 e1 = make_double2(cs, sn);
    sincospi(2.0 * ((double)a0 * fx), &sn, &cs);
    double2 x = make_double2(cs, sn);
    for (int a = a0; a < min(XS, a0 + 8); ++a) {
      Xt[n * XS + a] = x;
      x = cmul(x, e1);
    }
  }
  __syncthreads();
  if (warp < 8) {
    const int q = warp & 3, h = warp >> 2;
    const int r = 32 * q + lane;
    const int rg = mtile * 128 + r;
    const bool live = rg < n_rows && nkb > 0;
    const T3Row R = live ? rows[rg] : T3Row{0, 0};
    const double rsc = live ? row_scale[rg] / (T3_SC * T3_SC) : 0.0;
    const int comp = R.type >> 1;
    const bool im_row = (R.type & 1) == 0;
    const double wx = comp == 0 ? (double)R.a : 1.0;
#pragma unroll 1
    for (int c0 = 0; c0 < TS_NP / 2; c0 += 8) {
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = 0.0;
#pragma unroll
      for (int l = T3_NL - 1; l >= 0; --l) {
        int rr[8];
        tc_ld8(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(l * TS_NP + (TS_NP / 2) * h + c0), rr);
        tc_wait_ld();
        const double wl = ldexp(1.0, 8 * (T3_W0 + l));
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = fma((double)rr[k], wl, v[k]);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int n = (TS_NP / 2) * h + c0 + k;
        const double2 x = Xt[n * XS + R.a];
        E[r * ES + n] = live ? v[k] * rsc * (im_row ? x.x : x.y) * wx : 0.0;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
  const int ks_index = split * n_mtiles + mtile;
  for (int t = threadIdx.x; t < 3 * TS_NP; t += TS_THREADS) {
    const int c = t / TS_NP, n = t % TS_NP;
    const int64_t i = (int64_t)ptile * TS_NP + n;
    if (i >= n_local) continue;
    const int4 cr = comp_rows[mtile];
    const int lo = c == 0 ? 0 : (c == 1 ? cr.x : cr.y), hi = c == 0 ? cr.x : (c == 1 ? cr.y : cr.z);
    double s = 0.0;
    for (int rr = lo; rr < hi; ++rr) s += E[rr * ES + n];
    fpart[(size_t)ks_index * 3 * n_local + (size_t)c * n_local + i] = s;
  }
}

// TS-mode throughput probe: A (M=128 x K=32 int8) read from TMEM columns
// [256, 264), B from shared memory, N = n_mma, back-to-back MMAs into
// accumulator columns [0, n_mma).
__global__ void __launch_bounds__(128, 1) k_i8_probe_ts(int iters, int n_mma, int *__restrict__ sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t done;
  __shared__ uint32_t tmem_base_s;
  for (int i = threadIdx.x; i < 32 * TC_SBO / 4; i += blockDim.x)
    reinterpret_cast<uint32_t *>(smem)[i] = 0x01010101u * (uint32_t)(i & 3);
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&tmem_base_s))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  {
    const uint32_t w[8] = {0x01010101u, 0x02020202u, 0x01010101u, 0x03030303u,
                           0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u};
    tc_st8(tmem + ((uint32_t)(32 * ((threadIdx.x >> 5) & 3)) << 16) + 256u, w);
    tc_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n_mma >> 3) << 17) | (8u << 24);
    const uint64_t bd = tc_desc(smem_u32(smem));
    for (int i = 0; i < iters; ++i) tc_mma_ts(tmem, tmem + 256u, bd + (uint64_t)((i & 1) * 16), idesc, i > 0 ? 1u : 0u);
    tc_commit(smem_u32(&done));
  }
  mbar_wait(smem_u32(&done), 0);
  tc_fence_after();
  if ((threadIdx.x >> 5) == 0) {
    int r[8];
    tc_ld8(tmem, r);
    tc_wait_ld();
    if (r[0] == 123456789) sink[0] = r[1];
  }
  tc_fence_before();
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}
