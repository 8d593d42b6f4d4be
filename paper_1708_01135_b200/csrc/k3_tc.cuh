// k3_tc.cuh -- reciprocal-space forces (Algorithm 2, ewald.py:306-331) on the
// int8 tensor cores.  Included by ewald_b200.cu after k1_tc.cuh (same
// fixed-point slicing, TMEM levels and pipeline primitives).
//
// F_c(j) = sum_k m_c Im(e^{+ik.r_j} W_k),  W_k = C_k S_k  (the K3 convention:
// k3_combine applies 4 pi q_j / L).  With e^{ik.r} = X(m_x) YZ(m_y, m_z) and
// the +-a = |m_x| columns folded into Wsum = W(a,p) + W(-a,p) and
// Wdiff = W(a,p) - W(-a,p) (p = yz pair):
//   Fx = sum_a a  [Xr(a) Im V(Wdiff)    + Xi(a) Re V(Wsum)]
//   Fy = sum_a    [Xr(a) Im V(my Wsum)  + Xi(a) Re V(my Wdiff)]
//   Fz = sum_a    [Xr(a) Im V(mz Wsum)  + Xi(a) Re V(mz Wdiff)]
// where V(w) = sum_p YZ_j(p) w(p) and X(a) = e^{+i 2pi a f_x}.  Every
// Re/Im V(.) is one row of a real GEMM over K = (Re YZ, Im YZ) of all pairs:
//   D[row, j] = sum_k Arow[k] * B[j, k],  B[j, 2p] = Re YZ_j(p), B[j, 2p+1] = Im YZ_j(p)
//   Im-row: A[2p] = Im w(p), A[2p+1] = Re w(p);  Re-row: A[2p] = Re w(p), A[2p+1] = -Im w(p)
// Rows per a > 0: 6; a = 0: Im V(my W), Im V(mz W) (X(0) = 1).  A rows are
// scaled per row (the scale factors out of the sum), B = unit phases.
//
// CTA = (64 particles, M tile of 128 rows, k split); warps 0-7 generate the
// YZ slices of a K-block (32 pairs = 4 runs of 8 consecutive m_y: one
// sincospi + a recurrence per run), warp 8 issues the 26 x 2 MMAs
// (M=128, N=64, K=32), warp 9 bulk-copies the pre-split A slices.  The
// epilogue combines the 7 levels, multiplies by the particle's X(a) and
// reduces over the rows (warp shuffles + shared memory).

constexpr int T3_NP = 64;         // particles per CTA (MMA N)
constexpr int T3_AS = 3;          // A ring depth
constexpr int T3_BSL = (T3_NP / 8) * TC_SBO;  // one B slice (64 rows x 64 B)
constexpr int T3_KMAX = 16384;    // K (bytes) per CTA: int32 exactness
__host__ __device__ constexpr int t3_smem_bytes() {
  return T3_AS * TC_S * TC_GSL + 2 * TC_S * T3_BSL;
}

// rows: type 0 Im V(Wdiff) [x], 1 Re V(Wsum) [x], 2 Im V(my Wsum), 3 Re V(my Wdiff),
//       4 Im V(mz Wsum), 5 Re V(mz Wdiff)
struct T3Row {
  int a, type;
};

// k3t_wprep: one block per A row: the row's values over all K entries,
// its max |value| (row scale), then the six digit slices in the K-block
// shared-memory image: wsl[((mtile * nkb + kb) * 6 + s) * TC_GSL + tc_off(r, k)]
__global__ void __launch_bounds__(256)
    k3t_wprep(const double2 *__restrict__ sp, const int *__restrict__ slotmap, int A,
              const int2 *__restrict__ pair_yz, int n_pairs_pad, const T3Row *__restrict__ rows,
              int n_rows, int nkb, double *__restrict__ row_scale, uint8_t *__restrict__ wsl) {
  __shared__ double red[8];
  const int r = blockIdx.x;
  const int mtile = r / 128, rl = r % 128;
  const bool live = r < n_rows;
  const T3Row R = live ? rows[r] : T3Row{0, 0};
  const bool im_row = (R.type & 1) == 0;  // types 0, 2, 4
  const bool use_sum = R.type == 1 || R.type == 2 || R.type == 4;
  auto value = [&](int k) -> double {
    if (!live) return 0.0;
    const int p = k >> 1;
    if (p >= n_pairs_pad) return 0.0;
    const int2 yz = pair_yz[p];
    if (yz.x == INT_MIN) return 0.0;  // padding pair
    const int sp_ = slotmap[(size_t)(A + R.a) * n_pairs_pad + p];
    const int sm_ = slotmap[(size_t)(A - R.a) * n_pairs_pad + p];
    double2 w = make_double2(0.0, 0.0);
    const double2 wp = sp_ >= 0 ? sp[sp_] : make_double2(0.0, 0.0);
    if (R.a == 0) {
      w = wp;
    } else {
      const double2 wm = sm_ >= 0 ? sp[sm_] : make_double2(0.0, 0.0);
      w = use_sum ? make_double2(wp.x + wm.x, wp.y + wm.y) : make_double2(wp.x - wm.x, wp.y - wm.y);
    }
    const double cw = R.type <= 1 ? 1.0 : (R.type <= 3 ? (double)yz.x : (double)yz.y);
    w.x *= cw;
    w.y *= cw;
    if (im_row) return (k & 1) ? w.x : w.y;
    return (k & 1) ? -w.y : w.x;
  };
  const int K = 2 * n_pairs_pad;
  double m = 0.0;
  for (int k = threadIdx.x; k < K; k += blockDim.x) m = fmax(m, fabs(value(k)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  double mx = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) mx = fmax(mx, red[i]);
  const double inv = mx > 0.0 ? 1.0 / mx : 0.0;
  if (threadIdx.x == 0) row_scale[r] = mx;
  // digits: one word (4 consecutive k) per thread and slice
  for (int k4 = threadIdx.x * 4; k4 < nkb * TC_KB; k4 += blockDim.x * 4) {
    uint2 b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) b[u] = tc_bits(fmin(1.0, fmax(-1.0, value(k4 + u) * inv)));
    uint32_t w[TC_S];
    tc_digits4(b[0], b[1], b[2], b[3], w);
    const int kb = k4 / TC_KB, kin = k4 % TC_KB;
    uint8_t *base = wsl + ((size_t)mtile * nkb + kb) * TC_S * TC_GSL;
    const int off = tc_off(rl, kin);
#pragma unroll
    for (int s = 0; s < TC_S; ++s) *reinterpret_cast<uint32_t *>(base + s * TC_GSL + off) = w[s];
  }
}

// k3t_gemm: grid (particle tiles of 64, M tiles, k splits).
//   pair_yz[p] = (m_y, m_z) of K pair p (runs of 8 consecutive m_y, padded
//   entries INT_MIN); fpart[(ks_index) * 3 * n_local + c * n_local + i].
__global__ void __launch_bounds__(TC_NTHREADS, 1)
    k3t_gemm(const double4 *__restrict__ frac, const double2 *__restrict__ base,
             const uint8_t *__restrict__ wsl, const double *__restrict__ row_scale,
             const T3Row *__restrict__ rows, int n_rows, const int2 *__restrict__ pair_yz,
             int nkb_all, int kb_per_split, int64_t p_begin, int64_t p_end,
             double *__restrict__ fpart, int dbg) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t b_full[2], b_empty[2], a_full[T3_AS], a_empty[T3_AS], acc_full;
  __shared__ uint32_t tmem_base_s;
  const int ptile = blockIdx.x, mtile = blockIdx.y, split = blockIdx.z;
  const int n_mtiles = gridDim.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_local = p_end - p_begin;
  const int kb0 = split * kb_per_split;
  const int nkb = max(0, min(nkb_all, kb0 + kb_per_split) - kb0);
  uint8_t *abuf = smem;
  uint8_t *bbuf = smem + T3_AS * TC_S * TC_GSL;
  constexpr int ABLK = TC_S * TC_GSL;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&b_full[i]), TC_THREADS / 32);
      mbar_init(smem_u32(&b_empty[i]), 1);
    }
    for (int i = 0; i < T3_AS; ++i) {
      mbar_init(smem_u32(&a_full[i]), 1);
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

  if (warp == 9) {
    if (lane == 0) {
      for (int it = 0; it < nkb; ++it) {
        const int as = it % T3_AS;
        if (it >= T3_AS) mbar_wait(smem_u32(&a_empty[as]), ((it / T3_AS) - 1) & 1);
        const uint8_t *src = wsl + ((size_t)mtile * nkb_all + kb0 + it) * (size_t)ABLK;
        const uint32_t fb = smem_u32(&a_full[as]);
        mbar_expect_tx(fb, (uint32_t)ABLK);
        bulk_g2s(smem_u32(abuf + as * ABLK), src, (uint32_t)ABLK, fb);
      }
    }
  } else if (warp == 8) {
    if (lane == 0) {
      const uint32_t idesc =
          (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(T3_NP >> 3) << 17) | (8u << 24);
      for (int it = 0; it < nkb; ++it) {
        const int bs = it & 1, as = it % T3_AS;
        mbar_wait(smem_u32(&b_full[bs]), (it >> 1) & 1);
        mbar_wait(smem_u32(&a_full[as]), (it / T3_AS) & 1);
        tc_fence_after();
        if (!(dbg & 2)) {
          const uint64_t ad = tc_desc(smem_u32(abuf + as * ABLK));
          const uint64_t bd = tc_desc(smem_u32(bbuf + bs * TC_S * T3_BSL));
          const uint32_t acc0 = it > 0 ? 1u : 0u;
#pragma unroll
          for (int l = 0; l < TC_NL; ++l) {
            const int w = TC_W0 + l;
            const int s_lo = w - (TC_S - 1) > 0 ? w - (TC_S - 1) : 0;
#pragma unroll
            for (int s = 0; s < TC_S; ++s) {
              const int t = w - s;
              if (t < 0 || t >= TC_S) continue;
#pragma unroll
              for (int ks = 0; ks < TC_KB / 32; ++ks)
                tc_mma(tmem + (uint32_t)(l * T3_NP), ad + (uint64_t)((s * TC_GSL + ks * 256) >> 4),
                       bd + (uint64_t)((t * T3_BSL + ks * 256) >> 4), idesc,
                       (s > s_lo || ks > 0) ? 1u : acc0);
            }
          }
          tc_commit(smem_u32(&b_empty[bs]));
          tc_commit(smem_u32(&a_empty[as]));
        } else {
          mbar_arrive(smem_u32(&b_empty[bs]));
          mbar_arrive(smem_u32(&a_empty[as]));
        }
      }
      if (!(dbg & 2) && nkb > 0)
        tc_commit(smem_u32(&acc_full));
      else
        mbar_arrive(smem_u32(&acc_full));
    }
  } else {
    // ---- B producers: particle n, run g of the K-block (8 pairs = 16 k) ----
    // lanes: 8 particles (lane & 7) x 4 runs (lane >> 3); warps: 8 particle octets
    const int pn = warp * 8 + (lane & 7);
    const int g = lane >> 3;
    const int64_t jg = p_begin + (int64_t)ptile * T3_NP + pn;
    const bool pvalid = jg < p_end;
    const int64_t jc = pvalid ? jg : p_begin;
    const double4 f = frac[jc];
    const double2 by = base[3 * jc + 1];
    const double2 ey = make_double2(by.x, -by.y);  // e^{+i 2pi f_y}
    for (int it = 0; it < nkb; ++it) {
      const int bs = it & 1;
      uint8_t *sb = bbuf + bs * TC_S * T3_BSL;
      if (it >= 2) mbar_wait(smem_u32(&b_empty[bs]), ((it >> 1) - 1) & 1);
      if (!(dbg & 1)) {
        const int p0 = (kb0 + it) * (TC_KB / 2) + 8 * g;  // first pair of this run
        const int2 yz = pair_yz[p0];
        double2 cur = make_double2(0.0, 0.0);
        if (pvalid && yz.x != INT_MIN) {
          double sn, cs;
          sincospi(2.0 * ((double)yz.x * f.y + (double)yz.y * f.z), &sn, &cs);
          cur = make_double2(cs, sn);
        }
        uint32_t w4[TC_S][4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {  // pairs 2q4, 2q4+1 -> k = 4q4 .. 4q4+3
          const double2 v0 = cur;
          cur = cmul(cur, ey);
          const double2 v1 = cur;
          cur = cmul(cur, ey);
          uint32_t w[TC_S];
          tc_digits4(tc_bits(v0.x), tc_bits(v0.y), tc_bits(v1.x), tc_bits(v1.y), w);
#pragma unroll
          for (int s = 0; s < TC_S; ++s) w4[s][q4] = w[s];
        }
        const int off = tc_off(pn, 16 * g);
#pragma unroll
        for (int s = 0; s < TC_S; ++s)
          *reinterpret_cast<uint4 *>(sb + s * T3_BSL + off) =
              make_uint4(w4[s][0], w4[s][1], w4[s][2], w4[s][3]);
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&b_full[bs]));
    }
  }

  // ---- epilogue ----
  mbar_wait(smem_u32(&acc_full), 0);
  tc_fence_after();
  __syncthreads();
  // E[r][n] = this row's contribution to particle n's force component
  // comp(r): the level sum times the row scale times X-coefficient
  // (Xr for Im rows, Xi for Re rows, x a for the x component)
  constexpr int ES = T3_NP + 1;
  double *E = reinterpret_cast<double *>(smem);
  int *rcomp = reinterpret_cast<int *>(smem + 128 * ES * sizeof(double));
  if (warp < 8) {
    const int q = warp & 3, h = warp >> 2;
    const int r = 32 * q + lane;
    const int rg = mtile * 128 + r;
    const bool live = rg < n_rows && nkb > 0;
    const T3Row R = live ? rows[rg] : T3Row{0, 0};
    const double rsc = live ? row_scale[rg] / (TC_SC * TC_SC) : 0.0;
    const int comp = R.type >> 1;  // 0 x, 1 y, 2 z
    const bool im_row = (R.type & 1) == 0;
    if (h == 0) rcomp[r] = live ? comp : -1;
#pragma unroll 1
    for (int c0 = 0; c0 < 32; c0 += 8) {
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = 0.0;
#pragma unroll
      for (int l = TC_NL - 1; l >= 0; --l) {
        int rr[8];
        tc_ld8(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(l * T3_NP + 32 * h + c0), rr);
        tc_wait_ld();
        const double wl = ldexp(1.0, 8 * (TC_W0 + l));
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = fma((double)rr[k], wl, v[k]);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int n = 32 * h + c0 + k;
        const int64_t jg = p_begin + (int64_t)ptile * T3_NP + n;
        double coef = 0.0;
        if (live && jg < p_end) {
          double sn = 0.0, cs = 1.0;
          if (R.a != 0) sincospi(2.0 * ((double)R.a * frac[jg].x), &sn, &cs);
          coef = (im_row ? cs : sn) * (comp == 0 ? (double)R.a : 1.0);
        }
        E[r * ES + n] = v[k] * rsc * coef;
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
  for (int t = threadIdx.x; t < 3 * T3_NP; t += TC_NTHREADS) {
    const int c = t / T3_NP, n = t % T3_NP;
    const int64_t i = (int64_t)ptile * T3_NP + n;
    if (i >= n_local) continue;
    double s = 0.0;
    for (int r = 0; r < 128; ++r)
      if (rcomp[r] == c) s += E[r * ES + n];
    fpart[(size_t)ks_index * 3 * n_local + (size_t)c * n_local + i] = s;
  }
}

// k_i8_probe: the roofline denominator for the tensor-core kernels.  One CTA
// per SM issues `iters` back-to-back int8 MMAs (M=128, N=256, K=32, both
// operands in shared memory, the same no-swizzle K-major layout as the
// kernels above) into TMEM and waits for them.
__global__ void __launch_bounds__(128, 1) k_i8_probe(int iters, int *__restrict__ sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t done;
  __shared__ uint32_t tmem_base_s;
  for (int i = threadIdx.x; i < (16 + 32) * TC_SBO / 4; i += blockDim.x)
    reinterpret_cast<uint32_t *>(smem)[i] = 0x01010101u * (uint32_t)(i & 3);
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                     smem_u32(&tmem_base_s))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | (8u << 24);
    const uint64_t ad = tc_desc(smem_u32(smem)), bd = tc_desc(smem_u32(smem + 16 * TC_SBO));
    for (int i = 0; i < iters; ++i) tc_mma(tmem, ad + (uint64_t)((i & 1) * 16), bd, idesc, i > 0 ? 1u : 0u);
    tc_commit(smem_u32(&done));
  }
  mbar_wait(smem_u32(&done), 0);
  tc_fence_after();
  if ((threadIdx.x >> 5) == 0) {
    int r[8];
    tc_ld8(tmem + ((uint32_t)(32 * 0) << 16), r);
    tc_wait_ld();
    if (r[0] == 123456789) sink[0] = r[1];
  }
  tc_fence_before();
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  }
}
