// k3_pair.cuh -- the force GEMM of k3_tc.cuh on CTA PAIRS that split the
// accumulator levels.  Included after k3_tc.cuh.  Correct (tests), but
// measured slower than k3t_gemm (c5 124 vs 101 ms; with neither operand
// production nor MMAs the pair kernel already takes 83 ms against 37: each
// SM copies the full W block for half of the MMA work, the ring is two
// deep, and the CTAs run in lock step), so off by default (T3_PAIR).
//
// Why: an SS int8 MMA reads (M + N) x 32 bytes of shared memory for
// M x N x 32 MACs, and at N = 80 (the widest the 6 int32 levels x N <= 512
// TMEM columns allow) the MMA operand reads plus the operand stores use the
// whole shared-memory bandwidth of the SM (measured: MMA-only runs at the
// issue floor, full runs ~55% of it).  Two CTAs of a cluster process the
// SAME 144 particles and W rows and split the six levels (rank 0: w = 5, 8,
// 9 -- 11 slice pairs; rank 1: w = 6, 7, 10 -- 10 pairs), so each holds 3
// levels x 144 = 432 TMEM columns: N = 144 cuts the shared-memory bytes per
// MAC by 27% (1/144 + 1/128 vs 1/80 + 1/128) and runs the MMAs at the full
// rate (tools/i8_shapes.py: ~4560 vs 3503 TOP/s).
//
// The B operand (YZ phases of the 144 particles) is produced once: each CTA
// generates 72 particles and writes them to its own shared memory and, with
// st.async (complete_tx on the peer's mbarrier), to the peer's.  A stage of
// B may be overwritten only when BOTH CTAs' MMAs have read it: every MMA
// completion is multicast to the B-empty barriers of the pair.  Each CTA
// writes the partial sums of its own levels; k3_combine adds them.

constexpr int P3_NP = 144;                     // particles per pair (MMA N)
constexpr int P3_HALF = P3_NP / 2;             // produced per CTA
constexpr int P3_PW = P3_HALF / 8;             // producer warps (9)
constexpr int P3_MMA_WARP = P3_PW;
constexpr int P3_LD_WARP = P3_PW + 1;
constexpr int P3_THREADS = (P3_PW + 2) * 32;   // 352
constexpr int P3_AS = 2, P3_BS = 2;
constexpr int P3_BSL = (P3_NP / 8) * TC_SBO;   // one B slice (144 rows x 64 B)
constexpr int P3_ABLK = T3_S * TC_GSL;
constexpr int P3_BBLK = T3_S * P3_BSL;
constexpr int P3_NLV = 3;                      // levels per CTA
static_assert(T3_S == 6 && T3_W0 == 5, "level split written for 6 slices, w >= 5");
static_assert(P3_NLV * P3_NP <= 512, "TMEM budget");
constexpr int P3_REMOTE_BYTES = T3_S * P3_HALF * 64;  // the peer's half of a B stage

__host__ __device__ constexpr int p3_smem_bytes() { return P3_AS * P3_ABLK + P3_BS * P3_BBLK; }
__host__ __device__ constexpr int p3_level(int rank, int l) {
  return rank == 0 ? (l == 0 ? 5 : (l == 1 ? 8 : 9)) : (l == 0 ? 6 : (l == 1 ? 7 : 10));
}

__device__ __forceinline__ uint32_t mapa_u32(uint32_t local_addr, uint32_t cta) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(cta));
  return remote;
}
__device__ __forceinline__ void st_async_v4(uint32_t remote_addr, uint4 v, uint32_t remote_mbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::
          "r"(remote_addr),
      "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(remote_mbar)
      : "memory");
}

__global__ void __launch_bounds__(P3_THREADS, 1)
    k3p_gemm(const double4 *__restrict__ frac, const double2 *__restrict__ base,
             const uint8_t *__restrict__ wsl, const double *__restrict__ row_scale,
             const T3Row *__restrict__ rows, int n_rows, const int2 *__restrict__ pair_yz,
             int nkb_all, int kb_per_split, int64_t p_begin, int64_t p_end, int A,
             const int4 *__restrict__ comp_rows, double *__restrict__ fpart, int dbg) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t b_full[P3_BS], b_empty[P3_BS], a_full[P3_AS], a_empty[P3_AS], acc_full;
  __shared__ uint32_t tmem_base_s;
  const uint32_t rank = cluster_rank();
  const uint32_t peer = rank ^ 1u;
  const int ptile = blockIdx.x >> 1, mtile = blockIdx.y, split = blockIdx.z;
  const int n_mtiles = gridDim.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_local = p_end - p_begin;
  const int kb0 = split * kb_per_split;
  const int nkb = max(0, min(nkb_all, kb0 + kb_per_split) - kb0);
  uint8_t *abuf = smem;
  uint8_t *bbuf = smem + P3_AS * P3_ABLK;

  if (threadIdx.x == 0) {
    for (int i = 0; i < P3_BS; ++i) {
      mbar_init(smem_u32(&b_full[i]), P3_PW + 1);  // local producer warps + the expect_tx
      mbar_init(smem_u32(&b_empty[i]), 2);         // both CTAs' MMAs
    }
    for (int i = 0; i < P3_AS; ++i) {
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
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;

  if (warp == P3_LD_WARP) {
    if (lane == 0) {
      for (int it = 0; it < nkb; ++it) {
        const int as = it % P3_AS;
        if (it >= P3_AS) mbar_wait(smem_u32(&a_empty[as]), ((it / P3_AS) - 1) & 1);
        const uint8_t *src = wsl + ((size_t)mtile * nkb_all + kb0 + it) * (size_t)P3_ABLK;
        const uint32_t fb = smem_u32(&a_full[as]);
        mbar_expect_tx(fb, (uint32_t)P3_ABLK);
        bulk_g2s(smem_u32(abuf + as * P3_ABLK), src, (uint32_t)P3_ABLK, fb);
      }
    }
  } else if (warp == P3_MMA_WARP) {
    const uint32_t idesc =
        (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(P3_NP >> 3) << 17) | (8u << 24);
    for (int it = 0; it < nkb; ++it) {
      const int bs = it % P3_BS, as = it % P3_AS;
      mbar_wait(smem_u32(&b_full[bs]), (it / P3_BS) & 1);
      mbar_wait(smem_u32(&a_full[as]), (it / P3_AS) & 1);
      tc_fence_after();
      __syncwarp();
      if (!(dbg & 2) && elect_one()) {
        const uint64_t ad = tc_desc(smem_u32(abuf + as * P3_ABLK));
        const uint64_t bd = tc_desc(smem_u32(bbuf + bs * P3_BBLK));
        const uint32_t acc0 = it > 0 ? 1u : 0u;
        auto issue = [&](auto rank_tag) {
          constexpr int R = decltype(rank_tag)::value;
#pragma unroll
          for (int l = 0; l < P3_NLV; ++l) {
            const int w = p3_level(R, l);
            const int s_lo = w - (T3_S - 1) > 0 ? w - (T3_S - 1) : 0;
#pragma unroll
            for (int s = 0; s < T3_S; ++s) {
              const int t = w - s;
              if (t < 0 || t >= T3_S) continue;
#pragma unroll
              for (int ks = 0; ks < TC_KB / 32; ++ks)
                tc_mma(tmem + (uint32_t)(l * P3_NP), ad + (uint64_t)((s * TC_GSL + ks * 256) >> 4),
                       bd + (uint64_t)((t * P3_BSL + ks * 256) >> 4), idesc,
                       (s > s_lo || ks > 0) ? 1u : acc0);
            }
          }
        };
        if (rank == 0)
          issue(std::integral_constant<int, 0>{});
        else
          issue(std::integral_constant<int, 1>{});
        tc_commit(smem_u32(&a_empty[as]));
        tc_commit_mc(smem_u32(&b_empty[bs]), (uint16_t)0x3);
      } else if ((dbg & 2) && lane == 0) {
        mbar_arrive(smem_u32(&a_empty[as]));
        mbar_arrive(smem_u32(&b_empty[bs]));
        mbar_arrive_cluster(smem_u32(&b_empty[bs]), peer);
      }
      __syncwarp();
    }
    if (lane == 0) {
      if (!(dbg & 2) && nkb > 0)
        tc_commit(smem_u32(&acc_full));
      else
        mbar_arrive(smem_u32(&acc_full));
    }
  } else {
    // ---- producers: this CTA's 72 particles (rows 72*rank + pl), run g ----
    const int pl = warp * 8 + (lane & 7);
    const int prow = P3_HALF * (int)rank + pl;
    const int g = lane >> 3;
    const int64_t jg = p_begin + (int64_t)ptile * P3_NP + prow;
    const bool pvalid = jg < p_end;
    const int64_t jc = pvalid ? jg : p_begin;
    const double4 f = frac[jc];
    const double2 by = base[3 * jc + 1];
    const double2 ey = make_double2(by.x, -by.y);  // e^{+i 2pi f_y}
    const int off = tc_off(prow, 16 * g);
    for (int it = 0; it < nkb; ++it) {
      const int bs = it % P3_BS;
      uint8_t *sb = bbuf + bs * P3_BBLK;
      if (it >= P3_BS) mbar_wait(smem_u32(&b_empty[bs]), ((it / P3_BS) - 1) & 1);
      if (warp == 0 && lane == 0) mbar_expect_tx(smem_u32(&b_full[bs]), (uint32_t)P3_REMOTE_BYTES);
      const uint32_t rmbar = mapa_u32(smem_u32(&b_full[bs]), peer);
      const uint32_t rbase = mapa_u32(smem_u32(sb), peer);
      uint32_t w4[T3_S][4];
      if (!(dbg & 1)) {
        const int p0 = (kb0 + it) * (TC_KB / 2) + 8 * g;
        const int2 yz = pair_yz[p0];
        double2 cur = make_double2(0.0, 0.0);
        if (pvalid && yz.x != INT_MIN) {
          double sn, cs;
          sincospi(2.0 * ((double)yz.x * f.y + (double)yz.y * f.z), &sn, &cs);
          cur = make_double2(cs, sn);
        }
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
      } else {
#pragma unroll
        for (int s = 0; s < T3_S; ++s) w4[s][0] = w4[s][1] = w4[s][2] = w4[s][3] = 0u;
      }
#pragma unroll
      for (int s = 0; s < T3_S; ++s) {
        const uint4 v = make_uint4(w4[s][0], w4[s][1], w4[s][2], w4[s][3]);
        *reinterpret_cast<uint4 *>(sb + s * P3_BSL + off) = v;
        st_async_v4(rbase + (uint32_t)(s * P3_BSL + off), v, rmbar);
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&b_full[bs]));
    }
  }

  // ---- epilogue: this CTA's levels, two passes of 72 particles ----
  mbar_wait(smem_u32(&acc_full), 0);
  tc_fence_after();
  __syncthreads();
  constexpr int PC = P3_HALF;  // particles per pass
  constexpr int ES = PC + 1;
  double *E = reinterpret_cast<double *>(smem);
  const int XS = A + 1;
  double2 *Xt = reinterpret_cast<double2 *>(smem + 128 * ES * sizeof(double));
  const int ks_index = ((split * n_mtiles + mtile) << 1) + (int)rank;
  for (int pass = 0; pass < 2; ++pass) {
    const int n0 = pass * PC;
    for (int t = threadIdx.x; t < PC * ((XS + 7) / 8); t += P3_THREADS) {
      const int n = t % PC, a0 = 8 * (t / PC);
      const int64_t jg = p_begin + (int64_t)ptile * P3_NP + n0 + n;
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
      // 9 chunks of 8 columns: h = 0 takes chunks 0..4, h = 1 chunks 5..8
#pragma unroll 1
      for (int ch = h * 5; ch < (h == 0 ? 5 : 9); ++ch) {
        const int c0 = ch * 8;
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = 0.0;
#pragma unroll
        for (int l = 0; l < P3_NLV; ++l) {
          int rr[8];
          tc_ld8(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(l * P3_NP + n0 + c0), rr);
          tc_wait_ld();
          const double wl = ldexp(1.0, 8 * (rank == 0 ? p3_level(0, l) : p3_level(1, l)));
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = fma((double)rr[k], wl, v[k]);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int n = c0 + k;
          const double2 x = Xt[n * XS + R.a];
          E[r * ES + n] = live ? v[k] * rsc * (im_row ? x.x : x.y) * wx : 0.0;
        }
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 3 * PC; t += P3_THREADS) {
      const int c = t / PC, n = t % PC;
      const int64_t i = (int64_t)ptile * P3_NP + n0 + n;
      if (i >= n_local) continue;
      const int4 cr = comp_rows[mtile];
      const int lo = c == 0 ? 0 : (c == 1 ? cr.x : cr.y), hi = c == 0 ? cr.x : (c == 1 ? cr.y : cr.z);
      double s = 0.0;
      for (int rr = lo; rr < hi; ++rr) s += E[rr * ES + n];
      fpart[(size_t)ks_index * 3 * n_local + (size_t)c * n_local + i] = s;
    }
    __syncthreads();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
  cluster_sync_all();  // the peer may still signal our barriers until here
}
