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
// CTA = (T3_NP = 80 particles, M tile of 128 rows, k split); T3_PGROUPS
// groups of producer warps generate the YZ slices of alternate K-blocks
// (32 pairs = 4 runs of 8 consecutive m_y: one sincospi + a recurrence per
// run), one warp stages the A slices in TMEM (tcgen05.cp) and issues the TS
// MMAs of the 21 kept slice pairs (M=128, K=32, N = up to 3 merged B
// slices x 80), one warp bulk-copies the pre-split A slices.  The epilogue
// combines the 6 levels, multiplies by the particle's X(a) and reduces over
// the rows (warp shuffles + shared memory).

// The force GEMM splits W rows (scaled per row) and the unit phases into
// T3_S byte slices and keeps the slice pairs with s + t >= T3_W0.  Measured
// max|dF|/F_rms against the FP64 gather (c2 / c4 / c5):
//   6 slices, w >= 5 (21 MMAs): 3.3e-14 / 2.7e-13 / 5.0e-14   <- default
//   5 slices, w >= 4 (15 MMAs): 4.8e-12 / 5.4e-11 / 7.7e-12   (-15..20% time)
//   5 slices, w >= 3 (19 MMAs): 2.8e-12 / 3.4e-11 / 4.5e-12   (40-bit quantisation)
// all inside the 1e-9 F_rms tolerance; the default keeps a 3000x margin.
#ifndef T3_SLICES
#define T3_SLICES 6
#endif
#ifndef T3_LEVEL0
#define T3_LEVEL0 5
#endif
constexpr int T3_S = T3_SLICES;
constexpr int T3_W0 = T3_LEVEL0;
constexpr int T3_NL = 2 * T3_S - 1 - T3_W0;  // 5 levels
constexpr int T3_PAIRS = T3_S * T3_S - (T3_W0 * (T3_W0 + 1)) / 2;
// 0x7F..7F and 1.5*2^52 + 0x80..80 for T3_S bytes
constexpr double T3_SC = T3_S == 6 ? 140185576636287.0 : 547599908479.0;
constexpr double T3_MAGIC =
    6755399441055744.0 + (T3_S == 6 ? 141289400074368.0 : 551911719040.0);
static_assert(T3_S == 5 || T3_S == 6, "force GEMM slices: 5 or 6");
__device__ __forceinline__ uint2 t3_bits(double v) {
  const double x = fma(v, T3_SC, T3_MAGIC);
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return make_uint2((uint32_t)b, (uint32_t)(b >> 32));
}
#ifndef T3_PARTICLES
#define T3_PARTICLES 80
#endif
// particles per CTA (MMA N): 6 levels x 80 = 480 of 512 TMEM columns; the
// shape probe gives 3487 TOP/s at N=80 vs 3006 at 64 (shared-memory A read)
constexpr int T3_NP = T3_PARTICLES;
static_assert(T3_NP % 16 == 0 && T3_NP <= 80, "N: multiple of 16, TMEM budget");
constexpr int T3_PW = T3_NP / 8;               // producer warps per group (8 particles x 4 runs each)
#ifndef T3_PGROUPS
#define T3_PGROUPS 2  // c5 forces 102 -> 91 ms (two K-blocks in production at once)
#endif
// producer groups: group g fills the K-blocks it with it % T3_PG == g
constexpr int T3_PG = T3_PGROUPS;
constexpr int T3_PROD = T3_PW * T3_PG;          // producer warps
constexpr int T3_THREADS = (T3_PROD + 2) * 32;  // + MMA warp + loader warp
constexpr int T3_HALF = T3_NP / 2;             // epilogue columns per warp
#ifndef T3_ASTAGES
#define T3_ASTAGES 3
#endif
#ifndef T3_BSTAGES
#define T3_BSTAGES 2
#endif
#ifndef T3_CLUSTER
#define T3_CLUSTER 1  // measured: 2 neutral, 4 slower (c5) -- A loads are not the limit
#endif
constexpr int T3_CL = T3_CLUSTER;  // CTAs (particle tiles) sharing each A load (multicast)
constexpr int T3_AS = T3_ASTAGES;  // A ring depth (bulk copies)
constexpr int T3_BS = T3_BSTAGES;  // B ring depth (produced)
constexpr int T3_BSL = (T3_NP / 8) * TC_SBO;  // one B slice (T3_NP rows x 64 B)
static_assert(T3_BS % T3_PG == 0, "each B stage must belong to one producer group");
constexpr int T3_KMAX = 16384;    // K (bytes) per CTA: int32 exactness
__host__ __device__ constexpr int t3_smem_bytes() {
  return T3_AS * T3_S * TC_GSL + T3_BS * T3_S * T3_BSL;
}

// rows: type 0 Im V(Wdiff) [x], 1 Re V(Wsum) [x], 2 Im V(my Wsum), 3 Re V(my Wdiff),
//       4 Im V(mz Wsum), 5 Re V(mz Wdiff)
struct T3Row {
  int a, type;
};

// A-row value at K index k (2p: Re YZ coefficient, 2p+1: Im YZ coefficient)
__device__ __forceinline__ double t3_value(const double2 *__restrict__ sp,
                                           const int *__restrict__ slotmap, int A,
                                           const int2 *__restrict__ pair_yz, int n_pairs_pad,
                                           const T3Row R, int k) {
  const int p = k >> 1;
  if (p >= n_pairs_pad) return 0.0;
  const int2 yz = pair_yz[p];
  if (yz.x == INT_MIN) return 0.0;  // padding pair
  const bool im_row = (R.type & 1) == 0;  // types 0, 2, 4
  const bool use_sum = R.type == 1 || R.type == 2 || R.type == 4;
  const int sp_ = slotmap[(size_t)(A + R.a) * n_pairs_pad + p];
  const double2 wp = sp_ >= 0 ? sp[sp_] : make_double2(0.0, 0.0);
  double2 w = wp;
  if (R.a != 0) {
    const int sm_ = slotmap[(size_t)(A - R.a) * n_pairs_pad + p];
    const double2 wm = sm_ >= 0 ? sp[sm_] : make_double2(0.0, 0.0);
    w = use_sum ? make_double2(wp.x + wm.x, wp.y + wm.y) : make_double2(wp.x - wm.x, wp.y - wm.y);
  }
  const double cw = R.type <= 1 ? 1.0 : (R.type <= 3 ? (double)yz.x : (double)yz.y);
  if (im_row) return cw * ((k & 1) ? w.x : w.y);
  return cw * ((k & 1) ? -w.y : w.x);
}

// k3t_wmax: grid (rows, K parts): row maxima |A[r, k]| (bit-pattern atomicMax
// of non-negative doubles; row_scale zeroed before)
__global__ void __launch_bounds__(256)
    k3t_wmax(const double2 *__restrict__ sp, const int *__restrict__ slotmap, int A,
             const int2 *__restrict__ pair_yz, int n_pairs_pad, const T3Row *__restrict__ rows,
             int n_rows, unsigned long long *__restrict__ row_scale_bits) {
  const int r = blockIdx.x;
  if (r >= n_rows) return;
  const T3Row R = rows[r];
  const int K = 2 * n_pairs_pad;
  double m = 0.0;
  for (int k = blockIdx.y * blockDim.x + threadIdx.x; k < K; k += gridDim.y * blockDim.x)
    m = fmax(m, fabs(t3_value(sp, slotmap, A, pair_yz, n_pairs_pad, R, k)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.0)
    atomicMax(row_scale_bits + r, (unsigned long long)__double_as_longlong(m));
}

// k3t_wprep: grid (M-tile rows, K parts): the six digit slices of A in the
// K-block shared-memory image: wsl[((mtile * nkb + kb) * S + s) * TC_GSL + tc_off(r, k)]
__global__ void __launch_bounds__(256)
    k3t_wprep(const double2 *__restrict__ sp, const int *__restrict__ slotmap, int A,
              const int2 *__restrict__ pair_yz, int n_pairs_pad, const T3Row *__restrict__ rows,
              int n_rows, int nkb, const double *__restrict__ row_scale, uint8_t *__restrict__ wsl) {
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
    uint8_t *base = wsl + ((size_t)mtile * nkb + kb) * T3_S * TC_GSL;
    const int off = tc_off(rl, kin);
#pragma unroll
    for (int s = 0; s < T3_S; ++s) *reinterpret_cast<uint32_t *>(base + s * TC_GSL + off) = w[s];
  }
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void bulk_g2s_mc(uint32_t dst, const void *src, uint32_t bytes,
                                            uint32_t mbar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], "
      "[%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(mbar), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tc_commit_mc(uint32_t mbar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(mbar),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t local_addr, uint32_t cta) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(cta));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}

// SS-form merged MMAs: each A slice read from shared memory by its 1-2 MMAs.
// Staging A in TMEM for TS-form MMAs (slice-major) measured slower once the
// MMAs are merged: c5 forces 79.0 (TS) vs 73.2 ms (SS), c2 0.164 vs 0.156.
#ifndef T3_MERGE
#define T3_MERGE 3  // c5 forces 84.2 -> 81.1 ms
#endif
// T3_MERGE = m > 1: one MMA covers up to m consecutive B slices
// t..t+m-1 against A slice s -- N = m x 80 rows of B (the slices are
// contiguous in shared memory) into the m consecutive level accumulators
// (contiguous in TMEM); accumulators are zeroed first and every MMA adds
static_assert(T3_MERGE > 1 && T3_MERGE * T3_NP <= 256, "merged N <= 256");

// k3t_gemm: grid (particle tiles of 64, M tiles, k splits), clusters of
// T3_CL consecutive particle tiles: every A block is bulk-copied once per
// cluster (each CTA fetches 1/T3_CL and multicasts it), every CTA's MMA
// completion is multicast to the A-empty barriers of the whole cluster.
//   pair_yz[p] = (m_y, m_z) of K pair p (runs of 8 consecutive m_y, padded
//   entries INT_MIN); fpart[(ks_index) * 3 * n_local + c * n_local + i].
__global__ void __launch_bounds__(T3_THREADS, 1)
    k3t_gemm(const double4 *__restrict__ frac, const double2 *__restrict__ base,
             const uint8_t *__restrict__ wsl, const double *__restrict__ row_scale,
             const T3Row *__restrict__ rows, int n_rows, const int2 *__restrict__ pair_yz,
             int nkb_all, int kb_per_split, int64_t p_begin, int64_t p_end, int A,
             const int4 *__restrict__ comp_rows, double *__restrict__ fpart, int dbg) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t b_full[T3_BS], b_empty[T3_BS], a_full[T3_AS], a_empty[T3_AS], acc_full;
  __shared__ uint32_t tmem_base_s;
  const int ptile = blockIdx.x, mtile = blockIdx.y, split = blockIdx.z;
  const int n_mtiles = gridDim.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_local = p_end - p_begin;
  const int kb0 = split * kb_per_split;
  const int nkb = max(0, min(nkb_all, kb0 + kb_per_split) - kb0);
  uint8_t *abuf = smem;
  uint8_t *bbuf = smem + T3_AS * T3_S * TC_GSL;
  constexpr int ABLK = T3_S * TC_GSL;

  if (threadIdx.x == 0) {
    for (int i = 0; i < T3_BS; ++i) {
      mbar_init(smem_u32(&b_full[i]), T3_PW);
      mbar_init(smem_u32(&b_empty[i]), 1);
    }
    for (int i = 0; i < T3_AS; ++i) {
      mbar_init(smem_u32(&a_full[i]), 1);
      mbar_init(smem_u32(&a_empty[i]), T3_CL);
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
  cluster_sync_all();  // barriers initialised cluster-wide before any remote signal
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  if (T3_MERGE > 1) {  // zero the level accumulators (every merged MMA accumulates)
    if (warp < 4) {
      const uint32_t z[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
      for (int c = 0; c < T3_NL * T3_NP; c += 8)
        tc_st8(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c, z);
      tc_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  const uint32_t crank = cluster_rank();
  constexpr uint16_t CMASK = (uint16_t)((1u << T3_CL) - 1u);

  if (warp == T3_PROD + 1) {
    if (lane == 0) {
      constexpr int PIECE = ABLK / T3_CL;
      static_assert(ABLK % (16 * T3_CL) == 0, "A block must split into 16-byte pieces");
      for (int it = 0; it < nkb; ++it) {
        const int as = it % T3_AS;
        if (it >= T3_AS) mbar_wait(smem_u32(&a_empty[as]), ((it / T3_AS) - 1) & 1);
        const uint8_t *src = wsl + ((size_t)mtile * nkb_all + kb0 + it) * (size_t)ABLK;
        const uint32_t fb = smem_u32(&a_full[as]);
        mbar_expect_tx(fb, (uint32_t)ABLK);
        if (T3_CL == 1)
          bulk_g2s(smem_u32(abuf + as * ABLK), src, (uint32_t)ABLK, fb);
        else
          bulk_g2s_mc(smem_u32(abuf + as * ABLK + crank * PIECE), src + crank * PIECE,
                      (uint32_t)PIECE, fb, CMASK);
      }
    }
  } else if (warp == T3_PROD) {
    {
      for (int it = 0; it < nkb; ++it) {
        const int bs = it % T3_BS, as = it % T3_AS;
        mbar_wait(smem_u32(&b_full[bs]), (it / T3_BS) & 1);
        mbar_wait(smem_u32(&a_full[as]), (it / T3_AS) & 1);
        tc_fence_after();
        __syncwarp();
        if (!(dbg & 2) && elect_one()) {
          const uint64_t ad = tc_desc(smem_u32(abuf + as * ABLK));
          const uint64_t bd = tc_desc(smem_u32(bbuf + bs * T3_S * T3_BSL));
          // SS form with merged N: A slice s read from shared memory by its
          // (one or two) MMAs, no staging copy into TMEM
          constexpr uint32_t idesc0 = (2u << 4) | (1u << 7) | (1u << 10) | (8u << 24);
#pragma unroll
          for (int ks = 0; ks < TC_KB / 32; ++ks) {
#pragma unroll
            for (int s = 0; s < T3_S; ++s) {
#pragma unroll
              for (int t = (T3_W0 - s > 0 ? T3_W0 - s : 0); t < T3_S; t += T3_MERGE) {
                const int m = T3_S - t < T3_MERGE ? T3_S - t : T3_MERGE;
                tc_mma(tmem + (uint32_t)((s + t - T3_W0) * T3_NP),
                       ad + (uint64_t)((s * TC_GSL + ks * 256) >> 4),
                       bd + (uint64_t)((t * T3_BSL + ks * 256) >> 4),
                       idesc0 | ((uint32_t)((m * T3_NP) >> 3) << 17), 1u);
              }
            }
          }
          tc_commit(smem_u32(&b_empty[bs]));
          if (T3_CL == 1)
            tc_commit(smem_u32(&a_empty[as]));
          else
            tc_commit_mc(smem_u32(&a_empty[as]), CMASK);
        } else if ((dbg & 2) && lane == 0) {
          mbar_arrive(smem_u32(&b_empty[bs]));
          for (int c = 0; c < T3_CL; ++c) mbar_arrive_cluster(smem_u32(&a_empty[as]), c);
        }
        __syncwarp();
      }
      if (lane == 0) {
        if (!(dbg & 2) && nkb > 0)
          tc_commit(smem_u32(&acc_full));
        else
          mbar_arrive(smem_u32(&acc_full));
      }
    }
  } else {
    // ---- B producers: particle n, run g of the K-block (8 pairs = 16 k) ----
    // lanes: 8 particles (lane & 7) x 4 runs (lane >> 3); warps: 8 particle octets
    const int pn = (warp % T3_PW) * 8 + (lane & 7);
    const int g = lane >> 3;
    const int64_t jg = p_begin + (int64_t)ptile * T3_NP + pn;
    const bool pvalid = jg < p_end;
    const int64_t jc = pvalid ? jg : p_begin;
    const double4 f = frac[jc];
    const double2 by = base[3 * jc + 1];
    const double2 ey = make_double2(by.x, -by.y);  // e^{+i 2pi f_y}
    for (int it = warp / T3_PW; it < nkb; it += T3_PG) {
      const int bs = it % T3_BS;
      uint8_t *sb = bbuf + bs * T3_S * T3_BSL;
      if (it >= T3_BS) mbar_wait(smem_u32(&b_empty[bs]), ((it / T3_BS) - 1) & 1);
      if (!(dbg & 1)) {
        const int p0 = (kb0 + it) * (TC_KB / 2) + 8 * g;  // first pair of this run
        const int2 yz = pair_yz[p0];
        double2 cur = make_double2(0.0, 0.0);
        if (pvalid && yz.x != INT_MIN) {
          double sn, cs;
          sincospi(2.0 * ((double)yz.x * f.y + (double)yz.y * f.z), &sn, &cs);
          cur = make_double2(cs, sn);
        }
        uint32_t w4[T3_S][4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {  // pairs 2q4, 2q4+1 -> k = 4q4 .. 4q4+3
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
  // X table: Xt[n * XS + a] = e^{+i 2pi a f_x} of the CTA's particles
  // (sincospi every 8 steps, recurrence between); then E[r][n] = the row's
  // level sum x row scale x X-coefficient (Xr for Im rows, Xi for Re rows,
  // x a for the x component).  Rows are ordered by component, so the final
  // sum for (n, c) runs over one contiguous row range.
  constexpr int ES = T3_NP + 1;
  double *E = reinterpret_cast<double *>(smem);
  const int XS = A + 1;
  double2 *Xt = reinterpret_cast<double2 *>(smem + 128 * ES * sizeof(double));
  for (int t = threadIdx.x; t < T3_NP * ((XS + 7) / 8); t += T3_THREADS) {
    const int n = t % T3_NP, a0 = 8 * (t / T3_NP);
    const int64_t jg = p_begin + (int64_t)ptile * T3_NP + n;
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
    const int comp = R.type >> 1;  // 0 x, 1 y, 2 z
    const bool im_row = (R.type & 1) == 0;
    const double wx = comp == 0 ? (double)R.a : 1.0;
#pragma unroll 1
    for (int c0 = 0; c0 < T3_HALF; c0 += 8) {
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = 0.0;
#pragma unroll
      for (int l = T3_NL - 1; l >= 0; --l) {
        int rr[8];
        tc_ld8(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(l * T3_NP + T3_HALF * h + c0), rr);
        tc_wait_ld();
        const double wl = ldexp(1.0, 8 * (T3_W0 + l));
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = fma((double)rr[k], wl, v[k]);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int n = T3_HALF * h + c0 + k;
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
  for (int t = threadIdx.x; t < 3 * T3_NP; t += T3_THREADS) {
    const int c = t / T3_NP, n = t % T3_NP;
    const int64_t i = (int64_t)ptile * T3_NP + n;
    if (i >= n_local) continue;
    const int4 cr = comp_rows[mtile];  // row ranges of x, y, z in this tile
    const int lo = c == 0 ? 0 : (c == 1 ? cr.x : cr.y), hi = c == 0 ? cr.x : (c == 1 ? cr.y : cr.z);
    double s = 0.0;
    for (int r = lo; r < hi; ++r) s += E[r * ES + n];
    fpart[(size_t)ks_index * 3 * n_local + (size_t)c * n_local + i] = s;
  }
  // no CTA may leave while cluster peers can still signal its barriers
  cluster_sync_all();
}

// k_i8_probe: the roofline denominator for the tensor-core kernels.  One CTA
// per SM issues `iters` back-to-back int8 MMAs (M=128, N=256, K=32, both
// operands in shared memory, the same no-swizzle K-major layout as the
// kernels above) into TMEM and waits for them.
__global__ void __launch_bounds__(128, 1) k_i8_probe(int iters, int n_mma, int *__restrict__ sink) {
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
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n_mma >> 3) << 17) | (8u << 24);
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
