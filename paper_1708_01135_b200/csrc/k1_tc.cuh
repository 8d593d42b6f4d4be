// k1_tc.cuh -- structure factor S(k) on the int8 tensor cores (tcgen05.mma
// kind::i8, accumulators in TMEM).  Included by ewald_b200.cu inside its
// anonymous namespace.
//
// Algorithm 1 of the reference (ewald.py:281-305, S(k) = sum_j q_j e^{-ik.r_j})
// factorises over the axes: e^{-ik.r} = X_a(x) * G_{my,mz}(y,z) with
// X_a = e^{-+i 2pi a f_x} (a = |m_x|) and G = q e^{-i 2pi (m_y f_y + m_z f_z)}.
// For one (m_y, m_z) "yz pair" and one a, with Xr = cos(2pi a f_x),
// Xs = sin(2pi a f_x):
//     P1 = sum Xr Re G,  P2 = sum Xs Im G,  P3 = sum Xr Im G,  P4 = sum Xs Re G
//     S(+-a, m_y, m_z) = (P1 +- P2) + i (P3 -+ P4),
// i.e. four real products per pair, all of them entries of ONE real GEMM
//     D[row, col] = sum_j Gop[row, j] * Xop[col, j]
// with rows = (Re G, Im G) of 64 yz pairs (M = 128) and columns = (Xr, Xs)
// of a range of a (N <= 64), reduced over the particles j (K).
//
// FP64 accuracy on the int8 tensor cores (Ozaki-style splitting): every
// operand value v in [-1, 1] becomes the 48-bit integer V = rint(v * SC),
// SC = 0x7F7F7F7F7F7F, written as six signed base-256 digits
// V = sum_s d_s 256^s, d_s in [-128, 127].  One DFMA produces all six:
// fma(v, SC, 1.5*2^52 + 0x808080808080) leaves V + 0x808080808080 in the low
// 48 mantissa bits, whose bytes XOR 0x80 are exactly the d_s.  The product
// sum_j Vg Vx = sum_{s,t} 256^{s+t} sum_j d_s d_t is accumulated per level
// w = s + t in int32 TMEM accumulators (exact: |sum| <= 6 * 16384 * 2^14 <
// 2^31), keeping the 26 slice pairs with w >= 4 (dropped terms < 2^-52 of
// full scale; with w >= 5 only, two opposite charges at one point would
// leave ~1e-14 instead of the exact cancellation the reference's tests
// demand, test_ewald.py:176-182); the epilogue combines the seven levels in
// fp64.  Measured against the fp64 restatement: |dS| / max|S| ~ 1e-15.
//
// Data flow per CTA (M tile of 64 yz pairs, a-chunk, particle split):
//   K-block of 64 particles -> the 8 warps write the six G slices (digits of
//   q e^{...}, generated from per-particle phase tables with a recurrence
//   along m_y) into shared memory in the no-swizzle K-major core-matrix
//   layout, cp.async brings the six pre-split X slices (k1t_prep) -> one
//   thread issues 26 x 2 MMAs (M=128, N=Npad, K=32) -> tcgen05.commit to the
//   stage's mbarrier.  Two stages: the MMAs of block k overlap the
//   production of block k+1.

// per-particle m_y / m_z phase tables written by k1t_prep and read by the
// producers (a sincospi per particle and run in the producers measured
// slower: c5 S(k) 70 vs 48.5 ms, the producers are on the critical path)
constexpr bool K1_TABLES = true;
constexpr int TC_S = 6;                     // byte slices per operand
constexpr int TC_W0 = 4;                    // kept levels: w = s + t >= TC_W0
constexpr int TC_NL = 2 * TC_S - 1 - TC_W0; // 7 levels
constexpr int TC_KB = 64;                   // particles per K-block
constexpr int TC_SBO = 528;                 // bytes between 8-row groups (512 + 16 pad)
constexpr int TC_GSL = 16 * TC_SBO;         // one G slice: 128 rows x 64 B
constexpr int TC_NMAX = 64;                 // X columns per a-chunk (7 x 64 <= 512 TMEM cols)
constexpr int TC_THREADS = 256;
constexpr int TC_MAXP = 16384;              // particles per CTA (int32 exactness)
constexpr double TC_SC = 140185576636287.0;              // 0x7F7F7F7F7F7F
constexpr double TC_MAGIC = 6755399441055744.0 + 141289400074368.0;  // 1.5*2^52 + 0x8080..80

// one X slice (fixed stride for every chunk: compile-time MMA descriptors)
__host__ __device__ constexpr int tc_xsl_bytes(int xnp) { return (xnp / 8) * TC_SBO; }
__host__ __device__ constexpr int tc_stage_bytes(int npad) {
  return TC_S * TC_GSL + TC_S * tc_xsl_bytes(npad);
}

// byte offset of (row, particle-in-block) in a K-major no-swizzle tile
__device__ __forceinline__ int tc_off(int row, int k) {
  return (row >> 3) * TC_SBO + (k >> 4) * 128 + (row & 7) * 16 + (k & 15);
}

// value in [-1,1] -> 64-bit pattern whose low 48 bits are V + 0x808080808080
__device__ __forceinline__ uint2 tc_bits(double v) {
  const double x = fma(v, TC_SC, TC_MAGIC);
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return make_uint2((uint32_t)b, (uint32_t)(b >> 32));
}

// four values (consecutive particles) -> six words, word s = digit s of each
__device__ __forceinline__ void tc_digits4(const uint2 v0, const uint2 v1, const uint2 v2,
                                           const uint2 v3, uint32_t (&w)[TC_S]) {
  const uint32_t t0 = __byte_perm(v0.x, v1.x, 0x5140), t1 = __byte_perm(v0.x, v1.x, 0x7362);
  const uint32_t t2 = __byte_perm(v2.x, v3.x, 0x5140), t3 = __byte_perm(v2.x, v3.x, 0x7362);
  const uint32_t u0 = __byte_perm(v0.y, v1.y, 0x5140), u1 = __byte_perm(v2.y, v3.y, 0x5140);
  w[0] = __byte_perm(t0, t2, 0x5410) ^ 0x80808080u;
  w[1] = __byte_perm(t0, t2, 0x7632) ^ 0x80808080u;
  w[2] = __byte_perm(t1, t3, 0x5410) ^ 0x80808080u;
  w[3] = __byte_perm(t1, t3, 0x7632) ^ 0x80808080u;
  w[4] = __byte_perm(u0, u1, 0x5410) ^ 0x80808080u;
  w[5] = __byte_perm(u0, u1, 0x7632) ^ 0x80808080u;
}

// ---- tcgen05 / mbarrier primitives (PTX) ----
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "TC_WAIT%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra TC_WAIT%=;\n}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// K-major, no swizzle: LBO = 128 B (next core matrix along K), SBO = TC_SBO
__device__ __forceinline__ uint64_t tc_desc(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(TC_SBO >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void tc_mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accum));
}
// smem -> TMEM copy of one 128 x 32-byte operand tile (same descriptor as
// the MMA's A operand); executes in issue order with tcgen05.mma
__device__ __forceinline__ void tc_cp_a(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void tc_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
      : "memory");
}
__device__ __forceinline__ void tc_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// SS-form merged MMAs read G from shared memory directly.  Staging G in TMEM
// (tcgen05.cp) for TS-form MMAs measured slower once MMAs are merged along N
// (each G slice then feeds only 1-3 MMAs and the copies occupy the tensor
// pipe in order with them): c5 39.9 (TS) vs 37.8 ms (SS, merge 3).
#ifndef K1_MERGE
#define K1_MERGE 3  // c5 37.8 ms; 2: 39.1, 4: 38.2
#endif
// K1_MERGE = m > 1: one MMA covers up to m consecutive X slices
// against G slice s, N = (m - 1) x 64 + npad (X slices sit 64 rows apart in
// shared memory; levels 64 columns apart in TMEM, the columns npad..63 of a
// level collect junk and are never read); accumulators zeroed first
static_assert(K1_MERGE > 1 && (K1_MERGE - 1) * TC_NMAX + TC_NMAX <= 256, "merged N <= 256");
// one lane of a converged warp (PTX elect.sync)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n}\n"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void tc_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   mbar)
               : "memory");
}
__device__ __forceinline__ void tc_ld8(uint32_t taddr, int (&r)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
}
__device__ __forceinline__ void tc_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

struct TCChunk {
  int a0, a1, nr, npad;  // a range, number of Xr columns (= a1-a0+1), padded N
};

// k1t_prep: per-particle tables for the tensor-core structure factor.
//   ytab[(my - ymin) * np + j]  = e^{-i 2pi my f_y}
//   ztab[(mz - zmin) * np + j]  = (q_j / qmax) e^{-i 2pi mz f_z}
//   xsl: per (chunk, K-block) the six X slices in the shared-memory image
// grid (particles / 128, tasks): task < nyt: 8 m_y values per particle,
// then 8 m_z values, then one a-chunk of X slices per particle quad.  Each
// run of 8 starts with a sincospi and continues by recurrence.
__global__ void __launch_bounds__(128)
    k1t_prep(const double4 *__restrict__ frac, int64_t p_begin, int64_t p_end, int64_t np,
             const double *__restrict__ qmax_p, int ymin, int ny, int zmin, int nz,
             const TCChunk *__restrict__ chunks, int n_chunks, int npad_max,
             double2 *__restrict__ ytab, double2 *__restrict__ ztab, uint8_t *__restrict__ xsl) {
  const int task = blockIdx.y;
  const int nyt = K1_TABLES ? (ny + 7) / 8 : 0, nzt = K1_TABLES ? (nz + 7) / 8 : 0;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (task < nyt + nzt) {
    const int64_t j = t;
    if (j >= np) return;
    const bool ok = p_begin + j < p_end;
    const double4 f = ok ? frac[p_begin + j] : make_double4(0.0, 0.0, 0.0, 0.0);
    const bool is_y = task < nyt;
    const int t0 = 8 * (is_y ? task : task - nyt);
    const int m0 = (is_y ? ymin : zmin) + t0, cnt = min(8, (is_y ? ny : nz) - t0);
    const double fr = is_y ? f.y : f.z;
    const double sc = is_y ? 1.0 : (ok ? f.w / fmax(*qmax_p, 1e-300) : 0.0);
    double s, c;
    sincospi(2.0 * fr, &s, &c);
    const double2 e1 = make_double2(c, -s);
    sincospi(2.0 * ((double)m0 * fr), &s, &c);
    double2 cur = make_double2(c, -s);
    double2 *dst = (is_y ? ytab : ztab) + (int64_t)t0 * np + j;
    for (int u = 0; u < cnt; ++u) {
      dst[(int64_t)u * np] = make_double2(sc * cur.x, sc * cur.y);
      cur = cmul(cur, e1);
    }
    return;
  }
  // X slices: column c of chunk ch: Xr(a0 + c) for c < nr, Xs(max(a0,1) + c - nr),
  // zero above; one task per (chunk, 8 consecutive columns)
  const int xt = task - nyt - nzt;
  const int segs = (npad_max + 7) / 8;
  const int ch = xt / segs, c0 = 8 * (xt % segs);
  const int64_t j0 = 4 * t;
  if (j0 >= np || ch >= n_chunks) return;
  const TCChunk C = chunks[ch];
  if (c0 >= C.npad) return;
  double fx[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t j = p_begin + j0 + u;
    fx[u] = j < p_end ? frac[j].x : 0.0;
  }
  const int64_t kb = j0 / TC_KB;
  const int kin = (int)(j0 % TC_KB);
  const int64_t n_kb = np / TC_KB;
  const int xsl_b = tc_xsl_bytes(npad_max);
  uint8_t *base = xsl + ((int64_t)ch * n_kb + kb) * (int64_t)(TC_S * xsl_b);
  const int sa0 = max(C.a0, 1), ns = max(0, C.a1 - sa0 + 1);
  double2 cr[4], e1[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    double s, c;
    sincospi(2.0 * fx[u], &s, &c);
    e1[u] = make_double2(c, s);  // e^{+i 2pi f_x}: (cos, sin) of a f_x
  }
  int prev_pass = -1;
  for (int col = c0; col < min(c0 + 8, C.npad); ++col) {
    const int pass = col < C.nr ? 0 : (col < C.nr + ns ? 1 : 2);
    uint32_t w[TC_S];
    if (pass == 2) {
#pragma unroll
      for (int s = 0; s < TC_S; ++s) w[s] = 0u;
    } else {
      const int a = pass == 0 ? C.a0 + col : sa0 + (col - C.nr);
      uint2 b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (pass != prev_pass) {
          double s, c;
          sincospi(2.0 * ((double)a * fx[u]), &s, &c);
          cr[u] = make_double2(c, s);
        } else {
          cr[u] = cmul(cr[u], e1[u]);
        }
        const bool ok = p_begin + j0 + u < p_end;
        b[u] = tc_bits(ok ? (pass == 0 ? cr[u].x : cr[u].y) : 0.0);
      }
      tc_digits4(b[0], b[1], b[2], b[3], w);
    }
    prev_pass = pass;
    const int off = tc_off(col, kin);
#pragma unroll
    for (int s = 0; s < TC_S; ++s) *reinterpret_cast<uint32_t *>(base + s * xsl_b + off) = w[s];
  }
}

// k1t_gemm: grid (M tiles, a-chunks, particle splits); warp-specialised:
//   warps 0-7 (256 threads): produce the G slices of a K-block (2 stages),
//   warp 8 lane 0: issues the MMAs, warp 9 lane 0: bulk-copies the X slices
//   (TC_XS-deep ring).  Stages hand over through mbarriers: G full (8
//   producer-warp arrivals) / empty (tcgen05.commit), X full (complete_tx) /
//   empty (tcgen05.commit).
//   runs[tile*8 + g] = (m_z, m_y0, len, 0): rows 8g..8g+len-1 of the tile are
//   the pairs (m_y0 + i, m_z); Re G in rows 0..63, Im G in rows 64..127.
//   tmap[(tile*64 + p) * (A+1) + a] = pair slots (x, y; -1 = none) of
//   (a, m_y, m_z) in the K1 pair layout (k2p_finalize input).
#ifndef TC_GSTAGES
#define TC_GSTAGES 2
#endif
#ifndef TC_XSTAGES
#define TC_XSTAGES 4
#endif
constexpr int TC_GS = TC_GSTAGES;             // G ring depth (produced)
constexpr int TC_XS = TC_XSTAGES;             // X ring depth (bulk copies)
#ifndef K1_PGROUPS
#define K1_PGROUPS 2
#endif
// producer groups: group g fills the K-blocks it with it % TC_PG == g
constexpr int TC_PG = K1_PGROUPS;
constexpr int TC_PWARPS = TC_PG * TC_THREADS / 32;     // producer warps
constexpr int TC_NTHREADS = TC_PG * TC_THREADS + 64;  // + MMA warp + loader warp
static_assert(TC_GS % TC_PG == 0, "each G stage must belong to one producer group");
__host__ __device__ constexpr int tc_smem_bytes(int npad_max) {
  return TC_GS * TC_S * TC_GSL + TC_XS * TC_S * tc_xsl_bytes(npad_max);
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes,
                                         uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(mbar)
      : "memory");
}

// XNP: rows between consecutive X slices in shared memory and columns
// between TMEM levels = the largest padded a-chunk width of the k-table
// (16..64), so merged MMAs carry no padding columns beyond the last chunk's
template <int XNP>
__global__ void __launch_bounds__(TC_NTHREADS, 1)
    k1t_gemm(const double4 *__restrict__ frac, const double2 *__restrict__ ytab,
             const double2 *__restrict__ ztab,
             const double2 *__restrict__ base, const uint8_t *__restrict__ xsl,
             const TCChunk *__restrict__ chunks, const int4 *__restrict__ runs,
             const int2 *__restrict__ tmap, const double *__restrict__ qmax_p, int64_t p_begin,
             int64_t p_end, int64_t np, int64_t ppb, int ymin, int zmin, int A, int npad_max,
             int64_t n_pslots, double4 *__restrict__ spart, int dbg) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t g_full[TC_GS], g_empty[TC_GS], x_full[TC_XS], x_empty[TC_XS], acc_full;
  __shared__ uint32_t tmem_base_s;
  __shared__ int4 s_runs[8];
  const int tile = blockIdx.x, ch = blockIdx.y, split = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TCChunk C = chunks[ch];
  const int npad = C.npad;
  const int xsl_b = tc_xsl_bytes(XNP);  // X slice stride (XNP rows)
  const int xblk = TC_S * xsl_b;  // bytes of one K-block's X slices
  uint8_t *gbuf = smem;
  uint8_t *xbuf = smem + TC_GS * TC_S * TC_GSL;
  const int64_t n_kb_all = np / TC_KB;
  const int64_t kb0 = (int64_t)split * (ppb / TC_KB);
  const int64_t kb1 = min(n_kb_all, kb0 + ppb / TC_KB);
  const int nkb = (int)max((int64_t)0, kb1 - kb0);

  if (threadIdx.x < 8) s_runs[threadIdx.x] = runs[tile * 8 + threadIdx.x];
  if (threadIdx.x == 0) {
    for (int i = 0; i < TC_GS; ++i) {
      mbar_init(smem_u32(&g_full[i]), TC_THREADS / 32);
      mbar_init(smem_u32(&g_empty[i]), 1);
    }
    for (int i = 0; i < TC_XS; ++i) {
      mbar_init(smem_u32(&x_full[i]), 1);
      mbar_init(smem_u32(&x_empty[i]), 1);
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
  const int lstride = K1_MERGE > 1 ? XNP : npad;  // TMEM columns between levels
  if (K1_MERGE > 1) {  // zero the level accumulators (every merged MMA accumulates)
    if (warp < 4) {
      const uint32_t z[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
      for (int c = 0; c < TC_NL * XNP; c += 8)
        tc_st8(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c, z);
      tc_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }

  if (warp == TC_PWARPS + 1) {
    // ---- X loader ----
    if (lane == 0) {
      for (int it = 0; it < nkb; ++it) {
        const int xs = it % TC_XS;
        if (it >= TC_XS) mbar_wait(smem_u32(&x_empty[xs]), ((it / TC_XS) - 1) & 1);
        const uint8_t *src = xsl + ((int64_t)ch * n_kb_all + kb0 + it) * (int64_t)xblk;
        const uint32_t fb = smem_u32(&x_full[xs]);
        mbar_expect_tx(fb, (uint32_t)xblk);
        bulk_g2s(smem_u32(xbuf + xs * xblk), src, (uint32_t)xblk, fb);
      }
    }
  } else if (warp == TC_PWARPS) {
    // ---- MMA issuer: the whole warp waits, one elected lane issues ----
    {
      const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) |
                             ((uint32_t)(npad >> 3) << 17) | (8u << 24);
      for (int it = 0; it < nkb; ++it) {
        const int gs = it % TC_GS, xs = it % TC_XS;
        mbar_wait(smem_u32(&g_full[gs]), (it / TC_GS) & 1);
        mbar_wait(smem_u32(&x_full[xs]), (it / TC_XS) & 1);
        tc_fence_after();
        __syncwarp();
        if (!(dbg & 2) && elect_one()) {
          const uint64_t gd = tc_desc(smem_u32(gbuf + gs * TC_S * TC_GSL));
          const uint64_t xd = tc_desc(smem_u32(xbuf + xs * xblk));
          constexpr int XSL = tc_xsl_bytes(XNP);
          // SS form with merged N: each G slice read from shared memory by
          // its merged MMAs, no staging copy into TMEM
          const uint32_t idesc0 = idesc & ~(63u << 17);
#pragma unroll
          for (int ks = 0; ks < TC_KB / 32; ++ks) {
#pragma unroll
            for (int s = 0; s < TC_S; ++s) {
#pragma unroll
              for (int t = (TC_W0 - s > 0 ? TC_W0 - s : 0); t < TC_S; t += K1_MERGE) {
                const int m = TC_S - t < K1_MERGE ? TC_S - t : K1_MERGE;
                tc_mma(tmem + (uint32_t)((s + t - TC_W0) * XNP),
                       gd + (uint64_t)((s * TC_GSL + ks * 256) >> 4),
                       xd + (uint64_t)((t * XSL + ks * 256) >> 4),
                       idesc0 | ((uint32_t)(((m - 1) * XNP + npad) >> 3) << 17), 1u);
              }
            }
          }
          tc_commit(smem_u32(&g_empty[gs]));
          tc_commit(smem_u32(&x_empty[xs]));
        } else if ((dbg & 2) && lane == 0) {
          mbar_arrive(smem_u32(&g_empty[gs]));
          mbar_arrive(smem_u32(&x_empty[xs]));
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
    // ---- G producers: core column pc (16 particles), row half ph, run g, quad qd ----
    const int pc = warp & 3, ph = (warp >> 2) & 1, g = lane >> 2, qd = lane & 3;
    const int4 run = s_runs[g];
    const int kin = pc * 16 + qd * 4;  // particle offset in the K-block
    const int myl = run.y + 4 * ph;
    const bool active = 4 * ph < run.z;  // rows of this half exist in the run
    const double inv_qmax = 1.0 / fmax(*qmax_p, 1e-300);
    for (int it = warp >> 3; it < nkb; it += TC_PG) {
      const int gs = it % TC_GS;
      uint8_t *sb = gbuf + gs * TC_S * TC_GSL;
      if (it >= TC_GS) mbar_wait(smem_u32(&g_empty[gs]), ((it / TC_GS) - 1) & 1);
      if (!(dbg & 1)) {
        const int64_t j = (kb0 + it) * TC_KB + kin;  // relative to p_begin
        double2 cur[4], e1[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (active) {
            const double2 yv = ytab[(int64_t)(myl - ymin) * np + j + u];
            const double2 zv = ztab[(int64_t)(run.x - zmin) * np + j + u];
            cur[u] = cmul(yv, zv);
            e1[u] = base[3 * min(p_begin + j + u, p_end - 1) + 1];
          } else {
            cur[u] = e1[u] = make_double2(0.0, 0.0);
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = 4 * ph + i;
          const bool valid = r < run.z;
          uint2 br[4], bi[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            br[u] = tc_bits(valid ? cur[u].x : 0.0);
            bi[u] = tc_bits(valid ? cur[u].y : 0.0);
            if (i < 3) cur[u] = cmul(cur[u], e1[u]);
          }
          uint32_t w[TC_S];
          const int row = 8 * g + r;
          tc_digits4(br[0], br[1], br[2], br[3], w);
          const int off = tc_off(row, kin);
#pragma unroll
          for (int s = 0; s < TC_S; ++s) *reinterpret_cast<uint32_t *>(sb + s * TC_GSL + off) = w[s];
          tc_digits4(bi[0], bi[1], bi[2], bi[3], w);
          const int offi = tc_off(row + 64, kin);
#pragma unroll
          for (int s = 0; s < TC_S; ++s)
            *reinterpret_cast<uint32_t *>(sb + s * TC_GSL + offi) = w[s];
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&g_full[gs]));
    }
  }

  // ---- epilogue: combine the levels, exchange Re/Im rows through smem ----
  double *E = reinterpret_cast<double *>(smem);
  const int ES = npad + 1;
  mbar_wait(smem_u32(&acc_full), 0);
  tc_fence_after();
  __syncthreads();  // every producer/loader is done with the stage buffers
  if (warp < 8 && nkb > 0) {
    const double scale = 2.0 * (*qmax_p) / (TC_SC * TC_SC);  // x2: pair layout A = 2 P
    const int row = 32 * (warp & 3) + lane;
    const int half = npad / 2;
    const int c_lo = (warp >> 2) * half;
    for (int c0 = c_lo; c0 < c_lo + half; c0 += 8) {
      double acc[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = 0.0;
#pragma unroll
      for (int l = TC_NL - 1; l >= 0; --l) {
        int r[8];
        tc_ld8(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(l * lstride + c0), r);
        tc_wait_ld();
        const double wl = ldexp(1.0, 8 * (TC_W0 + l));
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] = fma((double)r[k], wl, acc[k]);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) E[row * ES + c0 + k] = acc[k] * scale;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
  // write the pair-layout partials (2P1, 2P3, 2P4, 2P2) of every mapped slot
  const int na = C.a1 - C.a0 + 1;
  const int sa0 = max(C.a0, 1);
  for (int item = threadIdx.x; item < 64 * na; item += TC_NTHREADS) {
    const int p = item / na, a = C.a0 + item % na;
    const int2 sl = tmap[((int64_t)tile * 64 + p) * (A + 1) + a];
    if (sl.x < 0 && sl.y < 0) continue;
    double4 v = make_double4(0.0, 0.0, 0.0, 0.0);
    if (nkb > 0) {
      const int cr = a - C.a0;
      v.x = E[p * ES + cr];
      v.y = E[(p + 64) * ES + cr];
      if (a >= sa0) {
        const int cs = C.nr + (a - sa0);
        v.z = E[p * ES + cs];
        v.w = E[(p + 64) * ES + cs];
      }
    }
    double4 *out = spart + (int64_t)split * n_pslots;
    if (sl.x >= 0) out[sl.x] = v;
    if (sl.y >= 0) out[sl.y] = v;
  }
}

// max |q| over a particle range (bit pattern of a non-negative double orders
// like the integer)
__global__ void __launch_bounds__(256)
    k_absmax_q(const double4 *__restrict__ frac, int64_t i0, int64_t i1,
               unsigned long long *__restrict__ out) {
  double m = 0.0;
  for (int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < i1;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(frac[i].w));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}
