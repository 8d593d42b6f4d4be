// ewald_b200.cu -- B200-native (sm_100a) classical Ewald energy + forces.
//
// Hot path of arXiv 1708.01135 as restated by the reference package ewaldmd
// (/root/reference/pkg/src/ewaldmd).  See include/ewald_b200.h for the C-ABI
// and DESIGN.md for the data layout and rooflines.  This file holds the
// per-particle set-up kernels, the k-space planner, the evaluation pipeline
// (two streams, CUDA graphs) and the C-ABI; the kernels live in:
//
//   k1_tc.cuh       Alg. 1 (ewald.py:281-305) S(k) as an int8 tensor-core GEMM
//                   (tcgen05.mma kind::i8, six 48-bit slices, TMEM levels)
//   k3_tc.cuh       Alg. 2 (ewald.py:308-349) reciprocal forces as an int8 GEMM
//                   (W = C S rows x YZ phases, X(a) contraction in the epilogue)
//   recip_fp64.cuh  Alg. 1/2 on the FP64 pipe (small systems, tensor cores off,
//                   per-particle energies of the foreign-rho API)
//   rs_cells.cuh    cell list (celllist.py:75-108), deterministic in-cell order
//   rs_pairs.cuh    real-space pair kernel (ewald.py:208-221, engine.py:102-159):
//                   FP32 box/centre prefilter, exact FP64 predicate, erfc via
//                   exp x erfcx table, half shell with cell-sorted atomics;
//                   image-shell kernel for r_c > L/2 (ewald.py:490-576)
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <tuple>
#include <type_traits>
#include <cmath>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "ewald_b200.h"

#define EWB_VERSION 100

namespace {

constexpr int ERR_UNWRAPPED = 1;
constexpr int ERR_COINCIDENT = 2;
constexpr int64_t WIDE_MAX_N = 4096;  // _WIDE_CUTOFF_MAX_N (ewald.py:490)

constexpr int MAXM = 32;          // longest k-column segment (template range)
constexpr int MAXM1 = 20;         // longest K1 pair segment (two accumulator sets)
constexpr int K1_THREADS = 128;   // k-items per structure-factor block
constexpr int K1_PMAX = 32;       // particles per shared-memory phase chunk
#ifndef K1_ILP
#define K1_ILP 2                  // particles (independent chains) per K1 step
#endif
#ifndef K1_TAB_BYTES
#define K1_TAB_BYTES (24 * 1024)  // one of the two phase-table buffers
#endif
#ifndef K1_PPB
#define K1_PPB 256                // target particles per structure-factor block
#endif
constexpr size_t K1_PART_BYTES = (size_t)512 << 20;  // cap of the partial S(k) buffers
#ifndef K3_WAVES
#define K3_WAVES 4
#endif
#ifndef K3C_MIN_WAVES
#define K3C_MIN_WAVES 2           // constant-bank K3 when >= this many blocks per SM
#endif
constexpr int K3_THREADS = 128;
constexpr int K3_PPT = 2;         // particles per thread in the gather
constexpr int K3_CH = 32;         // k-items per shared-memory chunk
#ifndef K6_WARPS
#define K6_WARPS 4
#endif
#ifndef K6_RSPLIT
#define K6_RSPLIT 1               // warps per real-space unit (stencil rows split between them)
#endif
#ifndef K6_G
#define K6_G 8                    // centre particles per real-space warp
#endif
#ifndef K6_SLAB_BLOCKS
#define K6_SLAB_BLOCKS 2          // few-unit real space: split rows until this many blocks per SM
#endif
#ifndef K6_RAD_MAX
#define K6_RAD_MAX 3              // largest stencil radius in cells (3: r_c/3 cells)
#endif
#ifndef K6_RAD3_F
#define K6_RAD3_F 3.0             // radius-3 cells: edge L / floor(F L / r_c) >= r_c / 3
#endif
#ifndef K6_RAD3_MINOCC
#define K6_RAD3_MINOCC 16.0       // ... used when cells hold at least this many particles
#endif
#ifndef K6_HI_WAVES
#define K6_HI_WAVES 3             // fused pair kernel at 5 blocks/SM from this many waves up
#endif
#ifndef K6_SPLIT
#define K6_SPLIT 0                // real space as traversal + evaluation passes (measured slower)
#endif
constexpr int SORT_CAP = 4096;    // in-cell deterministic sort capacity
constexpr int RED_THREADS = 256;

// tab_desc flags
constexpr int TF_QSCALE = 1;
constexpr int TF_LINK = 2;
constexpr int TF_SCALE2 = 16;  // x2 (the 2 cos / 2 sin of a pair item)

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

__device__ __forceinline__ double4 ldcs4(const double4 *p) {
  const double2 *q = reinterpret_cast<const double2 *>(p);
  const double2 a = __ldcs(q), b = __ldcs(q + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block reduction; result valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double *sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NT / 32; ++i) r += sh[i];
  }
  return r;
}

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

// ---------------------------------------------------------------------------
// template dispatch tables
#define EWB_M_CASES(X)                                                                           \
  X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) X(17) \
      X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26) X(27) X(28) X(29) X(30) X(31) X(32)

typedef void (*k1_fn)(const double4 *, const double2 *, int64_t, int64_t, int64_t, int,
                      const int4 *, int, const int4 *, const int *, const int *, double4 *);
typedef void (*k3_fn)(const double4 *, const double2 *, int64_t, int64_t, const int4 *,
                      const int *, const int *, const int *, const double2 *, int, double *,
                      double *);

#define EWB_M1_CASES(X)                                                                          \
  X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) X(17) \
      X(18) X(19) X(20)
k1_fn k1_table(int M) {
  switch (M) {
#define X(m) \
  case m:    \
    return k1_structure_factor<m>;
    EWB_M1_CASES(X)
#undef X
  }
  return nullptr;
}

typedef void (*k3c_fn)(const double4 *, const double2 *, int64_t, int64_t, int, int, double *,
                       double *);
k3c_fn k3c_table(int M, bool energy, int buf) {
  switch (M) {
#define X(m)                                                                        \
  case m:                                                                           \
    return buf ? (energy ? k3c_force_gather<m, true, 1> : k3c_force_gather<m, false, 1>) \
               : (energy ? k3c_force_gather<m, true, 0> : k3c_force_gather<m, false, 0>);
    EWB_M_CASES(X)
#undef X
  }
  return nullptr;
}

k3_fn k3_table(int M, bool energy) {
  switch (M) {
#define X(m) \
  case m:    \
    return energy ? k3_force_gather<m, true> : k3_force_gather<m, false>;
    EWB_M_CASES(X)
#undef X
  }
  return nullptr;
}

// ---------------------------------------------------------------------------
// host side
// bumped on every device reallocation: captured graphs bake in pointers
uint64_t g_realloc_epoch = 0;

struct DBuf {
  void *p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap && p) return cudaSuccess;
    if (p) {
      // growth is rare; make sure no queued kernel still uses the old buffer
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) return e;
      cudaFree(p);
    }
    p = nullptr;
    cap = 0;
    if (bytes == 0) bytes = 16;
    ++g_realloc_epoch;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) cap = bytes;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <class T>
  T *as() const {
    return reinterpret_cast<T *>(p);
  }
};

struct Plan {
  int64_t K = 0;
  // K3 (force gather) layout: items = z-segments of <= M k-vectors
  int M = 0, n_items = 0, n_rows = 0;
  std::vector<int> row_item_prefix;  // n_rows+1
  DBuf item_my, item_row, rows, slot_k, slot_coeff, k3meta;
  // K1 (structure factor) layout: pair items = the +m_x and -m_x segments of
  // one (|m_x|, m_y, m_z-run) sharing one z recurrence
  int M1 = 0, n_pitems = 0, n_tiles = 0, ts_max = 0, pchunk = K1_PMAX;
  DBuf pitem_tab, tab_desc, tile_off, tile_ts, pslot_map;  // pslot_map: int4 (kp, km, k3p, k3m)
  // tensor-core structure factor (k1_tc.cuh): M tiles of 8 (m_z, m_y-run)
  // runs, a-chunks of <= TC_NMAX X columns, (tile, pair, a) -> pair slots
  bool tc_ok = false;
  int tc_A = 0, tc_mtiles = 0, tc_nchunks = 0, tc_npad_max = 0;
  int tc_ymin = 0, tc_ny = 0, tc_zmin = 0, tc_nz = 0;
  DBuf tc_runs, tc_map, tc_chunks;
  std::vector<TCChunk> tc_chunks_host;
  // tensor-core force gather (k3_tc.cuh): A rows (a, type), K pairs, slot map
  bool t3_ok = false;
  int t3_rows = 0, t3_mtiles = 0, t3_npairs = 0, t3_nkb = 0;
  DBuf t3_rowtab, t3_pair_yz, t3_slotmap, t3_comp;
  std::vector<std::pair<int, DBuf>> ks_cache;  // n_ks -> row boundaries
  void release() {
    for (DBuf *b : {&item_my, &item_row, &rows, &slot_k, &slot_coeff, &k3meta, &pitem_tab, &tab_desc,
                    &tile_off, &tile_ts, &pslot_map, &tc_runs, &tc_map, &tc_chunks, &t3_rowtab,
                    &t3_pair_yz, &t3_slotmap, &t3_comp})
      b->release();
    for (auto &c : ks_cache) c.second.release();
    ks_cache.clear();
  }
};

}  // namespace

constexpr int N_SEG = 6;  // pipeline: load | cells | pairs | S(k) | forces | combine + self

struct ewb_handle {
  int device = 0;
  int n_sm = 148;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t aux_stream = nullptr;  // second stream of the constant-bank gather
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // reciprocal space concurrently with real space (tensor-core path)
  cudaStream_t rstream = nullptr;
  cudaEvent_t ev_rfork = nullptr, ev_rjoin = nullptr;
  int overlap = 1;
  bool ov_active = false;       // this evaluation runs the two streams
  int t3_pend_nks = 0;          // deferred k3_combine (overlap mode)
  int64_t t3_pend_i0 = 0, t3_pend_n = 0;
  double *t3_pend_force = nullptr;
  // host-API copies overlapped with the pipeline (ewb_evaluate): the force
  // upload is waited for before the pair segment, rho is copied out as soon
  // as S(k) is final
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_fup = nullptr, ev_rho = nullptr, ev_rhodone = nullptr;
  bool fup_pending = false;
  double *rho_host = nullptr;
  cudaEvent_t ev[6] = {};
  std::string err;
  int mcap = 28;   // K3 segment cap
  int mcap1 = 20;  // K1 pair segment cap
  int stencil_rad = 0;  // 0 auto, 1 force r_c cells (testing)
  int deterministic = 0;  // 1: full-shell real space, no atomics (bitwise reproducible)
  int k3_const = 1;       // constant-bank force gather for large systems
  int use_tc = 2;         // int8 tensor-core reciprocal space: 0 off, 1 forced, 2 auto (N*K)
  int tc_dbg = 0;  // compile-time -DEWB_TC_DBG=1|2 only: skip G production | the MMAs
  DBuf tc_qmax, tc_ytab, tc_ztab, tc_xsl;
  DBuf t3_wsl, t3_rscale;
  DBuf pairc;  // in-cutoff pairs visited by the last real-space pass
  int64_t geom_n = 0;           // particle count deciding the cell grid (0: the loaded one)
  int row_lo = -1, row_hi = -1;  // explicit centre rows of the next real-space pass
  int rs_split = K6_SPLIT;        // two-pass real space (pair lists in HBM), off by default
  DBuf rs_list, rs_count;         // per-unit pair lists and their lengths
  DBuf eblk_r;  // energy scratch of the reciprocal stages (own stream)
  DBuf fsorted;  // real-space forces in cell-sorted order
  void *tc_spart_zeroed = nullptr;  // spart buffer whose unmapped slots were zeroed
  int64_t launches = 0;
  // system
  bool have_system = false;
  double L = 0, alpha = 0, rc = 0, rc2 = 0;
  // force-field switches (ForceAssembler, driver.py:81-126): Coulomb (Ewald)
  // and the shifted 12-6 LJ fused into the real-space pair traversal
  bool coul_on = true, lj_on = false;
  double rc_lj = 0, rc2_lj = 0, lj_s2 = 0, lj_4e = 0, lj_shift = 0, lj_24e = 0;
  // k-space
  bool have_kspace = false;
  Plan plan;
  // particles
  int64_t n = 0;
  bool loaded = false;
  DBuf pos, q, force, rho;                   // host-API staging (caller layout)
  DBuf force_in;  // the caller's forces as uploaded (restored on a device-side error)
  double *hscr = nullptr;  // pinned host scratch: energies [0..2], error flag [3]
  DBuf frac, base, xyzq;                     // derived
  DBuf spart, sslot, sp, fpart, upart, eblk, eblk2, eblk_lj, energy, errflag;
  DBuf cell_of, slot, count, start, gstart, order_tmp, order, sorted, sorted_cell, row_ustart;
  DBuf sorted_f;  // FP32 copy of the sorted positions (candidate prefilter)
  // CUDA graph of the device pipeline (prep + real space + S(k) + forces +
  // self energy), captured on the second call with an unchanged key
  struct GKey {
    const void *pos = nullptr, *q = nullptr;
    void *force = nullptr, *rho = nullptr;
    int64_t n = -1;
    bool timed = false;
    uint64_t gen = 0, epoch = 0;
    bool operator==(const GKey &o) const {
      return pos == o.pos && q == o.q && force == o.force && rho == o.rho && n == o.n &&
             timed == o.timed && gen == o.gen && epoch == o.epoch;
    }
  };
  bool use_graphs = true;
  uint64_t gen = 0;  // bumped by every configuration change
  GKey gkey, warm_key;
  cudaGraphExec_t gexec[N_SEG] = {};
  int64_t glaunch[N_SEG] = {};
  int occ_k1[MAXM + 1] = {};
  int occ_k3[MAXM + 1][2] = {};
  bool k1_attr[MAXM + 1] = {};

  int fail(int code, const std::string &msg) {
    err = msg;
    return code;
  }
};

namespace {

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return h->fail(EWB_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));      \
  } while (0)

#define CKL()                                                                                 \
  do {                                                                                        \
    ++h->launches;                                                                            \
    cudaError_t e_ = cudaGetLastError();                                                      \
    if (e_ != cudaSuccess)                                                                    \
      return h->fail(EWB_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e_));    \
  } while (0)

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

template <class T>
int upload(ewb_handle *h, DBuf &b, const std::vector<T> &v) {
  CK(b.ensure(v.size() * sizeof(T)));
  if (!v.empty()) CK(cudaMemcpy(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return EWB_OK;
}

// Host planning of the k-space work decomposition.
int build_plan(ewb_handle *h, const int64_t *m, int64_t K, const double *coeff) {
  Plan &P = h->plan;
  CK(cudaStreamSynchronize(h->stream));  // queued kernels may read the old plan
  if (K <= 0) return h->fail(EWB_EKSPACE, "empty reciprocal-space table");
  for (int64_t i = 0; i < 3 * K; ++i)
    if (m[i] > 1000000 || m[i] < -1000000)
      return h->fail(EWB_EINVAL, "m_int entries must satisfy |m| <= 1e6");
  std::vector<int64_t> idx(K);
  std::iota(idx.begin(), idx.end(), 0);
  std::sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) {
    for (int c = 0; c < 3; ++c)
      if (m[3 * a + c] != m[3 * b + c]) return m[3 * a + c] < m[3 * b + c];
    return a < b;
  });
  struct Item {
    int mx, my, s, len;
    int64_t off;
  };
  std::vector<Item> items;
  const int mcap = std::max(1, std::min(MAXM, h->mcap));
  int64_t a = 0;
  while (a < K) {
    const int64_t i0 = idx[a];
    int64_t b = a + 1;
    while (b < K) {
      const int64_t ib = idx[b], ip = idx[b - 1];
      if (m[3 * ib] != m[3 * i0] || m[3 * ib + 1] != m[3 * i0 + 1] ||
          m[3 * ib + 2] != m[3 * ip + 2] + 1)
        break;
      ++b;
    }
    const int64_t len = b - a;
    const int64_t nseg = (len + mcap - 1) / mcap;
    const int64_t base_len = len / nseg, rem = len % nseg;
    int64_t off = a;
    for (int64_t sg = 0; sg < nseg; ++sg) {
      const int sl = (int)(base_len + (sg < rem ? 1 : 0));
      items.push_back(Item{(int)m[3 * i0], (int)m[3 * i0 + 1], (int)m[3 * idx[off] + 2], sl, off});
      off += sl;
    }
    a = b;
  }
  std::sort(items.begin(), items.end(), [](const Item &x, const Item &y) {
    if (x.s != y.s) return x.s < y.s;
    if (x.mx != y.mx) return x.mx < y.mx;
    return x.my < y.my;
  });
  const int n_items = (int)items.size();
  int M = 0;
  for (auto &it : items) M = std::max(M, it.len);

  // rows: maximal runs of equal (s, mx)
  std::vector<int> item_row(n_items), item_my(n_items);
  std::vector<int4> rows;
  for (int i = 0; i < n_items; ++i) {
    if (i == 0 || items[i].s != items[i - 1].s || items[i].mx != items[i - 1].mx)
      rows.push_back(make_int4(items[i].mx, items[i].s, i, 0));
    rows.back().w++;
    item_row[i] = (int)rows.size() - 1;
    item_my[i] = items[i].my;
  }
  const int n_rows = (int)rows.size();
  std::vector<int4> k3meta(n_items);
  for (int i = 0; i < n_items; ++i) {
    const bool new_row = i == 0 || item_row[i] != item_row[i - 1];
    const bool jump = !new_row && items[i].my != items[i - 1].my + 1;
    k3meta[i] = make_int4(items[i].mx, items[i].s, items[i].my, (new_row ? 1 : 0) | (jump ? 2 : 0));
  }
  P.row_item_prefix.assign(n_rows + 1, 0);
  for (int r = 0; r < n_rows; ++r) P.row_item_prefix[r + 1] = P.row_item_prefix[r] + rows[r].w;

  // gather slots (item-major layout: slot = item * M + m)
  const size_t n_slots = (size_t)M * n_items;
  std::vector<int> slot_k(n_slots, -1);
  std::vector<double> slot_coeff(n_slots, 0.0);
  for (int i = 0; i < n_items; ++i)
    for (int mm = 0; mm < items[i].len; ++mm) {
      const int64_t k = idx[items[i].off + mm];
      slot_k[(size_t)i * M + mm] = (int)k;  // item-major: a k-chunk is contiguous
      slot_coeff[(size_t)i * M + mm] = coeff ? coeff[k] : 0.0;
    }

  // ---- K1 pair plan (own segmentation, cap mcap1) ----
  struct Seg {
    int mx, my, s, len;
    int64_t off;
  };
  std::vector<Seg> segs;
  const int mcap1 = std::max(1, std::min(MAXM1, h->mcap1));
  {
    int64_t a1 = 0;
    while (a1 < K) {
      const int64_t i0 = idx[a1];
      int64_t b1 = a1 + 1;
      while (b1 < K) {
        const int64_t ib = idx[b1], ip = idx[b1 - 1];
        if (m[3 * ib] != m[3 * i0] || m[3 * ib + 1] != m[3 * i0 + 1] ||
            m[3 * ib + 2] != m[3 * ip + 2] + 1)
          break;
        ++b1;
      }
      const int64_t len = b1 - a1;
      // <= mcap1 per segment; long columns (>= 3 segments) use ~14: the
      // two accumulator sets of longer segments cost occupancy
      int64_t nseg = (len + mcap1 - 1) / mcap1;
      if (nseg >= 3 && mcap1 > 14) nseg = (len + 13) / 14;
      const int64_t base_len = len / nseg, rem = len % nseg;
      int64_t off = a1;
      for (int64_t sg = 0; sg < nseg; ++sg) {
        const int sl = (int)(base_len + (sg < rem ? 1 : 0));
        segs.push_back(Seg{(int)m[3 * i0], (int)m[3 * i0 + 1], (int)m[3 * idx[off] + 2], sl, off});
        off += sl;
      }
      a1 = b1;
    }
  }
  struct PItem {
    int ax, my, s, len;
    int64_t offp, offm;
  };
  std::vector<PItem> pitems;
  {
    std::map<std::tuple<int, int, int, int>, int> by_key;
    for (int i = 0; i < (int)segs.size(); ++i)
      by_key[std::make_tuple(segs[i].mx, segs[i].my, segs[i].s, segs[i].len)] = i;
    std::vector<char> used(segs.size(), 0);
    for (int i = 0; i < (int)segs.size(); ++i) {
      const Seg &g = segs[i];
      if (used[i] || g.mx <= 0) continue;
      auto it = by_key.find(std::make_tuple(-g.mx, g.my, g.s, g.len));
      if (it != by_key.end() && !used[it->second]) {
        used[i] = used[it->second] = 1;
        pitems.push_back(PItem{g.mx, g.my, g.s, g.len, g.off, segs[it->second].off});
      }
    }
    for (int i = 0; i < (int)segs.size(); ++i) {
      if (used[i]) continue;
      const Seg &g = segs[i];
      if (g.mx >= 0)
        pitems.push_back(PItem{g.mx, g.my, g.s, g.len, g.off, -1});
      else
        pitems.push_back(PItem{-g.mx, g.my, g.s, g.len, -1, g.off});
    }
  }
  std::sort(pitems.begin(), pitems.end(), [](const PItem &x, const PItem &y) {
    if (x.s != y.s) return x.s < y.s;
    if (x.ax != y.ax) return x.ax < y.ax;
    return x.my < y.my;
  });
  const int n_pitems = (int)pitems.size();
  int M1 = 0;
  for (auto &it : pitems) M1 = std::max(M1, it.len);
  // caller index -> K3 slot
  std::vector<int> k3slot(K, -1);
  for (size_t sl = 0; sl < n_slots; ++sl)
    if (slot_k[sl] >= 0) k3slot[slot_k[sl]] = (int)sl;
  std::vector<int4> pslot((size_t)M1 * n_pitems, make_int4(-1, -1, -1, -1));
  for (int i = 0; i < n_pitems; ++i)
    for (int mm = 0; mm < pitems[i].len; ++mm) {
      int4 &e = pslot[(size_t)mm * n_pitems + i];
      if (pitems[i].offp >= 0) {
        e.x = (int)idx[pitems[i].offp + mm];
        e.z = k3slot[e.x];
      }
      if (pitems[i].offm >= 0) {
        e.y = (int)idx[pitems[i].offm + mm];
        e.w = k3slot[e.y];
      }
    }

  // ---- tensor-core structure factor plan ----
  std::vector<int4> tc_runs;
  std::vector<int2> tc_map;
  std::vector<TCChunk> tc_chunks;
  int tc_A = 0, tc_ymin = 0, tc_ymax = 0, tc_zmin = 0, tc_zmax = 0, tc_mtiles = 0, tc_npad_max = 16;
  {
    std::map<int, std::vector<int>> by_z;  // m_z -> distinct m_y
    tc_ymin = tc_ymax = (int)m[1];
    tc_zmin = tc_zmax = (int)m[2];
    for (int64_t k = 0; k < K; ++k) {
      const int mx = (int)m[3 * k], my = (int)m[3 * k + 1], mz = (int)m[3 * k + 2];
      tc_A = std::max(tc_A, std::abs(mx));
      tc_ymin = std::min(tc_ymin, my);
      tc_ymax = std::max(tc_ymax, my);
      tc_zmin = std::min(tc_zmin, mz);
      tc_zmax = std::max(tc_zmax, mz);
      by_z[mz].push_back(my);
    }
    std::map<std::pair<int, int>, int> row_of;  // (m_y, m_z) -> tile*64 + p
    int n_runs = 0;
    for (auto &kv : by_z) {
      auto &v = kv.second;
      std::sort(v.begin(), v.end());
      v.erase(std::unique(v.begin(), v.end()), v.end());
      size_t i = 0;
      while (i < v.size()) {
        size_t e = i + 1;
        while (e < v.size() && e - i < 8 && v[e] == v[e - 1] + 1) ++e;
        tc_runs.push_back(make_int4(kv.first, v[i], (int)(e - i), 0));
        for (size_t u = i; u < e; ++u)
          row_of[std::make_pair(v[u], kv.first)] = (n_runs / 8) * 64 + (n_runs % 8) * 8 + (int)(u - i);
        ++n_runs;
        i = e;
      }
    }
    tc_mtiles = (n_runs + 7) / 8;
    tc_runs.resize((size_t)tc_mtiles * 8, make_int4(0, 0, 0, 0));
    const int A1 = tc_A + 1;
    tc_map.assign((size_t)tc_mtiles * 64 * A1, make_int2(-1, -1));
    for (int i = 0; i < n_pitems; ++i)
      for (int mm = 0; mm < pitems[i].len; ++mm) {
        const int r = row_of.at(std::make_pair(pitems[i].my, pitems[i].s + mm));
        int2 &e = tc_map[(size_t)r * A1 + pitems[i].ax];
        const int slot = mm * n_pitems + i;
        if (e.x < 0) e.x = slot; else e.y = slot;
      }
    // a-chunks: Xr columns then Xs columns, <= TC_NMAX in total.  Two
    // candidate splits -- greedy (full chunks, a narrow last one) and the
    // same number of chunks with the a-range split evenly -- priced by the
    // merged-MMA columns they execute (every chunk runs at the widest
    // chunk's slice stride XNP: a merge of m slices costs (m-1) XNP + npad;
    // per K-step 7 merges of 3, 2 of 2, 1 single): c3's 64 + 16 columns
    // become 48 + 48 (-12% MMA columns), c5 keeps 64 + 48.
    auto ncols = [&](int lo, int hi) { return (hi - lo + 1) + std::max(0, hi - std::max(lo, 1) + 1); };
    auto pad16 = [](int nc) { return ((nc + 15) / 16) * 16; };
    std::vector<TCChunk> greedy, even;
    for (int a0 = 0; a0 <= tc_A;) {
      int a1 = a0;
      while (a1 + 1 <= tc_A && ncols(a0, a1 + 1) <= TC_NMAX) ++a1;
      greedy.push_back(TCChunk{a0, a1, a1 - a0 + 1, pad16(ncols(a0, a1))});
      a0 = a1 + 1;
    }
    {
      const int nch = (int)greedy.size();
      bool ok = true;
      for (int c = 0; c < nch && ok; ++c) {
        const int a0 = (int)((int64_t)(tc_A + 1) * c / nch), a1 = (int)((int64_t)(tc_A + 1) * (c + 1) / nch) - 1;
        ok = a1 >= a0 && ncols(a0, a1) <= TC_NMAX;
        if (ok) even.push_back(TCChunk{a0, a1, a1 - a0 + 1, pad16(ncols(a0, a1))});
      }
      if (!ok) even.clear();
    }
    auto cost = [&](const std::vector<TCChunk> &v) {
      int xnp = 16;
      for (const auto &c : v) xnp = std::max(xnp, c.npad);
      int64_t t = 0;
      for (const auto &c : v) t += 7 * (2 * xnp + c.npad) + 2 * (xnp + c.npad) + c.npad;
      return t;
    };
    tc_chunks = (!even.empty() && cost(even) < cost(greedy)) ? even : greedy;
    for (const auto &c : tc_chunks) tc_npad_max = std::max(tc_npad_max, c.npad);
  }

  // ---- tensor-core force-gather plan ----
  std::vector<T3Row> t3_rows;
  std::vector<int4> t3_comp;
  std::vector<int2> t3_pair_yz;
  std::vector<int> t3_slotmap;
  {
    // rows ordered by force component (x: types 0,1; y: 2,3 and a=0; z: 4,5
    // and a=0) so that each component is a contiguous row range per M tile
    for (int c = 0; c < 3; ++c) {
      if (c > 0) t3_rows.push_back(T3Row{0, 2 * c});
      for (int t = 1; t <= tc_A; ++t)
        for (int ty = 2 * c; ty < 2 * c + 2; ++ty) t3_rows.push_back(T3Row{t, ty});
    }
    const int n_t3 = (int)t3_rows.size();
    for (int mt = 0; mt < (n_t3 + 127) / 128; ++mt) {
      int4 cr = make_int4(0, 0, 0, 0);
      int *ends[3] = {&cr.x, &cr.y, &cr.z};
      for (int c = 0; c < 3; ++c) {
        int e = 0;
        for (int r = 0; r < 128 && mt * 128 + r < n_t3; ++r)
          if ((t3_rows[mt * 128 + r].type >> 1) <= c) e = r + 1;
        *ends[c] = e;
      }
      t3_comp.push_back(cr);
    }
    const int n_runs_all = (int)tc_runs.size();
    const int npp = ((n_runs_all * 8 + 31) / 32) * 32;
    t3_pair_yz.assign(npp, make_int2(INT_MIN, INT_MIN));
    for (int r = 0; r < n_runs_all; ++r)
      for (int i = 0; i < tc_runs[r].z; ++i)
        t3_pair_yz[r * 8 + i] = make_int2(tc_runs[r].y + i, tc_runs[r].x);
    std::map<std::pair<int, int>, int> p_of;
    for (int p = 0; p < npp; ++p)
      if (t3_pair_yz[p].x != INT_MIN) p_of[std::make_pair(t3_pair_yz[p].x, t3_pair_yz[p].y)] = p;
    t3_slotmap.assign((size_t)(2 * tc_A + 1) * npp, -1);
    for (int64_t k = 0; k < K; ++k) {
      const int p = p_of.at(std::make_pair((int)m[3 * k + 1], (int)m[3 * k + 2]));
      t3_slotmap[(size_t)(m[3 * k] + tc_A) * npp + p] = k3slot[k];
    }
  }

  // K1 tiles and their phase-table descriptors: q e^{-i s th_z} for the
  // distinct segment starts, e^{-i m_y th_y} over the m_y range,
  // 2 e^{-i |m_x| th_x} for the distinct |m_x| (linked along x), e^{-i th_z}
  const int n_tiles = (n_pitems + K1_THREADS - 1) / K1_THREADS;
  std::vector<int4> ptab(n_pitems);
  std::vector<int4> desc;
  std::vector<int> tile_off(n_tiles), tile_ts(n_tiles);
  int ts_max = 0;
  for (int t = 0; t < n_tiles; ++t) {
    const int i0 = t * K1_THREADS, i1 = std::min(n_pitems, i0 + K1_THREADS);
    std::vector<int> svals, axs;
    int my_lo = pitems[i0].my, my_hi = pitems[i0].my;
    for (int i = i0; i < i1; ++i) {
      svals.push_back(pitems[i].s);
      axs.push_back(pitems[i].ax);
      my_lo = std::min(my_lo, pitems[i].my);
      my_hi = std::max(my_hi, pitems[i].my);
    }
    std::sort(svals.begin(), svals.end());
    svals.erase(std::unique(svals.begin(), svals.end()), svals.end());
    std::sort(axs.begin(), axs.end());
    axs.erase(std::unique(axs.begin(), axs.end()), axs.end());
    const int n_z = (int)svals.size(), n_y = my_hi - my_lo + 1, n_x = (int)axs.size();
    const int TS = n_z + n_y + n_x + 1;
    if (TS > 8192) return h->fail(EWB_EINVAL, "k-table too sparse for the tile planner");
    tile_off[t] = (int)desc.size();
    tile_ts[t] = TS;
    ts_max = std::max(ts_max, TS);
    for (int v : svals) desc.push_back(make_int4(0, 0, v, TF_QSCALE));
    for (int y = my_lo; y <= my_hi; ++y)
      desc.push_back(make_int4(0, y, 0, y > my_lo ? (TF_LINK | (1 << 2)) : 0));
    for (int xi = 0; xi < n_x; ++xi)
      desc.push_back(make_int4(axs[xi], 0, 0,
                               TF_SCALE2 | ((xi > 0 && axs[xi] == axs[xi - 1] + 1) ? TF_LINK : 0)));
    desc.push_back(make_int4(0, 0, 1, 0));
    for (int i = i0; i < i1; ++i) {
      const int iz = (int)(std::lower_bound(svals.begin(), svals.end(), pitems[i].s) - svals.begin());
      const int ix = (int)(std::lower_bound(axs.begin(), axs.end(), pitems[i].ax) - axs.begin());
      ptab[i] = make_int4(iz, n_z + pitems[i].my - my_lo, n_z + n_y + ix, 0);
    }
  }

  P.K = K;
  P.M = M;
  P.n_items = n_items;
  P.n_rows = n_rows;
  P.M1 = M1;
  P.n_pitems = n_pitems;
  P.n_tiles = n_tiles;
  P.ts_max = ts_max;
  P.pchunk = std::max(1, std::min(K1_PMAX, (K1_TAB_BYTES) / (16 * (ts_max | 1))));
  for (auto &c : P.ks_cache) c.second.release();
  P.ks_cache.clear();
  int rc;
  P.tc_A = tc_A;
  P.tc_mtiles = tc_mtiles;
  P.tc_nchunks = (int)tc_chunks.size();
  P.tc_npad_max = tc_npad_max;
  P.tc_ymin = tc_ymin;
  P.tc_ny = tc_ymax - tc_ymin + 1;
  P.tc_zmin = tc_zmin;
  P.tc_nz = tc_zmax - tc_zmin + 1;
  if ((rc = upload(h, P.tc_runs, tc_runs))) return rc;
  if ((rc = upload(h, P.tc_map, tc_map))) return rc;
  if ((rc = upload(h, P.tc_chunks, tc_chunks))) return rc;
  P.tc_ok = true;
  P.tc_chunks_host = tc_chunks;
  P.t3_rows = (int)t3_rows.size();
  P.t3_mtiles = (P.t3_rows + 127) / 128;
  P.t3_npairs = (int)t3_pair_yz.size();
  P.t3_nkb = 2 * P.t3_npairs / TC_KB;
  if ((rc = upload(h, P.t3_rowtab, t3_rows))) return rc;
  if ((rc = upload(h, P.t3_comp, t3_comp))) return rc;
  if ((rc = upload(h, P.t3_pair_yz, t3_pair_yz))) return rc;
  if ((rc = upload(h, P.t3_slotmap, t3_slotmap))) return rc;
  // the epilogue's shared X table must fit next to the level sums
  P.t3_ok = 128 * (T3_NP + 1) * (int)sizeof(double) + T3_NP * (tc_A + 1) * (int)sizeof(double2) <=
            t3_smem_bytes();
  h->tc_spart_zeroed = nullptr;
  if ((rc = upload(h, P.pitem_tab, ptab))) return rc;
  if ((rc = upload(h, P.item_my, item_my))) return rc;
  if ((rc = upload(h, P.item_row, item_row))) return rc;
  if ((rc = upload(h, P.rows, rows))) return rc;
  if ((rc = upload(h, P.tab_desc, desc))) return rc;
  if ((rc = upload(h, P.tile_off, tile_off))) return rc;
  if ((rc = upload(h, P.tile_ts, tile_ts))) return rc;
  if ((rc = upload(h, P.slot_k, slot_k))) return rc;
  if ((rc = upload(h, P.slot_coeff, slot_coeff))) return rc;
  if ((rc = upload(h, P.pslot_map, pslot))) return rc;
  if ((rc = upload(h, P.k3meta, k3meta))) return rc;
  // C*S for the gather: padding slots stay zero for the lifetime of the plan
  CK(h->sp.ensure(n_slots * sizeof(double2)));
  CK(cudaMemset(h->sp.p, 0, n_slots * sizeof(double2)));
  return EWB_OK;
}

// k-split row boundaries for n_ks splits; cached per n_ks so a buffer a
// queued kernel may still read is never overwritten
const int *ensure_ks(ewb_handle *h, int n_ks, int *status) {
  Plan &P = h->plan;
  for (auto &c : P.ks_cache)
    if (c.first == n_ks) return c.second.as<int>();
  std::vector<int> b(n_ks + 1);
  b[0] = 0;
  b[n_ks] = P.n_rows;
  for (int q = 1; q < n_ks; ++q) {
    const int64_t target = (int64_t)q * P.n_items / n_ks;
    int r = (int)(std::lower_bound(P.row_item_prefix.begin(), P.row_item_prefix.end(), target) -
                  P.row_item_prefix.begin());
    b[q] = std::max(b[q - 1], std::min(r, P.n_rows));
  }
  P.ks_cache.emplace_back(n_ks, DBuf());
  DBuf &buf = P.ks_cache.back().second;
  cudaError_t e = buf.ensure(b.size() * sizeof(int));
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(buf.p, b.data(), b.size() * sizeof(int), cudaMemcpyHostToDevice,
                        h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);  // b is a local vector
  if (e != cudaSuccess) {
    *status = h->fail(EWB_ECUDA, std::string("k-split upload: ") + cudaGetErrorString(e));
    return nullptr;
  }
  return buf.as<int>();
}

int require_state(ewb_handle *h, bool need_kspace, bool need_loaded) {
  if (!h) return EWB_EINVAL;
  if (!h->have_system) return h->fail(EWB_ESTATE, "ewb_set_system not called");
  if (need_kspace && !h->have_kspace) return h->fail(EWB_ESTATE, "ewb_set_kspace not called");
  if (need_loaded && !h->loaded) return h->fail(EWB_ESTATE, "no particles loaded");
  return EWB_OK;
}

// ---- stages (all asynchronous on h->stream) ----
int stage_load(ewb_handle *h, const double *d_pos, const double *d_q, int64_t n) {
  if (n < 1) return h->fail(EWB_EINVAL, "particle count must be >= 1");
  if (n >= (int64_t)1 << 25) return h->fail(EWB_EINVAL, "particle count must be < 2^25");
  CK(h->frac.ensure(n * sizeof(double4)));
  CK(h->xyzq.ensure(n * sizeof(double4)));
  CK(h->base.ensure(n * 3 * sizeof(double2)));
  CK(h->errflag.ensure(sizeof(int)));
  CK(cudaMemsetAsync(h->errflag.p, 0, sizeof(int), h->stream));
  k_prep<<<blocks_for(n, 256), 256, 0, h->stream>>>(d_pos, d_q, n, h->L, h->frac.as<double4>(),
                                                    h->base.as<double2>(), h->xyzq.as<double4>(),
                                                    h->errflag.as<int>());
  CKL();
  h->n = n;
  h->loaded = true;
  return EWB_OK;
}

int occupancy_k1(ewb_handle *h, int M, size_t smem, int *occ_out) {
  if (!h->k1_attr[M]) {
    CK(cudaFuncSetAttribute((const void *)k1_table(M), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            200 * 1024));
    h->k1_attr[M] = true;
  }
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void *)k1_table(M), K1_THREADS,
                                                   smem));
  *occ_out = std::max(1, occ);
  return EWB_OK;
}

// S(k) over particles [i0, i1): partials over particle chunks reduced into
// d_slots (if non-null) or left in h->spart with *n_part set.
// Tensor-core reciprocal space for this particle count?  Auto mode: the
// GEMM set-up (prep kernels, operand splits, epilogues) costs a few tens of
// microseconds, so tiny systems (c1: N K = 2.5e6) stay on the FP64 kernels.
constexpr double TC_AUTO_MIN_WORK = 67108864.0;  // N * K
bool tc_wanted(const ewb_handle *h, int64_t n) {
  if (h->use_tc == 0) return false;
  if (h->use_tc == 1) return true;
  return (double)n * (double)h->plan.K >= TC_AUTO_MIN_WORK;
}

// Tensor-core structure factor (k1_tc.cuh): same pair-layout partials as K1.
int stage_rho_tc(ewb_handle *h, int64_t i0, int64_t i1, int *n_part_out) {
  Plan &P = h->plan;
  const int64_t n = std::max<int64_t>(0, i1 - i0);
  const size_t n_pslots = (size_t)P.M1 * P.n_pitems;
  const int64_t np = std::max<int64_t>(TC_KB, ((n + TC_KB - 1) / TC_KB) * TC_KB);
  const int64_t nkb = np / TC_KB;
  const int T = P.tc_mtiles * P.tc_nchunks;
  const int64_t kb_cap = TC_MAXP / TC_KB;
  const int64_t ns_min = (nkb + kb_cap - 1) / kb_cap;
  const int64_t waves = std::max<int64_t>(1, (T * ns_min + h->n_sm - 1) / h->n_sm);
  int64_t ns = std::max<int64_t>(ns_min, (waves * h->n_sm) / std::max(1, T));
  ns = std::min<int64_t>(ns, nkb);
  const int64_t kbps = (nkb + ns - 1) / ns;
  ns = (nkb + kbps - 1) / kbps;
  const int xsl_b = tc_xsl_bytes(P.tc_npad_max);
  CK(h->tc_qmax.ensure(sizeof(double)));
  CK(h->tc_ytab.ensure(K1_TABLES ? (size_t)P.tc_ny * np * sizeof(double2) : 16));
  CK(h->tc_ztab.ensure(K1_TABLES ? (size_t)P.tc_nz * np * sizeof(double2) : 16));
  CK(h->tc_xsl.ensure((size_t)P.tc_nchunks * nkb * TC_S * xsl_b));
  CK(h->spart.ensure((size_t)ns * n_pslots * sizeof(double4)));
  if (h->tc_spart_zeroed != h->spart.p) {  // slots no k maps to stay zero
    CK(cudaMemsetAsync(h->spart.p, 0, h->spart.cap, h->stream));
    h->tc_spart_zeroed = h->spart.p;
  }
  CK(cudaMemsetAsync(h->tc_qmax.p, 0, sizeof(double), h->stream));
  if (n > 0) {
    k_absmax_q<<<(unsigned)std::min<int64_t>(1184, (n + 255) / 256), 256, 0, h->stream>>>(
        h->frac.as<double4>(), i0, i1, h->tc_qmax.as<unsigned long long>());
    CKL();
  }
  k1t_prep<<<dim3((unsigned)((np + 127) / 128),
                  (K1_TABLES ? (P.tc_ny + 7) / 8 + (P.tc_nz + 7) / 8 : 0) +
                      P.tc_nchunks * ((P.tc_npad_max + 7) / 8)),
             128, 0, h->stream>>>(
      h->frac.as<double4>(), i0, std::max(i0, i1), np, h->tc_qmax.as<double>(), P.tc_ymin, P.tc_ny,
      P.tc_zmin, P.tc_nz, P.tc_chunks.as<TCChunk>(), P.tc_nchunks, P.tc_npad_max,
      h->tc_ytab.as<double2>(), h->tc_ztab.as<double2>(), h->tc_xsl.as<uint8_t>());
  CKL();
  const size_t smem = (size_t)tc_smem_bytes(P.tc_npad_max);
  // X slice stride = the widest padded a-chunk (multiple of 16, <= 64)
  auto kern = P.tc_npad_max <= 16   ? k1t_gemm<16>
              : P.tc_npad_max <= 32 ? k1t_gemm<32>
              : P.tc_npad_max <= 48 ? k1t_gemm<48>
                                    : k1t_gemm<64>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<dim3(P.tc_mtiles, P.tc_nchunks, (unsigned)ns), TC_NTHREADS, smem, h->stream>>>(
      h->frac.as<double4>(), h->tc_ytab.as<double2>(), h->tc_ztab.as<double2>(),
      h->base.as<double2>(), h->tc_xsl.as<uint8_t>(), P.tc_chunks.as<TCChunk>(),
      P.tc_runs.as<int4>(),
      P.tc_map.as<int2>(), h->tc_qmax.as<double>(), i0, std::max(i0, i1), np, kbps * TC_KB,
      P.tc_ymin, P.tc_zmin, P.tc_A, P.tc_npad_max, (int64_t)n_pslots, h->spart.as<double4>(),
      h->tc_dbg);
  CKL();
  *n_part_out = (int)ns;
  return EWB_OK;
}

int stage_rho(ewb_handle *h, int64_t i0, int64_t i1, int *n_part_out) {
  Plan &P = h->plan;
  if (P.tc_ok && tc_wanted(h, h->n)) return stage_rho_tc(h, i0, i1, n_part_out);
  const int M1 = P.M1;
  const size_t smem = 2 * (size_t)P.pchunk * (P.ts_max | 1) * sizeof(double2) +
                      (size_t)P.ts_max * sizeof(int4);
  int occ = 1;
  int rc = occupancy_k1(h, M1, smem, &occ);
  if (rc) return rc;
  const int64_t n = std::max<int64_t>(0, i1 - i0);
  // many short blocks (they desynchronise the table-build phases of
  // co-resident blocks), bounded by the partial-sum buffer size
  const size_t slot_bytes = (size_t)M1 * P.n_pitems * sizeof(double4);
  const int64_t slots1 = (int64_t)h->n_sm * occ;
  int64_t n_pc = std::max<int64_t>(1, (n + K1_PPB - 1) / K1_PPB);
  n_pc = std::min<int64_t>(n_pc, std::max<int64_t>(1, (int64_t)(K1_PART_BYTES / slot_bytes)));
  // round the grid to whole waves of resident blocks (no partial last wave)
  {
    const int64_t waves = std::max<int64_t>(1, (P.n_tiles * n_pc + slots1 - 1) / slots1);
    const int64_t fit = (waves * slots1) / P.n_tiles;
    if (fit >= 1) n_pc = std::min<int64_t>(fit, std::max<int64_t>(1, (int64_t)(K1_PART_BYTES / slot_bytes)));
  }
  n_pc = std::min<int64_t>(n_pc, std::max<int64_t>(1, n / K1_PMAX));  // >= one chunk per block
  int64_t ppb = (n + n_pc - 1) / std::max<int64_t>(1, n_pc);
  ppb = std::max<int64_t>(1, ppb);
  n_pc = std::max<int64_t>(1, (n + ppb - 1) / ppb);
  const size_t n_pslots = (size_t)M1 * P.n_pitems;
  CK(h->spart.ensure((size_t)n_pc * n_pslots * sizeof(double4)));
  dim3 grid(P.n_tiles, (unsigned)n_pc);
  k1_table(M1)<<<grid, K1_THREADS, smem, h->stream>>>(
      h->frac.as<double4>(), h->base.as<double2>(), i0, std::max(i0, i1), ppb, P.pchunk,
      P.pitem_tab.as<int4>(), P.n_pitems, P.tab_desc.as<int4>(), P.tile_off.as<int>(),
      P.tile_ts.as<int>(), h->spart.as<double4>());
  CKL();
  *n_part_out = (int)n_pc;
  return EWB_OK;
}

// finalize from a gather-layout S (caller-supplied rho, ewb_long_range)
int stage_finalize(ewb_handle *h, const double2 *src, int n_part, double *d_rho_out,
                   double *d_u_out) {
  Plan &P = h->plan;
  const int64_t n_slots = (int64_t)P.M * P.n_items;
  const unsigned nb = blocks_for(n_slots, RED_THREADS);
  CK(h->sp.ensure(n_slots * sizeof(double2)));
  CK(h->eblk.ensure(nb * sizeof(double)));
  k2_finalize<<<nb, RED_THREADS, 0, h->stream>>>(src, n_part, n_slots, P.slot_k.as<int>(),
                                                 P.slot_coeff.as<double>(), P.K, d_rho_out,
                                                 nullptr, h->sp.as<double2>(),
                                                 h->eblk.as<double>(), 1);
  CKL();
  k_sum<<<1, 1024, 0, h->stream>>>(h->eblk.as<double>(), nb, 1.0, d_u_out);
  CKL();
  return EWB_OK;
}

// finalize from n_part pair-layout partials (the structure-factor output)
int stage_finalize_pairs(ewb_handle *h, const double4 *src, int n_part, double *d_rho_out,
                         double *d_u_out) {
  Plan &P = h->plan;
  const int64_t n_pslots = (int64_t)P.M1 * P.n_pitems;
  const unsigned nb = blocks_for(n_pslots, RED_THREADS);
  CK(h->eblk_r.ensure(nb * sizeof(double)));
  k2p_finalize<<<nb, RED_THREADS, 0, h->stream>>>(src, n_part, n_pslots, P.pslot_map.as<int4>(),
                                                  P.slot_coeff.as<double>(), P.K, d_rho_out,
                                                  nullptr, h->sp.as<double2>(),
                                                  h->eblk_r.as<double>(), 1);
  CKL();
  k_sum<<<1, 1024, 0, h->stream>>>(h->eblk_r.as<double>(), nb, 1.0, d_u_out);
  CKL();
  return EWB_OK;
}

// Tensor-core force gather (k3_tc.cuh); forces only (the per-particle
// energy of the foreign-rho API stays on the FP64 gather).
int stage_recip_tc(ewb_handle *h, int64_t i0, int64_t i1, double *d_force) {
  Plan &P = h->plan;
  const int64_t n_local = i1 - i0;
  const int nkb = P.t3_nkb;
  const int NP = T3_NP;
  CK(h->t3_wsl.ensure((size_t)P.t3_mtiles * nkb * T3_S * TC_GSL));
  CK(h->t3_rscale.ensure((size_t)P.t3_mtiles * 128 * sizeof(double)));
  {
    const unsigned kparts = (unsigned)std::max(1, std::min(16, (2 * P.t3_npairs + 1023) / 1024));
    CK(cudaMemsetAsync(h->t3_rscale.p, 0, (size_t)P.t3_mtiles * 128 * sizeof(double), h->stream));
    k3t_wmax<<<dim3(P.t3_rows, kparts), 256, 0, h->stream>>>(
        h->sp.as<double2>(), P.t3_slotmap.as<int>(), P.tc_A, P.t3_pair_yz.as<int2>(), P.t3_npairs,
        P.t3_rowtab.as<T3Row>(), P.t3_rows, h->t3_rscale.as<unsigned long long>());
    CKL();
    k3t_wprep<<<dim3(P.t3_mtiles * 128, kparts), 256, 0, h->stream>>>(
          h->sp.as<double2>(), P.t3_slotmap.as<int>(), P.tc_A, P.t3_pair_yz.as<int2>(),
          P.t3_npairs, P.t3_rowtab.as<T3Row>(), P.t3_rows, nkb, h->t3_rscale.as<double>(),
          h->t3_wsl.as<uint8_t>());
    CKL();
  }
  const int64_t ptiles = (n_local + NP - 1) / NP;
  const int64_t T = ptiles * P.t3_mtiles;  // CTAs per split
  const int kb_cap = T3_KMAX / TC_KB;
  const int ns_min = std::max(1, (nkb + kb_cap - 1) / kb_cap);
  // K splits: as few as int32 exactness allows -- each split adds a CTA
  // prologue/epilogue and a partial-force pass, which costs more than the
  // partial last wave it could fill (measured: forcing 1 instead of the
  // wave-filling choice, c4 0.837 -> 0.762 ms, c3 6.25 -> 5.88, c5 81.2 ->
  // 78.6); more only when one split leaves SMs idle
  int ns = ns_min;
  if ((int64_t)T * ns < h->n_sm)
    ns = std::max(ns_min, (int)std::min<int64_t>(std::max(1, nkb / 4),
                                                  (h->n_sm + T - 1) / std::max<int64_t>(1, T)));
  const int kbps = (nkb + ns - 1) / ns;
  ns = (nkb + kbps - 1) / kbps;
  const int n_ks = ns * P.t3_mtiles;
  CK(h->fpart.ensure((size_t)n_ks * 3 * n_local * sizeof(double)));
  const size_t smem = (size_t)t3_smem_bytes();
  CK(cudaFuncSetAttribute(k3t_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  {
    // clusters of T3_CL particle tiles share the A loads (padding tiles
    // carry no particles)
    const int64_t ptiles_pad = ((ptiles + T3_CL - 1) / T3_CL) * T3_CL;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)ptiles_pad, P.t3_mtiles, ns);
    lc.blockDim = dim3(T3_THREADS);
    lc.dynamicSmemBytes = smem;
    lc.stream = h->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = T3_CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    CK(cudaLaunchKernelEx(&lc, k3t_gemm, (const double4 *)h->frac.as<double4>(),
                          (const double2 *)h->base.as<double2>(), (const uint8_t *)h->t3_wsl.as<uint8_t>(),
                          (const double *)h->t3_rscale.as<double>(),
                          (const T3Row *)P.t3_rowtab.as<T3Row>(), P.t3_rows,
                          (const int2 *)P.t3_pair_yz.as<int2>(), nkb, kbps, i0, i1, P.tc_A,
                          (const int4 *)P.t3_comp.as<int4>(), h->fpart.as<double>(), h->tc_dbg));
    ++h->launches;
  }
  if (h->ov_active) {  // the combine adds into forces: after the real-space join
    h->t3_pend_nks = n_ks;
    h->t3_pend_i0 = i0;
    h->t3_pend_n = n_local;
    h->t3_pend_force = d_force;
    return EWB_OK;
  }
  const unsigned nbc = blocks_for(n_local, RED_THREADS);
  k3_combine<<<nbc, RED_THREADS, 0, h->stream>>>(h->fpart.as<double>(), nullptr, n_ks, i0, n_local,
                                                  h->frac.as<double4>(), 4.0 * M_PI / h->L,
                                                  d_force, nullptr, 0);
  CKL();
  return EWB_OK;
}

int stage_recip_forces(ewb_handle *h, int64_t i0, int64_t i1, double *d_force, bool energy,
                       double *d_u_out) {
  Plan &P = h->plan;
  const int64_t n_local = std::max<int64_t>(0, i1 - i0);
  if (n_local == 0) {
    if (energy) CK(cudaMemsetAsync(d_u_out, 0, sizeof(double), h->stream));
    return EWB_OK;
  }
  if (!energy && P.t3_ok && tc_wanted(h, h->n)) return stage_recip_tc(h, i0, i1, d_force);
  const int M = P.M;
  k3_fn fn = k3_table(M, energy);
  int &occ = h->occ_k3[M][energy ? 1 : 0];
  if (occ == 0) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void *)fn, K3_THREADS, 0));
    occ = std::max(1, occ);
  }
  const int64_t ptiles = (n_local + K3_THREADS * K3_PPT - 1) / (K3_THREADS * K3_PPT);
  const int64_t slots3 = (int64_t)h->n_sm * occ;
  const unsigned nbc = blocks_for(n_local, RED_THREADS);
  if (h->k3_const && ptiles >= K3C_MIN_WAVES * (int64_t)h->n_sm) {
    // constant-bank variant: enough particles to fill the GPU without
    // k-splits; walk the k-space in constant-bank chunks
    const int cap = std::max(1, std::min(K3C_ITEMS, K3C_CAP / M));
    CK(h->fpart.ensure((size_t)2 * 3 * n_local * sizeof(double)));
    if (energy) CK(h->upart.ensure((size_t)2 * n_local * sizeof(double)));
    const int n_chunks = (P.n_items + cap - 1) / cap;
    cudaStream_t st[2] = {h->stream, h->aux_stream};
    // fork the auxiliary stream off the main one (graph-capture safe)
    CK(cudaEventRecord(h->ev_fork, h->stream));
    CK(cudaStreamWaitEvent(h->aux_stream, h->ev_fork, 0));
    if (n_chunks < 2) {  // the second accumulator must still be defined
      CK(cudaMemsetAsync(h->fpart.as<double>() + 3 * n_local, 0, 3 * n_local * sizeof(double),
                         h->aux_stream));
      if (energy)
        CK(cudaMemsetAsync(h->upart.as<double>() + n_local, 0, n_local * sizeof(double),
                           h->aux_stream));
    }
    for (int c = 0; c < n_chunks; ++c) {
      const int it0 = c * cap, nc = std::min(cap, P.n_items - it0), b = c & 1;
      CK(cudaMemcpyToSymbolAsync(c_k3sp, h->sp.as<double2>() + (size_t)it0 * M,
                                 (size_t)nc * M * sizeof(double2),
                                 (size_t)b * K3C_CAP * sizeof(double2), cudaMemcpyDeviceToDevice,
                                 st[b]));
      CK(cudaMemcpyToSymbolAsync(c_k3meta, P.k3meta.as<int4>() + it0, (size_t)nc * sizeof(int4),
                                 (size_t)b * K3C_ITEMS * sizeof(int4), cudaMemcpyDeviceToDevice,
                                 st[b]));
      k3c_table(M, energy, b)<<<(unsigned)ptiles, K3_THREADS, 0, st[b]>>>(
          h->frac.as<double4>(), h->base.as<double2>(), i0, i1, nc, c < 2 ? 1 : 0,
          h->fpart.as<double>() + (size_t)b * 3 * n_local,
          energy ? h->upart.as<double>() + (size_t)b * n_local : nullptr);
      CKL();
    }
    // join
    CK(cudaEventRecord(h->ev_join, h->aux_stream));
    CK(cudaStreamWaitEvent(h->stream, h->ev_join, 0));
    if (h->ov_active && !energy) {  // the combine adds into forces: after the real-space join
      h->t3_pend_nks = 2;
      h->t3_pend_i0 = i0;
      h->t3_pend_n = n_local;
      h->t3_pend_force = d_force;
      return EWB_OK;
    }
    if (energy) CK(h->eblk2.ensure(nbc * sizeof(double)));
    k3_combine<<<nbc, RED_THREADS, 0, h->stream>>>(
        h->fpart.as<double>(), energy ? h->upart.as<double>() : nullptr, 2, i0, n_local,
        h->frac.as<double4>(), 4.0 * M_PI / h->L, d_force,
        energy ? h->eblk2.as<double>() : nullptr, energy ? 1 : 0);
    CKL();
    if (energy) {
      k_sum<<<1, 1024, 0, h->stream>>>(h->eblk2.as<double>(), nbc, 1.0, d_u_out);
      CKL();
    }
    return EWB_OK;
  }
  // enough k-splits for K3_WAVES waves of resident blocks (short blocks
  // balance the tail), each split keeping >= 2 rows
  int n_ks = (int)std::max<int64_t>(1, (K3_WAVES * slots3 + ptiles - 1) / ptiles);
  n_ks = std::max(1, std::min(n_ks, std::max(1, P.n_rows / 2)));
  int rc = EWB_OK;
  const int *ks_rows = ensure_ks(h, n_ks, &rc);
  if (!ks_rows) return rc;
  CK(h->fpart.ensure((size_t)n_ks * 3 * n_local * sizeof(double)));
  if (energy) CK(h->upart.ensure((size_t)n_ks * n_local * sizeof(double)));
  dim3 grid((unsigned)ptiles, n_ks);
  fn<<<grid, K3_THREADS, 0, h->stream>>>(h->frac.as<double4>(), h->base.as<double2>(), i0, i1,
                                         P.rows.as<int4>(), ks_rows,
                                         P.item_my.as<int>(), P.item_row.as<int>(),
                                         h->sp.as<double2>(), P.n_items, h->fpart.as<double>(),
                                         energy ? h->upart.as<double>() : nullptr);
  CKL();
  if (h->ov_active && !energy) {  // the combine adds into forces: after the real-space join
    h->t3_pend_nks = n_ks;
    h->t3_pend_i0 = i0;
    h->t3_pend_n = n_local;
    h->t3_pend_force = d_force;
    return EWB_OK;
  }
  const unsigned nb = blocks_for(n_local, RED_THREADS);
  if (energy) CK(h->eblk2.ensure(nb * sizeof(double)));
  k3_combine<<<nb, RED_THREADS, 0, h->stream>>>(
      h->fpart.as<double>(), energy ? h->upart.as<double>() : nullptr, n_ks, i0, n_local,
      h->frac.as<double4>(), 4.0 * M_PI / h->L, d_force, energy ? h->eblk2.as<double>() : nullptr,
      energy ? 1 : 0);
  CKL();
  if (energy) {
    k_sum<<<1, 1024, 0, h->stream>>>(h->eblk2.as<double>(), nb, 1.0, d_u_out);
    CKL();
  }
  return EWB_OK;
}

// Cell geometry of the real-space pass at traversal cutoff rc_t.  Reference
// binning: cpd = floor(L / r_c), edge = L / cpd (celllist.py:96-98); with
// cpd < 3 the 27-stencil folds onto every cell and the reference scans all
// particles with a per-pair fold (engine.py:111-134) -- FOLD mode here.
// Cells of edge >= r_c/2 with a 5^3 stencil when the box holds >= 5 of them
// (42% fewer candidate pairs than r_c cells with 3^3), r_c/3 cells with 7^3
// while they hold >= 16 particles on average, else r_c cells with 3^3, else
// (fewer than 3 cells) the reference's scan-all branch.  Any cell size whose
// stencil covers the cutoff sphere visits the same pair set: the predicate,
// not the binning, decides membership.  The particle count deciding the
// r_c/3 grid is the global one of a sharded evaluation (ewb_set_geometry_n),
// so every rank bins on the same grid.
struct RSGeom {
  int rad, cpd, cpd_eff;
  bool fold;
  double edge;
};
RSGeom rs_geometry(const ewb_handle *h, double rc_t, int64_t n_local) {
  const int64_t n = h->geom_n > 0 ? h->geom_n : n_local;
  int rad = 2;
  int cpd = (int)std::floor(2.0 * h->L / rc_t);
  {
    // r_c/3 cells with a 7^3 stencil: tighter candidate pieces, but only
    // while a cell still holds >= 16 particles on average (c4, r_c = 8:
    // 19 per cell, real space -3.4%; r_c = 6 at unit density: 8 per cell,
    // +2..8%)
    const int cpd3 = (int)std::floor(K6_RAD3_F * h->L / rc_t);
    if (K6_RAD_MAX >= 3 && h->stencil_rad == 0 && cpd3 >= 7 && cpd3 <= 64 &&
        (double)n >= K6_RAD3_MINOCC * (double)cpd3 * cpd3 * cpd3) {
      rad = 3;
      cpd = cpd3;
    }
  }
  if (cpd < 5 || h->stencil_rad == 1) {
    rad = 1;
    cpd = (int)std::floor(h->L / rc_t);
  }
  if (cpd < 1) cpd = 1;
  if (cpd > 64) cpd = 64;  // edge stays >= r_c/rad; bounds the cell arrays
  const bool fold = cpd < 2 * rad + 1;
  return RSGeom{rad, cpd, fold ? 1 : cpd, fold, h->L / cpd};
}

// traversal cutoff (and its square) of the real-space pass: the larger of
// the Coulomb and LJ cutoffs of the terms the pair kernel evaluates
void rs_cutoff(const ewb_handle *h, double &rc_t, double &rc2_t) {
  const bool pair_coul = h->coul_on && !(h->rc > 0.5 * h->L);
  rc_t = std::max(pair_coul ? h->rc : 0.0, h->lj_on ? h->rc_lj : 0.0);
  rc2_t = std::max(pair_coul ? h->rc2 : 0.0, h->lj_on ? h->rc2_lj : 0.0);
}

// Cell list + real space for z-slab part/nparts; u_sr into d_u_out.
constexpr int RS_CELLS = 1, RS_PAIRS = 2;
int stage_real_space(ewb_handle *h, int part, int nparts, double *d_force, double *d_u_out,
                     cudaEvent_t ev_cell, int which = RS_CELLS | RS_PAIRS,
                     double *d_ulj_out = nullptr) {
  const int64_t n = h->n;
  const bool coul_on = h->coul_on, lj_on = h->lj_on;
  if (coul_on && !(h->rc > 0.0)) return h->fail(EWB_EINVAL, "cutoff must be positive");
  const bool wide = coul_on && h->rc > 0.5 * h->L;
  if (wide) {
    // r_c > L/2: the reference's image-shell path (ewald.py:553-576)
    if (h->rc > h->L)
      return h->fail(EWB_EBOX, "r_cutoff exceeds the box edge; a single image shell no longer "
                               "covers the interaction range");
    if (n > WIDE_MAX_N)
      return h->fail(EWB_ESIZE, "wide-cutoff real-space path is O(N^2); N exceeds the 4096 guard");
    if (which & RS_PAIRS) {
      if (h->row_hi >= 0 ? h->row_lo > 0 : part != 0) {  // not sharded: part 0 owns every centre
        CK(cudaMemsetAsync(d_u_out, 0, sizeof(double), h->stream));
      } else {
        CK(h->eblk.ensure(n * sizeof(double)));
        k6w_wide<<<(unsigned)n, 128, 0, h->stream>>>(h->xyzq.as<double4>(), n, h->L, h->rc2,
                                                     std::sqrt(h->alpha), h->alpha,
                                                     2.0 * std::sqrt(h->alpha / M_PI), d_force,
                                                     h->eblk.as<double>(), h->errflag.as<int>());
        CKL();
        k_sum<<<1, 1024, 0, h->stream>>>(h->eblk.as<double>(), n, 1.0, d_u_out);
        CKL();
      }
    }
  } else if ((which & RS_PAIRS) && !coul_on) {
    CK(cudaMemsetAsync(d_u_out, 0, sizeof(double), h->stream));
  }
  if (!((coul_on && !wide) || lj_on)) {
    if ((which & RS_PAIRS) && d_ulj_out) CK(cudaMemsetAsync(d_ulj_out, 0, sizeof(double), h->stream));
    return EWB_OK;
  }
  if (lj_on && !(h->rc_lj > 0.0)) return h->fail(EWB_EINVAL, "cutoff must be positive");
  if (lj_on && h->rc_lj > 0.5 * h->L)
    return h->fail(EWB_ECUTOFF, "LJ cutoff exceeds L/2 (minimum-image bound)");
  // one traversal at the larger cutoff; each term keeps its own exact predicate
  const bool pair_coul = coul_on && !wide;
  const double rc_t = std::max(pair_coul ? h->rc : 0.0, lj_on ? h->rc_lj : 0.0);
  const double rc2_t = std::max(pair_coul ? h->rc2 : 0.0, lj_on ? h->rc2_lj : 0.0);
  const RSGeom g = rs_geometry(h, rc_t, n);
  const int rad = g.rad, cpd_eff = g.cpd_eff;
  const bool fold = g.fold;
  const int n_cells = cpd_eff * cpd_eff * cpd_eff;
  const double edge = g.edge;
  if (which & RS_CELLS) {
  CK(h->cell_of.ensure(n * sizeof(int)));
  CK(h->slot.ensure(n * sizeof(int)));
  CK(h->count.ensure((n_cells + 1) * sizeof(int)));
  CK(h->start.ensure((n_cells + 1) * sizeof(int)));
  CK(h->gstart.ensure((n_cells + 1) * sizeof(int)));
  CK(h->order_tmp.ensure(n * sizeof(int)));
  CK(h->order.ensure(n * sizeof(int)));
  CK(h->sorted.ensure(n * sizeof(double4)));
  CK(h->sorted_f.ensure(n * sizeof(float4)));
  CK(h->sorted_cell.ensure(n * sizeof(int)));
  const int n_rows = fold ? 1 : cpd_eff * cpd_eff;
  CK(h->row_ustart.ensure((n_rows + 1) * sizeof(int)));
  if (fold) {  // every particle is a candidate: identity order, one launch
    k_fold_prep<<<blocks_for(n, 256), 256, 0, h->stream>>>(
        h->xyzq.as<double4>(), n, (int)((n + K6_G - 1) / K6_G), h->sorted.as<double4>(),
        h->sorted_f.as<float4>(), h->sorted_cell.as<int>(), h->order.as<int>(),
        h->start.as<int>(), h->row_ustart.as<int>());
    CKL();
  } else {
  CK(cudaMemsetAsync(h->count.p, 0, (n_cells + 1) * sizeof(int), h->stream));
  k4_bin_count<<<blocks_for(n, 256), 256, 0, h->stream>>>(h->xyzq.as<double4>(), n, edge, cpd_eff,
                                                          h->cell_of.as<int>(), h->slot.as<int>(),
                                                          h->count.as<int>());
  CKL();
  k_scan_cells<<<1, 1024, 0, h->stream>>>(h->count.as<int>(), n_cells, h->start.as<int>(),
                                          h->gstart.as<int>());
  CKL();
  {
    k5_scatter<<<blocks_for(n, 256), 256, 0, h->stream>>>(h->cell_of.as<int>(), h->slot.as<int>(),
                                                          n, h->start.as<int>(),
                                                          h->order_tmp.as<int>());
    CKL();
    k5_cell_sort<<<n_cells, 256, 0, h->stream>>>(h->start.as<int>(), h->order_tmp.as<int>(),
                                                 h->order.as<int>());
    CKL();
  }
  k5_gather<<<blocks_for(n, 256), 256, 0, h->stream>>>(h->order.as<int>(), h->xyzq.as<double4>(),
                                                       h->cell_of.as<int>(), n,
                                                       h->sorted.as<double4>(),
                                                       h->sorted_f.as<float4>(),
                                                       h->sorted_cell.as<int>());
  CKL();
  // units: K6_G consecutive particles of one row of cells (fixed cy, cz)
  k_scan_rows<<<1, 1024, 0, h->stream>>>(h->start.as<int>(), cpd_eff, n_rows,
                                         h->row_ustart.as<int>());
  CKL();
  }
  if (ev_cell) CK(cudaEventRecord(ev_cell, h->stream));
  }
  if (!(which & RS_PAIRS)) return EWB_OK;

  RSParams rp;
  rp.L = h->L;
  rp.hl = 0.5 * h->L;
  rp.rc2 = rc2_t;
  rp.coul = pair_coul ? 1 : 0;
  rp.rc2c = h->rc2;
  rp.rc2lj = h->rc2_lj;
  rp.lj_s2 = h->lj_s2;
  rp.lj_4e = h->lj_4e;
  rp.lj_shift = h->lj_shift;
  rp.lj_24e = h->lj_24e;
  {
    // |error of the FP32 r^2| <= 2^-24 (14 L r_c + 3 r_c^2) for |x| < L,
    // |shift| <= L (positions, shifted centres, differences and the FMA
    // chain rounded once each); doubled and rounded up
    const double rc_t = std::sqrt(rc2_t);
    const double margin = std::ldexp(2.0 * (16.0 * h->L * rc_t + 8.0 * rc2_t), -24);
    rp.rc2f = std::nextafter((float)(rc2_t + margin), INFINITY);
  }
  rp.sa = std::sqrt(h->alpha);
  rp.al = h->alpha;
  rp.tsap = 2.0 * std::sqrt(h->alpha / M_PI);
  rp.cpd = cpd_eff;
  rp.fold = fold;
  rp.rad = rad;
  rp.half = h->deterministic ? 0 : 1;
  rp.n = n;
  // rows of cells (fixed cy, cz; cz-major, so a contiguous range is a
  // z-slab with at most two partial layers) owned by this part: split by
  // rows, not whole layers (c2 on 8 parts: 12-13 of 100 rows each instead
  // of 1-2 of 10 layers, max slab 20% -> 13% of the pairs)
  const int64_t rows_all = (int64_t)cpd_eff * cpd_eff;
  rp.c_lo = fold ? (part == 0 ? 0 : 1) : (int)(rows_all * part / nparts);
  rp.c_hi = fold ? 1 : (int)(rows_all * (part + 1) / nparts);
  if (h->row_hi >= 0) {  // explicit row range (domain-decomposed evaluation)
    rp.c_lo = (int)std::min<int64_t>(rows_all, h->row_lo);
    rp.c_hi = (int)std::min<int64_t>(rows_all, std::max(h->row_lo, h->row_hi));
  }
  const int64_t rows_slab = rp.c_hi - rp.c_lo;
  const int64_t units_max = n / K6_G + rows_slab + 1;
  // scan-all mode with few units: split every unit's candidates over
  // several warps (partial sums meet in the atomics of the half shell)
  rp.jsplit = 1;
  // units this slab actually owns (estimate: rows are about equally filled)
  const int64_t active = std::max<int64_t>(
      1, (n / K6_G + rows_slab) * rows_slab / std::max<int64_t>(1, (int64_t)cpd_eff * cpd_eff));
  if (!fold && rp.half) {
    // few units (a z-slab of a multi-GPU step, small boxes): split each
    // unit's stencil rows over up to 4 warps so that >= 2 blocks per SM are
    // active (at full occupancy splitting costs: c2 +9% for 2 warps)
    const int64_t want = (int64_t)K6_SLAB_BLOCKS * h->n_sm * K6_WARPS;
    rp.jsplit = (int)std::min<int64_t>(4, std::max<int64_t>(K6_RSPLIT, (want + active - 1) / active));
  }
  if (fold && rp.half) {
    const int64_t want = 4 * (int64_t)h->n_sm * K6_WARPS;
    rp.jsplit = (int)std::max<int64_t>(1, std::min<int64_t>(64, want / std::max<int64_t>(1, units_max)));
    rp.jsplit = (int)std::min<int64_t>(rp.jsplit, std::max<int64_t>(1, n / 64));
  }
  const unsigned nb = (unsigned)std::max<int64_t>(
      1, (units_max * rp.jsplit + K6_WARPS - 1) / K6_WARPS);
  const int64_t n_eslots = (int64_t)nb * K6_WARPS;  // one energy slot per warp
  // two-pass real space: lists of 32-bit entries (j < 2^23), capacity per
  // unit twice the mean half-shell pair count of K6_G centres plus slack
  const bool split = h->rs_split && !fold && n < ((int64_t)1 << K6_LIST_JBITS) &&
                     rp.jsplit == 1;
  int cap = 0;
  if (split) {
    const double rho = (double)n / (h->L * h->L * h->L);
    const double est = K6_G * rho * (2.0 * M_PI / 3.0) * std::pow(rc2_t, 1.5);
    cap = (int)std::min<double>(1 << 20, 32.0 * std::ceil((2.0 * est + 256.0) / 32.0));
    if (h->rs_split == 2) cap = 32;  // testing: most units take the overflow pass
    CK(h->rs_list.ensure((size_t)units_max * cap * sizeof(uint32_t)));
    CK(h->rs_count.ensure((size_t)units_max * sizeof(int)));
  }
  const int64_t n_eslot_all = split ? 2 * n_eslots : n_eslots;  // + overflow pass
  CK(h->eblk.ensure(n_eslot_all * sizeof(double)));
  if (lj_on) CK(h->eblk_lj.ensure(n_eslot_all * sizeof(double)));
  if (rows_slab <= 0) {
    if (pair_coul) CK(cudaMemsetAsync(d_u_out, 0, sizeof(double), h->stream));
    if (lj_on && d_ulj_out) CK(cudaMemsetAsync(d_ulj_out, 0, sizeof(double), h->stream));
    return EWB_OK;
  }
  CK(h->pairc.ensure(sizeof(unsigned long long)));
  if (part == 0) CK(cudaMemsetAsync(h->pairc.p, 0, sizeof(unsigned long long), h->stream));
  // cell-sorted force accumulator, un-permuted afterwards; in FOLD mode the
  // sorted order is the caller's, so the pair kernel adds into d_force
  // directly (the reciprocal forces are combined after the join)
  double *facc = d_force;
  if (!fold) {
    CK(h->fsorted.ensure((size_t)n * 3 * sizeof(double)));
    CK(cudaMemsetAsync(h->fsorted.p, 0, (size_t)n * 3 * sizeof(double), h->stream));
    facc = h->fsorted.as<double>();
  }
  {
    K6Lists lists{split ? h->rs_list.as<uint32_t>() : nullptr,
                  split ? h->rs_count.as<int>() : nullptr, cap};
    double *eb = h->eblk.as<double>();
    double *eb_lj = lj_on ? h->eblk_lj.as<double>() : nullptr;
    if (!split) {
      // more resident warps pay off only when the grid spans several waves
      const bool hi = active * rp.jsplit >= (int64_t)K6_HI_WAVES * h->n_sm * K6_MINB_HI * K6_WARPS;
      auto kern = hi ? (lj_on ? (rp.half ? k6_real_space<true, true, K6_MODE_FUSED_HI>
                                         : k6_real_space<true, false, K6_MODE_FUSED_HI>)
                              : (rp.half ? k6_real_space<false, true, K6_MODE_FUSED_HI>
                                         : k6_real_space<false, false, K6_MODE_FUSED_HI>))
                     : (lj_on ? (rp.half ? k6_real_space<true, true, K6_MODE_FUSED>
                                         : k6_real_space<true, false, K6_MODE_FUSED>)
                              : (rp.half ? k6_real_space<false, true, K6_MODE_FUSED>
                                         : k6_real_space<false, false, K6_MODE_FUSED>));
      kern<<<nb, K6_WARPS * 32, 0, h->stream>>>(
          h->sorted.as<double4>(), h->sorted_f.as<float4>(), h->sorted_cell.as<int>(),
          h->order.as<int>(), h->start.as<int>(), h->row_ustart.as<int>(), rp,
          facc, eb, eb_lj, h->errflag.as<int>(),
          h->pairc.as<unsigned long long>(), lists);
      CKL();
    } else {
      // pass 1: traversal -> per-unit pair lists (the LJ switch only
      // changes the evaluation; the traversal cutoff is in rp.rc2)
      auto trav = rp.half ? k6_real_space<false, true, K6_MODE_LIST>
                          : k6_real_space<false, false, K6_MODE_LIST>;
      trav<<<nb, K6_WARPS * 32, 0, h->stream>>>(
          h->sorted.as<double4>(), h->sorted_f.as<float4>(), h->sorted_cell.as<int>(),
          h->order.as<int>(), h->start.as<int>(), h->row_ustart.as<int>(), rp,
          facc, nullptr, nullptr, h->errflag.as<int>(),
          h->pairc.as<unsigned long long>(), lists);
      CKL();
      // pass 2: evaluation of the lists
      auto ev = lj_on ? (rp.half ? k6b_eval<true, true> : k6b_eval<true, false>)
                      : (rp.half ? k6b_eval<false, true> : k6b_eval<false, false>);
      ev<<<nb, K6_WARPS * 32, 0, h->stream>>>(h->sorted.as<double4>(), h->start.as<int>(),
                                              h->row_ustart.as<int>(), rp, lists,
                                              facc, eb, eb_lj,
                                              h->errflag.as<int>());
      CKL();
      // overflowed units (list longer than its capacity): fused kernel,
      // other units exit at once; energies into the second slot range
      auto ovf = lj_on ? (rp.half ? k6_real_space<true, true, K6_MODE_OVF>
                                  : k6_real_space<true, false, K6_MODE_OVF>)
                       : (rp.half ? k6_real_space<false, true, K6_MODE_OVF>
                                  : k6_real_space<false, false, K6_MODE_OVF>);
      ovf<<<nb, K6_WARPS * 32, 0, h->stream>>>(
          h->sorted.as<double4>(), h->sorted_f.as<float4>(), h->sorted_cell.as<int>(),
          h->order.as<int>(), h->start.as<int>(), h->row_ustart.as<int>(), rp,
          facc, eb + n_eslots, eb_lj ? eb_lj + n_eslots : nullptr,
          h->errflag.as<int>(), nullptr, lists);
      CKL();
    }
  }
  if (!fold) {
    k_unpermute_add<<<blocks_for(n, 256), 256, 0, h->stream>>>(h->order.as<int>(),
                                                               h->fsorted.as<double>(), n, d_force);
    CKL();
  }
  if (pair_coul) {
    k_sum<<<1, 1024, 0, h->stream>>>(h->eblk.as<double>(), n_eslot_all, 1.0, d_u_out);
    CKL();
  }
  if (lj_on && d_ulj_out) {
    k_sum<<<1, 1024, 0, h->stream>>>(h->eblk_lj.as<double>(), n_eslot_all, 1.0, d_ulj_out);
    CKL();
  }
  return EWB_OK;
}

int stage_self(ewb_handle *h, double *d_u_out, int64_t i0 = 0, int64_t i1 = -1) {
  if (i1 < 0) i1 = h->n;
  const int64_t cnt = i1 - i0;
  const unsigned nb = (unsigned)std::max<int64_t>(1, std::min<int64_t>(1024, blocks_for(cnt, RED_THREADS)));
  CK(h->eblk2.ensure(std::max<size_t>(nb, 1) * sizeof(double)));
  k7_sum_q2<<<nb, RED_THREADS, 0, h->stream>>>(h->frac.as<double4>() + i0, cnt, h->eblk2.as<double>());
  CKL();
  k_sum<<<1, 1024, 0, h->stream>>>(h->eblk2.as<double>(), nb, -std::sqrt(h->alpha / M_PI), d_u_out);
  CKL();
  return EWB_OK;
}

// device error bits a completed evaluation reports: the wide-cutoff (image
// shell) real space accepts unwrapped positions, as the reference's
// short_range_wide_cutoff does (ewald.py:553-576)
int err_mask(const ewb_handle *h) {
  return ((h->coul_on && h->rc > 0.5 * h->L && !h->lj_on) ? 0 : ERR_UNWRAPPED) | ERR_COINCIDENT;
}

int check_errflag(ewb_handle *h, int mask) {
  int e = 0;
  CK(cudaMemcpyAsync(&e, h->errflag.p, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  e &= mask;
  if (e & ERR_UNWRAPPED)
    return h->fail(EWB_EUNWRAPPED, "positions must be wrapped into [0, L) before binning");
  if (e & ERR_COINCIDENT)
    return h->fail(EWB_ECOINCIDENT, "coincident particles in Coulomb kernel");
  return EWB_OK;
}

int h2d_particles(ewb_handle *h, const double *pos, const double *q, int64_t n) {
  if (!pos || !q) return h->fail(EWB_EINVAL, "null particle arrays");
  CK(h->pos.ensure(n * 3 * sizeof(double)));
  CK(h->q.ensure(n * sizeof(double)));
  CK(cudaMemcpyAsync(h->pos.p, pos, n * 3 * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  CK(cudaMemcpyAsync(h->q.p, q, n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  return stage_load(h, h->pos.as<double>(), h->q.as<double>(), n);
}

int h2d_force(ewb_handle *h, const double *force, int64_t n) {
  CK(h->force.ensure(n * 3 * sizeof(double)));
  CK(cudaMemcpyAsync(h->force.p, force, n * 3 * sizeof(double), cudaMemcpyHostToDevice,
                     h->stream));
  return EWB_OK;
}

// full single-GPU pipeline on loaded particles; energies stay on device
// evaluation pipeline in five segments; timing events sit between them
// (outside any captured graph): ev0 | cells | ev1 | pairs | ev2 | S(k) |
// ev3 | forces + self | ev4
// N_SEG (pipeline segments) is defined with the handle
int pipeline_seg(ewb_handle *h, int seg, const double *d_pos, const double *d_q, int64_t n,
                 double *d_force, double *d_rho_out) {
  int rc;
  double *en = h->energy.as<double>();
  switch (seg) {
    case 0:
      return stage_load(h, d_pos, d_q, n);
    case 1:
      return stage_real_space(h, 0, 1, d_force, en + 0, nullptr, RS_CELLS);
    case 2:
      return stage_real_space(h, 0, 1, d_force, en + 0, nullptr, RS_PAIRS, en + 3);
    case 3: {
      if (!h->coul_on) {
        CK(cudaMemsetAsync(en + 1, 0, sizeof(double), h->stream));
        return EWB_OK;
      }
      int n_part = 0;
      if ((rc = stage_rho(h, 0, h->n, &n_part))) return rc;
      return stage_finalize_pairs(h, h->spart.as<double4>(), n_part, d_rho_out, en + 1);
    }
    case 4:
      if (!h->coul_on) {
        CK(cudaMemsetAsync(en + 2, 0, sizeof(double), h->stream));
        return EWB_OK;
      }
      if ((rc = stage_recip_forces(h, 0, h->n, d_force, false, nullptr))) return rc;
      // self energy (depends on q only): on the reciprocal stream, before the
      // join, so it stays off the tail of the evaluation
      return stage_self(h, en + 2);
    default:
      if (h->coul_on && h->ov_active && h->t3_pend_nks > 0) {
        const unsigned nbc = blocks_for(h->t3_pend_n, RED_THREADS);
        k3_combine<<<nbc, RED_THREADS, 0, h->stream>>>(
            h->fpart.as<double>(), nullptr, h->t3_pend_nks, h->t3_pend_i0, h->t3_pend_n,
            h->frac.as<double4>(), 4.0 * M_PI / h->L, h->t3_pend_force, nullptr, 0);
        CKL();
      }
      return EWB_OK;
  }
}

// prep + pipeline; segments are replayed from CUDA graphs when the key
// (pointers, size, configuration, buffer epoch) is unchanged
int run_eval(ewb_handle *h, const double *d_pos, const double *d_q, int64_t n, double *d_force,
             double *d_rho, bool timed) {
  CK(h->energy.ensure(8 * sizeof(double)));
  ewb_handle::GKey k;
  k.pos = d_pos;
  k.q = d_q;
  k.force = d_force;
  k.rho = d_rho;
  k.n = n;
  k.timed = false;  // events live outside the graphs
  k.gen = h->gen;
  k.epoch = g_realloc_epoch;
  const bool replay = h->use_graphs && h->gexec[0] && k == h->gkey;
  const bool capture = !replay && h->use_graphs && k == h->warm_key;
  const int64_t l0 = h->launches;
  int rc = EWB_OK;
  bool captured_all = capture;
  // reciprocal space (segments 3, 4) on its own stream, concurrently with
  // real space (1, 2): its kernels touch neither the forces nor the
  // real-space scratch; the force combine waits for the join in segment 5
  struct OvGuard {  // the stage APIs must never see a deferred combine
    ewb_handle *h;
    ~OvGuard() { h->ov_active = false; }
  } ov_guard{h};
  h->ov_active = h->overlap && h->coul_on && !h->lj_on;
  h->t3_pend_nks = 0;
  cudaStream_t main_stream = h->stream;
  for (int seg = 0; seg < N_SEG; ++seg) {
    const bool on_r = h->ov_active && (seg == 3 || seg == 4);
    cudaStream_t st = on_r ? h->rstream : main_stream;
    if (h->ov_active && seg == 1) {
      CK(cudaEventRecord(h->ev_rfork, main_stream));
      CK(cudaStreamWaitEvent(h->rstream, h->ev_rfork, 0));
    }
    if (h->ov_active && seg == 5) {
      if (timed) CK(cudaEventRecord(h->ev[2], main_stream));  // after the pairs, before the join
      CK(cudaEventRecord(h->ev_rjoin, h->rstream));
      CK(cudaStreamWaitEvent(main_stream, h->ev_rjoin, 0));
    }
    // timing events: 0 | cells | 1 | pairs | 2   3 | S(k) | 4 | forces | 5
    if (timed) {
      if (seg == 1) CK(cudaEventRecord(h->ev[0], st));
      if (seg == 2) CK(cudaEventRecord(h->ev[1], st));
      if (seg == 3) {
        if (!h->ov_active) CK(cudaEventRecord(h->ev[2], st));
        CK(cudaEventRecord(h->ev[3], st));
      }
      if (seg == 4) CK(cudaEventRecord(h->ev[4], st));
    }
    if (seg == 2 && h->fup_pending) {  // forces are first touched by the pair segment
      CK(cudaStreamWaitEvent(st, h->ev_fup, 0));
      h->fup_pending = false;
    }
    if (seg == 4 && h->rho_host && d_rho) {  // rho is final after segment 3
      CK(cudaEventRecord(h->ev_rho, on_r ? h->rstream : main_stream));
      CK(cudaStreamWaitEvent(h->cstream, h->ev_rho, 0));
      CK(cudaMemcpyAsync(h->rho_host, d_rho, 2 * h->plan.K * sizeof(double),
                         cudaMemcpyDeviceToHost, h->cstream));
      CK(cudaEventRecord(h->ev_rhodone, h->cstream));
    }
    h->stream = st;
    if (replay) {
      cudaError_t e = cudaGraphLaunch(h->gexec[seg], st);
      h->stream = main_stream;
      CK(e);
      if (timed && seg == 4) CK(cudaEventRecord(h->ev[5], st));
      continue;
    }
    if (capture && captured_all) {
      cudaError_t eb = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
      if (eb != cudaSuccess) {
        h->stream = main_stream;
        CK(eb);
      }
      const int64_t s0 = h->launches;
      rc = pipeline_seg(h, seg, d_pos, d_q, n, d_force, d_rho);
      cudaGraph_t g = nullptr;
      const cudaError_t e = cudaStreamEndCapture(st, &g);
      if (rc) {
        h->stream = main_stream;
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      if (e == cudaSuccess && k.epoch == g_realloc_epoch) {
        if (h->gexec[seg]) cudaGraphExecDestroy(h->gexec[seg]);
        h->gexec[seg] = nullptr;
        const cudaError_t ei = cudaGraphInstantiate(&h->gexec[seg], g, 0);
        cudaGraphDestroy(g);
        h->glaunch[seg] = h->launches - s0;
        const cudaError_t el = ei == cudaSuccess ? cudaGraphLaunch(h->gexec[seg], st) : ei;
        h->stream = main_stream;
        CK(el);
        if (timed && seg == 4) CK(cudaEventRecord(h->ev[5], st));
        continue;
      }
      // capture failed (or a buffer moved): finish this call eagerly
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      captured_all = false;
      h->launches = s0;
    }
    rc = pipeline_seg(h, seg, d_pos, d_q, n, d_force, d_rho);
    h->stream = main_stream;
    if (rc) return rc;
    if (timed && seg == 4) CK(cudaEventRecord(h->ev[5], st));
  }
  h->stream = main_stream;
  if (replay) {
    for (int seg = 0; seg < N_SEG; ++seg) h->launches += h->glaunch[seg];
    h->n = n;
    h->loaded = true;
  } else if (capture && captured_all) {
    h->gkey = k;
  } else {
    if (!capture) {
      k.epoch = g_realloc_epoch;  // the first call may have grown buffers
      h->warm_key = k;
    } else {
      h->warm_key = ewb_handle::GKey();
    }
    (void)l0;
  }
  return EWB_OK;
}

__global__ void k_rho_to_slots(const double *__restrict__ rho, int64_t K,
                               const int *__restrict__ slot_k, int64_t n_slots,
                               double2 *__restrict__ out) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n_slots) return;
  const int k = slot_k[s];
  out[s] = k >= 0 ? make_double2(rho[k], rho[K + k]) : make_double2(0.0, 0.0);
}

// rho (caller order, h->rho) -> slot layout (h->sslot)
int stage_rho_to_slots(ewb_handle *h) {
  const int64_t n_slots = (int64_t)h->plan.M * h->plan.n_items;
  k_rho_to_slots<<<blocks_for(n_slots, 256), 256, 0, h->stream>>>(
      h->rho.as<double>(), h->plan.K, h->plan.slot_k.as<int>(), n_slots, h->sslot.as<double2>());
  CKL();
  return EWB_OK;
}

int read_timings(ewb_handle *h, double *timings) {
  if (!timings) return EWB_OK;
  float a = 0, b = 0, c = 0, d = 0;
  CK(cudaEventSynchronize(h->ev[5]));
  CK(cudaEventSynchronize(h->ev[2]));
  CK(cudaEventElapsedTime(&a, h->ev[0], h->ev[1]));
  CK(cudaEventElapsedTime(&b, h->ev[0], h->ev[2]));
  CK(cudaEventElapsedTime(&c, h->ev[3], h->ev[4]));
  CK(cudaEventElapsedTime(&d, h->ev[4], h->ev[5]));
  timings[0] = a * 1e-3;
  timings[1] = b * 1e-3;
  timings[2] = c * 1e-3;
  timings[3] = d * 1e-3;
  return EWB_OK;
}

}  // namespace

// ===========================================================================
// C-ABI
extern "C" {

int ewb_version(void) { return EWB_VERSION; }

int ewb_create(int device, ewb_handle **out) {
  if (!out) return EWB_EINVAL;
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) return EWB_ECUDA;
  if (device < 0 || device >= ndev) return EWB_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return EWB_ECUDA;
  ewb_handle *h = new ewb_handle();
  h->device = device;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) h->n_sm = prop.multiProcessorCount;
  if (cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete h;
    return EWB_ECUDA;
  }
  h->stream = h->own_stream;
#ifdef EWB_TC_DBG
  h->tc_dbg = EWB_TC_DBG;  // component-timing builds only (tools/tc_dbg.sh)
#endif
  if (cudaStreamCreateWithFlags(&h->aux_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&h->rstream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_fup, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_rho, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_rhodone, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_rfork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_rjoin, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess) {
    delete h;
    return EWB_ECUDA;
  }
  for (auto &ev : h->ev)
    if (cudaEventCreate(&ev) != cudaSuccess) {
      delete h;
      return EWB_ECUDA;
    }
  *out = h;
  return EWB_OK;
}

void ewb_destroy(ewb_handle *h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (DBuf *b : {&h->pos, &h->q, &h->force, &h->rho, &h->frac, &h->base, &h->xyzq, &h->spart,
                  &h->sslot, &h->sp, &h->fpart, &h->upart, &h->eblk, &h->eblk2, &h->eblk_lj,
                  &h->energy,
                  &h->errflag, &h->cell_of, &h->slot, &h->count, &h->start, &h->gstart,
                  &h->order_tmp, &h->order, &h->sorted, &h->sorted_cell, &h->row_ustart,
                  &h->sorted_f, &h->tc_qmax, &h->tc_ytab, &h->tc_ztab, &h->tc_xsl, &h->t3_wsl,
                  &h->t3_rscale, &h->pairc, &h->eblk_r, &h->fsorted, &h->force_in,
                  &h->rs_list, &h->rs_count})
    b->release();
  if (h->hscr) cudaFreeHost(h->hscr);
  h->plan.release();
  for (auto &ge : h->gexec)
    if (ge) cudaGraphExecDestroy(ge);
  for (auto &ev : h->ev)
    if (ev) cudaEventDestroy(ev);
  if (h->ev_fup) cudaEventDestroy(h->ev_fup);
  if (h->ev_rho) cudaEventDestroy(h->ev_rho);
  if (h->ev_rhodone) cudaEventDestroy(h->ev_rhodone);
  if (h->cstream) cudaStreamDestroy(h->cstream);
  if (h->ev_rfork) cudaEventDestroy(h->ev_rfork);
  if (h->ev_rjoin) cudaEventDestroy(h->ev_rjoin);
  if (h->rstream) cudaStreamDestroy(h->rstream);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->aux_stream) cudaStreamDestroy(h->aux_stream);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  delete h;
}

const char *ewb_last_error(const ewb_handle *h) { return h ? h->err.c_str() : "null handle"; }

int ewb_set_stream(ewb_handle *h, uintptr_t stream) {
  if (!h) return EWB_EINVAL;
  ++h->gen;
  // 0 is the legacy default stream (torch's default stream), as for any
  // CUDA API; ewb_use_own_stream rebinds the handle's own stream
  h->stream = reinterpret_cast<cudaStream_t>(stream);
  return EWB_OK;
}

int ewb_use_own_stream(ewb_handle *h) {
  if (!h) return EWB_EINVAL;
  ++h->gen;
  h->stream = h->own_stream;
  return EWB_OK;
}

int ewb_set_max_pair_segment(ewb_handle *h, int mcap1) {
  if (!h) return EWB_EINVAL;
  ++h->gen;
  if (mcap1 < 1 || mcap1 > MAXM1) return h->fail(EWB_EINVAL, "pair segment length must be in [1, 20]");
  h->mcap1 = mcap1;
  return EWB_OK;
}

int ewb_set_max_segment(ewb_handle *h, int mcap) {
  if (!h) return EWB_EINVAL;
  ++h->gen;
  if (mcap < 1 || mcap > MAXM) return h->fail(EWB_EINVAL, "segment length must be in [1, 32]");
  h->mcap = mcap;
  return EWB_OK;
}

int ewb_set_stencil(ewb_handle *h, int rad) {
  if (!h) return EWB_EINVAL;
  ++h->gen;
  if (rad < 0 || rad > 2) return h->fail(EWB_EINVAL, "stencil radius must be 0 (auto), 1 or 2");
  h->stencil_rad = rad;
  return EWB_OK;
}

int ewb_set_coulomb(ewb_handle *h, int on) {
  if (!h) return EWB_EINVAL;
  h->coul_on = on != 0;
  ++h->gen;
  return EWB_OK;
}

int ewb_set_lj(ewb_handle *h, int on, double sigma2, double four_eps, double shift,
               double tf_eps, double rc_lj, double rc2_lj) {
  if (!h) return EWB_EINVAL;
  ++h->gen;
  if (on && !(rc_lj > 0.0)) return h->fail(EWB_EINVAL, "cutoff must be positive");
  h->lj_on = on != 0;
  h->lj_s2 = sigma2;
  h->lj_4e = four_eps;
  h->lj_shift = shift;
  h->lj_24e = tf_eps;
  h->rc_lj = rc_lj;
  h->rc2_lj = rc2_lj;
  return EWB_OK;
}

int ewb_last_energies(ewb_handle *h, double *out4) {
  if (!h || !out4) return EWB_EINVAL;
  CK(cudaSetDevice(h->device));
  CK(h->energy.ensure(8 * sizeof(double)));
  CK(cudaMemcpyAsync(out4, h->energy.p, 4 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return EWB_OK;
}

int ewb_dev_md_kick_drift(ewb_handle *h, double *d_pos, double *d_vel, const double *d_force,
                          const double *d_mass, int64_t n, double dt) {
  int rc = require_state(h, false, false);
  if (rc) return rc;
  if (n < 1) return h->fail(EWB_EINVAL, "particle count must be >= 1");
  CK(cudaSetDevice(h->device));
  k_md_kick_drift<<<blocks_for(n, 256), 256, 0, h->stream>>>(d_pos, d_vel, d_force, d_mass, n,
                                                             dt, h->L);
  CKL();
  return EWB_OK;
}

int ewb_dev_md_kick(ewb_handle *h, double *d_vel, const double *d_force, const double *d_mass,
                    int64_t n, double dt, int kick, double *kinetic) {
  if (!h) return EWB_EINVAL;
  if (n < 1) return h->fail(EWB_EINVAL, "particle count must be >= 1");
  CK(cudaSetDevice(h->device));
  const unsigned nb = blocks_for(n, RED_THREADS);
  CK(h->eblk2.ensure(nb * sizeof(double)));
  CK(h->energy.ensure(8 * sizeof(double)));
  k_md_kick<<<nb, RED_THREADS, 0, h->stream>>>(d_vel, d_force, d_mass, n, dt, kick ? 1 : 0,
                                               h->eblk2.as<double>());
  CKL();
  k_sum<<<1, 1024, 0, h->stream>>>(h->eblk2.as<double>(), nb, 0.5, h->energy.as<double>() + 4);
  CKL();
  if (kinetic) {
    CK(cudaMemcpyAsync(kinetic, h->energy.as<double>() + 4, sizeof(double), cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaStreamSynchronize(h->stream));
  }
  return EWB_OK;
}

int ewb_set_const_gather(ewb_handle *h, int on) {
  if (!h) return EWB_EINVAL;
  h->k3_const = on ? 1 : 0;
  ++h->gen;
  return EWB_OK;
}

int ewb_set_tensor_cores(ewb_handle *h, int on) {
  if (!h) return EWB_EINVAL;
  if (on < 0 || on > 2) return h->fail(EWB_EINVAL, "tensor-core mode must be 0, 1 or 2");
  h->use_tc = on;
  ++h->gen;
  return EWB_OK;
}

int ewb_set_overlap(ewb_handle *h, int on) {
  if (!h) return EWB_EINVAL;
  h->overlap = on ? 1 : 0;
  ++h->gen;
  return EWB_OK;
}

int ewb_set_graphs(ewb_handle *h, int on) {
  if (!h) return EWB_EINVAL;
  h->use_graphs = on != 0;
  ++h->gen;
  return EWB_OK;
}

int ewb_set_real_space_split(ewb_handle *h, int on) {
  if (!h) return EWB_EINVAL;
  ++h->gen;
  h->rs_split = on < 0 ? 0 : (on > 2 ? 2 : on);
  return EWB_OK;
}

int ewb_set_deterministic(ewb_handle *h, int on) {
  if (!h) return EWB_EINVAL;
  ++h->gen;
  h->deterministic = on ? 1 : 0;
  return EWB_OK;
}

int ewb_set_system(ewb_handle *h, double L, double alpha, double r_cutoff, double rc2) {
  if (!h) return EWB_EINVAL;
  if (!(L > 0.0) || !std::isfinite(L)) return h->fail(EWB_EINVAL, "box edge length must be positive");
  if (!(alpha > 0.0) || !std::isfinite(alpha)) return h->fail(EWB_EINVAL, "alpha must be positive");
  h->L = L;
  h->alpha = alpha;
  h->rc = r_cutoff;
  h->rc2 = rc2;
  h->have_system = true;
  ++h->gen;
  return EWB_OK;
}

int ewb_set_kspace(ewb_handle *h, const int64_t *m_int, int64_t K, const double *coeff) {
  if (!h) return EWB_EINVAL;
  if (!m_int && K > 0) return h->fail(EWB_EINVAL, "null m_int");
  CK(cudaSetDevice(h->device));
  int rc = build_plan(h, m_int, K, coeff);
  ++h->gen;
  if (rc) return rc;
  h->have_kspace = true;
  return EWB_OK;
}

int ewb_kspace_info(const ewb_handle *h, int64_t *info8) {
  if (!h || !info8) return EWB_EINVAL;
  info8[0] = h->plan.K;
  info8[1] = h->plan.n_items;
  info8[2] = h->plan.M;
  info8[3] = h->plan.n_rows;
  info8[4] = h->plan.n_tiles;
  info8[5] = h->plan.ts_max;
  info8[6] = h->plan.n_pitems;
  info8[7] = h->plan.M1;
  return EWB_OK;
}

int ewb_compute_rho_hat(ewb_handle *h, const double *pos, const double *q, int64_t n,
                        double *rho_out) {
  int rc = require_state(h, true, false);
  if (rc) return rc;
  CK(cudaSetDevice(h->device));
  if ((rc = h2d_particles(h, pos, q, n))) return rc;
  CK(h->rho.ensure(2 * h->plan.K * sizeof(double)));
  CK(h->energy.ensure(8 * sizeof(double)));
  int n_part = 0;
  if ((rc = stage_rho(h, 0, n, &n_part))) return rc;
  if ((rc = stage_finalize_pairs(h, h->spart.as<double4>(), n_part, h->rho.as<double>(),
                                 h->energy.as<double>() + 1)))
    return rc;
  CK(cudaMemcpyAsync(rho_out, h->rho.p, 2 * h->plan.K * sizeof(double), cudaMemcpyDeviceToHost,
                     h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return EWB_OK;
}

int ewb_long_range(ewb_handle *h, const double *pos, const double *q, int64_t n, const double *rho,
                   double *force_inout, double *u_lr) {
  int rc = require_state(h, true, false);
  if (rc) return rc;
  CK(cudaSetDevice(h->device));
  if ((rc = h2d_particles(h, pos, q, n))) return rc;
  if ((rc = h2d_force(h, force_inout, n))) return rc;
  // rho given by the caller (any values): scatter it into slot layout
  const int64_t K = h->plan.K;
  const int64_t n_slots = (int64_t)h->plan.M * h->plan.n_items;
  CK(h->rho.ensure(2 * K * sizeof(double)));
  CK(h->sslot.ensure(n_slots * sizeof(double2)));
  CK(h->energy.ensure(8 * sizeof(double)));
  CK(cudaMemcpyAsync(h->rho.p, rho, 2 * K * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  if ((rc = stage_rho_to_slots(h))) return rc;
  if ((rc = stage_finalize(h, h->sslot.as<double2>(), 1, nullptr, h->energy.as<double>() + 7)))
    return rc;
  if ((rc = stage_recip_forces(h, 0, n, h->force.as<double>(), true, h->energy.as<double>() + 1)))
    return rc;
  double u = 0.0;
  CK(cudaMemcpyAsync(&u, h->energy.as<double>() + 1, sizeof(double), cudaMemcpyDeviceToHost,
                     h->stream));
  CK(cudaMemcpyAsync(force_inout, h->force.p, n * 3 * sizeof(double), cudaMemcpyDeviceToHost,
                     h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (u_lr) *u_lr = u;
  return EWB_OK;
}

int ewb_short_range(ewb_handle *h, const double *pos, const double *q, int64_t n,
                    double *force_inout, double *u_sr) {
  int rc = require_state(h, false, false);
  if (rc) return rc;
  CK(cudaSetDevice(h->device));
  if (!(h->rc > 0.0)) return h->fail(EWB_EINVAL, "cutoff must be positive");
  if (h->rc > 0.5 * h->L)
    return h->fail(EWB_ECUTOFF, "cutoff exceeds L/2 (minimum-image bound)");
  if ((rc = h2d_particles(h, pos, q, n))) return rc;
  if ((rc = check_errflag(h, ERR_UNWRAPPED))) return rc;
  if ((rc = h2d_force(h, force_inout, n))) return rc;
  CK(h->energy.ensure(8 * sizeof(double)));
  if ((rc = stage_real_space(h, 0, 1, h->force.as<double>(), h->energy.as<double>(), nullptr)))
    return rc;
  double u = 0.0;
  CK(cudaMemcpyAsync(&u, h->energy.as<double>(), sizeof(double), cudaMemcpyDeviceToHost,
                     h->stream));
  if ((rc = check_errflag(h, ERR_COINCIDENT))) return rc;
  CK(cudaMemcpy(force_inout, h->force.p, n * 3 * sizeof(double), cudaMemcpyDeviceToHost));
  if (u_sr) *u_sr = u;
  return EWB_OK;
}

int ewb_self_energy(ewb_handle *h, const double *q, int64_t n, double *u_self) {
  int rc = require_state(h, false, false);
  if (rc) return rc;
  CK(cudaSetDevice(h->device));
  if (n < 1) return h->fail(EWB_EINVAL, "particle count must be >= 1");
  CK(h->q.ensure(n * sizeof(double)));
  CK(h->pos.ensure(n * 3 * sizeof(double)));
  CK(cudaMemcpyAsync(h->q.p, q, n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  CK(cudaMemsetAsync(h->pos.p, 0, n * 3 * sizeof(double), h->stream));
  if ((rc = stage_load(h, h->pos.as<double>(), h->q.as<double>(), n))) return rc;
  CK(h->energy.ensure(8 * sizeof(double)));
  if ((rc = stage_self(h, h->energy.as<double>() + 2))) return rc;
  double u = 0.0;
  CK(cudaMemcpyAsync(&u, h->energy.as<double>() + 2, sizeof(double), cudaMemcpyDeviceToHost,
                     h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (u_self) *u_self = u;
  return EWB_OK;
}

int ewb_evaluate(ewb_handle *h, const double *pos, const double *q, int64_t n,
                 double *force_inout, double *rho_out, double *energies, double *timings) {
  int rc = require_state(h, h && h->coul_on, false);
  if (rc) return rc;
  CK(cudaSetDevice(h->device));
  if (h->coul_on && !(h->rc > 0.0)) return h->fail(EWB_EINVAL, "cutoff must be positive");
  if (!pos || !q) return h->fail(EWB_EINVAL, "null particle arrays");
  if (n < 1) return h->fail(EWB_EINVAL, "particle count must be >= 1");
  CK(h->pos.ensure(n * 3 * sizeof(double)));
  CK(h->q.ensure(n * sizeof(double)));
  CK(h->force.ensure(n * 3 * sizeof(double)));
  if (rho_out && h->coul_on) CK(h->rho.ensure(2 * h->plan.K * sizeof(double)));
  if (!h->coul_on) rho_out = nullptr;
  CK(cudaMemcpyAsync(h->pos.p, pos, n * 3 * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  CK(cudaMemcpyAsync(h->q.p, q, n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  // the force upload overlaps the set-up and cell build (waited for before
  // the pair segment); the previous call's result copies must be done
  CK(cudaEventRecord(h->ev_fup, h->stream));
  CK(cudaStreamWaitEvent(h->cstream, h->ev_fup, 0));
  CK(cudaMemcpyAsync(h->force.p, force_inout, n * 3 * sizeof(double), cudaMemcpyHostToDevice,
                     h->cstream));
  // kept so that an error detected after the pipeline can restore the
  // caller's array (the result is copied out before the flag is read)
  CK(h->force_in.ensure(n * 3 * sizeof(double)));
  CK(cudaMemcpyAsync(h->force_in.p, h->force.p, n * 3 * sizeof(double), cudaMemcpyDeviceToDevice,
                     h->cstream));
  CK(cudaEventRecord(h->ev_fup, h->cstream));
  h->fup_pending = true;
  h->rho_host = rho_out;
  rc = run_eval(h, h->pos.as<double>(), h->q.as<double>(), n, h->force.as<double>(),
                rho_out ? h->rho.as<double>() : nullptr, true);
  h->rho_host = nullptr;
  if (h->fup_pending) {  // (not consumed: make the main stream depend on it anyway)
    CK(cudaStreamWaitEvent(h->stream, h->ev_fup, 0));
    h->fup_pending = false;
  }
  if (rc) {
    cudaStreamSynchronize(h->cstream);
    return rc;
  }
  // one synchronisation: energies, error flag and forces are copied out
  // together; on a device-side error the caller's forces are restored
  if (!h->hscr) CK(cudaHostAlloc(&h->hscr, 4 * sizeof(double), cudaHostAllocPortable));
  CK(cudaMemcpyAsync(h->hscr, h->energy.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaMemcpyAsync(h->hscr + 3, h->errflag.p, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaMemcpyAsync(force_inout, h->force.p, n * 3 * sizeof(double), cudaMemcpyDeviceToHost,
                     h->stream));
  CK(cudaStreamSynchronize(h->stream));
  CK(cudaStreamSynchronize(h->cstream));  // rho (copied after segment 3)
  int e = 0;
  std::memcpy(&e, h->hscr + 3, sizeof(int));
  e &= err_mask(h);
  if (e) {
    CK(cudaMemcpy(force_inout, h->force_in.p, n * 3 * sizeof(double), cudaMemcpyDeviceToHost));
    if (e & ERR_UNWRAPPED)
      return h->fail(EWB_EUNWRAPPED, "positions must be wrapped into [0, L) before binning");
    return h->fail(EWB_ECOINCIDENT, "coincident particles in Coulomb kernel");
  }
  if (energies) std::memcpy(energies, h->hscr, 3 * sizeof(double));
  return read_timings(h, timings);
}

// ---- device-pointer stages ----
int ewb_dev_load(ewb_handle *h, const double *d_pos, const double *d_q, int64_t n) {
  int rc = require_state(h, false, false);
  if (rc) return rc;
  CK(cudaSetDevice(h->device));
  return stage_load(h, d_pos, d_q, n);
}

int64_t ewb_dev_slot_doubles(const ewb_handle *h) {
  if (!h || !h->have_kspace) return -1;
  return 4 * (int64_t)h->plan.M1 * h->plan.n_pitems;
}

int ewb_dev_rho_partial(ewb_handle *h, int64_t i0, int64_t i1, double *d_slots) {
  int rc = require_state(h, true, true);
  if (rc) return rc;
  if (i0 < 0 || i1 > h->n || i0 > i1) return h->fail(EWB_EINVAL, "bad particle range");
  CK(cudaSetDevice(h->device));
  const int64_t n_pslots = (int64_t)h->plan.M1 * h->plan.n_pitems;
  if (i1 == i0) {
    CK(cudaMemsetAsync(d_slots, 0, n_pslots * sizeof(double4), h->stream));
    return EWB_OK;
  }
  int n_part = 0;
  if ((rc = stage_rho(h, i0, i1, &n_part))) return rc;
  const unsigned nb = blocks_for(n_pslots, RED_THREADS);
  k2p_finalize<<<nb, RED_THREADS, 0, h->stream>>>(h->spart.as<double4>(), n_part, n_pslots,
                                                  nullptr, nullptr, h->plan.K, nullptr,
                                                  reinterpret_cast<double4 *>(d_slots), nullptr,
                                                  nullptr, 0);
  CKL();
  return EWB_OK;
}

int ewb_dev_kspace_finalize(ewb_handle *h, const double *d_slots, double *d_rho_out, double *u_lr) {
  int rc = require_state(h, true, false);
  if (rc) return rc;
  CK(cudaSetDevice(h->device));
  CK(h->energy.ensure(8 * sizeof(double)));
  if ((rc = stage_finalize_pairs(h, reinterpret_cast<const double4 *>(d_slots), 1, d_rho_out,
                                 h->energy.as<double>() + 1)))
    return rc;
  if (u_lr) {
    CK(cudaMemcpyAsync(u_lr, h->energy.as<double>() + 1, sizeof(double), cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaStreamSynchronize(h->stream));
  }
  return EWB_OK;
}

int ewb_dev_recip_forces(ewb_handle *h, int64_t i0, int64_t i1, double *d_force) {
  int rc = require_state(h, true, true);
  if (rc) return rc;
  if (i0 < 0 || i1 > h->n || i0 > i1) return h->fail(EWB_EINVAL, "bad particle range");
  CK(cudaSetDevice(h->device));
  return stage_recip_forces(h, i0, i1, d_force, false, nullptr);
}

int ewb_dev_real_space(ewb_handle *h, int part, int nparts, double *d_force, double *u_sr) {
  int rc = require_state(h, false, true);
  if (rc) return rc;
  if (nparts < 1 || part < 0 || part >= nparts) return h->fail(EWB_EINVAL, "bad slab index");
  CK(cudaSetDevice(h->device));
  // u_sr == NULL: asynchronous (binning clamps cell indices, so unwrapped
  // input is memory-safe); u_sr stays in the device energy slot and errors
  // are reported by ewb_dev_check
  if (u_sr && (rc = check_errflag(h, ERR_UNWRAPPED))) return rc;
  CK(h->energy.ensure(8 * sizeof(double)));
  if ((rc = stage_real_space(h, part, nparts, d_force, h->energy.as<double>(), nullptr))) return rc;
  if (!u_sr) return EWB_OK;
  double u = 0.0;
  CK(cudaMemcpyAsync(&u, h->energy.as<double>(), sizeof(double), cudaMemcpyDeviceToHost,
                     h->stream));
  if ((rc = check_errflag(h, ERR_COINCIDENT))) return rc;
  if (u_sr) *u_sr = u;
  return EWB_OK;
}

int ewb_set_geometry_n(ewb_handle *h, int64_t n_global) {
  if (!h) return EWB_EINVAL;
  if (n_global < 0) return h->fail(EWB_EINVAL, "negative particle count");
  h->geom_n = n_global;
  ++h->gen;
  return EWB_OK;
}

int ewb_rs_geometry(ewb_handle *h, int64_t *info4) {
  if (!h || !info4) return EWB_EINVAL;
  if (!h->have_system) return h->fail(EWB_ESTATE, "ewb_set_system first");
  double rc_t, rc2_t;
  rs_cutoff(h, rc_t, rc2_t);
  const bool wide = h->coul_on && h->rc > 0.5 * h->L;
  if (!(rc_t > 0.0) || (wide && !h->lj_on)) {  // one "row": image shell or no pair term
    info4[0] = 1; info4[1] = 1; info4[2] = 1; info4[3] = 1;
    return EWB_OK;
  }
  const RSGeom g = rs_geometry(h, rc_t, h->n);
  info4[0] = g.cpd_eff;
  info4[1] = g.rad;
  info4[2] = (int64_t)g.cpd_eff * g.cpd_eff;
  info4[3] = g.fold ? 1 : 0;
  return EWB_OK;
}

// row of cells (cy + cpd cz) of every particle, binned exactly as the pair
// kernel's cell list (k4_bin_count)
__global__ void k_rows(const double *__restrict__ pos, int64_t n, double edge, int cpd,
                       int *__restrict__ rows) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int id[2] = {0, 0};
  if (cpd > 1) {
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const double f = floor(pos[3 * i + 1 + a] / edge);
      id[a] = (f >= 0.0) ? (f < (double)cpd ? (int)f : cpd - 1) : 0;  // NaN -> 0
    }
  }
  rows[i] = id[0] + cpd * id[1];
}

int ewb_dev_rows(ewb_handle *h, const double *d_pos, int64_t n, int *d_rows) {
  int64_t g[4];
  int rc = ewb_rs_geometry(h, g);
  if (rc) return rc;
  if (n < 0 || (n > 0 && (!d_pos || !d_rows))) return h->fail(EWB_EINVAL, "bad arrays");
  if (n == 0) return EWB_OK;
  CK(cudaSetDevice(h->device));
  k_rows<<<blocks_for(n, 256), 256, 0, h->stream>>>(d_pos, n, h->L / (double)g[0], (int)g[0],
                                                   d_rows);
  CKL();
  return EWB_OK;
}

int ewb_dev_real_space_rows(ewb_handle *h, int row_lo, int row_hi, double *d_force,
                            double *u_sr) {
  int rc = require_state(h, false, true);
  if (rc) return rc;
  if (row_lo < 0 || row_hi < row_lo) return h->fail(EWB_EINVAL, "bad row range");
  CK(cudaSetDevice(h->device));
  if (u_sr && (rc = check_errflag(h, ERR_UNWRAPPED))) return rc;
  CK(h->energy.ensure(8 * sizeof(double)));
  h->row_lo = row_lo;
  h->row_hi = row_hi;
  rc = stage_real_space(h, 0, 1, d_force, h->energy.as<double>(), nullptr);
  h->row_lo = h->row_hi = -1;
  if (rc) return rc;
  if (!u_sr) return EWB_OK;
  double u = 0.0;
  CK(cudaMemcpyAsync(&u, h->energy.as<double>(), sizeof(double), cudaMemcpyDeviceToHost,
                     h->stream));
  if ((rc = check_errflag(h, ERR_COINCIDENT))) return rc;
  *u_sr = u;
  return EWB_OK;
}

// The device energy slots (u_sr, u_lr, u_self of the last asynchronous
// stages) copied into caller device memory on the handle's stream.
int ewb_dev_energies(ewb_handle *h, double *d_out3) {
  int rc = require_state(h, false, false);
  if (rc) return rc;
  if (!d_out3) return h->fail(EWB_EINVAL, "null energy buffer");
  CK(cudaSetDevice(h->device));
  CK(h->energy.ensure(8 * sizeof(double)));
  CK(cudaMemcpyAsync(d_out3, h->energy.p, 3 * sizeof(double), cudaMemcpyDeviceToDevice,
                     h->stream));
  return EWB_OK;
}

// the masked device error flag of the last load/evaluation as a double in
// caller device memory (stream-ordered, no host synchronisation): a
// multi-rank driver reduces it with the energies so that every rank raises
// the same error together
__global__ void k_status(const int *__restrict__ err, int mask, double *__restrict__ out) {
  out[0] = (double)(*err & mask);
}

int ewb_dev_status(ewb_handle *h, double *d_out) {
  int rc = require_state(h, false, false);
  if (rc) return rc;
  if (!d_out) return h->fail(EWB_EINVAL, "null status buffer");
  CK(cudaSetDevice(h->device));
  CK(h->errflag.ensure(sizeof(int)));
  k_status<<<1, 1, 0, h->stream>>>(h->errflag.as<int>(), err_mask(h), d_out);
  CKL();
  return EWB_OK;
}

// Synchronise the handle's stream and report device-side errors of the
// asynchronous stages (unwrapped positions, coincident particles).
int ewb_dev_check(ewb_handle *h) {
  int rc = require_state(h, false, false);
  if (rc) return rc;
  CK(cudaSetDevice(h->device));
  CK(h->errflag.ensure(sizeof(int)));
  return check_errflag(h, err_mask(h));
}

int ewb_dev_self_energy(ewb_handle *h, double *u_self) {
  return ewb_dev_self_energy_range(h, 0, h ? h->n : 0, u_self);
}

int ewb_dev_self_energy_range(ewb_handle *h, int64_t i0, int64_t i1, double *u_self) {
  int rc = require_state(h, false, true);
  if (rc) return rc;
  if (i0 < 0 || i1 > h->n || i0 > i1) return h->fail(EWB_EINVAL, "bad particle range");
  CK(cudaSetDevice(h->device));
  CK(h->energy.ensure(8 * sizeof(double)));
  if ((rc = stage_self(h, h->energy.as<double>() + 2, i0, i1))) return rc;
  if (!u_self) return EWB_OK;  // asynchronous: stays in the device energy slot
  double u = 0.0;
  CK(cudaMemcpyAsync(&u, h->energy.as<double>() + 2, sizeof(double), cudaMemcpyDeviceToHost,
                     h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (u_self) *u_self = u;
  return EWB_OK;
}

int ewb_dev_evaluate(ewb_handle *h, const double *d_pos, const double *d_q, int64_t n,
                     double *d_force, double *d_rho_out, double *energies, double *timings) {
  int rc = require_state(h, h && h->coul_on, false);
  if (rc) return rc;
  CK(cudaSetDevice(h->device));
  if (h->coul_on && !(h->rc > 0.0)) return h->fail(EWB_EINVAL, "cutoff must be positive");
  if (!h->coul_on) d_rho_out = nullptr;
  if ((rc = run_eval(h, d_pos, d_q, n, d_force, d_rho_out, timings != nullptr))) return rc;
  double en[3];
  CK(cudaMemcpyAsync(en, h->energy.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  if ((rc = check_errflag(
           h, err_mask(h) |
                  ERR_COINCIDENT)))
    return rc;
  if (energies) std::memcpy(energies, en, sizeof en);
  return read_timings(h, timings);
}

int ewb_probe_fp64_peak(ewb_handle *h, double *tflops) {
  if (!h || !tflops) return EWB_EINVAL;
  CK(cudaSetDevice(h->device));
  CK(h->eblk2.ensure(64));
  const int iters = 4096;
  const unsigned blocks = (unsigned)h->n_sm * 8;
  k_fp64_probe<<<blocks, 256, 0, h->stream>>>(h->eblk2.as<double>(), iters, 0.999999, 1e-7);
  CKL();
  CK(cudaEventRecord(h->ev[0], h->stream));
  const int reps = 5;
  for (int r = 0; r < reps; ++r) {
    k_fp64_probe<<<blocks, 256, 0, h->stream>>>(h->eblk2.as<double>(), iters, 0.999999, 1e-7);
    CKL();
  }
  CK(cudaEventRecord(h->ev[1], h->stream));
  CK(cudaEventSynchronize(h->ev[1]));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]));
  const double flops = 2.0 * 8.0 * iters * 256.0 * blocks * reps;
  *tflops = flops / (ms * 1e-3) / 1e12;
  return EWB_OK;
}

int ewb_probe_i8_shape(ewb_handle *h, int n_mma, double *tops) {
  if (!h || !tops || n_mma < 16 || n_mma > 256 || n_mma % 16) return EWB_EINVAL;
  CK(cudaSetDevice(h->device));
  CK(h->eblk2.ensure(64));
  const int iters = 16384;
  const unsigned blocks = (unsigned)h->n_sm;
  const size_t smem = (size_t)(16 + 32) * TC_SBO;
  CK(cudaFuncSetAttribute(k_i8_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_i8_probe<<<blocks, 128, smem, h->stream>>>(iters, n_mma, h->eblk2.as<int>());
  CKL();
  CK(cudaEventRecord(h->ev[0], h->stream));
  const int reps = 3;
  for (int r = 0; r < reps; ++r) {
    k_i8_probe<<<blocks, 128, smem, h->stream>>>(iters, n_mma, h->eblk2.as<int>());
    CKL();
  }
  CK(cudaEventRecord(h->ev[1], h->stream));
  CK(cudaEventSynchronize(h->ev[1]));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]));
  const double ops = 2.0 * 128.0 * n_mma * 32.0 * iters * blocks * reps;
  *tops = ops / (ms * 1e-3) / 1e12;
  return EWB_OK;
}

int ewb_probe_i8_peak(ewb_handle *h, double *tops) { return ewb_probe_i8_shape(h, 256, tops); }

int ewb_probe_i8_shape_ts(ewb_handle *h, int n_mma, double *tops) {
  if (!h || !tops || n_mma < 16 || n_mma > 256 || n_mma % 16) return EWB_EINVAL;
  CK(cudaSetDevice(h->device));
  CK(h->eblk2.ensure(64));
  const int iters = 16384;
  const unsigned blocks = (unsigned)h->n_sm;
  const size_t smem = (size_t)32 * TC_SBO;
  CK(cudaFuncSetAttribute(k_i8_probe_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_i8_probe_ts<<<blocks, 128, smem, h->stream>>>(iters, n_mma, h->eblk2.as<int>());
  CKL();
  CK(cudaEventRecord(h->ev[0], h->stream));
  const int reps = 3;
  for (int r = 0; r < reps; ++r) {
    k_i8_probe_ts<<<blocks, 128, smem, h->stream>>>(iters, n_mma, h->eblk2.as<int>());
    CKL();
  }
  CK(cudaEventRecord(h->ev[1], h->stream));
  CK(cudaEventSynchronize(h->ev[1]));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]));
  const double ops = 2.0 * 128.0 * n_mma * 32.0 * iters * blocks * reps;
  *tops = ops / (ms * 1e-3) / 1e12;
  return EWB_OK;
}

int ewb_tc_info(const ewb_handle *h, int64_t *info8) {
  if (!h || !info8) return EWB_EINVAL;
  if (!h->have_kspace) return EWB_ESTATE;
  const Plan &P = h->plan;
  int64_t npad_sum = 0;
  for (const auto &c : P.tc_chunks_host) npad_sum += c.npad;
  info8[0] = P.tc_ok && tc_wanted(h, h->n) ? 1 : 0;
  info8[1] = P.tc_mtiles;
  info8[2] = npad_sum;         // sum of padded X columns over the a-chunks
  info8[3] = P.t3_mtiles;
  info8[4] = 2 * P.t3_npairs;  // K of the force GEMM
  info8[5] = T3_PAIRS;         // slice-pair MMAs per K step of the force GEMM
  info8[6] = 26;               // slice-pair MMAs per K step of the S(k) GEMM
  info8[7] = P.tc_A;
  return EWB_OK;
}

int ewb_last_pair_count(ewb_handle *h, int64_t *pairs) {
  if (!h || !pairs) return EWB_EINVAL;
  *pairs = 0;
  if (!h->pairc.p) return EWB_OK;
  unsigned long long v = 0;
  CK(cudaStreamSynchronize(h->stream));
  CK(cudaMemcpy(&v, h->pairc.p, sizeof(v), cudaMemcpyDeviceToHost));
  *pairs = (int64_t)v;
  return EWB_OK;
}

int ewb_host_alloc(size_t bytes, void **out) {
  if (!out) return EWB_EINVAL;
  *out = nullptr;
  if (cudaHostAlloc(out, bytes ? bytes : 16, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    *out = nullptr;
    return EWB_ECUDA;
  }
  return EWB_OK;
}

int ewb_host_free(void *p) {
  if (p && cudaFreeHost(p) != cudaSuccess) return EWB_ECUDA;
  return EWB_OK;
}

// page-lock a caller's host range in place (cudaHostRegister), so the
// evaluation's copies of it run as asynchronous DMA; the caller unregisters
// it before the memory is freed.  1: already registered (not an error).
int ewb_host_register(void *p, size_t bytes) {
  if (!p || !bytes) return EWB_EINVAL;
  const cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterPortable);
  if (e == cudaErrorHostMemoryAlreadyRegistered) {
    cudaGetLastError();
    return 1;
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    return EWB_ECUDA;
  }
  return EWB_OK;
}

int ewb_host_unregister(void *p) {
  if (!p) return EWB_EINVAL;
  if (cudaHostUnregister(p) != cudaSuccess) {
    cudaGetLastError();
    return EWB_ECUDA;
  }
  return EWB_OK;
}

int64_t ewb_launch_count(const ewb_handle *h) { return h ? h->launches : -1; }

}  // extern "C"

