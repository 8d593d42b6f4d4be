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

#include <cub/device/device_radix_sort.cuh>

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

#include "ewb_kernels.cuh"

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
  DBuf ro_key, ro_keyout, ro_idx, ro_cnt, ro_g, ro_tmp;  // ewb_dev_row_order scratch
  void *ipc_slots = nullptr;      // dedicated allocation of the S(k) partial (CUDA IPC export)
  size_t ipc_bytes = 0;
  // Verlet pair lists (ewb_set_skin): lists built at r_c + skin are reused
  // while no particle has moved more than skin/2 since the build
  double skin = 0.0;
  bool vl_valid = false, vl_reuse = false;
  uint64_t vl_gen = 0;
  int64_t vl_n = -1;
  int64_t vl_builds = 0, vl_reuses = 0;
  DBuf vl_xb, vl_dmax;            // build-time sorted positions; max displacement^2
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

#include "ewb_plan.cuh"
#include "ewb_stages.cuh"

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
                  &h->rs_list, &h->rs_count, &h->vl_xb, &h->vl_dmax, &h->ro_key, &h->ro_keyout,
                  &h->ro_idx, &h->ro_cnt, &h->ro_g, &h->ro_tmp})
    b->release();
  if (h->ipc_slots) cudaFree(h->ipc_slots);
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

int ewb_set_skin(ewb_handle *h, double skin) {
  if (!h || !(skin >= 0.0)) return EWB_EINVAL;
  ++h->gen;
  h->skin = skin;
  h->vl_valid = false;
  h->vl_reuse = false;
  h->vl_builds = h->vl_reuses = 0;
  return EWB_OK;
}

int ewb_dev_verlet_check(ewb_handle *h, const double *d_pos, int64_t n, int *rebuild) {
  if (!h || !rebuild || (n > 0 && !d_pos)) return EWB_EINVAL;
  *rebuild = 1;
  h->vl_reuse = false;
  if (!(h->skin > 0.0) || !h->vl_valid || h->vl_gen != h->gen || h->vl_n != n) return EWB_OK;
  CK(cudaSetDevice(h->device));
  CK(h->vl_dmax.ensure(sizeof(unsigned long long)));
  CK(cudaMemsetAsync(h->vl_dmax.p, 0, sizeof(unsigned long long), h->stream));
  k_verlet_disp<<<blocks_for(n, 256), 256, 0, h->stream>>>(
      d_pos, h->order.as<int>(), h->vl_xb.as<double4>(), n, h->L,
      h->vl_dmax.as<unsigned long long>());
  CKL();
  unsigned long long bits = 0;
  CK(cudaMemcpyAsync(&bits, h->vl_dmax.p, sizeof bits, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  double d2;
  std::memcpy(&d2, &bits, sizeof d2);
  const double half = 0.5 * h->skin;
  // strictly inside skin/2: pairs now within r_c were within r_c + skin
  *rebuild = d2 < half * half ? 0 : 1;
  h->vl_reuse = *rebuild == 0;
  return EWB_OK;
}

int ewb_verlet_info(const ewb_handle *h, int64_t *out2) {
  if (!h || !out2) return EWB_EINVAL;
  out2[0] = h->vl_builds;
  out2[1] = h->vl_reuses;
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
  const unsigned nb = blocks_for(n_pslots, K2P_THREADS);
  k2p_finalize<<<nb, K2P_THREADS, 0, h->stream>>>(h->spart.as<double4>(), n_part, n_pslots,
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

int ewb_dev_kspace_finalize_peer(ewb_handle *h, const double *const *d_slots, int n_ranks,
                                 double *d_rho_out) {
  int rc = require_state(h, true, false);
  if (rc) return rc;
  if (!d_slots || n_ranks < 1 || n_ranks > K2P_MAX_PEERS)
    return h->fail(EWB_EINVAL, "1..16 peer slot buffers");
  CK(cudaSetDevice(h->device));
  CK(h->energy.ensure(8 * sizeof(double)));
  Plan &P = h->plan;
  const int64_t n_pslots = (int64_t)P.M1 * P.n_pitems;
  PeerSlots ps{};
  for (int r = 0; r < n_ranks; ++r) {
    if (!d_slots[r]) return h->fail(EWB_EINVAL, "null peer slot buffer");
    ps.p[r] = reinterpret_cast<const double4 *>(d_slots[r]);
  }
  ps.n = n_ranks;
  const unsigned nb = blocks_for(n_pslots, K2P_THREADS);
  CK(h->eblk_r.ensure(nb * sizeof(double)));
  k2p_finalize_peer<<<nb, K2P_THREADS, 0, h->stream>>>(ps, n_pslots, P.pslot_map.as<int4>(),
                                                       P.slot_coeff.as<double>(), P.K, d_rho_out,
                                                       h->sp.as<double2>(), h->eblk_r.as<double>());
  CKL();
  k_sum<<<1, 1024, 0, h->stream>>>(h->eblk_r.as<double>(), nb, 1.0, h->energy.as<double>() + 1);
  CKL();
  return EWB_OK;
}

int ewb_ipc_slots(ewb_handle *h, void **d_ptr, unsigned char *handle64) {
  int rc = require_state(h, true, false);
  if (rc) return rc;
  if (!d_ptr || !handle64) return h->fail(EWB_EINVAL, "null output");
  CK(cudaSetDevice(h->device));
  const size_t bytes = (size_t)h->plan.M1 * h->plan.n_pitems * sizeof(double4);
  if (bytes != h->ipc_bytes) {
    if (h->ipc_slots) CK(cudaFree(h->ipc_slots));
    h->ipc_slots = nullptr;
    h->ipc_bytes = 0;
    CK(cudaMalloc(&h->ipc_slots, bytes ? bytes : 16));
    h->ipc_bytes = bytes;
  }
  cudaIpcMemHandle_t hd;
  CK(cudaIpcGetMemHandle(&hd, h->ipc_slots));
  std::memcpy(handle64, &hd, sizeof hd < 64 ? sizeof hd : 64);
  *d_ptr = h->ipc_slots;
  return EWB_OK;
}

int ewb_ipc_open(ewb_handle *h, const unsigned char *handle64, void **d_ptr) {
  if (!h || !handle64 || !d_ptr) return EWB_EINVAL;
  CK(cudaSetDevice(h->device));
  cudaIpcMemHandle_t hd;
  std::memcpy(&hd, handle64, sizeof hd);
  CK(cudaIpcOpenMemHandle(d_ptr, hd, cudaIpcMemLazyEnablePeerAccess));
  return EWB_OK;
}

int ewb_ipc_close(ewb_handle *h, void *d_ptr) {
  if (!h || !d_ptr) return EWB_EINVAL;
  CK(cudaSetDevice(h->device));
  CK(cudaIpcCloseMemHandle(d_ptr));
  return EWB_OK;
}

int ewb_enable_peer_access(ewb_handle *h, int peer_device) {
  if (!h) return EWB_EINVAL;
  if (peer_device == h->device) return EWB_OK;
  CK(cudaSetDevice(h->device));
  int can = 0;
  CK(cudaDeviceCanAccessPeer(&can, h->device, peer_device));
  if (!can) return h->fail(EWB_ECUDA, "no peer access between the devices");
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return EWB_OK;
  }
  CK(e);
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

}  // extern "C"
namespace {
__global__ void k_iota_hist(const int *__restrict__ key, int64_t n, int *__restrict__ idx,
                            int *__restrict__ count) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  idx[i] = (int)i;
  atomicAdd(count + key[i], 1);
}
}  // namespace
extern "C" {

// particles grouped by row of cells, ascending index within a row (stable
// radix sort on the row), and the row offsets: the ownership and halo lists
// of the multi-GPU decomposition are slices of d_order
int ewb_dev_row_order(ewb_handle *h, const double *d_pos, int64_t n, int *d_order,
                      int *d_row_start) {
  int64_t g[4];
  int rc = ewb_rs_geometry(h, g);
  if (rc) return rc;
  if (n < 1 || !d_pos || !d_order || !d_row_start) return h->fail(EWB_EINVAL, "bad arrays");
  if (n >= ((int64_t)1 << 31)) return h->fail(EWB_EINVAL, "particle count too large");
  CK(cudaSetDevice(h->device));
  const int cpd = (int)g[0], n_rows = (int)g[2];
  CK(h->ro_key.ensure(n * sizeof(int)));
  CK(h->ro_keyout.ensure(n * sizeof(int)));
  CK(h->ro_idx.ensure(n * sizeof(int)));
  CK(h->ro_cnt.ensure((n_rows + 1) * sizeof(int)));
  CK(h->ro_g.ensure((n_rows + 1) * sizeof(int)));
  k_rows<<<blocks_for(n, 256), 256, 0, h->stream>>>(d_pos, n, h->L / (double)cpd, cpd,
                                                   h->ro_key.as<int>());
  CKL();
  CK(cudaMemsetAsync(h->ro_cnt.p, 0, (n_rows + 1) * sizeof(int), h->stream));
  k_iota_hist<<<blocks_for(n, 256), 256, 0, h->stream>>>(h->ro_key.as<int>(), n,
                                                          h->ro_idx.as<int>(), h->ro_cnt.as<int>());
  CKL();
  k_scan_cells<<<1, 1024, 0, h->stream>>>(h->ro_cnt.as<int>(), n_rows, d_row_start,
                                          h->ro_g.as<int>());
  CKL();
  int bits = 1;
  while ((1 << bits) < n_rows) ++bits;
  size_t tmp = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, h->ro_key.as<int>(), h->ro_keyout.as<int>(),
                                     h->ro_idx.as<int>(), d_order, (int)n, 0, bits, h->stream));
  CK(h->ro_tmp.ensure(tmp));
  CK(cub::DeviceRadixSort::SortPairs(h->ro_tmp.p, tmp, h->ro_key.as<int>(),
                                     h->ro_keyout.as<int>(), h->ro_idx.as<int>(), d_order, (int)n,
                                     0, bits, h->stream));
  ++h->launches;
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

