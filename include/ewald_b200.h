/*
 * ewald_b200.h -- C-ABI of the B200-native classical Ewald library
 * (libewaldb200.so).  Plain pointers and sizes only; no torch types.
 *
 * Every entry point replaces one reference interface of the Python package
 * ewaldmd (paths are relative to /root/reference/pkg/src/ewaldmd):
 *
 *   ewb_set_system        EwaldParams / coulomb_short_range_kernel consts
 *                         (ewald.py:40-72, 243-259)
 *   ewb_set_kspace        ReciprocalSpace.__init__ (ewald.py:150-168)
 *   ewb_compute_rho_hat   compute_rho_hat           (ewald.py:457-464)
 *   ewb_long_range        long_range_energy_forces  (ewald.py:467-479)
 *   ewb_short_range       PairLoop(coulomb_short_range) over build_cell_list
 *                         (ewald.py:639-643, engine.py:283-324,
 *                          celllist.py:75-108)
 *   ewb_self_energy       self_energy               (ewald.py:482-484)
 *   ewb_evaluate          EwaldSolver.evaluate      (ewald.py:629-655)
 *
 * Host-pointer entry points copy inputs host->device and results back; they
 * follow the reference's argument meaning exactly: pos is (N,3) C-order
 * xyz-interleaved float64, q is (N,), force is (N,3) and is ACCUMULATED
 * (+=, ewald.py:603-605), rho is the GlobalAccumulator layout: K real parts
 * followed by K imaginary parts, rho(k) = sum_j q_j exp(-i k.r_j), K in the
 * caller's m_int order (ewald.py:170-173, 303-305).
 *
 * ewb_dev_* entry points take DEVICE pointers and run on the stream set by
 * ewb_set_stream; they are the stages a multi-GPU driver composes around its
 * collectives (particle-sharded S(k) partials -> all-reduce -> force gather).
 *
 * All functions return an ewb_status; ewb_last_error() gives the message.
 * A handle is not thread-safe (same contract as the reference engine,
 * SPEC.md:181).
 */
#ifndef EWALD_B200_H
#define EWALD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ewb_handle ewb_handle;

typedef enum {
    EWB_OK = 0,
    EWB_EINVAL = 1,      /* ValueError                       */
    EWB_ECOINCIDENT = 2, /* CoincidentParticlesError (r^2==0) */
    EWB_ECUTOFF = 3,     /* CutoffTooLargeError (r_c > L/2)  */
    EWB_EUNWRAPPED = 4,  /* ValueError: positions not in [0,L) */
    EWB_ECUDA = 5,       /* RuntimeError: CUDA failure        */
    EWB_EBOX = 6,        /* BoxTooSmallError (r_c > L)        */
    EWB_EKSPACE = 7,     /* KSpaceEmptyError                  */
    EWB_ESTATE = 8,      /* RuntimeError: call order violated */
    EWB_ESIZE = 9        /* OracleSizeError (image-shell path, N > 4096) */
} ewb_status;

/* library / handle lifetime */
int ewb_version(void);
int ewb_create(int device, ewb_handle **out);
void ewb_destroy(ewb_handle *h);
const char *ewb_last_error(const ewb_handle *h);
/* stream used by every later call (a cudaStream_t; 0 = the legacy default
 * stream).  A new handle runs on its own non-blocking stream;
 * ewb_use_own_stream returns to it. */
int ewb_set_stream(ewb_handle *h, uintptr_t stream);
int ewb_use_own_stream(ewb_handle *h);
/* tuning knobs (take effect at the next ewb_set_kspace): maximum k-column
 * segment length of the force gather (1..32; default 28) and of the
 * structure factor's +-m_x pair items (1..20; default 20) */
int ewb_set_max_segment(ewb_handle *h, int mcap);
int ewb_set_max_pair_segment(ewb_handle *h, int mcap1);

/* real-space cell grid: 0 = auto (r_c/2 cells, 5^3 stencil, when >= 5 cells
 * per edge), 1 = r_c cells with the 3^3 stencil (the reference's grid). */
int ewb_set_stencil(ewb_handle *h, int rad);

/* Force gather with C*S in the constant bank (uniform-register operands)
 * for systems with >= 2 particle blocks per SM (default on).  The constant
 * bank is per process: handles must not run evaluations concurrently on
 * different streams of the same device. */
int ewb_set_const_gather(ewb_handle *h, int on);
/* Reciprocal space (Algorithms 1 and 2) on the int8 tensor cores: 48-bit
 * fixed-point operands split into six int8 slices, exact int32 accumulation
 * in TMEM, fp64 recombination (|dS| ~ 1e-15 max|S|, forces ~1e-13 F_rms).
 * mode 0: FP64-pipe kernels; 1: tensor cores; 2 (default): tensor cores when
 * N*K >= 2^26, else the FP64 kernels (faster for tiny systems). */
int ewb_set_tensor_cores(ewb_handle *h, int mode);
/* Run reciprocal space on a second stream concurrently with real space
 * (default on; applies when both reciprocal stages use the tensor cores).
 * The stage times of ewb_evaluate then overlap. */
int ewb_set_overlap(ewb_handle *h, int on);
/* CUDA-graph replay of the evaluation pipeline (default on): the second
 * evaluate with unchanged shapes/pointers/configuration is captured, later
 * ones replay the graph.  0 runs every kernel eagerly. */
int ewb_set_graphs(ewb_handle *h, int on);
/* Verlet pair lists with a skin (the reference rebuilds its cell list every
 * step, SPEC.md:179 and driver.py:119-124, 227-245): with skin > 0 the
 * real-space pass bins and builds per-unit pair lists at r_c + skin and
 * later evaluations reuse them (exact r < r_c predicates per pair) while no
 * particle has moved skin/2 since the build.  ewb_dev_verlet_check (one
 * small kernel + synchronisation) decides for the NEXT evaluation of d_pos:
 * *rebuild = 0 arms one reuse.  ewb_verlet_info: {builds, reuses}.  skin 0
 * (default) rebuilds every evaluation. */
int ewb_set_skin(ewb_handle *h, double skin);
int ewb_dev_verlet_check(ewb_handle *h, const double *d_pos, int64_t n, int *rebuild);
int ewb_verlet_info(const ewb_handle *h, int64_t *out2);

/* 0 (default): real space visits each unordered pair once and scatters
 * the partner's force with fp64 atomics (fastest; summation order varies
 * run to run at the 1e-16 level).  1: ordered pairs, write-to-centre only
 * (engine.py:10-14) -- bitwise reproducible, ~1.6x more real-space work. */
int ewb_set_deterministic(ewb_handle *h, int on);
/* Real space in two passes (default 0: measured slower than the fused kernel,
 * kept as an option and tested for equality): a traversal kernel writes each
 * unit's accepted pairs to a list in HBM, an evaluation kernel (fewer
 * registers, more warps per SM) evaluates them; units whose list overflows
 * its capacity fall back to the fused kernel.  0: one fused kernel.  2:
 * split with a 32-entry capacity (testing: exercises the overflow pass).
 * Same pairs and per-pair arithmetic either way (ewald.py:208-221). */
int ewb_set_real_space_split(ewb_handle *h, int on);

/* EwaldParams: box edge L, screening alpha (A^-2, erfc(sqrt(alpha) r)),
 * real-space cutoff.  rc2 is r_cutoff**2 as the caller computed it, so the
 * cutoff predicate r2 < rc2 is bit-identical to the reference's. */
int ewb_set_system(ewb_handle *h, double L, double alpha, double r_cutoff,
                   double rc2);

/* ReciprocalSpace: m_int (K,3) int64 in caller order, coeff (K,) C_k. */
int ewb_set_kspace(ewb_handle *h, const int64_t *m_int, int64_t K,
                   const double *coeff);
/* plan summary: [K, n_items, M, n_rows, n_tiles, max_table, n_pair_items, M1] */
int ewb_kspace_info(const ewb_handle *h, int64_t *info8);

/* Force-field switches of the reference's ForceAssembler (driver.py:81-126):
 * Coulomb (Ewald) on/off, and the energy-shifted 12-6 Lennard-Jones pair
 * term fused into the real-space traversal.  LJ constants are the
 * reference's lj_kernel consts (potentials.py:74-79): sigma^2, 4 eps,
 * energy_shift(), 24 eps; rc2_lj = r_cutoff_lj**2 as computed by the caller. */
int ewb_set_coulomb(ewb_handle *h, int on);
int ewb_set_lj(ewb_handle *h, int on, double sigma2, double four_eps, double shift,
               double tf_eps, double rc_lj, double rc2_lj);
/* energies of the last evaluation: u_sr, u_lr, u_self, u_lj */
int ewb_last_energies(ewb_handle *h, double *out4);

/* ---- host-pointer entry points (reference-facing) ---- */
int ewb_compute_rho_hat(ewb_handle *h, const double *pos, const double *q,
                        int64_t n, double *rho_out);
int ewb_long_range(ewb_handle *h, const double *pos, const double *q,
                   int64_t n, const double *rho, double *force_inout,
                   double *u_lr);
int ewb_short_range(ewb_handle *h, const double *pos, const double *q,
                    int64_t n, double *force_inout, double *u_sr);
int ewb_self_energy(ewb_handle *h, const double *q, int64_t n,
                    double *u_self);
/* energies[3] = u_sr, u_lr, u_self; timings[4] = t_cell, t_sr, t_alg1,
 * t_alg2 in seconds (device events); rho_out may be NULL. */
int ewb_evaluate(ewb_handle *h, const double *pos, const double *q,
                 int64_t n, double *force_inout, double *rho_out,
                 double *energies, double *timings);

/* ---- device-pointer stages (multi-GPU driver, device-resident bench) ---- */
/* Load particles (device pos (N,3), q (N,)); validates wrapping. */
int ewb_dev_load(ewb_handle *h, const double *d_pos, const double *d_q,
                 int64_t n);
/* Number of doubles of the pair-slot S(k) partial buffer (4 * M1 * n_pair_items). */
int64_t ewb_dev_slot_doubles(const ewb_handle *h);
/* S(k) partial over particles [i0, i1) into d_slots (slot layout). */
int ewb_dev_rho_partial(ewb_handle *h, int64_t i0, int64_t i1,
                        double *d_slots);
/* From complete slot-layout S(k): rho_out (device, 2K, may be NULL),
 * internal C*S for the force gather, and u_lr = sum_k C_k |S_k|^2. */
int ewb_dev_kspace_finalize(ewb_handle *h, const double *d_slots,
                            double *d_rho_out, double *u_lr);
/* The multi-GPU S(k) reduction fused with the finalisation: d_slots[r]
 * (host array of n_ranks <= 16 device pointers) are the ranks' partial
 * pair-slot buffers (ewb_dev_rho_partial), read straight from peer memory
 * (NVLink; enable with ewb_enable_peer_access) and summed in rank order
 * inside the finalising kernel -- no separate all-reduce.  Every rank gets
 * the same S; u_lr lands in the device energy slot (ewb_dev_energies).
 * Replaces the reduce_global + finalize of engine.py:85-91 / ewald.py:457. */
int ewb_dev_kspace_finalize_peer(ewb_handle *h, const double *const *d_slots, int n_ranks,
                                 double *d_rho_out);
int ewb_enable_peer_access(ewb_handle *h, int peer_device);
/* One process per GPU: the S(k) partial in a dedicated allocation whose CUDA
 * IPC handle (64 bytes) the ranks exchange once; each rank opens the others'
 * (ewb_ipc_open) and ewb_dev_kspace_finalize_peer reads them over NVLink. */
int ewb_ipc_slots(ewb_handle *h, void **d_ptr, unsigned char *handle64);
int ewb_ipc_open(ewb_handle *h, const unsigned char *handle64, void **d_ptr);
int ewb_ipc_close(ewb_handle *h, void *d_ptr);
/* Reciprocal forces of particles [i0, i1), added into d_force (N,3). */
int ewb_dev_recip_forces(ewb_handle *h, int64_t i0, int64_t i1,
                         double *d_force);
/* Real-space forces of the particles whose home cell lies in z-slab
 * part/nparts, added into d_force (N,3); u_sr of those particles.  With
 * u_sr == NULL the call only enqueues work (no synchronisation): the energy
 * stays in the device slot read by ewb_dev_energies and device-side errors
 * are reported by ewb_dev_check. */
int ewb_dev_real_space(ewb_handle *h, int part, int nparts, double *d_force,
                       double *u_sr);
/* Self energy -sqrt(alpha/pi) * sum q^2 over all loaded particles
 * (u_self == NULL: asynchronous, device slot only). */
int ewb_dev_self_energy(ewb_handle *h, double *u_self);
/* Self energy of the loaded particles [i0, i1) only (the owned particles of
 * a domain-decomposed rank; self_energy, ewald.py:482-484). */
int ewb_dev_self_energy_range(ewb_handle *h, int64_t i0, int64_t i1, double *u_self);

/* Domain decomposition of the real space (distributed.SlabEwald): every rank
 * bins on the grid of the GLOBAL particle count n_global (the r_c/3 grid is
 * chosen by occupancy), so all ranks agree on cells and rows. */
int ewb_set_geometry_n(ewb_handle *h, int64_t n_global);
/* Real-space cell grid of the current system: info4 = (cells per edge,
 * stencil radius in cells, rows of cells = cpd^2, scan-all flag).  A row is
 * the line of cells (cy, cz) along x, numbered cy + cpd cz. */
int ewb_rs_geometry(ewb_handle *h, int64_t *info4);
/* Row of cells of each of n particles (device pointers), binned exactly as
 * the pair kernel's cell list (celllist.py:75-108 binning). */
int ewb_dev_rows(ewb_handle *h, const double *d_pos, int64_t n, int *d_rows);
/* Particles grouped by row of cells (a stable sort on the row: ascending
 * index within a row) into d_order[n], and the row offsets d_row_start
 * [n_rows + 1]: every rank's own particles and halo of the multi-GPU
 * decomposition are slices of d_order (the reference partitions particles
 * into worker blocks, engine.py:75-82). */
int ewb_dev_row_order(ewb_handle *h, const double *d_pos, int64_t n, int *d_order,
                      int *d_row_start);
/* Real space of the loaded particles with centres restricted to the rows
 * [row_lo, row_hi): the rank's own rows, partners from its own rows and the
 * halo rows it received.  Half shell: forces also land on halo partners
 * (returned to their owners by the caller).  u_sr as ewb_dev_real_space. */
int ewb_dev_real_space_rows(ewb_handle *h, int row_lo, int row_hi, double *d_force,
                            double *u_sr);
/* Device energy slots (u_sr, u_lr, u_self of the last stages) copied into
 * d_out3 (device, 3 doubles) on the handle's stream.  Replaces the three
 * scalar returns of the engine's kernels (ewald.py:609-655) for a
 * synchronisation-free multi-GPU step. */
int ewb_dev_energies(ewb_handle *h, double *d_out3);
/* Synchronise and raise the deferred device-side errors: unwrapped
 * positions (celllist.py:90-91) and coincident particles (ewald.py:212-213). */
/* The masked device error flag (1: unwrapped positions, 2: coincident
 * particles) written as a double into d_out on the handle's stream, without
 * a host synchronisation (multi-rank drivers reduce it with the energies). */
int ewb_dev_status(ewb_handle *h, double *d_out);
int ewb_dev_check(ewb_handle *h);
/* Whole evaluation on device-resident data (single GPU); force +=. */
int ewb_dev_evaluate(ewb_handle *h, const double *d_pos, const double *d_q,
                     int64_t n, double *d_force, double *d_rho_out,
                     double *energies, double *timings);
/* Device-resident velocity Verlet (driver.py:134-153), arrays (N,3)/(N,):
 * kick_drift: v += dt/2 F/m, r += dt v, wrap into [0, L);
 * kick: (if kick) v += dt/2 F/m, then kinetic = 0.5 sum m v.v. */
int ewb_dev_md_kick_drift(ewb_handle *h, double *d_pos, double *d_vel, const double *d_force,
                          const double *d_mass, int64_t n, double dt);
int ewb_dev_md_kick(ewb_handle *h, double *d_vel, const double *d_force, const double *d_mass,
                    int64_t n, double dt, int kick, double *kinetic);
/* Sustained FP64 DFMA throughput of this device (TFLOP/s), measured with
 * independent fma chains; the FP64 roofline denominator. */
int ewb_probe_fp64_peak(ewb_handle *h, double *tflops);
/* Roofline denominator of the tensor-core kernels: dense int8 tcgen05.mma
 * (M=128, N=256, K=32, shared-memory operands) issued back to back on every
 * SM; *tops = measured int8 TOP/s. */
int ewb_probe_i8_peak(ewb_handle *h, double *tops);
/* The same probe for MMA shape M=128, N=n_mma (16..256, multiple of 16). */
int ewb_probe_i8_shape(ewb_handle *h, int n_mma, double *tops);
/* The same with the A operand read from tensor memory (TS form). */
int ewb_probe_i8_shape_ts(ewb_handle *h, int n_mma, double *tops);
/* Tensor-core plan of the current k-table (for MMA-work accounting):
 * info8 = {enabled, S(k) M tiles, sum of padded X columns, force M tiles,
 *          force GEMM K, levels, slice-pair MMAs per K step, max |m_x|}. */
int ewb_tc_info(const ewb_handle *h, int64_t *info8);
/* Pairs inside the traversal cutoff visited by the last real-space pass
 * (unordered pairs in the default half-shell mode, ordered pairs in the
 * deterministic full-shell mode); synchronises the handle's stream. */
int ewb_last_pair_count(ewb_handle *h, int64_t *pairs);
/* Kernels launched by this handle since creation (evidence counter). */
int64_t ewb_launch_count(const ewb_handle *h);
/* Page-locked host memory for arrays the evaluation copies into (e.g.
 * ReciprocalSpace.rho): device-to-host copies land directly. */
int ewb_host_alloc(size_t bytes, void **out);
int ewb_host_free(void *p);
/* Page-lock / release a caller-owned host range in place (cudaHostRegister):
 * the facade pins a ParticleSet's arrays on their second evaluation so the
 * copies of EwaldSolver.evaluate (reference ewald.py:629-655, pageable numpy
 * arrays allocated at core.py:111-115) run as asynchronous DMA.  Returns 1
 * if the range was registered already.  The caller unregisters before the
 * memory is freed. */
int ewb_host_register(void *p, size_t bytes);
int ewb_host_unregister(void *p);

/* ---- harness helper (csrc/workloads.c, separate library) ----
 * int ewb_gen_hardcore_gas(int64_t n, double L, double min_sep,
 *                          uint64_t seed, int64_t max_attempts,
 *                          double *pos_out, int64_t *attempts_out);
 */

#ifdef __cplusplus
}
#endif
#endif /* EWALD_B200_H */
