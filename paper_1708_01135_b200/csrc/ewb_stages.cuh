// ewb_stages.cuh -- host orchestration of the evaluation: the stages
// (load, real space, S(k), finalisation, forces, self energy), the two-stream
// pipeline with CUDA-graph segments, error-flag checks and timings.  All
// asynchronous on h->stream.  Included by ewald_b200.cu inside its anonymous
// namespace (after ewb_plan.cuh).

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
  const unsigned nb = blocks_for(n_pslots, K2P_THREADS);
  CK(h->eblk_r.ensure(nb * sizeof(double)));
  k2p_finalize<<<nb, K2P_THREADS, 0, h->stream>>>(src, n_part, n_pslots, P.pslot_map.as<int4>(),
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
  const double rc_i = std::max(pair_coul ? h->rc : 0.0, lj_on ? h->rc_lj : 0.0);
  // Verlet lists: traverse (cells, stencil, lists) at r_c + skin; every
  // term keeps its exact predicate in the evaluation.  Not with the scan-all
  // geometry (tiny boxes), a sharded row range or a skin beyond L/2.
  bool verlet = h->skin > 0.0 && h->row_hi < 0 && nparts == 1 &&
                rc_i + h->skin <= 0.5 * h->L && n < ((int64_t)1 << K6_LIST_JBITS);
  RSGeom g = rs_geometry(h, verlet ? rc_i + h->skin : rc_i, n);
  if (verlet && g.fold) {
    verlet = false;
    g = rs_geometry(h, rc_i, n);
  }
  const double rc_t = verlet ? rc_i + h->skin : rc_i;
  const double rc2_t = verlet ? rc_t * rc_t
                              : std::max(pair_coul ? h->rc2 : 0.0, lj_on ? h->rc2_lj : 0.0);
  const bool reuse = verlet && h->vl_reuse && h->vl_valid && h->vl_gen == h->gen && h->vl_n == n;
  const int rad = g.rad, cpd_eff = g.cpd_eff;
  const bool fold = g.fold;
  const int n_cells = cpd_eff * cpd_eff * cpd_eff;
  const double edge = g.edge;
  if ((which & RS_CELLS) && reuse) {
    // the build's cells, order and lists; positions refreshed in build order
    k_verlet_gather<<<blocks_for(n, 256), 256, 0, h->stream>>>(
        h->xyzq.as<double4>(), h->order.as<int>(), h->vl_xb.as<double4>(), n, h->L,
        h->sorted.as<double4>(), h->sorted_f.as<float4>(), h->errflag.as<int>());
    CKL();
    if (ev_cell) CK(cudaEventRecord(ev_cell, h->stream));
  } else if (which & RS_CELLS) {
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
  if (verlet) {  // the build's positions: reference for displacements and images
    CK(h->vl_xb.ensure(n * sizeof(double4)));
    CK(cudaMemcpyAsync(h->vl_xb.p, h->sorted.p, n * sizeof(double4), cudaMemcpyDeviceToDevice,
                       h->stream));
  }
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
    // chain rounded once each); doubled and rounded up.  Verlet reuse:
    // positions lie within skin/2 < L/4 of [0, L), covered by 1.5 L
    const double rc_t = std::sqrt(rc2_t);
    const double Lm = verlet ? 1.5 * h->L : h->L;
    const double margin = std::ldexp(2.0 * (16.0 * Lm * rc_t + 8.0 * rc2_t), -24);
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
  if (!fold && rp.half && !verlet) {
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
  // one energy slot per work item (unit x split), zeroed before the pass:
  // items past the slab's real unit count are never written
  const int64_t n_eslots = (int64_t)nb * K6_WARPS;
  // two-pass real space: lists of 32-bit entries (j < 2^23), capacity per
  // unit twice the mean half-shell pair count of K6_G centres plus slack
  // two-pass real space: the Verlet lists, or the list/evaluation split on request
  const bool split = (verlet || h->rs_split) && !fold && n < ((int64_t)1 << K6_LIST_JBITS) &&
                     (verlet || rp.jsplit == 1);
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
  const int64_t n_esum = n_eslot_all;
  if (pair_coul || lj_on)
    CK(cudaMemsetAsync(h->eblk.p, 0, n_eslot_all * sizeof(double), h->stream));
  if (lj_on) CK(cudaMemsetAsync(h->eblk_lj.p, 0, n_eslot_all * sizeof(double), h->stream));
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
      // changes the evaluation; the traversal cutoff is in rp.rc2); a
      // reused Verlet build keeps its lists
      if (!reuse) {
        auto trav = rp.half ? k6_real_space<false, true, K6_MODE_LIST>
                            : k6_real_space<false, false, K6_MODE_LIST>;
        trav<<<nb, K6_WARPS * 32, 0, h->stream>>>(
            h->sorted.as<double4>(), h->sorted_f.as<float4>(), h->sorted_cell.as<int>(),
            h->order.as<int>(), h->start.as<int>(), h->row_ustart.as<int>(), rp,
            facc, nullptr, nullptr, h->errflag.as<int>(),
            h->pairc.as<unsigned long long>(), lists);
        CKL();
      }
      if (verlet) {
        if (reuse) {
          ++h->vl_reuses;
        } else {
          ++h->vl_builds;
          h->vl_valid = true;
          h->vl_gen = h->gen;
          h->vl_n = n;
        }
      }
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
  h->vl_reuse = false;  // every reuse needs a fresh ewb_dev_verlet_check
  if (!fold) {
    k_unpermute_add<<<blocks_for(n, 256), 256, 0, h->stream>>>(h->order.as<int>(),
                                                               h->fsorted.as<double>(), n, d_force);
    CKL();
  }
  if (pair_coul) {
    k_sum<<<1, 1024, 0, h->stream>>>(h->eblk.as<double>(), n_esum, 1.0, d_u_out);
    CKL();
  }
  if (lj_on && d_ulj_out) {
    k_sum<<<1, 1024, 0, h->stream>>>(h->eblk_lj.as<double>(), n_esum, 1.0, d_ulj_out);
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
  // Verlet lists switch between build and reuse launches: no graphs
  const bool graphs = h->use_graphs && !(h->skin > 0.0);
  const bool replay = graphs && h->gexec[0] && k == h->gkey;
  const bool capture = !replay && graphs && k == h->warm_key;
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

