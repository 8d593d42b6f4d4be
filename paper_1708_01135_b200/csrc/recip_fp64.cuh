// recip_fp64.cuh -- reciprocal space on the FP64 pipe (Algorithms 1 and 2:
// pair-item structure factor, finalize, force gathers, force combine).  Included by ewald_b200.cu inside its anonymous
// namespace (shared helpers: cmul, warp_sum, block_sum, constants).

// K1 inner loop for G particles at once (G independent recurrence chains).
// One pair item = the z-segments of (+|m_x|, m_y) and (-|m_x|, m_y): with
// YZ_m = q e^{-i(m_y th_y + m_z th_z)} (three-term recurrence along m_z),
// A+[m] += 2cos(m_x th_x) YZ_m and A-[m] += 2sin(m_x th_x) YZ_m, so that
// S(+-m_x) = (A+ -+ i A-)/2: 6 FP64 instructions per two k-vectors.
template <int M, int G>
__device__ __forceinline__ void k1_accumulate(double2 (&ap)[M], double2 (&am)[M],
                                              const double2 *t, int TSp, int4 it, int eidx) {
  double2 bp[G], bc[G];
  double c2[G], cx[G], sx[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const double2 *tg = t + g * TSp;
    const double2 e = tg[eidx];
    const double2 x = tg[it.z];  // 2 e^{-i |m_x| th_x}
    cx[g] = x.x;
    sx[g] = -x.y;
    bp[g] = cmul(tg[it.x], tg[it.y]);  // m = 0: q e^{-i s th_z} e^{-i m_y th_y}
    bc[g] = cmul(bp[g], e);            // m = 1
    c2[g] = e.x + e.x;                 // 2 cos(theta_z)
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
    ap[0].x = fma(cx[g], bp[g].x, ap[0].x);
    ap[0].y = fma(cx[g], bp[g].y, ap[0].y);
    am[0].x = fma(sx[g], bp[g].x, am[0].x);
    am[0].y = fma(sx[g], bp[g].y, am[0].y);
    if (M > 1) {
      ap[1].x = fma(cx[g], bc[g].x, ap[1].x);
      ap[1].y = fma(cx[g], bc[g].y, ap[1].y);
      am[1].x = fma(sx[g], bc[g].x, am[1].x);
      am[1].y = fma(sx[g], bc[g].y, am[1].y);
    }
  }
#pragma unroll
  for (int m = 2; m < M; ++m) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const double2 bn = make_double2(fma(c2[g], bc[g].x, -bp[g].x), fma(c2[g], bc[g].y, -bp[g].y));
      bp[g] = bc[g];
      bc[g] = bn;
      ap[m].x = fma(cx[g], bn.x, ap[m].x);
      ap[m].y = fma(cx[g], bn.y, ap[m].y);
      am[m].x = fma(sx[g], bn.x, am[m].x);
      am[m].y = fma(sx[g], bn.y, am[m].y);
    }
  }
}

// ---------------------------------------------------------------------------
// K1: structure factor.  Block = (k-tile of K1_THREADS items, particle chunk).
template <int M>
__global__ void __launch_bounds__(K1_THREADS)
    k1_structure_factor(const double4 *__restrict__ frac, const double2 *__restrict__ base,
                        int64_t p_begin, int64_t p_end, int64_t ppb, int pchunk,
                        const int4 *__restrict__ item_tab, int n_items,
                        const int4 *__restrict__ tab_desc, const int *__restrict__ tile_off,
                        const int *__restrict__ tile_ts, double4 *__restrict__ spart) {
  extern __shared__ double2 tab[];
  const int tile = blockIdx.x;
  const int item = tile * K1_THREADS + threadIdx.x;
  const bool valid = item < n_items;
  const int4 it = item_tab[valid ? item : n_items - 1];
  const int TS = tile_ts[tile];
  const int4 *desc = tab_desc + tile_off[tile];
  const int eidx = TS - 1;

  double2 ap[M], am[M];
#pragma unroll
  for (int m = 0; m < M; ++m) ap[m] = am[m] = make_double2(0.0, 0.0);

  const int64_t c_begin = p_begin + (int64_t)blockIdx.y * ppb;
  const int64_t c_end = min(p_end, c_begin + ppb);
  const int nch = (int)((c_end - c_begin + pchunk - 1) / pchunk);
  const int TSp = TS | 1;  // odd stride: conflict-free per-particle rows
  double2 *tabs[2] = {tab, tab + pchunk * TSp};
  int4 *s_desc = reinterpret_cast<int4 *>(tab + 2 * pchunk * TSp);
  for (int e = threadIdx.x; e < TS; e += K1_THREADS) s_desc[e] = desc[e];
  __syncthreads();

  // per-particle phase tables of this tile: rows q e^{-i(mx th_x + s th_z)},
  // columns e^{-i my th_y}, and e^{-i th_z} (last entry).  The np*TS entries
  // are split evenly over the block; each thread walks a contiguous run,
  // starting every run (and every unlinked entry) with one sincospi and
  // extending it by complex multiplication with the particle's axis phase.
  auto build = [&](const int k, double2 *dst) {
    const int64_t c0 = c_begin + (int64_t)k * pchunk;
    const int np = (int)min((int64_t)pchunk, c_end - c0);
    const int total = np * TS;
    const int per = (total + K1_THREADS - 1) / K1_THREADS;
    int t = threadIdx.x * per;
    const int t1 = min(total, t + per);
    if (t >= t1) return;
    int p = t / TS, e = t - p * TS;
    double4 f = frac[c0 + p];
    double2 bx = base[3 * (c0 + p)], by = base[3 * (c0 + p) + 1];
    double2 prev = make_double2(1.0, 0.0);
    bool fresh = true;
    for (; t < t1; ++t) {
      if (e == TS) {
        e = 0;
        ++p;
        f = frac[c0 + p];
        bx = base[3 * (c0 + p)];
        by = base[3 * (c0 + p) + 1];
        fresh = true;
      }
      const int4 d = s_desc[e];
      double2 v;
      if (fresh || !(d.w & TF_LINK)) {
        const double arg = (double)d.x * f.x + (double)d.y * f.y + (double)d.z * f.z;
        double sn, cs;
        sincospi(2.0 * arg, &sn, &cs);
        v = make_double2(cs, -sn);
        const double sc = (d.w & TF_QSCALE) ? f.w : ((d.w & TF_SCALE2) ? 2.0 : 1.0);
        v.x *= sc;
        v.y *= sc;
      } else {
        v = cmul(prev, ((d.w >> 2) & 3) ? by : bx);
      }
      dst[p * TSp + e] = v;
      prev = v;
      fresh = false;
      ++e;
    }
  };

  if (nch > 0) build(0, tabs[0]);
  __syncthreads();
  for (int k = 0; k < nch; ++k) {
    // the next chunk's table is built by the same warps while (or before)
    // they consume this one; warps that finish early start computing, so the
    // latency-bound build overlaps other warps' FP64 work
    if (k + 1 < nch) build(k + 1, tabs[(k + 1) & 1]);
    const double2 *tab_k = tabs[k & 1];
    const int np = (int)min((int64_t)pchunk, c_end - (c_begin + (int64_t)k * pchunk));
    int p = 0;
    for (; p + K1_ILP <= np; p += K1_ILP)
      k1_accumulate<M, K1_ILP>(ap, am, tab_k + p * TSp, TSp, it, eidx);
    for (; p < np; ++p) k1_accumulate<M, 1>(ap, am, tab_k + p * TSp, TSp, it, eidx);
    __syncthreads();
  }
  if (valid) {
    double4 *out = spart + (size_t)blockIdx.y * M * n_items + item;
#pragma unroll
    for (int m = 0; m < M; ++m)
      out[(size_t)m * n_items] = make_double4(ap[m].x, ap[m].y, am[m].x, am[m].y);
  }
}

// K2: reduce particle-chunk partials; optionally finalize (rho scatter,
// C*S for the gather, energy partials).
__global__ void __launch_bounds__(RED_THREADS)
    k2_finalize(const double2 *__restrict__ spart, int n_part, int64_t n_slots,
                const int *__restrict__ slot_k, const double *__restrict__ slot_coeff, int64_t K,
                double *__restrict__ rho_out, double2 *__restrict__ s_out,
                double2 *__restrict__ sp, double *__restrict__ epart, int finalize) {
  __shared__ double sh[RED_THREADS / 32];
  const int64_t s = blockIdx.x * (int64_t)RED_THREADS + threadIdx.x;
  double e = 0.0;
  if (s < n_slots) {
    double2 S = make_double2(0.0, 0.0);
    int pc = 0;
    for (; pc + 8 <= n_part; pc += 8) {  // 8 independent loads in flight
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcs(spart + (size_t)(pc + u) * n_slots + s);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        S.x += v[u].x;
        S.y += v[u].y;
      }
    }
    for (; pc < n_part; ++pc) {
      const double2 v = __ldcs(spart + (size_t)pc * n_slots + s);
      S.x += v.x;
      S.y += v.y;
    }
    if (s_out) s_out[s] = S;
    if (finalize) {
      const int k = slot_k[s];
      if (k >= 0) {
        if (rho_out) {
          rho_out[k] = S.x;
          rho_out[K + k] = S.y;
        }
        const double C = slot_coeff[s];
        sp[s] = make_double2(C * S.x, C * S.y);
        e = C * (S.x * S.x + S.y * S.y);
      } else {
        sp[s] = make_double2(0.0, 0.0);
      }
    }
  }
  if (finalize) {
    const double b = block_sum<RED_THREADS>(e, sh);
    if (threadIdx.x == 0) epart[blockIdx.x] = b;
  }
}

// K2 for the K1 pair layout: sum particle-chunk partials (A+, A-) of a pair
// slot, S(+-m_x) = (A+ -+ i A-)/2, scatter rho to the caller's k order, C*S to
// the gather's slot layout, and u_lr partials.  finalize=0: only the summed
// pair slots (multi-GPU partial S before the all-reduce).
#ifndef K2P_THREADS
#define K2P_THREADS 64  // small blocks: the slots spread over every SM (c2: 54 -> 216 blocks)
#endif
// finalisation of one summed pair slot A = (A+, A-): S(+-m_x), rho into the
// caller's k order, C*S into the gather's layout; returns its C |S|^2
__device__ __forceinline__ double k2p_emit(const double4 A, int64_t s,
                                           const int4 *__restrict__ pmap,
                                           const double *__restrict__ slot_coeff, int64_t K,
                                           double *__restrict__ rho_out,
                                           double2 *__restrict__ sp) {
  double e = 0.0;
  const int4 mp = pmap[s];
  const double2 Sp_ = make_double2(0.5 * (A.x + A.w), 0.5 * (A.y - A.z));  // +m_x
  const double2 Sm_ = make_double2(0.5 * (A.x - A.w), 0.5 * (A.y + A.z));  // -m_x
  if (mp.x >= 0) {
    if (rho_out) {
      rho_out[mp.x] = Sp_.x;
      rho_out[K + mp.x] = Sp_.y;
    }
    const double C = slot_coeff[mp.z];
    sp[mp.z] = make_double2(C * Sp_.x, C * Sp_.y);
    e += C * (Sp_.x * Sp_.x + Sp_.y * Sp_.y);
  }
  if (mp.y >= 0) {
    if (rho_out) {
      rho_out[mp.y] = Sm_.x;
      rho_out[K + mp.y] = Sm_.y;
    }
    const double C = slot_coeff[mp.w];
    sp[mp.w] = make_double2(C * Sm_.x, C * Sm_.y);
    e += C * (Sm_.x * Sm_.x + Sm_.y * Sm_.y);
  }
  return e;
}

// The ranks' S(k) partials (pair-slot layout) summed straight from their
// buffers -- peer memory over NVLink (or the same device) -- in rank order,
// then finalised: the all-reduce and the finalisation in ONE kernel.  Every
// rank runs it over the same pointers, so every rank gets bitwise the same S.
constexpr int K2P_MAX_PEERS = 16;
struct PeerSlots {
  const double4 *p[K2P_MAX_PEERS];
  int n;
};
__global__ void __launch_bounds__(K2P_THREADS)
    k2p_finalize_peer(PeerSlots parts, int64_t n_pslots, const int4 *__restrict__ pmap,
                      const double *__restrict__ slot_coeff, int64_t K,
                      double *__restrict__ rho_out, double2 *__restrict__ sp,
                      double *__restrict__ epart) {
  __shared__ double sh[K2P_THREADS / 32];
  const int64_t s = blockIdx.x * (int64_t)K2P_THREADS + threadIdx.x;
  double e = 0.0;
  if (s < n_pslots) {
    double4 v[K2P_MAX_PEERS];
#pragma unroll
    for (int r = 0; r < K2P_MAX_PEERS; ++r)
      if (r < parts.n) v[r] = ldcs4(parts.p[r] + s);
    double4 A = make_double4(0.0, 0.0, 0.0, 0.0);
#pragma unroll
    for (int r = 0; r < K2P_MAX_PEERS; ++r) {
      if (r < parts.n) {
        A.x += v[r].x;
        A.y += v[r].y;
        A.z += v[r].z;
        A.w += v[r].w;
      }
    }
    e = k2p_emit(A, s, pmap, slot_coeff, K, rho_out, sp);
  }
  const double b = block_sum<K2P_THREADS>(e, sh);
  if (threadIdx.x == 0) epart[blockIdx.x] = b;
}
__global__ void __launch_bounds__(K2P_THREADS)
    k2p_finalize(const double4 *__restrict__ spart, int n_part, int64_t n_pslots,
                 const int4 *__restrict__ pmap, const double *__restrict__ slot_coeff, int64_t K,
                 double *__restrict__ rho_out, double4 *__restrict__ s_out,
                 double2 *__restrict__ sp, double *__restrict__ epart, int finalize) {
  __shared__ double sh[K2P_THREADS / 32];
  const int64_t s = blockIdx.x * (int64_t)K2P_THREADS + threadIdx.x;
  double e = 0.0;
  if (s < n_pslots) {
    double4 A = make_double4(0.0, 0.0, 0.0, 0.0);
    int pc = 0;
    for (; pc + 8 <= n_part; pc += 8) {
      double4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = ldcs4(spart + (size_t)(pc + u) * n_pslots + s);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        A.x += v[u].x;
        A.y += v[u].y;
        A.z += v[u].z;
        A.w += v[u].w;
      }
    }
    for (; pc < n_part; ++pc) {
      const double4 v = ldcs4(spart + (size_t)pc * n_pslots + s);
      A.x += v.x;
      A.y += v.y;
      A.z += v.z;
      A.w += v.w;
    }
    if (s_out) s_out[s] = A;
    if (finalize) e = k2p_emit(A, s, pmap, slot_coeff, K, rho_out, sp);
  }
  if (finalize) {
    const double b = block_sum<K2P_THREADS>(e, sh);
    if (threadIdx.x == 0) epart[blockIdx.x] = b;
  }
}

// Deterministic single-block sum of an array into out[0].

// ---------------------------------------------------------------------------
// K3: reciprocal force gather.  Block = (K3_THREADS*K3_PPT particles, k-split).
__device__ __forceinline__ double2 phase_plus(int mx, int my, int s, double tx, double ty,
                                              double tz) {
  const double arg = (double)mx * tx + (double)my * ty + (double)s * tz;
  double sn, cs;
  sincospi(2.0 * arg, &sn, &cs);
  return make_double2(cs, sn);
}

#ifndef K3_MINB
#define K3_MINB 4
#endif
template <int M, bool ENERGY>
__global__ void __launch_bounds__(K3_THREADS, K3_MINB)
    k3_force_gather(const double4 *__restrict__ frac, const double2 *__restrict__ base,
                    int64_t p_begin, int64_t p_end, const int4 *__restrict__ rows,
                    const int *__restrict__ ks_rows, const int *__restrict__ item_my,
                    const int *__restrict__ item_row, const double2 *__restrict__ sp, int n_items,
                    double *__restrict__ fpart, double *__restrict__ upart) {
  __shared__ double2 s_spb[2][K3_CH * M];
  __shared__ int s_myb[2][K3_CH];
  __shared__ int s_rowb[2][K3_CH];
  const int64_t n_local = p_end - p_begin;
  const int ks = blockIdx.y;
  const int r_begin = ks_rows[ks], r_end = ks_rows[ks + 1];

  int64_t pi[K3_PPT];
  double tx[K3_PPT], ty[K3_PPT], tz[K3_PPT], c2z[K3_PPT];
  double2 ey[K3_PPT], ez[K3_PPT], P[K3_PPT];
  double Fx[K3_PPT], Fy[K3_PPT], Fz[K3_PPT], U[K3_PPT], SG[K3_PPT], SY[K3_PPT], SH[K3_PPT];
#pragma unroll
  for (int q = 0; q < K3_PPT; ++q) {
    pi[q] = (int64_t)blockIdx.x * (K3_THREADS * K3_PPT) + q * K3_THREADS + threadIdx.x;
    const int64_t g = p_begin + (pi[q] < n_local ? pi[q] : 0);
    const double4 f = frac[g];
    tx[q] = f.x;
    ty[q] = f.y;
    tz[q] = f.z;
    const double2 by = base[3 * g + 1], bz = base[3 * g + 2];
    ey[q] = make_double2(by.x, -by.y);
    ez[q] = make_double2(bz.x, -bz.y);
    c2z[q] = bz.x + bz.x;
    Fx[q] = Fy[q] = Fz[q] = U[q] = SG[q] = SY[q] = SH[q] = 0.0;
    P[q] = make_double2(1.0, 0.0);
  }

  int cur_row = -1, pmy = 0, cmx = 0, cs = 0;
  if (r_begin < r_end) {
    const int i_first = rows[r_begin].z;
    const int4 rl = rows[r_end - 1];
    const int i_last = rl.z + rl.w;
    // C_k S_k chunks are double-buffered through registers: chunk k+1 is
    // fetched from L2 before chunk k is consumed and stored after it
    constexpr int NPT = (K3_CH * M + K3_THREADS - 1) / K3_THREADS;
    double2 stage_sp[NPT];
    int stage_my = 0, stage_row = 0;
    auto fetch = [&](const int c0) {
      const int nc = min(K3_CH, i_last - c0);
#pragma unroll
      for (int u = 0; u < NPT; ++u) {
        const int t = threadIdx.x + u * K3_THREADS;
        if (t < nc * M) stage_sp[u] = sp[(size_t)c0 * M + t];
      }
      if (threadIdx.x < nc) {
        stage_my = item_my[c0 + threadIdx.x];
        stage_row = item_row[c0 + threadIdx.x];
      }
    };
    auto commit = [&](const int c0, const int b) {
      const int nc = min(K3_CH, i_last - c0);
#pragma unroll
      for (int u = 0; u < NPT; ++u) {
        const int t = threadIdx.x + u * K3_THREADS;
        if (t < nc * M) s_spb[b][t] = stage_sp[u];
      }
      if (threadIdx.x < nc) {
        s_myb[b][threadIdx.x] = stage_my;
        s_rowb[b][threadIdx.x] = stage_row;
      }
    };
    fetch(i_first);
    commit(i_first, 0);
    __syncthreads();
    int kb = 0;
    for (int c0 = i_first; c0 < i_last; c0 += K3_CH, kb ^= 1) {
      const int nc = min(K3_CH, i_last - c0);
      const bool more = c0 + K3_CH < i_last;
      if (more) fetch(c0 + K3_CH);
      const double2 *s_sp = s_spb[kb];
      const int *s_my = s_myb[kb];
      const int *s_row = s_rowb[kb];
      for (int itc = 0; itc < nc; ++itc) {
        const int row = s_row[itc], my = s_my[itc];
        if (row != cur_row) {
          if (cur_row >= 0) {
#pragma unroll
            for (int q = 0; q < K3_PPT; ++q) {
              Fx[q] = fma((double)cmx, SG[q], Fx[q]);
              Fy[q] += SY[q];
              Fz[q] += fma((double)(cs + M), SG[q], -SH[q]);
              SG[q] = SY[q] = SH[q] = 0.0;
            }
          }
          const int4 r = rows[row];
          cmx = r.x;
          cs = r.y;
          cur_row = row;
#pragma unroll
          for (int q = 0; q < K3_PPT; ++q) P[q] = phase_plus(cmx, my, cs, tx[q], ty[q], tz[q]);
        } else if (my != pmy + 1) {
#pragma unroll
          for (int q = 0; q < K3_PPT; ++q) P[q] = phase_plus(cmx, my, cs, tx[q], ty[q], tz[q]);
        } else {
#pragma unroll
          for (int q = 0; q < K3_PPT; ++q) P[q] = cmul(P[q], ey[q]);
        }
        pmy = my;
        const double2 *spi = s_sp + itc * M;
        double2 Ap[K3_PPT], Ac[K3_PPT];
        double G[K3_PPT], H[K3_PPT];
        {
          const double2 s0 = spi[0];
#pragma unroll
          for (int q = 0; q < K3_PPT; ++q) {
            Ap[q] = P[q];
            G[q] = fma(Ap[q].x, s0.y, Ap[q].y * s0.x);
            H[q] = G[q];
            if (ENERGY) U[q] = fma(Ap[q].x, s0.x, fma(-Ap[q].y, s0.y, U[q]));
          }
        }
        if (M > 1) {
          const double2 s1 = spi[1];
#pragma unroll
          for (int q = 0; q < K3_PPT; ++q) {
            Ac[q] = cmul(P[q], ez[q]);
            G[q] = fma(Ac[q].x, s1.y, fma(Ac[q].y, s1.x, G[q]));
            H[q] += G[q];
            if (ENERGY) U[q] = fma(Ac[q].x, s1.x, fma(-Ac[q].y, s1.y, U[q]));
          }
#pragma unroll
          for (int m = 2; m < M; ++m) {
            const double2 sm = spi[m];
#pragma unroll
            for (int q = 0; q < K3_PPT; ++q) {
              const double2 An = make_double2(fma(c2z[q], Ac[q].x, -Ap[q].x),
                                              fma(c2z[q], Ac[q].y, -Ap[q].y));
              Ap[q] = Ac[q];
              Ac[q] = An;
              G[q] = fma(An.x, sm.y, fma(An.y, sm.x, G[q]));
              H[q] += G[q];
              if (ENERGY) U[q] = fma(An.x, sm.x, fma(-An.y, sm.y, U[q]));
            }
          }
        }
#pragma unroll
        for (int q = 0; q < K3_PPT; ++q) {
          SG[q] += G[q];
          SY[q] = fma((double)my, G[q], SY[q]);
          SH[q] += H[q];
        }
      }
      if (more) commit(c0 + K3_CH, kb ^ 1);
      __syncthreads();
    }
    if (cur_row >= 0) {
#pragma unroll
      for (int q = 0; q < K3_PPT; ++q) {
        Fx[q] = fma((double)cmx, SG[q], Fx[q]);
        Fy[q] += SY[q];
        Fz[q] += fma((double)(cs + M), SG[q], -SH[q]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < K3_PPT; ++q) {
    if (pi[q] < n_local) {
      double *fp = fpart + (size_t)ks * 3 * n_local;
      fp[pi[q]] = Fx[q];
      fp[n_local + pi[q]] = Fy[q];
      fp[2 * n_local + pi[q]] = Fz[q];
      if (ENERGY) upart[(size_t)ks * n_local + pi[q]] = U[q];
    }
  }
}

// K3c: the force gather with C*S and the item metadata in the CONSTANT bank.
// Every thread of a warp reads the same C*S entry, so with a warp-uniform
// constant-bank index the operand lives in uniform registers (LDCU -> DFMA
// ..., URx, ...), relieving the vector register file, whose operand
// bandwidth bounds the shared-memory variant (measured: +27% FP64
// throughput on the K3 inner loop, tools/micro/fp64uniform.cu).  The
// k-space is walked in chunks of <= K3C_CAP slots, one launch per chunk
// (copy-to-symbol is stream ordered); partial rows are flushed at chunk
// ends and forces accumulate across launches.
// Two buffers (A/B) on two streams: consecutive chunks alternate, so one
// launch's partial last wave overlaps the next launch.
constexpr int K3C_CAP = 1700;    // C*S slots per chunk buffer (27.2 KB)
constexpr int K3C_ITEMS = 160;   // items per chunk (metadata)
__constant__ double2 c_k3sp[2][K3C_CAP];
__constant__ int4 c_k3meta[2][K3C_ITEMS];  // (m_x, s, m_y, flags: 1 new row, 2 m_y jump)

template <int M, bool ENERGY, int BUF>
__global__ void __launch_bounds__(K3_THREADS, K3_MINB)
    k3c_force_gather(const double4 *__restrict__ frac, const double2 *__restrict__ base,
                     int64_t p_begin, int64_t p_end, int nc, int first,
                     double *__restrict__ fpart, double *__restrict__ upart) {
  const int64_t n_local = p_end - p_begin;
  int64_t pi[K3_PPT];
  double tx[K3_PPT], ty[K3_PPT], tz[K3_PPT], c2z[K3_PPT];
  double2 ey[K3_PPT], ez[K3_PPT], P[K3_PPT];
  double Fx[K3_PPT], Fy[K3_PPT], Fz[K3_PPT], U[K3_PPT], SG[K3_PPT], SY[K3_PPT], SH[K3_PPT];
#pragma unroll
  for (int q = 0; q < K3_PPT; ++q) {
    pi[q] = (int64_t)blockIdx.x * (K3_THREADS * K3_PPT) + q * K3_THREADS + threadIdx.x;
    const int64_t g = p_begin + (pi[q] < n_local ? pi[q] : 0);
    const double4 f = frac[g];
    tx[q] = f.x;
    ty[q] = f.y;
    tz[q] = f.z;
    const double2 by = base[3 * g + 1], bz = base[3 * g + 2];
    ey[q] = make_double2(by.x, -by.y);
    ez[q] = make_double2(bz.x, -bz.y);
    c2z[q] = bz.x + bz.x;
    Fx[q] = Fy[q] = Fz[q] = U[q] = SG[q] = SY[q] = SH[q] = 0.0;
    P[q] = make_double2(1.0, 0.0);
  }
  int cmx = 0, cs = 0;
  for (int itc = 0; itc < nc; ++itc) {
    const int4 mt = c_k3meta[BUF][itc];
    const int my = mt.z;
    if (itc == 0 || (mt.w & 1)) {
      if (itc > 0) {
#pragma unroll
        for (int q = 0; q < K3_PPT; ++q) {
          Fx[q] = fma((double)cmx, SG[q], Fx[q]);
          Fy[q] += SY[q];
          Fz[q] += fma((double)(cs + M), SG[q], -SH[q]);
          SG[q] = SY[q] = SH[q] = 0.0;
        }
      }
      cmx = mt.x;
      cs = mt.y;
#pragma unroll
      for (int q = 0; q < K3_PPT; ++q) P[q] = phase_plus(cmx, my, cs, tx[q], ty[q], tz[q]);
    } else if (mt.w & 2) {
#pragma unroll
      for (int q = 0; q < K3_PPT; ++q) P[q] = phase_plus(cmx, my, cs, tx[q], ty[q], tz[q]);
    } else {
#pragma unroll
      for (int q = 0; q < K3_PPT; ++q) P[q] = cmul(P[q], ey[q]);
    }
    const double2 *spi = c_k3sp[BUF] + itc * M;
    double2 Ap[K3_PPT], Ac[K3_PPT];
    double G[K3_PPT], H[K3_PPT];
    {
      const double2 s0 = spi[0];
#pragma unroll
      for (int q = 0; q < K3_PPT; ++q) {
        Ap[q] = P[q];
        G[q] = fma(Ap[q].x, s0.y, Ap[q].y * s0.x);
        H[q] = G[q];
        if (ENERGY) U[q] = fma(Ap[q].x, s0.x, fma(-Ap[q].y, s0.y, U[q]));
      }
    }
    if (M > 1) {
      const double2 s1 = spi[1];
#pragma unroll
      for (int q = 0; q < K3_PPT; ++q) {
        Ac[q] = cmul(P[q], ez[q]);
        G[q] = fma(Ac[q].x, s1.y, fma(Ac[q].y, s1.x, G[q]));
        H[q] += G[q];
        if (ENERGY) U[q] = fma(Ac[q].x, s1.x, fma(-Ac[q].y, s1.y, U[q]));
      }
#pragma unroll
      for (int m = 2; m < M; ++m) {
        const double2 sm = spi[m];
#pragma unroll
        for (int q = 0; q < K3_PPT; ++q) {
          const double2 An = make_double2(fma(c2z[q], Ac[q].x, -Ap[q].x),
                                          fma(c2z[q], Ac[q].y, -Ap[q].y));
          Ap[q] = Ac[q];
          Ac[q] = An;
          G[q] = fma(An.x, sm.y, fma(An.y, sm.x, G[q]));
          H[q] += G[q];
          if (ENERGY) U[q] = fma(An.x, sm.x, fma(-An.y, sm.y, U[q]));
        }
      }
    }
#pragma unroll
    for (int q = 0; q < K3_PPT; ++q) {
      SG[q] += G[q];
      SY[q] = fma((double)my, G[q], SY[q]);
      SH[q] += H[q];
    }
  }
  if (nc > 0) {
#pragma unroll
    for (int q = 0; q < K3_PPT; ++q) {
      Fx[q] = fma((double)cmx, SG[q], Fx[q]);
      Fy[q] += SY[q];
      Fz[q] += fma((double)(cs + M), SG[q], -SH[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < K3_PPT; ++q) {
    if (pi[q] < n_local) {
      double *fx = fpart + pi[q], *fy = fpart + n_local + pi[q], *fz = fpart + 2 * n_local + pi[q];
      if (first) {
        *fx = Fx[q];
        *fy = Fy[q];
        *fz = Fz[q];
        if (ENERGY) upart[pi[q]] = U[q];
      } else {
        *fx += Fx[q];
        *fy += Fy[q];
        *fz += Fz[q];
        if (ENERGY) upart[pi[q]] += U[q];
      }
    }
  }
}

// Combine k-split partial forces: force[i] += (4 pi / L) q_i sum_ks F.
__global__ void __launch_bounds__(RED_THREADS)
    k3_combine(const double *__restrict__ fpart, const double *__restrict__ upart, int n_ks,
               int64_t p_begin, int64_t n_local, const double4 *__restrict__ frac, double scale,
               double *__restrict__ force, double *__restrict__ eblk, int energy) {
  __shared__ double sh[RED_THREADS / 32];
  const int64_t i = blockIdx.x * (int64_t)RED_THREADS + threadIdx.x;
  double e = 0.0;
  if (i < n_local) {
    double fx = 0.0, fy = 0.0, fz = 0.0, u = 0.0;
#pragma unroll 4
    for (int ks = 0; ks < n_ks; ++ks) {
      const double *fp = fpart + (size_t)ks * 3 * n_local;
      fx += __ldcs(fp + i);
      fy += __ldcs(fp + n_local + i);
      fz += __ldcs(fp + 2 * n_local + i);
      if (energy) u += upart[(size_t)ks * n_local + i];
    }
    const int64_t g = p_begin + i;
    const double qi = frac[g].w;
    const double sq = scale * qi;
    force[3 * g] += sq * fx;
    force[3 * g + 1] += sq * fy;
    force[3 * g + 2] += sq * fz;
    e = qi * u;
  }
  if (energy) {
    const double b = block_sum<RED_THREADS>(e, sh);
    if (threadIdx.x == 0) eblk[blockIdx.x] = b;
  }
}

