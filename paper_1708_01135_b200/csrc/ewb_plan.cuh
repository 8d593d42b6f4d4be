// ewb_plan.cuh -- host planning of the k-space work:
// pair items, yz runs, tensor-core tiles and slot maps for any m_int table.
// Included by ewald_b200.cu inside its anonymous namespace (after the handle).

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

