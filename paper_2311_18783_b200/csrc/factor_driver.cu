// Host drivers of the multifrontal factorisation and the level-scheduled
// supernodal triangular solves (kernels in kernels.cu).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <queue>

#include <cublas_v2.h>
#include <cusolverDn.h>

#include "device.h"

namespace mdd {


dev::PlanDev DevFactor::plan() const {
  dev::PlanDev P;
  P.sn_col0 = (const long long*)col0.p;
  P.sn_ncol = ncol.p;
  P.sn_noff = noff.p;
  P.sn_rowptr = (const long long*)rowptr.p;
  P.offrows = (const long long*)offrows.p;
  P.sn_lptr = (const long long*)lptr.p;
  P.sn_uptr = (const long long*)uptr.p;
  P.sn_fptr = (const long long*)fptr.p;
  P.sn_umptr = (const long long*)umptr.p;
  P.child_ptr = (const long long*)child_ptr.p;
  P.child_list = child_list.p;
  P.relmap = relmap.p;
  P.asm_ptr = (const long long*)asm_ptr.p;
  P.asm_src = (const long long*)asm_src.p;
  P.asm_pos = asm_pos.p;
  P.level_sn = level_sn.p;
  return P;
}

void DevFactor::upload(int prolong_n, const int64_t* pro_ptr_dev, const int32_t* pro_pos_dev,
                       const std::vector<int32_t>* gmap_host) {
  MDD_REQUIRE(role.empty() || (int)role.size() == fp.nsn, 5, "sweep roles: one per supernode");
  if (!base) {
  col0.upload(fp.sn_col0);
  ncol.upload(fp.sn_ncol);
  noff.upload(fp.sn_noff);
  rowptr.upload(fp.sn_rowptr);
  offrows.upload(fp.offrows);
  lptr.upload(fp.sn_lptr);
  uptr.upload(fp.sn_uptr);
  fptr.upload(fp.sn_fptr);
  umptr.upload(fp.sn_umptr);
  child_ptr.upload(fp.child_ptr);
  child_list.upload(fp.child_list);
  relmap.upload(fp.relmap);
  asm_ptr.upload(fp.asm_ptr);
  asm_src.upload(fp.asm_src);
  asm_pos.upload(fp.asm_pos);
  level_sn.upload(fp.level_sn);
  parent.upload(fp.sn_parent);
  L.alloc(fp.lsize);
  dinv.alloc(fp.ntot);
  }  // a view sweeps its base's factor (tiles, D^{-1}): no plan arrays, no panels
  upd.alloc(std::max<int64_t>(fp.usize, 1));
  xf.alloc(std::max<int64_t>(fp.ntot, 1));
  xb.alloc(std::max<int64_t>(fp.ntot, 1));
  // ---- tile geometry.  small: one CTA sweeps the whole panel (column tiles over
  // all nr rows, accumulated in shared memory).  strip (big, nr <= kVecMax):
  // forward row strips x all columns and backward all rows x column strips (two
  // copies of the panel; no partial sums).  2-D (nr > kVecMax): RB x CB tiles
  // whose partial sums the last tile of a row / column block combines.
  // tiles[] = {g, a, b, kind}: kind 0 = 2-D (a = rb, b = cb), 1 = forward strip
  // (a = first row, b = rows), 2 = backward strip (a = columns, b = first column),
  // 3 = small column tile
  const int nsn = fp.nsn;
  std::vector<int> vRB(nsn), vCB(nsn), vnrb(nsn, 1), vncb(nsn, 1);
  std::vector<uint8_t> mode(nsn);  // 0 small, 1 strip, 2 2-D
  std::vector<int64_t> vfp(nsn, 0), vbp(nsn, 0);
  std::vector<std::vector<int>> ft(nsn), bt(nsn);  // forward / backward tiles (2-D: same list)
  std::vector<int4> tl;
  std::vector<int2> rc;  // rows x cols of each tile
  std::vector<int64_t> toff;
  int64_t off = 0, nfp = 0, nbp = 0;
  auto add_tile = [&](int4 t, int rows, int cols) {
    tl.push_back(t);
    rc.push_back(make_int2(rows, cols));
    toff.push_back(off);
    off += ((int64_t)rows * cols + 1) & ~1LL;  // 16-byte aligned tiles
    return (int)tl.size() - 1;
  };
  const int64_t single_max = getenv("MDD_SINGLE_MAX") ? atoll(getenv("MDD_SINGLE_MAX")) : dev::kSingleMax;
  const int env_cb = getenv("MDD_TILE_CB") ? std::max(8, atoi(getenv("MDD_TILE_CB"))) : 64;  // 2-D tile columns
  for (int g = 0; g < nsn; ++g) {
    const int nc = fp.sn_ncol[g], nr = nc + fp.sn_noff[g];
    // a supernode one CTA sweeps alone must stay short (it is a phase's critical path
    // on the upper, latency-bound levels): at most ~kSingleMax stored entries
    mode[g] = nr <= dev::kVecMax ? ((int64_t)nr * nc <= single_max ? 0 : 1) : 2;
    if (mode[g] == 1 && getenv("MDD_FORCE_2D")) mode[g] = 2;  // debug: no strips
    if (mode[g] == 0) {
      // packed column tiles (no zeros above the diagonal), as many columns as fit
      vRB[g] = nr; vCB[g] = nc;
      for (int c0 = 0; c0 < nc;) {
        int cols = 0;
        int64_t sz = 0;
        while (c0 + cols < nc && sz + (nr - c0 - cols) <= dev::kTileMax) { sz += nr - c0 - cols; ++cols; }
        MDD_REQUIRE(cols > 0, 5, "small supernode column does not fit a tile");
        ft[g].push_back(add_tile(make_int4(g, cols, c0, 3), (int)sz, 1));
        c0 += cols;
      }
      bt[g] = ft[g];
    } else if (mode[g] == 1) {
      // strips store only the lower trapezoid they touch: forward row strip
      // [r0, r0+rows) x columns [0, min(nc, r0+rows)), backward column strip
      // [c0, c0+cols) x rows [c0, nr) (the panel is zero above its diagonal); as
      // many rows / columns per tile as fit kTileMax
      vRB[g] = nr; vCB[g] = nc;
      for (int r0 = 0; r0 < nr;) {
        int rows = 1;
        while (r0 + rows < nr && (int64_t)(rows + 1) * std::min(nc, r0 + rows + 1) <= dev::kTileMax) ++rows;
        ft[g].push_back(add_tile(make_int4(g, r0, rows, 1), rows, std::min(nc, r0 + rows)));
        r0 += rows;
      }
      for (int c0 = 0; c0 < nc;) {
        int cols = 1;
        while (c0 + cols < nc && (int64_t)(cols + 1) * (nr - c0) <= dev::kTileMax) ++cols;
        bt[g].push_back(add_tile(make_int4(g, cols, c0, 2), nr - c0, cols));
        c0 += cols;
      }
    } else {
      // a task's vector (up to kGroup row blocks / column blocks) must fit a
      // kVecMax shared-memory slot: RB, CB <= kVecMax / kGroup
      const int CB = std::min(nc, env_cb);
      // an odd row count keeps the column-strided reads of the forward 2-D tiles
      // (lanes down the columns, stride RB) free of shared-memory bank conflicts
      int RB = std::max(1, std::min(dev::kVecMax / 4, dev::kTileMax / CB));
      if (RB > 1 && !(RB & 1)) --RB;
      const int nrb = (nr + RB - 1) / RB, ncb = (nc + CB - 1) / CB;
      vRB[g] = RB; vCB[g] = CB; vnrb[g] = nrb; vncb[g] = ncb;
      vfp[g] = nfp; nfp += (int64_t)ncb * nr;   // sized for groups of one tile
      vbp[g] = nbp; nbp += (int64_t)nrb * nc;
      for (int rb = 0; rb < nrb; ++rb) {
        const int rend = std::min(nr, (rb + 1) * RB), rows = rend - rb * RB;
        for (int cb = 0; cb < ncb && cb * CB < rend; ++cb)
          ft[g].push_back(add_tile(make_int4(g, rb, cb, 0), rows, std::min(CB, nc - cb * CB)));
      }
      bt[g] = ft[g];
    }
  }
  ntiles = (int)tl.size();
  lt_size = off;
  n_packed = n_strip = n_2d = 0;
  for (int g = 0; g < nsn; ++g) (mode[g] == 0 ? n_packed : mode[g] == 1 ? n_strip : n_2d)++;
  auto tile_bytes = [&](int t) {
    return (int)((((int64_t)rc[t].x * rc[t].y + 1) & ~1LL) * (int64_t)sizeof(double));
  };
  // ---- plan levels: the supernodes each level's phases sweep, in forward order.
  // Whole factor: the factor's levels.  With roles (a rank of the sharded coarse
  // solve): the levels of the rank's subtrees (role 1, segment A), then the levels
  // of the replicated top (role 2, segment B); role 0 is not swept.
  std::vector<std::vector<int>> plev;
  int nlev_a = 0;
  for (int seg = 0; seg < (role.empty() ? 1 : 2); ++seg) {
    for (int l = 0; l < fp.nlevels; ++l) {
      std::vector<int> v;
      for (int k = fp.level_ptr[l]; k < fp.level_ptr[l + 1]; ++k) {
        const int g = fp.level_sn[k];
        if (role.empty() || role[g] == seg + 1) v.push_back(g);
      }
      if (!v.empty() || role.empty()) plev.push_back(std::move(v));
    }
    if (!role.empty() && seg == 0) nlev_a = (int)plev.size();
  }
  const int NL = (int)plev.size();
  // ---- per-level row vectors: rows of g at vb_off[g], each level contiguous
  std::vector<int64_t> vvo(nsn, 0), lev_row(NL + 1, 0);
  int64_t nrows = 0;
  for (int l = 0; l < NL; ++l) {
    lev_row[l] = nrows;
    for (const int g : plev[l]) {
      vvo[g] = nrows;
      nrows += fp.sn_ncol[g] + fp.sn_noff[g];
    }
  }
  lev_row[NL] = nrows;
  // forward gather: row -> b index (column rows) and children's update entries
  std::vector<int32_t> vgsrc(nrows, -1);
  std::vector<int64_t> vwsrc(nrows);
  std::vector<std::vector<int64_t>> contrib(nrows);
  for (int g = 0; g < nsn; ++g) {
    if (!role.empty() && !role[g]) continue;
    const int nc = fp.sn_ncol[g], no = fp.sn_noff[g];
    const int64_t c0 = fp.sn_col0[g];
    for (int r = 0; r < nc; ++r) {
      vgsrc[vvo[g] + r] = gmap_host ? (*gmap_host)[c0 + r] : (int32_t)(c0 + r);
      vwsrc[vvo[g] + r] = c0 + r;
    }
    for (int r = 0; r < no; ++r) vwsrc[vvo[g] + nc + r] = -(fp.offrows[fp.sn_rowptr[g] + r]) - 1;
    for (int64_t ci = fp.child_ptr[g]; ci < fp.child_ptr[g + 1]; ++ci) {
      const int c = fp.child_list[ci];
      for (int a = 0; a < fp.sn_noff[c]; ++a)
        contrib[vvo[g] + fp.relmap[fp.sn_rowptr[c] + a]].push_back(fp.sn_uptr[c] + a);
    }
  }
  std::vector<int64_t> vcptr(nrows + 1, 0), vcidx;
  for (int64_t q = 0; q < nrows; ++q) {
    vcidx.insert(vcidx.end(), contrib[q].begin(), contrib[q].end());
    vcptr[q + 1] = (int64_t)vcidx.size();
  }
  std::vector<std::vector<int64_t>>().swap(contrib);
  // ---- M tasks per level and direction (largest first), packed descriptors
  std::vector<dev::MTaskDesc> mtf, mtb;
  std::vector<int4> td;
  std::vector<int> lev_f(NL + 1, 0), lev_b(NL + 1, 0);
  std::vector<int> nreal[2] = {std::vector<int>(NL, 0), std::vector<int>(NL, 0)};  // tasks without padding
  // combine items (one per row block / column block of a 2-D supernode) per level
  std::vector<dev::CombDesc> cm;
  std::vector<int> cmf(NL + 1, 0), cmb_lev(NL + 1, 0);
  auto push_td = [&](int t) {
    // .x: tile id, or for packed small tiles first column | columns << 16 (the kernel
    // needs them per tile)
    const int x = tl[t].w == 3 ? (tl[t].z | (tl[t].y << 16)) : t;
    td.push_back(make_int4(x, tile_bytes(t), (int)(uint32_t)(toff[t] & 0xffffffffu), (int)(uint32_t)(toff[t] >> 32)));
  };
  auto set_vec = [](dev::MTaskDesc& X, int64_t lo, int64_t hi) {
    X.vlo2 = lo & ~1LL;
    X.voff = (int)(lo - X.vlo2);
    X.vbytes = (int)((((hi - X.vlo2) + 1) & ~1LL) * (int64_t)sizeof(double));
    X.vn = (int)(hi - lo);
  };
  // the fixed cost of one M task in byte equivalents (measured best of 12-64 KB on c1;
  // ~3 us of one CTA: task start, partial-sum store, atomic, combine)
  const int64_t kTaskCostBytes = getenv("MDD_TASK_COST") ? atoll(getenv("MDD_TASK_COST")) : 48 * 1024;
  struct Cand {
    int64_t bytes;
    dev::MTaskDesc d;
    std::vector<int> tiles;
  };
  // persistent grid (needed to size the 2-D tile groups; plan_grid, the full
  // resident grid, fixes the grouping and hence the summation order even when
  // MDD_SWEEP_GRID runs fewer CTAs)
  int plan_grid = 0;
  const int smem = dev::kSweepSmemDoubles * (int)sizeof(double);
  CUDA_CHECK(cudaFuncSetAttribute(dev::k_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  {
    int dev_id = 0, nsm = 0, per_sm = 0;
    CUDA_CHECK(cudaGetDevice(&dev_id));
    CUDA_CHECK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev_id));
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dev::k_sweep, dev::kSweepThreads, smem));
    MDD_REQUIRE(per_sm > 0, 5, "sweep kernel cannot be resident");
    sweep_grid = plan_grid = nsm * per_sm;
    if (const char* ev = getenv("MDD_SWEEP_GRID")) {  // debug: fewer persistent CTAs
      const int gr = atoi(ev);
      if (gr > 0 && gr < sweep_grid) sweep_grid = gr;
    }
  }
  for (int dir = 0; dir < 2; ++dir) {
    std::vector<dev::MTaskDesc>& out = dir == 0 ? mtf : mtb;
    std::vector<int>& lev = dir == 0 ? lev_f : lev_b;
    for (int l = 0; l < NL; ++l) {
      lev[l] = (int)out.size();
     // the level's tasks with 2-D groups of kGroup tiles
     auto build_level = [&](const int kGroup) {
      std::vector<Cand> lt;
      for (const int g : plev[l]) {
        const int nc = fp.sn_ncol[g], nr = nc + fp.sn_noff[g];
        dev::MTaskDesc D{};
        D.col0 = fp.sn_col0[g];
        D.vo = vvo[g];
        D.uptr = fp.sn_uptr[g];
        D.nr = nr; D.nc = nc; D.RB = vRB[g]; D.CB = vCB[g];
        const std::vector<int>& tiles_g = dir == 0 ? ft[g] : bt[g];
        if (mode[g] == 0) {
          // small: one task, all column tiles
          D.big = 0;
          D.rows = nr; D.cols = nc;
          set_vec(D, vvo[g], vvo[g] + nr);
          int64_t by = 0;
          for (int t : tiles_g) by += tile_bytes(t);
          lt.push_back({by, D, tiles_g});
        } else if (mode[g] == 1) {
          // strip: one task per strip, the whole t / w as vector
          for (int t : tiles_g) {
            dev::MTaskDesc X = D;
            X.big = 2;
            X.rows = rc[t].x; X.cols = rc[t].y;  // fwd: rows x columns [0, cols); bwd: nr - cb rows
            X.rb = dir == 0 ? tl[t].y : tl[t].z;  // first row
            X.cb = dir == 0 ? 0 : tl[t].z;        // first column
            set_vec(X, vvo[g], vvo[g] + nr);
            lt.push_back({tile_bytes(t), X, {t}});
          }
        } else {
          // 2-D: groups of <= kGroup tiles; fwd = one row block x consecutive column
          // blocks, bwd = one column block x consecutive row blocks
          const int RB = vRB[g], CB = vCB[g], nrb = vnrb[g], ncb = vncb[g];
          std::vector<std::vector<int>> tid_of(nrb, std::vector<int>(ncb, -1));
          for (int t : tiles_g) tid_of[tl[t].y][tl[t].z] = t;
          if (dir == 0) {
            for (int rb = 0; rb < nrb; ++rb) {
              const int rend = std::min(nr, (rb + 1) * RB);
              const int ntb = std::min(ncb, (rend + CB - 1) / CB);
              const int nch = (ntb + kGroup - 1) / kGroup;
              for (int ch = 0; ch < nch; ++ch) {
                dev::MTaskDesc X = D;
                X.big = 1;
                X.rb = rb;
                X.cb = ch * kGroup;
                const int cend = std::min(ntb, (ch + 1) * kGroup);
                X.rows = rend - rb * RB;
                X.part = vfp[g] + (int64_t)ch * nr + (int64_t)rb * RB;
                X.comb = vfp[g] + (int64_t)rb * RB;
                X.ntl = nch;
                set_vec(X, vvo[g] + (int64_t)X.cb * CB, vvo[g] + std::min<int64_t>(nc, (int64_t)cend * CB));
                Cand c{0, X, {}};
                for (int cb = X.cb; cb < cend; ++cb) { c.tiles.push_back(tid_of[rb][cb]); c.bytes += tile_bytes(tid_of[rb][cb]); }
                lt.push_back(c);
              }
            }
          } else {
            for (int cb = 0; cb < ncb; ++cb) {
              const int rb0 = (cb * CB) / RB;
              const int nch = (nrb - rb0 + kGroup - 1) / kGroup;
              for (int ch = 0; ch < nch; ++ch) {
                dev::MTaskDesc X = D;
                X.big = 1;
                X.cb = cb;
                X.rb = rb0 + ch * kGroup;
                const int rend_b = std::min(nrb, X.rb + kGroup);
                X.cols = std::min(CB, nc - cb * CB);
                X.part = vbp[g] + (int64_t)ch * nc + (int64_t)cb * CB;
                X.comb = vbp[g] + (int64_t)cb * CB;
                X.ntl = nch;
                set_vec(X, vvo[g] + (int64_t)X.rb * RB, vvo[g] + std::min<int64_t>(nr, (int64_t)rend_b * RB));
                Cand c{0, X, {}};
                for (int rb = X.rb; rb < rend_b; ++rb) { c.tiles.push_back(tid_of[rb][cb]); c.bytes += tile_bytes(tid_of[rb][cb]); }
                lt.push_back(c);
              }
            }
          }
        }
      }
      for (const Cand& c : lt)
        MDD_REQUIRE(c.d.vbytes <= (int)((dev::kVecMax + 2) * sizeof(double)), 5,
                    "sweep task vector exceeds its shared-memory slot");
      std::stable_sort(lt.begin(), lt.end(), [](const Cand& x, const Cand& y) { return x.bytes > y.bytes; });
      return lt;
     };
      // group size of the 2-D tiles: the one whose snake dealing gives the
      // smallest per-CTA load (bytes + a fixed cost per task: its start, the
      // partial sums and the atomic), larger groups on ties.  A phase ends with
      // its slowest CTA, so on the upper levels (few tiles) smaller groups win.
      std::vector<Cand> lt;
      int64_t best = INT64_MAX;
      const int only_group = getenv("MDD_GROUP") ? atoi(getenv("MDD_GROUP")) : 0;  // debug
      // MDD_DEAL=lpt: instead of the snake over the sorted tasks, each task (largest
      // first) goes to the CTA with the least load so far (longest-processing-time
      // rule); the kernel still deals position r * grid + q to CTA q (r even) or
      // grid - 1 - q (r odd), so the tasks are LAID OUT in that order, a CTA with
      // fewer tasks than rounds padded at its tail with empty tasks (no tiles, no
      // rows).  Which CTA runs a task never changes a result.
      // (a debug grid smaller than the planned one would deal padding between a
      // CTA's real tasks -- their vector slots assume none -- so it keeps the snake)
      const bool lpt = getenv("MDD_DEAL") && !strcmp(getenv("MDD_DEAL"), "lpt") && sweep_grid == plan_grid;
      std::vector<std::vector<int>> own_best;
      for (int kGroup : {4, 2, 1}) {
        if (only_group && kGroup != only_group) continue;
        std::vector<Cand> c = build_level(kGroup);
        std::vector<int64_t> load(plan_grid, 0);
        std::vector<std::vector<int>> own;
        if (lpt) {
          own.resize(plan_grid);
          // (load, cta) min-heap; ties to the lowest CTA index
          std::priority_queue<std::pair<int64_t, int>, std::vector<std::pair<int64_t, int>>,
                              std::greater<std::pair<int64_t, int>>> pq;
          for (int q = 0; q < plan_grid; ++q) pq.push({0, q});
          for (size_t i = 0; i < c.size(); ++i) {
            auto [ld, q] = pq.top();
            pq.pop();
            own[q].push_back((int)i);
            load[q] = ld + c[i].bytes + kTaskCostBytes;
            pq.push({load[q], q});
          }
        } else {
          for (size_t i = 0; i < c.size(); ++i) {
            const int64_t r = (int64_t)i / plan_grid, q = (int64_t)i % plan_grid;
            load[(r & 1) ? plan_grid - 1 - q : q] += c[i].bytes + kTaskCostBytes;
          }
        }
        const int64_t mk = *std::max_element(load.begin(), load.end());
        if (getenv("MDD_PLAN_STATS")) {
          int64_t sum = 0;
          for (int64_t v : load) sum += v;
          fprintf(stderr, "  [deal %s dir %d level %d group %d] tasks %zu max load %lld mean %lld\n", name.c_str(), dir,
                  l, kGroup, c.size(), (long long)mk, (long long)(sum / plan_grid));
        }
        if (mk < best) { best = mk; lt.swap(c); own_best.swap(own); }
        if (getenv("MDD_FIXED_GROUP")) break;  // debug: always groups of 4
      }
      nreal[dir][l] = (int)lt.size();
      if (lpt && !lt.empty()) {
        size_t rounds = 0;
        for (auto& o : own_best) rounds = std::max(rounds, o.size());
        std::vector<Cand> laid;
        laid.reserve(rounds * (size_t)plan_grid);
        size_t last = 0;
        for (size_t r = 0; r < rounds; ++r)
          for (int q = 0; q < plan_grid; ++q) {
            const int b = (r & 1) ? plan_grid - 1 - q : q;
            if (r < own_best[b].size()) {
              laid.push_back(std::move(lt[own_best[b][r]]));
              last = laid.size();
            } else {
              laid.push_back(Cand{});  // an empty task: k0 == k1, nr == 0, vn == 0
            }
          }
        laid.resize(last);
        lt.swap(laid);
      }
      if (dir == 0) cmf[l] = (int)cm.size(); else cmb_lev[l] = (int)cm.size();
      for (auto& c : lt) {
        const dev::MTaskDesc& X0 = c.d;
        if (X0.big == 1 && X0.part == X0.comb) {  // first chunk of its row / column block
          dev::CombDesc C{};
          C.comb = X0.comb;
          C.col0 = X0.col0;
          C.uptr = X0.uptr;
          C.vo = X0.vo;
          C.ld = dir == 0 ? X0.nr : X0.nc;
          C.ntl = X0.ntl;
          C.m = dir == 0 ? X0.rows : X0.cols;
          C.first = dir == 0 ? X0.rb * X0.RB : X0.cb * X0.CB;
          C.nc = X0.nc;
          cm.push_back(C);
        }
      }
      for (auto& c : lt) {
        dev::MTaskDesc X = c.d;
        X.k0 = (int)td.size();
        for (int t : c.tiles) push_td(t);
        X.k1 = (int)td.size();
        for (int q = 0; q < dev::kTdInline && X.k0 + q < X.k1; ++q) X.td[q] = td[X.k0 + q];
        out.push_back(X);
      }
    }
    lev[NL] = (int)out.size();
    if (dir == 0) cmf[NL] = (int)cm.size(); else cmb_lev[NL] = (int)cm.size();
  }
  // levels with few tasks per CTA gather their task vectors inside the tasks (no
  // flat G phase and no grid barrier before them); the leaf levels keep the
  // flat gather (many rows, many tasks per CTA).  Same sums in the same order.
  const int fuse_tasks = getenv("MDD_FUSE_TASKS") ? atoi(getenv("MDD_FUSE_TASKS")) : 2;
  auto fused = [&](const std::vector<int>& lev, int l) {
    return nreal[&lev == &lev_f ? 0 : 1][l] <= fuse_tasks * plan_grid;
  };
  // a combine phase goes one CTA per item (bit 1) when its items are few (<= 2 per
  // CTA) and their partial chains long (>= 8): a warp per item would walk ntl / 4
  // dependent loads while most of the grid idles
  auto cta_comb = [&](const std::vector<int>& lev, int l) {
    int mx = 0;
    for (int k = lev[l]; k < lev[l + 1]; ++k) mx = std::max(mx, cm[k].ntl);
    for (int k = lev[l]; k < lev[l + 1]; ++k)
      MDD_REQUIRE(cm[k].m <= 2 * dev::kVecMax / 4, 5, "combine item wider than its reduction slot");
    return (lev[l + 1] - lev[l] <= 2 * plan_grid && mx >= 8) ? 2 : 0;
  };
  std::vector<int4> ph;
  nph_a = 0;
  for (int l = 0; l < NL; ++l) {
    if (l == nlev_a && nlev_a > 0) nph_a = (int)ph.size();  // segment A ends: the rank's subtrees swept forward
    const bool fz = fused(lev_f, l);
    if (!fz) ph.push_back(make_int4(dev::PH_GF, (int)lev_row[l], (int)lev_row[l + 1], 0));
    ph.push_back(make_int4(dev::PH_MF, lev_f[l], lev_f[l + 1], fz ? 1 : 0));
    // the level's 2-D partial sums, added before any later phase reads xf / upd
    if (cmf[l + 1] > cmf[l]) ph.push_back(make_int4(dev::PH_CF, cmf[l], cmf[l + 1], (fz ? 1 : 0) | cta_comb(cmf, l)));
  }
  if (nlev_a == NL && nlev_a > 0) nph_a = (int)ph.size();
  for (int l = NL - 1; l >= 0; --l) {
    const bool fz = fused(lev_b, l);
    if (!fz) ph.push_back(make_int4(dev::PH_GB, (int)lev_row[l], (int)lev_row[l + 1], 0));
    ph.push_back(make_int4(dev::PH_MB, lev_b[l], lev_b[l + 1], fz ? 1 : 0));
    if (cmb_lev[l + 1] > cmb_lev[l]) ph.push_back(make_int4(dev::PH_CB, cmb_lev[l], cmb_lev[l + 1], cta_comb(cmb_lev, l)));
  }
  if (prolong_n > 0) {
    ph.push_back(make_int4(dev::PH_PR, 0, prolong_n, 0));
    pro_ptr = pro_ptr_dev;
    pro_pos = pro_pos_dev;
    n_out = prolong_n;
  }
  nphases = (int)ph.size();
  MDD_REQUIRE(nrows < INT32_MAX, 5, "sweep row space too large for 32-bit phase bounds");
  phases.upload(ph);
  mt_f.upload(mtf);
  mt_b.upload(mtb);
  cmb.upload(cm.empty() ? std::vector<dev::CombDesc>(1) : cm);
  tdesc.upload(td);
  tiles.upload(tl);
  tile_off.upload(toff);
  sn_RB.upload(vRB); sn_CB.upload(vCB); sn_nrb.upload(vnrb); sn_ncb.upload(vncb);
  sn_fpart.upload(vfp); sn_bpart.upload(vbp);
  vb_off.upload(vvo);
  gsrc.upload(vgsrc);
  cptr.upload(vcptr);
  cidx.upload(vcidx.empty() ? std::vector<int64_t>{0} : vcidx);
  wsrc.upload(vwsrc);
  vb.alloc(nrows + 2);  // +2: the even-aligned bulk copies may read one past the end
  fpart.alloc(std::max<int64_t>(nfp, 1));
  bpart.alloc(std::max<int64_t>(nbp, 1));
  ctl.alloc(dev::SW_COUNT);
  reset_counters(nullptr);
  CUDA_CHECK(cudaDeviceSynchronize());
  if (getenv("MDD_SWEEP_TRACE")) {
    trace.alloc((size_t)dev::kTraceWords * nphases * sweep_grid);
    CUDA_CHECK(cudaMemset(trace.p, 0, trace.n * sizeof(unsigned long long)));
  }
  if (base) MDD_REQUIRE(lt_size == base->lt_size && ntiles == base->ntiles, 5, "sweep view: tile layout differs from its base");
  swept_entries = 0;
  for (int g = 0; g < nsn; ++g)
    if (role.empty() || role[g]) {
      const int64_t nc = fp.sn_ncol[g], no = fp.sn_noff[g];
      swept_entries += nc * (nc + 1) / 2 + nc * no;
    }
  if (getenv("MDD_PLAN_STATS")) {
    int nbig = 0;
    for (int g = 0; g < nsn; ++g) nbig += mode[g] != 0;
    fprintf(stderr, "[mdd plan %s] nsn %d (big %d) levels %d entries %lld tiles %d (%.1f%% stored) mtasks %d "
            "rows %lld contrib %lld grid %d\n", name.c_str(), nsn, nbig, fp.nlevels, (long long)fp.factor_nnz(),
            ntiles, 100.0 * (double)lt_size / std::max<double>(1.0, (double)fp.factor_nnz()), (int)mtf.size(),
            (long long)nrows, (long long)vcidx.size(), sweep_grid);
    for (int l = 0; l < NL; ++l) {
      long long ent = 0;
      int big = 0;
      for (const int g : plev[l]) {
        ent += (long long)fp.sn_ncol[g] * (fp.sn_ncol[g] + fp.sn_noff[g]);
        big += mode[g] != 0;
      }
      fprintf(stderr, "  level %2d: sn %6d (big %4d) stored %10lld rows %8lld mtasks %6d\n", l,
              (int)plev[l].size(), big, ent, (long long)(lev_row[l + 1] - lev_row[l]),
              lev_f[l + 1] - lev_f[l]);
    }
  }
}

void DevFactor::reset_counters(cudaStream_t s) {
  std::vector<unsigned long long> c0(dev::SW_COUNT, 0ull);
  c0[dev::SW_T0] = ~0ull;
  CUDA_CHECK(cudaMemcpyAsync(ctl.p, c0.data(), c0.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
}

dev::SweepDev DevFactor::sweep_dev() const {
  dev::SweepDev S;
  S.P = plan();
  S.dinv = base ? base->dinv.p : dinv.p;
  S.phases = phases.p;
  S.nphases = nphases;
  S.ph0 = 0;
  S.ph1 = nphases;
  S.flags = 0;
  S.mtf = mt_f.p;
  S.mtb = mt_b.p;
  S.tdesc = tdesc.p;
  S.tiles = tiles.p;
  S.tile_off = tile_off.p;
  S.Lt = base ? base->Lt.p : Lt.p;
  S.sn_RB = sn_RB.p; S.sn_CB = sn_CB.p; S.sn_nrb = sn_nrb.p; S.sn_ncb = sn_ncb.p;
  S.sn_fpart = sn_fpart.p; S.sn_bpart = sn_bpart.p;
  S.fpart = fpart.p; S.bpart = bpart.p;
  S.cmb = cmb.p;
  S.vb = vb.p;
  S.vb_off = vb_off.p;
  S.gsrc = gsrc.p;
  S.cptr = cptr.p;
  S.cidx = cidx.p;
  S.wsrc = wsrc.p;
  S.ctl = ctl.p;
  S.upd = upd.p;
  S.xf = xf.p;
  S.xb = xb.p;
  S.b = nullptr;
  S.pro_ptr = pro_ptr;
  S.pro_pos = pro_pos;
  S.out = nullptr;
  S.n_out = n_out;
  S.stop = nullptr;
  S.trace = trace.p;
  return S;
}

DevFactor::~DevFactor() {
  if (trace.p && getenv("MDD_SWEEP_TRACE") && !name.empty()) {
    std::vector<unsigned long long> v(trace.n);
    std::vector<int4> phh(nphases);
    if (cudaMemcpy(v.data(), trace.p, v.size() * 8, cudaMemcpyDeviceToHost) == cudaSuccess &&
        cudaMemcpy(phh.data(), phases.p, phh.size() * sizeof(int4), cudaMemcpyDeviceToHost) == cudaSuccess) {
      std::string path = std::string(getenv("MDD_SWEEP_TRACE")) + "/trace_" + name + ".bin";
      if (FILE* f = fopen(path.c_str(), "wb")) {
        int hdr[3] = {nphases, sweep_grid, dev::kTraceWords};
        fwrite(hdr, sizeof(int), 3, f);
        fwrite(phh.data(), sizeof(int4), phh.size(), f);
        fwrite(v.data(), 8, v.size(), f);
        fclose(f);
      }
    }
  }
}

void DevFactor::sweep_timing(unsigned long long* ns, unsigned long long* cnt, cudaStream_t s) const {
  unsigned long long v[dev::SW_COUNT];
  CUDA_CHECK(cudaMemcpyAsync(v, ctl.p, sizeof(v), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  *ns = v[dev::SW_TSUM];
  *cnt = v[dev::SW_TCNT];
}

void DevFactor::sweep(const double* b, double* out, cudaStream_t s, const int* stop, int seg) const {
  dev::SweepDev S = sweep_dev();
  // without `out` the prolongation phase runs empty
  S.nphases = nphases;
  const char* fl = getenv("MDD_SWEEP_FLAGS");  // per launch (experiments toggle it)
  S.flags = fl ? atoi(fl) : 0;
  S.ph0 = seg == 1 ? nph_a : 0;
  S.ph1 = seg == 0 ? nph_a : nphases;
  if (S.ph1 <= S.ph0) return;
  S.n_out = out ? n_out : 0;
  S.b = b;
  S.out = out;
  S.stop = stop;
  // a cooperative launch: the persistent CTAs spin on grid barriers, so they must
  // all be co-resident -- guaranteed by the launch (or it fails), not assumed from
  // the occupancy calculator (other streams' kernels, MPS); the grid-barrier
  // timeout stays as a backstop.  Captured into the solve graph like any launch.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sweep_grid);
  cfg.blockDim = dim3(dev::kSweepThreads);
  cfg.dynamicSmemBytes = dev::kSweepSmemDoubles * sizeof(double);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_CHECK(cudaLaunchKernelEx(&cfg, dev::k_sweep, S));
}

void DevFactor::check_abort(cudaStream_t s) {
  unsigned long long ab = 0;
  CUDA_CHECK(cudaMemcpyAsync(&ab, ctl.p + dev::SW_ABORT, sizeof(ab), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  if (ab) {
    reset_counters(s);
    throw Error(5, "supernodal sweep aborted (barrier wait timed out)");
  }
}

namespace {
#define CUBLAS_OK(x)                                                                                \
  do {                                                                                              \
    cublasStatus_t s__ = (x);                                                                       \
    if (s__ != CUBLAS_STATUS_SUCCESS)                                                               \
      throw Error(1, std::string(#x) + ": cublas status " + std::to_string((int)s__));              \
  } while (0)
#define CUSOLVER_OK(x)                                                                              \
  do {                                                                                              \
    cusolverStatus_t s__ = (x);                                                                     \
    if (s__ != CUSOLVER_STATUS_SUCCESS)                                                             \
      throw Error(1, std::string(#x) + ": cusolver status " + std::to_string((int)s__));            \
  } while (0)
constexpr int kBigFront = 1024;  // fronts with more rows take the blocked path
constexpr int kPanel = 64;
}  // namespace

int DevFactor::factor(const double* src, int mode, double tol, uint8_t* dropped, cudaStream_t s) {
  DBuf<double> fronts, umat;
  fronts.alloc(std::max<int64_t>(fp.fsize, 1));
  umat.alloc(std::max<int64_t>(fp.umsize, 1));
  DBuf<int> err;
  err.alloc(1);
  err.zero(s);
  L.zero(s);
  dev::PlanDev P = plan();
  // per level: small fronts in one launch (one CTA each), big fronts blocked with
  // cuBLAS trailing updates, cuSOLVER triangular inverse and cuBLAS M21 = L21 L11^{-1}
  std::vector<int> small_list;
  std::vector<int> small_ptr(fp.nlevels + 1, 0);
  std::vector<std::vector<int>> big(fp.nlevels);
  int64_t wmax = 1;
  int n_blocked_now = 0;
  for (int l = 0; l < fp.nlevels; ++l) {
    small_ptr[l] = (int)small_list.size();
    for (int k = fp.level_ptr[l]; k < fp.level_ptr[l + 1]; ++k) {
      const int g = fp.level_sn[k];
      const int nr = fp.sn_ncol[g] + fp.sn_noff[g];
      if (nr > kBigFront) {
        big[l].push_back(g);
        ++n_blocked_now;
        wmax = std::max<int64_t>(wmax, (int64_t)nr * kPanel);
      } else {
        small_list.push_back(g);
      }
    }
  }
  small_ptr[fp.nlevels] = (int)small_list.size();
  n_blocked = n_blocked_now;
  DBuf<int> dsmall;
  dsmall.upload(small_list.empty() ? std::vector<int>{0} : small_list);
  bool any_big = false;
  for (auto& b : big) any_big |= !b.empty();
  cublasHandle_t cb = nullptr;
  cusolverDnHandle_t cs = nullptr;
  DBuf<double> W;
  DBuf<char> trw;
  DBuf<int> info;
  if (any_big) {
    CUBLAS_OK(cublasCreate(&cb));
    CUBLAS_OK(cublasSetStream(cb, s));
    CUSOLVER_OK(cusolverDnCreate(&cs));
    CUSOLVER_OK(cusolverDnSetStream(cs, s));
    W.alloc(wmax);
    info.alloc(std::max(n_blocked, 1));  // one trtri info word per blocked front
    info.zero(s);
  }
  int iblk = 0;
  try {
    for (int l = 0; l < fp.nlevels; ++l) {
      const int cnt = small_ptr[l + 1] - small_ptr[l];
      if (cnt > 0) {
        dev::k_mf_factor_level<<<cnt, 256, 0, s>>>(P, dsmall.p + small_ptr[l], src, fronts.p, L.p, dinv.p,
                                                   umat.p, mode, tol, dropped, err.p);
        CUDA_CHECK(cudaGetLastError());
      }
      for (int g : big[l]) {
        const int nc = fp.sn_ncol[g], no = fp.sn_noff[g], nr = nc + no;
        double* F = fronts.p + fp.sn_fptr[g];
        double* Lp = L.p + fp.sn_lptr[g];
        dev::k_front_assemble<<<256, 256, 0, s>>>(P, g, src, fronts.p, umat.p);
        dev::k_front_assemble2<<<1, 1024, 0, s>>>(P, g, src, fronts.p, umat.p);
        for (int j0 = 0; j0 < nc; j0 += kPanel) {
          const int nb = std::min(kPanel, nc - j0);
          dev::k_panel_factor<<<1, 512, 0, s>>>(P, g, j0, nb, fronts.p, dinv.p, W.p, mode, tol, dropped, err.p);
          const int rest = nr - (j0 + nb);
          if (rest > 0) {
            const double m1 = -1.0, one = 1.0;
            // F22 -= W L_p^T (lower triangle), W = L_p D_p
            CUBLAS_OK(cublasDsyrkx(cb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, rest, nb, &m1, W.p, rest,
                                   F + (int64_t)j0 * nr + (j0 + nb), nr, &one,
                                   F + (int64_t)(j0 + nb) * nr + (j0 + nb), nr));
          }
        }
        dev::k_front_finish_copy<<<256, 256, 0, s>>>(P, g, fronts.p, L.p, umat.p);
        // L11^{-1} in place (unit lower), then M21 = L21 L11^{-1}
        size_t dws = 0, hws = 0;
        CUSOLVER_OK(cusolverDnXtrtri_bufferSize(cs, CUBLAS_FILL_MODE_LOWER, CUBLAS_DIAG_UNIT, nc, CUDA_R_64F, Lp,
                                                nr, &dws, &hws));
        if (trw.n < dws + 8) trw.alloc(dws + 8);
        std::vector<char> hbuf(std::max<size_t>(hws, 1));
        CUSOLVER_OK(cusolverDnXtrtri(cs, CUBLAS_FILL_MODE_LOWER, CUBLAS_DIAG_UNIT, nc, CUDA_R_64F, Lp, nr, trw.p,
                                     dws, hbuf.data(), hws, info.p + iblk++));
        if (no > 0) {
          const double one = 1.0;
          CUBLAS_OK(cublasDtrmm(cb, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_UNIT, no, nc,
                                &one, Lp, nr, F + nc, nr, Lp + nc, nr));
        }
        dev::k_front_fold_d<<<256, 256, 0, s>>>(P, g, L.p, dinv.p);
        CUDA_CHECK(cudaGetLastError());
      }
    }
    CUDA_CHECK(cudaStreamSynchronize(s));
  } catch (...) {
    if (cb) cublasDestroy(cb);
    if (cs) cusolverDnDestroy(cs);
    throw;
  }
  if (cb) cublasDestroy(cb);
  if (cs) cusolverDnDestroy(cs);
  if (any_big) {
    std::vector<int> ti = info.download();
    for (int v : ti) MDD_REQUIRE(v == 0, 1, "triangular inverse (trtri) of a blocked front failed");
  }
  int e = 0;
  CUDA_CHECK(cudaMemcpy(&e, err.p, sizeof(int), cudaMemcpyDeviceToHost));
  if (mode != 2) MDD_REQUIRE(e == 0, 3, "nonpositive pivot in an SPD factorisation");
  // P-form panels -> contiguous sweep tiles; the column-major panels are dropped
  Lt.alloc(std::max<int64_t>(lt_size, 2));
  if (ntiles > 0) {
    dev::k_tile_relayout<<<ntiles, 256, 0, s>>>(sweep_dev(), ntiles, L.p, lptr.p);
    CUDA_CHECK(cudaGetLastError());
  }
  CUDA_CHECK(cudaStreamSynchronize(s));
  L.release();
  return mode == 2 ? e : 0;
}

}  // namespace mdd
