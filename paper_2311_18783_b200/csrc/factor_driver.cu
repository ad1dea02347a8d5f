// Host drivers of the multifrontal factorisation and the level-scheduled
// supernodal triangular solves (kernels in kernels.cu).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

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

namespace {
constexpr int kProlongChunk = 2048;
}  // namespace

void DevFactor::upload(int prolong_n, const int64_t* pro_ptr_dev, const int32_t* pro_pos_dev) {
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
  upd.alloc(std::max<int64_t>(fp.usize, 1));
  xf.alloc(std::max<int64_t>(fp.ntot, 1));
  xb.alloc(std::max<int64_t>(fp.ntot, 1));
  // ---- tile geometry per supernode.  "single": swept by one CTA (column tiles
  // over all nr rows, accumulated in shared memory); "big": RB x CB tiles spread
  // over CTAs with partial sums
  const int nsn = fp.nsn;
  std::vector<int> vRB(nsn), vCB(nsn), vnrb(nsn), vncb(nsn), vrbc(nsn, 0), vcbc(nsn, 0);
  std::vector<uint8_t> single(nsn);
  std::vector<int64_t> vfp(nsn, 0), vbp(nsn, 0), vtg(nsn, 0), stored(nsn);
  std::vector<std::vector<int>> sn_tiles(nsn);
  std::vector<int4> tl;
  std::vector<int64_t> toff;
  int64_t off = 0, nfp = 0, nbp = 0, ntg = 0;
  int nrbc = 0, ncbc = 0;
  for (int g = 0; g < nsn; ++g) {
    const int nc = fp.sn_ncol[g], nr = nc + fp.sn_noff[g];
    stored[g] = (int64_t)nr * nc;
    single[g] = nr <= dev::kVecMax && stored[g] <= dev::kSingleMax;
    int RB, CB;
    if (single[g]) {
      RB = nr;
      CB = std::max(1, std::min(nc, dev::kTileMax / nr));
    } else {
      CB = std::min(nc, 64);
      RB = std::min(dev::kVecMax, std::max(32, (dev::kTileMax / CB) / 32 * 32));
    }
    const int nrb = (nr + RB - 1) / RB, ncb = (nc + CB - 1) / CB;
    vRB[g] = RB; vCB[g] = CB; vnrb[g] = nrb; vncb[g] = ncb;
    if (!single[g]) {
      vfp[g] = nfp; nfp += (int64_t)ncb * nr;
      vbp[g] = nbp; nbp += (int64_t)nrb * nc;
      vtg[g] = ntg; ntg += nr;
      vrbc[g] = nrbc; nrbc += nrb;
      vcbc[g] = ncbc; ncbc += ncb;
    }
    for (int rb = 0; rb < nrb; ++rb) {
      const int rend = std::min(nr, (rb + 1) * RB), rows = rend - rb * RB;
      for (int cb = 0; cb < ncb && cb * CB < rend; ++cb) {
        const int cols = std::min(CB, nc - cb * CB);
        sn_tiles[g].push_back((int)tl.size());
        tl.push_back(make_int4(g, rb, cb, 0));
        toff.push_back(off);
        off += ((int64_t)rows * cols + 1) & ~1LL;  // 16-byte aligned tiles
      }
    }
  }
  ntiles = (int)tl.size();
  lt_size = off;
  // ---- clusters: a single-only subtree of <= kClusterMax stored entries is one
  // task (postorder); a single supernode above such subtrees is its own cluster
  std::vector<std::vector<int>> kids(nsn);
  for (int g = 0; g < nsn; ++g)
    if (fp.sn_parent[g] >= 0) kids[fp.sn_parent[g]].push_back(g);
  std::vector<uint8_t> sub_ok(nsn);
  std::vector<int64_t> sub_sz(nsn);
  for (int g = 0; g < nsn; ++g) {  // children precede parents
    bool okg = single[g];
    int64_t sz = stored[g];
    for (int c : kids[g]) { okg = okg && sub_ok[c]; sz += sub_sz[c]; }
    sub_ok[g] = okg;
    sub_sz[g] = sz;
  }
  struct Cl { int root; int wait; std::vector<int> members; };
  std::vector<Cl> clusters;
  std::vector<int> bigs;
  std::vector<int> stack;
  for (int g = 0; g < nsn; ++g)
    if (fp.sn_parent[g] < 0) stack.push_back(g);
  while (!stack.empty()) {
    const int g = stack.back();
    stack.pop_back();
    if (single[g] && sub_ok[g] && sub_sz[g] <= dev::kClusterMax) {
      Cl c{g, 0, {}};
      std::vector<int> st{g}, order;
      while (!st.empty()) {  // preorder, reversed below into a postorder
        const int v = st.back();
        st.pop_back();
        order.push_back(v);
        for (int k : kids[v]) st.push_back(k);
      }
      c.members.assign(order.rbegin(), order.rend());
      clusters.push_back(std::move(c));
      continue;
    }
    if (single[g]) clusters.push_back(Cl{g, kids[g].empty() ? 0 : 1, {g}});
    else bigs.push_back(g);
    for (int k : kids[g]) stack.push_back(k);
  }
  // ---- schedule: forward work by level of its top supernode, backward work in
  // the reverse order, prolongation last.  Every wait targets an earlier ticket.
  std::vector<std::vector<int>> cl_at(fp.nlevels), big_at(fp.nlevels);
  for (int c = 0; c < (int)clusters.size(); ++c) cl_at[fp.sn_level[clusters[c].root]].push_back(c);
  for (int g : bigs) big_at[fp.sn_level[g]].push_back(g);
  std::vector<int4> tk;
  std::vector<int> ttp(1, 0), ttl;
  auto add_task = [&](int4 t, const std::vector<int>& tiles_) {
    tk.push_back(t);
    ttl.insert(ttl.end(), tiles_.begin(), tiles_.end());
    ttp.push_back((int)ttl.size());
  };
  const std::vector<int> none;
  for (int l = 0; l < fp.nlevels; ++l) {
    for (int c : cl_at[l]) {
      std::vector<int> ts;
      for (int g : clusters[c].members) ts.insert(ts.end(), sn_tiles[g].begin(), sn_tiles[g].end());
      add_task(make_int4(4, clusters[c].root, clusters[c].wait, 0), ts);
    }
    for (int g : big_at[l]) {
      add_task(make_int4(3, g, 0, 0), none);
      for (int t : sn_tiles[g]) add_task(make_int4(0, t, 0, 0), std::vector<int>{t});
    }
  }
  total_bwd = 0;
  for (int g = 0; g < nsn; ++g) total_bwd += vncb[g];
  for (int l = fp.nlevels - 1; l >= 0; --l) {
    for (int g : big_at[l])
      for (int t : sn_tiles[g]) add_task(make_int4(1, t, 0, 0), std::vector<int>{t});
    for (int c : cl_at[l]) {
      std::vector<int> ts;
      for (auto it2 = clusters[c].members.rbegin(); it2 != clusters[c].members.rend(); ++it2)
        ts.insert(ts.end(), sn_tiles[*it2].begin(), sn_tiles[*it2].end());
      int ncbs = 0;
      for (int g : clusters[c].members) ncbs += vncb[g];
      add_task(make_int4(5, clusters[c].root, clusters[c].wait, ncbs), ts);
    }
  }
  ntasks_noprolong = (int)tk.size();
  if (prolong_n > 0) {
    for (int e0 = 0; e0 < prolong_n; e0 += kProlongChunk)
      add_task(make_int4(2, 0, e0, std::min(prolong_n, e0 + kProlongChunk)), none);
    pro_ptr = pro_ptr_dev;
    pro_pos = pro_pos_dev;
  }
  ntasks = (int)tk.size();
  tasks.upload(tk);
  tt_ptr.upload(ttp);
  {
    std::vector<int4> td(ttl.size());
    for (size_t k = 0; k < ttl.size(); ++k) {
      const int t = ttl[k];
      const int4 q = tl[t];
      const int g = q.x;
      const int nr = fp.sn_ncol[g] + fp.sn_noff[g], nc = fp.sn_ncol[g];
      const int rows = std::min(vRB[g], nr - q.y * vRB[g]), cols = std::min(vCB[g], nc - q.z * vCB[g]);
      const int bytes = (int)((((int64_t)rows * cols + 1) & ~1LL) * (int64_t)sizeof(double));
      td[k] = make_int4(t, bytes, (int)(uint32_t)(toff[t] & 0xffffffffu), (int)(uint32_t)(toff[t] >> 32));
    }
    tdesc.upload(td);
  }
  tiles.upload(tl);
  tile_off.upload(toff);
  sn_RB.upload(vRB); sn_CB.upload(vCB); sn_nrb.upload(vnrb); sn_ncb.upload(vncb);
  sn_rbc.upload(vrbc); sn_cbc.upload(vcbc);
  sn_fpart.upload(vfp); sn_bpart.upload(vbp); sn_tg.upload(vtg);
  fpart.alloc(std::max<int64_t>(nfp, 1));
  bpart.alloc(std::max<int64_t>(nbp, 1));
  tg.alloc(std::max<int64_t>(ntg, 1));
  rb_cnt.alloc(std::max(nrbc, 1));
  cb_cnt.alloc(std::max(ncbc, 1));
  asm_cnt.alloc(std::max(nsn, 1));
  fwd_cnt.alloc(std::max(nsn, 1));
  bwd_cnt.alloc(std::max(nsn, 1));
  ctl.alloc(dev::SW_COUNT);
  reset_counters(nullptr);
  CUDA_CHECK(cudaDeviceSynchronize());
  if (getenv("MDD_SWEEP_TRACE")) {
    trace.alloc((size_t)4 * ntasks);
    CUDA_CHECK(cudaMemset(trace.p, 0, trace.n * sizeof(unsigned long long)));
  }
  if (getenv("MDD_SWEEP_STATS")) {
    stats.alloc(10);
    CUDA_CHECK(cudaMemset(stats.p, 0, 10 * sizeof(unsigned long long)));
  }
  if (getenv("MDD_PLAN_STATS")) {
    int nbig = 0;
    for (int g = 0; g < nsn; ++g) nbig += !single[g];
    fprintf(stderr, "[mdd plan %s] nsn %d (big %d) levels %d entries %lld tiles %d (%.1f%% stored) tasks %d "
            "clusters %d\n", name.c_str(), nsn, nbig, fp.nlevels, (long long)fp.factor_nnz(), ntiles,
            100.0 * (double)lt_size / std::max<double>(1.0, (double)fp.factor_nnz()), ntasks, (int)clusters.size());
    for (int l = 0; l < fp.nlevels; ++l) {
      long long ent = 0, emax = 0;
      int ncmax = 0, nrmax = 0, tcount = 0, big = 0;
      for (int k = fp.level_ptr[l]; k < fp.level_ptr[l + 1]; ++k) {
        const int g = fp.level_sn[k];
        const long long nc = fp.sn_ncol[g], no = fp.sn_noff[g];
        const long long e = nc * (nc + 1) / 2 + nc * no;
        ent += e;
        emax = std::max(emax, e);
        ncmax = std::max(ncmax, (int)nc);
        nrmax = std::max(nrmax, (int)(nc + no));
        tcount += (int)sn_tiles[g].size();
        big += !single[g];
      }
      fprintf(stderr, "  level %2d: sn %6d (big %4d) entries %10lld max %8lld ncmax %5d nrmax %5d tiles %6d\n", l,
              fp.level_ptr[l + 1] - fp.level_ptr[l], big, ent, emax, ncmax, nrmax, tcount);
    }
  }
  const int smem = dev::kSweepSmemDoubles * (int)sizeof(double);
  CUDA_CHECK(cudaFuncSetAttribute(dev::k_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int dev_id = 0, nsm = 0, per_sm = 0;
  CUDA_CHECK(cudaGetDevice(&dev_id));
  CUDA_CHECK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev_id));
  CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dev::k_sweep, dev::kSweepThreads, smem));
  MDD_REQUIRE(per_sm > 0, 5, "sweep kernel cannot be resident");
  sweep_grid = nsm * per_sm;
}

void DevFactor::reset_counters(cudaStream_t s) {
  for (DBuf<unsigned long long>* c : {&fwd_cnt, &bwd_cnt, &rb_cnt, &cb_cnt, &asm_cnt})
    CUDA_CHECK(cudaMemsetAsync(c->p, 0, c->n * sizeof(unsigned long long), s));
  std::vector<unsigned long long> c0(dev::SW_COUNT, 0ull);
  c0[dev::SW_T0] = ~0ull;
  CUDA_CHECK(cudaMemcpyAsync(ctl.p, c0.data(), c0.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
}

dev::SweepDev DevFactor::sweep_dev() const {
  dev::SweepDev S;
  S.P = plan();
  S.dinv = dinv.p;
  S.tasks = tasks.p;
  S.tt_ptr = tt_ptr.p;
  S.tdesc = tdesc.p;
  S.ntasks = ntasks;
  S.total_bwd = total_bwd;
  S.parent = parent.p;
  S.tiles = tiles.p;
  S.tile_off = tile_off.p;
  S.Lt = Lt.p;
  S.sn_RB = sn_RB.p; S.sn_CB = sn_CB.p; S.sn_nrb = sn_nrb.p; S.sn_ncb = sn_ncb.p;
  S.sn_fpart = sn_fpart.p; S.sn_bpart = sn_bpart.p; S.sn_tg = sn_tg.p;
  S.sn_rbc = sn_rbc.p; S.sn_cbc = sn_cbc.p;
  S.fpart = fpart.p; S.bpart = bpart.p; S.tg = tg.p;
  S.rb_cnt = rb_cnt.p; S.cb_cnt = cb_cnt.p; S.asm_cnt = asm_cnt.p;
  S.fwd_cnt = fwd_cnt.p;
  S.bwd_cnt = bwd_cnt.p;
  S.ctl = ctl.p;
  S.upd = upd.p;
  S.xf = xf.p;
  S.xb = xb.p;
  S.b = nullptr;
  S.gmap = nullptr;
  S.pro_ptr = pro_ptr;
  S.pro_pos = pro_pos;
  S.out = nullptr;
  S.stop = nullptr;
  S.stats = stats.p;
  S.trace = trace.p;
  return S;
}

DevFactor::~DevFactor() {
  if (trace.p && getenv("MDD_SWEEP_TRACE") && !name.empty()) {
    std::vector<unsigned long long> v(trace.n);
    std::vector<int4> tk(ntasks);
    if (cudaMemcpy(v.data(), trace.p, v.size() * 8, cudaMemcpyDeviceToHost) == cudaSuccess &&
        cudaMemcpy(tk.data(), tasks.p, tk.size() * sizeof(int4), cudaMemcpyDeviceToHost) == cudaSuccess) {
      std::string path = std::string(getenv("MDD_SWEEP_TRACE")) + "/trace_" + name + ".bin";
      if (FILE* f = fopen(path.c_str(), "wb")) {
        int nt = ntasks;
        fwrite(&nt, sizeof(int), 1, f);
        fwrite(tk.data(), sizeof(int4), tk.size(), f);
        fwrite(v.data(), 8, v.size(), f);
        fclose(f);
      }
    }
  }
  if (stats.p) {
    unsigned long long v[10];
    if (cudaMemcpy(v, stats.p, sizeof(v), cudaMemcpyDeviceToHost) == cudaSuccess)
      fprintf(stderr, "[mdd sweep stats %s] cycles: fwd wait %llu work %llu | bwd wait %llu work %llu | "
              "prolong wait %llu work %llu | assemble wait %llu work %llu | ticket %llu | tasks %llu\n",
              name.c_str(), v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[8], v[9]);
  }
}

void DevFactor::sweep_timing(unsigned long long* ns, unsigned long long* cnt, cudaStream_t s) const {
  unsigned long long v[dev::SW_COUNT];
  CUDA_CHECK(cudaMemcpyAsync(v, ctl.p, sizeof(v), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  *ns = v[dev::SW_TSUM];
  *cnt = v[dev::SW_TCNT];
}

void DevFactor::sweep(const double* b, const int32_t* gmap, double* out, cudaStream_t s,
                      const int* stop) const {
  dev::SweepDev S = sweep_dev();
  S.ntasks = out ? ntasks : ntasks_noprolong;
  S.b = b;
  S.gmap = gmap;
  S.out = out;
  S.stop = stop;
  const int grid = std::max(1, std::min(sweep_grid, S.ntasks));
  dev::k_sweep<<<grid, dev::kSweepThreads, dev::kSweepSmemDoubles * sizeof(double), s>>>(S);
}

void DevFactor::check_abort(cudaStream_t s) {
  unsigned long long ab = 0;
  CUDA_CHECK(cudaMemcpyAsync(&ab, ctl.p + dev::SW_ABORT, sizeof(ab), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  if (ab) {
    reset_counters(s);
    throw Error(5, "supernodal sweep aborted (dependency wait timed out)");
  }
}

int DevFactor::factor(const double* src, int mode, double tol, uint8_t* dropped, cudaStream_t s) {
  DBuf<double> fronts, umat;
  fronts.alloc(std::max<int64_t>(fp.fsize, 1));
  umat.alloc(std::max<int64_t>(fp.umsize, 1));
  DBuf<int> err;
  err.alloc(1);
  err.zero(s);
  L.zero(s);
  dev::PlanDev P = plan();
  for (int l = 0; l < fp.nlevels; ++l) {
    int cnt = fp.level_ptr[l + 1] - fp.level_ptr[l];
    dev::k_mf_factor_level<<<cnt, 256, 0, s>>>(P, fp.level_ptr[l], src, fronts.p, L.p, dinv.p,
                                               umat.p, mode, tol, dropped, err.p);
    CUDA_CHECK(cudaGetLastError());
  }
  CUDA_CHECK(cudaStreamSynchronize(s));
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
