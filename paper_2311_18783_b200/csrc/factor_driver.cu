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
// tasks of roughly kTaskEntries panel entries (~192 KB) so top-of-tree supernodes
// spread over several SMs while leaves stay one task each
constexpr int64_t kTaskEntries = 32768;
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
  // ---- sweep schedule
  std::vector<int4> tk;
  std::vector<int> vf(fp.nsn), vb(fp.nsn);
  int smem_d = 1;
  for (int l = 0; l < fp.nlevels; ++l)
    for (int k = fp.level_ptr[l]; k < fp.level_ptr[l + 1]; ++k) {
      const int g = fp.level_sn[k];
      const int nc = fp.sn_ncol[g], no = fp.sn_noff[g], nr = nc + no;
      const int64_t ent = (int64_t)nc * (nc + 1) / 2 + (int64_t)nc * no;
      int rb = nr;
      if (nr > dev::kSweepThreads || ent > kTaskEntries) {
        rb = (int)std::min<int64_t>(dev::kSweepThreads, std::max<int64_t>(32, kTaskEntries / nc));
        rb = rb / 32 * 32;
      }
      int cnt = 0;
      for (int r0 = 0; r0 < nr; r0 += rb, ++cnt) tk.push_back(make_int4(0, g, r0, std::min(nr, r0 + rb)));
      vf[g] = cnt;
      smem_d = std::max(smem_d, nc + std::min(nr, rb) + dev::kSweepThreads);
    }
  ntasks_noprolong = 0;
  total_bwd = 0;
  for (int l = fp.nlevels - 1; l >= 0; --l)
    for (int k = fp.level_ptr[l + 1] - 1; k >= fp.level_ptr[l]; --k) {
      const int g = fp.level_sn[k];
      const int nc = fp.sn_ncol[g], no = fp.sn_noff[g], nr = nc + no;
      const int64_t ent = (int64_t)nc * (nc + 1) / 2 + (int64_t)nc * no;
      int cb = nc;
      if (ent > kTaskEntries) cb = (int)std::max<int64_t>(16, kTaskEntries / nr / 16 * 16);
      int cnt = 0;
      for (int c0 = 0; c0 < nc; c0 += cb, ++cnt) tk.push_back(make_int4(1, g, c0, std::min(nc, c0 + cb)));
      vb[g] = cnt;
      total_bwd += cnt;
      smem_d = std::max(smem_d, nr + (dev::kSweepThreads / 32) * 16);
    }
  ntasks_noprolong = (int)tk.size();
  if (prolong_n > 0) {
    for (int e0 = 0; e0 < prolong_n; e0 += kProlongChunk)
      tk.push_back(make_int4(2, 0, e0, std::min(prolong_n, e0 + kProlongChunk)));
    pro_ptr = pro_ptr_dev;
    pro_pos = pro_pos_dev;
  }
  ntasks = (int)tk.size();
  tasks.upload(tk);
  if (getenv("MDD_SWEEP_STATS")) {
    stats.alloc(8);
    CUDA_CHECK(cudaMemset(stats.p, 0, 8 * sizeof(unsigned long long)));
  }
  if (getenv("MDD_PLAN_STATS")) {
    fprintf(stderr, "[mdd plan %s] nsn %d levels %d entries %lld tasks %d (bwd %d)\n", name.c_str(), fp.nsn,
            fp.nlevels, (long long)fp.factor_nnz(), ntasks, total_bwd);
    for (int l = 0; l < fp.nlevels; ++l) {
      long long ent = 0, emax = 0;
      int ncmax = 0, nrmax = 0, tf = 0, tb = 0;
      for (int k = fp.level_ptr[l]; k < fp.level_ptr[l + 1]; ++k) {
        const int g = fp.level_sn[k];
        const long long nc = fp.sn_ncol[g], no = fp.sn_noff[g];
        const long long e = nc * (nc + 1) / 2 + nc * no;
        ent += e;
        emax = std::max(emax, e);
        ncmax = std::max(ncmax, (int)nc);
        nrmax = std::max(nrmax, (int)(nc + no));
        tf += vf[g];
        tb += vb[g];
      }
      fprintf(stderr, "  level %2d: sn %6d entries %10lld max %8lld ncmax %5d nrmax %5d fwd tasks %6d bwd tasks %6d\n",
              l, fp.level_ptr[l + 1] - fp.level_ptr[l], ent, emax, ncmax, nrmax, tf, tb);
    }
  }
  nbf.upload(vf);
  nbb.upload(vb);
  fwd_cnt.alloc(std::max(fp.nsn, 1));
  bwd_cnt.alloc(std::max(fp.nsn, 1));
  ctl.alloc(dev::SW_COUNT);
  CUDA_CHECK(cudaMemset(fwd_cnt.p, 0, fwd_cnt.n * sizeof(unsigned long long)));
  CUDA_CHECK(cudaMemset(bwd_cnt.p, 0, bwd_cnt.n * sizeof(unsigned long long)));
  {
    std::vector<unsigned long long> c0(dev::SW_COUNT, 0ull);
    c0[dev::SW_T0] = ~0ull;
    CUDA_CHECK(cudaMemcpy(ctl.p, c0.data(), c0.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice));
  }
  CUDA_CHECK(cudaDeviceSynchronize());
  sweep_smem = smem_d * (int)sizeof(double);
  MDD_REQUIRE(sweep_smem <= 200 * 1024, 5, "supernode too large for shared-memory staging");
  if (sweep_smem > 48 * 1024)
    CUDA_CHECK(cudaFuncSetAttribute(dev::k_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, sweep_smem));
  int dev_id = 0, nsm = 0, per_sm = 0;
  CUDA_CHECK(cudaGetDevice(&dev_id));
  CUDA_CHECK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev_id));
  CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dev::k_sweep, dev::kSweepThreads, sweep_smem));
  MDD_REQUIRE(per_sm > 0, 5, "sweep kernel cannot be resident");
  sweep_grid = nsm * per_sm;
}

DevFactor::~DevFactor() {
  if (stats.p) {
    unsigned long long v[8];
    if (cudaMemcpy(v, stats.p, sizeof(v), cudaMemcpyDeviceToHost) == cudaSuccess)
      fprintf(stderr, "[mdd sweep stats %s] cycles: fwd wait %llu work %llu | bwd wait %llu work %llu | "
              "prolong wait %llu work %llu | ticket %llu | tasks %llu\n", name.c_str(), v[0], v[1], v[2],
              v[3], v[4], v[5], v[6], v[7]);
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
  dev::SweepDev S;
  S.P = plan();
  S.L = L.p;
  S.dinv = dinv.p;
  S.tasks = tasks.p;
  S.ntasks = out ? ntasks : ntasks_noprolong;
  S.total_bwd = total_bwd;
  S.nbf = nbf.p;
  S.nbb = nbb.p;
  S.parent = parent.p;
  S.fwd_cnt = fwd_cnt.p;
  S.bwd_cnt = bwd_cnt.p;
  S.ctl = ctl.p;
  S.upd = upd.p;
  S.xf = xf.p;
  S.xb = xb.p;
  S.b = b;
  S.gmap = gmap;
  S.pro_ptr = pro_ptr;
  S.pro_pos = pro_pos;
  S.out = out;
  S.stop = stop;
  S.stats = stats.p;
  const int grid = std::max(1, std::min(sweep_grid, S.ntasks));
  dev::k_sweep<<<grid, dev::kSweepThreads, sweep_smem, s>>>(S);
}

void DevFactor::check_abort(cudaStream_t s) {
  unsigned long long ab = 0;
  CUDA_CHECK(cudaMemcpyAsync(&ab, ctl.p + dev::SW_ABORT, sizeof(ab), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  if (ab) {
    CUDA_CHECK(cudaMemsetAsync(fwd_cnt.p, 0, fwd_cnt.n * sizeof(unsigned long long), s));
    CUDA_CHECK(cudaMemsetAsync(bwd_cnt.p, 0, bwd_cnt.n * sizeof(unsigned long long), s));
    std::vector<unsigned long long> c0(dev::SW_COUNT, 0ull);
    c0[dev::SW_T0] = ~0ull;
    CUDA_CHECK(cudaMemcpyAsync(ctl.p, c0.data(), c0.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
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
  if (mode == 2) return e;
  MDD_REQUIRE(e == 0, 3, "nonpositive pivot in an SPD factorisation");
  return 0;
}

}  // namespace mdd
