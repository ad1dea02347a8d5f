// Host drivers of the multifrontal factorisation and the level-scheduled
// supernodal triangular solves (kernels in kernels.cu).
#include <algorithm>

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

void DevFactor::upload() {
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
  fwd_smem.assign(fp.nlevels, 0);
  bwd_smem.assign(fp.nlevels, 0);
  for (int l = 0; l < fp.nlevels; ++l)
    for (int k = fp.level_ptr[l]; k < fp.level_ptr[l + 1]; ++k) {
      int g = fp.level_sn[k];
      int nc = fp.sn_ncol[g], no = fp.sn_noff[g];
      fwd_smem[l] = std::max(fwd_smem[l], (int)((nc + no + nc) * sizeof(double)));
      bwd_smem[l] = std::max(bwd_smem[l], (int)((no + nc) * sizeof(double)));
    }
  int mx = 0;
  for (int l = 0; l < fp.nlevels; ++l) mx = std::max(mx, std::max(fwd_smem[l], bwd_smem[l]));
  MDD_REQUIRE(mx <= 227 * 1024, 5, "supernode too large for shared-memory staging");
  if (mx > 48 * 1024) {
    CUDA_CHECK(cudaFuncSetAttribute(dev::k_fwd_level, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CUDA_CHECK(cudaFuncSetAttribute(dev::k_bwd_level, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  }
  L.alloc(fp.lsize);
  dinv.alloc(fp.ntot);
  upd.alloc(std::max<int64_t>(fp.usize, 1));
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

void DevFactor::forward(const double* b, const int32_t* gmap, double* x, cudaStream_t s) const {
  dev::PlanDev P = plan();
  for (int l = 0; l < fp.nlevels; ++l) {
    int cnt = fp.level_ptr[l + 1] - fp.level_ptr[l];
    dev::k_fwd_level<<<cnt, threads, fwd_smem[l], s>>>(P, fp.level_ptr[l], L.p, dinv.p, b, gmap, x, upd.p);
  }
}

void DevFactor::backward(double* x, cudaStream_t s) const {
  dev::PlanDev P = plan();
  for (int l = fp.nlevels - 1; l >= 0; --l) {
    int cnt = fp.level_ptr[l + 1] - fp.level_ptr[l];
    dev::k_bwd_level<<<cnt, threads, bwd_smem[l], s>>>(P, fp.level_ptr[l], L.p, x);
  }
}

}  // namespace mdd
