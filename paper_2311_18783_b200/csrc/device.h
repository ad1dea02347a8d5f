// Device-side helpers shared by the orchestration files.
#pragma once
#include <cuda_runtime.h>
#include <cusparse.h>

#include <string>
#include <vector>

#include "common.h"
#include "kernels.cuh"

namespace mdd {

#define CUDA_CHECK(x)                                                                     \
  do {                                                                                    \
    cudaError_t e__ = (x);                                                                \
    if (e__ != cudaSuccess)                                                               \
      throw ::mdd::Error(1, std::string(#x) + ": " + cudaGetErrorString(e__));            \
  } while (0)
#define CUSPARSE_CHECK(x)                                                                 \
  do {                                                                                    \
    cusparseStatus_t s__ = (x);                                                           \
    if (s__ != CUSPARSE_STATUS_SUCCESS)                                                   \
      throw ::mdd::Error(1, std::string(#x) + ": cusparse status " + std::to_string((int)s__)); \
  } while (0)

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() {}
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) CUDA_CHECK(cudaMalloc(&p, count * sizeof(T)));
  }
  void zero(cudaStream_t s) {
    if (n) CUDA_CHECK(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  // Setup-time transfers.  A pageable cudaMemcpy may return before its DMA lands
  // and is not ordered with the library's non-blocking stream, so both directions
  // synchronise the whole device.
  void upload(const std::vector<T>& v) { upload(v.data(), v.size()); }
  void upload(const T* v, size_t count) {
    alloc(count);
    if (n) {
      CUDA_CHECK(cudaMemcpy(p, v, n * sizeof(T), cudaMemcpyHostToDevice));
      CUDA_CHECK(cudaDeviceSynchronize());
    }
  }
  std::vector<T> download() const {
    std::vector<T> v(n);
    CUDA_CHECK(cudaDeviceSynchronize());
    if (n) CUDA_CHECK(cudaMemcpy(v.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost));
    return v;
  }
};

// A FactorPlan on the device plus its numeric factor and its sweep schedule.
struct DevFactor {
  FactorPlan fp;
  DBuf<int64_t> col0, rowptr, offrows, lptr, uptr, fptr, umptr, child_ptr, asm_ptr, asm_src;
  DBuf<int> ncol, noff, child_list, relmap, asm_pos, level_sn, parent;
  DBuf<double> L, dinv, upd, xf, xb;
  // persistent level-synchronous sweep (sweep.cu)
  DBuf<int4> phases, tdesc, tiles;
  DBuf<dev::MTaskDesc> mt_f, mt_b;
  DBuf<dev::CombDesc> cmb;
  DBuf<int64_t> tile_off, sn_fpart, sn_bpart, vb_off, cptr, cidx, wsrc;
  DBuf<int> sn_RB, sn_CB, sn_nrb, sn_ncb;
  DBuf<int32_t> gsrc;
  DBuf<double> Lt, fpart, bpart, vb;
  DBuf<unsigned long long> ctl, trace;
  int nphases = 0, ntiles = 0, sweep_grid = 0, n_out = 0;
  // plan statistics (mdd_info): supernodes swept as packed / strip / 2-D tasks,
  // fronts factorised by the blocked (cuBLAS trailing update) path
  int n_packed = 0, n_strip = 0, n_2d = 0, n_blocked = 0;
  int64_t lt_size = 0;
  const int64_t* pro_ptr = nullptr;
  const int32_t* pro_pos = nullptr;
  std::string name;
  // a rank's view of a replicated factor (sharded coarse solve, sharded.cu):
  // `base` holds the tiles and D^{-1}; role[g] = 1 the rank's subtrees (segment A),
  // 2 the replicated top (segment B), 0 not swept.  Empty role: the whole factor.
  const DevFactor* base = nullptr;
  std::vector<int8_t> role;
  int nph_a = 0;               // segment A = phases [0, nph_a), segment B = [nph_a, nphases)
  int64_t swept_entries = 0;   // factor entries this schedule sweeps
  DevFactor() = default;
  DevFactor(const DevFactor&) = delete;
  ~DevFactor();
  dev::PlanDev plan() const;
  dev::SweepDev sweep_dev() const;
  // Builds the sweep schedule.  prolong_n > 0 appends the prolongation onto
  // prolong_n global dofs; gmap_host maps positions to indices of the sweep's
  // right-hand side (NULL: the right-hand side is indexed by position).
  void upload(int prolong_n = 0, const int64_t* pro_ptr_dev = nullptr,
              const int32_t* pro_pos_dev = nullptr, const std::vector<int32_t>* gmap_host = nullptr);
  // numeric multifrontal factorisation from a device value array `src`; the
  // panels are then re-laid out into the sweep tiles
  int factor(const double* src, int mode, double tol, uint8_t* dropped, cudaStream_t s);
  // x = A^{-1} b in one persistent launch; with `out` the result is prolongated
  // (out[e] = sum of its copies; needs upload(prolong_n > 0)), else it stays in xb.
  // seg: -1 every phase, 0 / 1 segment A / B of a view (empty segments launch nothing)
  void sweep(const double* b, double* out, cudaStream_t s, const int* stop = nullptr, int seg = -1) const;
  // accumulated device time (ns) and count of sweep launches (SW_TSUM / SW_TCNT)
  void sweep_timing(unsigned long long* ns, unsigned long long* cnt, cudaStream_t s) const;
  // throws if a sweep aborted (barrier timeout); resets the schedule state
  void check_abort(cudaStream_t s);
  void reset_counters(cudaStream_t s);
};

}  // namespace mdd
