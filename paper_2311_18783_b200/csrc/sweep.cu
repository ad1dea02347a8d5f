// Persistent, level-synchronous supernodal triangular sweep (sm_100a, FP64).
//
// One launch applies A_i^{-1} for ALL subdomains at once (north_star: "local
// solves A_i^{-1} as supernodal sparse LDL^T factors applied by hand-written
// level-scheduled triangular-solve kernels, with dense supernode blocks as
// warp-tiled TRSV"), fusing the restriction R_i, the forward sweep L y = b, the
// diagonal D^{-1}, the backward sweep L^T x = z and the prolongation
// sum_i R_i^T x_i (PAPER.md eq. AS: M_AS = sum_i R_i^T A_i^{-1} R_i).  The same
// kernel applies E^{-1} for the coarse correction Z E^{-1} Z^T.
//
// Panels are in "partitioned-inverse" form P = [D^{-1} L11^{-1}; L21 L11^{-1}], so
// per supernode
//   forward :  z_c = (D^{-1} L11^{-1}) t_c,     u = t_off - (L21 L11^{-1}) t_c
//   backward:  x_c = (D^{-1} L11^{-1})^T (D z_c) - (L21 L11^{-1})^T x_off
// are plain dense mat-vecs over contiguous tiles (<= kTileMax doubles), each
// streamed from HBM by ONE TMA bulk copy (cp.async.bulk + mbarrier) with one
// task of look-ahead.
//
// The launch walks a fixed list of phases separated by grid barriers (all CTAs
// are co-resident: one persistent CTA set sized by the occupancy calculator):
//   for each level, leaves first:   G_f  (flat gather of every supernode's
//     right-hand side t = [b_c ; 0] + children's update vectors, a precomputed
//     row -> contributions list, so no scatter and no atomics)  |  M_f (tiles)
//     |  C_f (the partial sums of the level's 2-D supernodes)
//   for each level, root first:     G_b  (w = [D z_c ; -x_off])  |  M_b  |  C_b
//   prolongation.
// Levels with few tasks per CTA skip their G phase: each task gathers its own
// vector rows (same sums, same order).  Within M phases the tasks, sorted
// largest first, are dealt to the CTAs in snake order (no atomics).  A task is a
// small supernode (all its packed column tiles, accumulated in shared memory by
// one CTA), a strip of a wide supernode, or a group of 1-4 RB x CB tiles of a big
// supernode, which stores its partial sums; the C phase after the tiles adds them
// in a fixed order (one barrier instead of a publishing atomic and a deferred
// combine per group: those cost ~2 us of CTA time per group, measured on c4) --
// every reduction is bit-reproducible and independent of the grid size.  The
// barrier counter is cumulative across launches (SW_EPOCH: the barriers of the
// earlier launches, so launches may run different phase ranges); a barrier wait that
// exceeds kSpinTimeoutNs raises an abort flag reported by the host.
#include "kernels.cuh"

namespace mdd {
namespace dev {

#ifdef MDD_DEBUG_NOCOMPUTE
// experiment builds only (tools/time_sweeps.py --nocompute): set after the setup
__device__ int g_nocompute = 0;
#endif
namespace {
constexpr unsigned long long kSpinTimeoutNs = 4000000000ull;  // 4 s
constexpr int kWarps = kSweepThreads / 32;
constexpr int kGatherRows = 4;  // rows per thread in flight in the flat gather phases

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* m) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(m)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(m)),
      "r"(parity)
      : "memory");
}

// one row of the forward task vector: t = [b_c ; 0] + children's updates
__device__ __forceinline__ double gather_t(const SweepDev& S, long long q) {
  const int src = S.gsrc[q];
  double v = src >= 0 ? __ldg(S.b + src) : 0.0;
  for (i64 k = S.cptr[q]; k < S.cptr[q + 1]; ++k) v += __ldcg(S.upd + S.cidx[k]);
  return v;
}
// one row of the backward task vector: w = [D z_c ; -x_off]; a pivot dropped by
// the rank-revealing factorisation has D^{-1} = 0 and z_c = 0: its D z_c is 0
__device__ __forceinline__ double gather_w(const SweepDev& S, long long q) {
  const i64 w = S.wsrc[q];
  if (w < 0) return -__ldcg(S.xb + (-w - 1));
  const double di = __ldg(S.dinv + w);
  return di != 0.0 ? __ldcg(S.xf + w) / di : 0.0;
}

// grid-wide barrier over co-resident CTAs (cumulative counter, no reset); *abort
// (shared) receives the abort flag as thread 0 saw it, uniform across the CTA
__device__ void grid_barrier(unsigned long long* ctl, unsigned long long target, int* abort) {
  // bar.sync orders the CTA's writes before thread 0's release add; thread 0's
  // acquire load and the second bar.sync order every later read after the other
  // CTAs' writes (release/acquire at gpu scope, no full fence)
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(&ctl[SW_BAR]) : "memory");
    if (ld_acquire(&ctl[SW_BAR]) < target) {
      const unsigned long long t0 = globaltimer();
      for (int it = 0;; ++it) {
        __nanosleep(it < 64 ? 16 : 64);
        if (ld_acquire(&ctl[SW_BAR]) >= target) break;
        if ((it & 255) == 255) {
          if (*(volatile unsigned long long*)&ctl[SW_ABORT]) break;
          if (globaltimer() - t0 > kSpinTimeoutNs) {
            atomicExch(&ctl[SW_ABORT], 1ull);
            break;
          }
        }
      }
    }
    *abort = *(volatile unsigned long long*)&ctl[SW_ABORT] != 0;
  }
  __syncthreads();
}

// y_i = sum_j T[j*R + i] v[j] for i < R (T col-major in smem); fin(i, y_i) is called
// once per row by one thread.  Fixed-order reduction over column slices.
template <class Fin>
__device__ __forceinline__ void tile_matvec(const double* T, int R, int C, const double* v, double* red,
                                            Fin fin) {
  const int tid = threadIdx.x;
  if (R > kSweepThreads / 2) {
    for (int i = tid; i < R; i += kSweepThreads) {
      double s0 = 0.0, s1 = 0.0;
      int j = 0;
      for (; j + 2 <= C; j += 2) {
        s0 += T[j * R + i] * v[j];
        s1 += T[(j + 1) * R + i] * v[j + 1];
      }
      if (j < C) s0 += T[j * R + i] * v[j];
      fin(i, s0 + s1);
    }
    return;
  }
  if (R <= 16) {
    // few rows (a fwd strip of a wide supernode): R-row slices over the columns
    const int Rp = R > 8 ? 16 : R > 4 ? 8 : R > 2 ? 4 : R;
    const int nsl = min(kSweepThreads / Rp, C);
    const int i = tid % Rp, sl = tid / Rp;
    if (sl < nsl && i < R) {
      const int ja = (sl * C) / nsl, jb = ((sl + 1) * C) / nsl;
      double s0 = 0.0, s1 = 0.0;
      int j = ja;
      for (; j + 2 <= jb; j += 2) {
        s0 += T[j * R + i] * v[j];
        s1 += T[(j + 1) * R + i] * v[j + 1];
      }
      if (j < jb) s0 += T[j * R + i] * v[j];
      red[sl * Rp + i] = s0 + s1;
    }
    __syncthreads();
    if (tid < R) {
      double s = 0.0;
      for (int q = 0; q < nsl; ++q) s += red[q * Rp + tid];
      fin(tid, s);
    }
    return;
  }
  // 16 < R <= 128: 2^lg rows per slice, 2^(8-lg) column slices; all index math
  // in shifts (no integer division on the per-tile path)
  static_assert(kSweepThreads == 256, "slice mapping assumes 256 threads");
  const int lg = R <= 32 ? 5 : R <= 64 ? 6 : 7;
  const int lgs = min(8 - lg, C > 1 ? 32 - __clz(C - 1) : 0);  // no more slices than columns
  const int i = tid & ((1 << lg) - 1), sl = tid >> lg;
  if (i < R && sl < (1 << lgs)) {
    const int ja = (sl * C) >> lgs, jb = ((sl + 1) * C) >> lgs;
    double s0 = 0.0, s1 = 0.0;
    int j = ja;
    for (; j + 2 <= jb; j += 2) {
      s0 += T[j * R + i] * v[j];
      s1 += T[(j + 1) * R + i] * v[j + 1];
    }
    if (j < jb) s0 += T[j * R + i] * v[j];
    red[tid] = s0 + s1;  // slice sl, row i
  }
  __syncthreads();
  if (tid < R) {
    double s = 0.0;
    for (int q = 0; q < (1 << lgs); ++q) s += red[(q << lg) + tid];
    fin(tid, s);
  }
}

// Butterfly reduce-scatter of 8 per-lane partial sums (one per column of a group
// of 8) over the 32 lanes of a warp: 9 shuffles instead of 8 x 5.  Returns, in
// every lane, the full sum of column (lane >> 2); a fixed order (deterministic).
__device__ __forceinline__ double warp_reduce8(const double (&p)[8], int lane) {
  double q[4], r[2];
  {
    const bool hi = (lane >> 4) & 1;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double keep = hi ? p[k + 4] : p[k], send = hi ? p[k] : p[k + 4];
      q[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
  }
  {
    const bool hi = (lane >> 3) & 1;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double keep = hi ? q[k + 2] : q[k], send = hi ? q[k] : q[k + 2];
      r[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
  }
  const bool hi = (lane >> 2) & 1;
  const double keep = hi ? r[1] : r[0], send = hi ? r[0] : r[1];
  double s = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  return s;
}

// The same for 4 columns: the full sum of column (lane >> 3) in every lane.
__device__ __forceinline__ double warp_reduce4(const double (&p)[4], int lane) {
  double q[2];
  {
    const bool hi = (lane >> 4) & 1;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double keep = hi ? p[k + 2] : p[k], send = hi ? p[k] : p[k + 2];
      q[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
  }
  const bool hi = (lane >> 3) & 1;
  const double keep = hi ? q[1] : q[0], send = hi ? q[0] : q[1];
  double s = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  s += __shfl_xor_sync(0xffffffffu, s, 4);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  return s;
}

// y_j = sum_i T[j*R + i] w[i] for j < C (T col-major in smem).  Work unit: a
// warp x (a group of 8 columns, a slice of the rows); lanes run down the rows
// with 8 partial sums, then warp_reduce8; several row slices (when the columns
// are too few to occupy the warps) are added in order through `red`.  fin(j, y_j)
// once per column.  Callers __syncthreads after.
template <int W, class Fin>
__device__ __forceinline__ void tile_matvec_t_w(const double* T, int R, int C, const double* w, double* red,
                                                Fin fin) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = (C + W - 1) / W;
  const int nsl = G >= kWarps ? 1 : kWarps / G;
  constexpr int kSh = W == 8 ? 2 : 3;  // lane >> kSh = the column a lane ends with
  for (int jb = warp; jb < G * nsl; jb += kWarps) {
    const int g = jb % G, sl = jb / G;
    const int r0 = (sl * R) / nsl, r1 = ((sl + 1) * R) / nsl;
    double p[W];
#pragma unroll
    for (int k = 0; k < W; ++k) p[k] = 0.0;
    for (int i = r0 + lane; i < r1; i += 32) {
      const double wi = w[i];
#pragma unroll
      for (int k = 0; k < W; ++k)
        if (g * W + k < C) p[k] += T[(g * W + k) * R + i] * wi;
    }
    double v;
    if constexpr (W == 8) v = warp_reduce8(p, lane);
    else v = warp_reduce4(p, lane);
    const int j = g * W + (lane >> kSh);
    if ((lane & ((1 << kSh) - 1)) == 0 && j < C) {
      if (nsl == 1) fin(j, v);
      else red[sl * C + j] = v;
    }
  }
  if (nsl > 1) {
    __syncthreads();
    for (int j = threadIdx.x; j < C; j += kSweepThreads) {
      double y = 0.0;
      for (int q = 0; q < nsl; ++q) y += red[q * C + j];
      fin(j, y);
    }
  }
}
// Forward 2-D tile, rows in groups of 8 per warp (warp w: rows 8w.. and 64+8w..),
// lanes down the columns with 8 row partials each, then warp_reduce8: every lane
// ends with the full sum of row r0 + (lane >> 2), added to its register
// accumulator -- no shared-memory reduction and no block barrier inside the tile,
// so the partial sums of a group of tiles stay in registers.  Fixed order.
__device__ __forceinline__ void tile_rows8(const double* T, int R, int C, const double* v, double& acc0,
                                           double& acc1) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int gi = 0; gi < 2; ++gi) {
    const int r0 = 8 * (warp + 8 * gi);
    if (r0 >= R) break;  // warp-uniform
    double p[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) p[k] = 0.0;
    for (int c = lane; c < C; c += 32) {
      const double vc = v[c];
      const double* col = T + c * R + r0;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (r0 + k < R) p[k] += col[k] * vc;
    }
    const double sm8 = warp_reduce8(p, lane);
    if (gi == 0) acc0 += sm8;
    else acc1 += sm8;
  }
}

// groups of 8 columns for wide tiles (2-D: 64 columns), of 4 for narrow ones
template <class Fin>
__device__ __forceinline__ void tile_matvec_t(const double* T, int R, int C, const double* w, double* red,
                                              Fin fin) {
  if (C >= 48) tile_matvec_t_w<8>(T, R, C, w, red, fin);
  else tile_matvec_t_w<4>(T, R, C, w, red, fin);
}

// Packed lower-trapezoidal column tile of a small supernode: columns c0 .. c0+C-1
// of an nr-row panel, column jj holding rows c0+jj .. nr-1 (the zeros above the
// diagonal are not stored), column offsets coff(jj) = jj (nr - c0) - jj (jj - 1) / 2.
// Forward: y_i = sum_{jj <= i - c0} T(i, c0 + jj) v[jj] for rows i in [c0, nr);
// fin(i, y) once per row.
template <class Fin>
__device__ __forceinline__ void tile_matvec_packed(const double* T, int nr, int c0, int C, const double* v,
                                                   double* red, Fin fin) {
  const int tid = threadIdx.x;
  const int R = nr - c0;  // rows this tile touches
  if (R > kSweepThreads / 2) {
    for (int ip = tid; ip < R; ip += kSweepThreads) {
      const int jb = min(C, ip + 1);
      double s0 = 0.0, s1 = 0.0;
      int addr = ip, jj = 0;
      for (; jj + 2 <= jb; jj += 2) {
        s0 += T[addr] * v[jj];
        addr += R - jj - 1;
        s1 += T[addr] * v[jj + 1];
        addr += R - jj - 2;
      }
      if (jj < jb) s0 += T[addr] * v[jj];
      fin(c0 + ip, s0 + s1);
    }
    return;
  }
  // 2^lg rows per slice, 2^(8-lg) column slices (shifts only)
  const int lg = R <= 4 ? 2 : R <= 8 ? 3 : R <= 16 ? 4 : R <= 32 ? 5 : R <= 64 ? 6 : 7;
  const int lgs = min(8 - lg, C > 1 ? 32 - __clz(C - 1) : 0), Rp = 1 << lg, nsl = 1 << lgs;
  const int ip = tid & (Rp - 1), sl = tid >> lg;
  if (ip < R && sl < nsl) {
    const int ja = (sl * C) >> lgs, jb = min(((sl + 1) * C) >> lgs, ip + 1);
    double s0 = 0.0;
    // address of (row c0+ip, column jj): coff(jj) + ip - jj
    int addr = ja * R - (ja * (ja - 1)) / 2 + ip - ja;
    for (int jj = ja; jj < jb; ++jj) {
      s0 += T[addr] * v[jj];
      addr += R - jj - 1;
    }
    red[sl * Rp + ip] = s0;
  }
  __syncthreads();
  for (int q2 = tid; q2 < R; q2 += kSweepThreads) {
    double s = 0.0;
    for (int q = 0; q < nsl; ++q) s += red[q * Rp + q2];
    fin(c0 + q2, s);
  }
}

// Backward on a packed tile: x_jj = sum_{i >= c0+jj} T(i, c0+jj) w[i]; fin(jj, x)
#ifdef MDD_PACKED_T_WARP
// experiment: one warp per column
template <class Fin>
__device__ __forceinline__ void tile_matvec_t_packed(const double* T, int nr, int c0, int C, const double* w,
                                                     double*, Fin fin) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int R = nr - c0;
  for (int jj = warp; jj < C; jj += kWarps) {
    const double* col = T + (jj * R - (jj * (jj - 1)) / 2);
    const double* wj = w + c0 + jj;
    const int len = R - jj;
    double s0 = 0.0, s1 = 0.0;
    int i = lane;
    for (; i + 32 < len; i += 64) {
      s0 += col[i] * wj[i];
      s1 += col[i + 32] * wj[i + 32];
    }
    if (i < len) s0 += col[i] * wj[i];
    const double s = warp_sum(s0 + s1);
    if (lane == 0) fin(jj, s);
  }
}
#else
template <class Fin>
__device__ __forceinline__ void tile_matvec_t_packed(const double* T, int nr, int c0, int C, const double* w,
                                                     double* red, Fin fin) {
  // groups of 4 columns (a small tile has few columns: more warps busy)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int R = nr - c0;
  const int G = (C + 3) >> 2;
  const int nsl = G >= kWarps ? 1 : kWarps / G;
  for (int jb = warp; jb < G * nsl; jb += kWarps) {
    const int g = jb % G, sl = jb / G;
    const int len0 = R - g * 4;  // rows of the group's first (longest) column
    const int r0 = (sl * len0) / nsl, r1 = ((sl + 1) * len0) / nsl;
    double p[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i = r0 + lane; i < r1; i += 32) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int jj = g * 4 + k;
        // column jj holds rows c0+jj .. nr-1 at coff(jj) = jj R - jj (jj - 1) / 2
        if (jj < C && i < R - jj) p[k] += T[jj * R - (jj * (jj - 1)) / 2 + i] * w[c0 + jj + i];
      }
    }
    const double v = warp_reduce4(p, lane);
    const int jj = g * 4 + (lane >> 3);
    if ((lane & 7) == 0 && jj < C) {
      if (nsl == 1) fin(jj, v);
      else red[sl * C + jj] = v;
    }
  }
  if (nsl > 1) {
    __syncthreads();
    for (int j = threadIdx.x; j < C; j += kSweepThreads) {
      double y = 0.0;
      for (int q = 0; q < nsl; ++q) y += red[q * C + j];
      fin(j, y);
    }
  }
}
#endif
}  // namespace

__global__ void __launch_bounds__(kSweepThreads, kSweepCtasPerSm) k_sweep(SweepDev S) {
  extern __shared__ __align__(128) double sm[];
  // kStages tile slots (a ring: kStages - 1 tiles stream while one is computed on),
  // kVecSlots task-vector slots, accumulators, reduction scratch
  double* const vbase = sm + kStages * kTileMax;  // kVecSlots x (kVecMax + 2)
  double* const vec2 = vbase + kVecSlots * (kVecMax + 2);  // kVecMax: accumulators
  double* const red = vec2 + kVecMax;                       // kSweepThreads
  __shared__ __align__(8) uint64_t mbar[kStages];
  __shared__ __align__(16) MTaskDesc s_desc[kDescRing];
  __shared__ int s_tinfo[kStages];
  __shared__ int s_abort;  // the abort flag as of the last grid barrier (CTA-uniform)
  const int tid = threadIdx.x;
  if (S.stop && *S.stop) return;  // PCG already stopped: the whole sweep is a no-op
  // barriers of earlier launches (cumulative counter: the targets of this launch
  // continue from them)
  const unsigned long long base = S.ctl[SW_EPOCH];
  const unsigned long long grid = gridDim.x;
  if (tid == 0) {
    atomicMin(&S.ctl[SW_T0], globaltimer());
    for (int q = 0; q < kStages; ++q) mbar_init(&mbar[q]);
    s_abort = *(volatile unsigned long long*)&S.ctl[SW_ABORT] != 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t parbits = 0u;  // phase parity of every ring slot
  const size_t gthreads = (size_t)gridDim.x * kSweepThreads;
  const size_t gtid = (size_t)blockIdx.x * kSweepThreads + tid;

  for (int ph = S.ph0; ph < S.ph1; ++ph) {
    const int4 PH = S.phases[ph];
    const int kind = PH.x;
    const unsigned long long t_ph = (S.trace && tid == 0) ? globaltimer() : 0ull;
    // trace (thread 0): time in tile waits, tiles, task starts, tile bodies, tasks
    unsigned long long t_wait = 0, t_tiles = 0, t_start = 0, t_body = 0, t_tasks = 0;
    const bool trc = S.trace && tid == 0;
    if (kind == PH_GF) {
      // t = [b_c ; 0] + children's updates: 4 rows per thread interleaved (their
      // dependent loads in flight together), each row's sum in its fixed order
      const size_t lo = PH.y, hi = PH.z;
      for (size_t q0 = lo + gtid; q0 < hi; q0 += kGatherRows * gthreads) {
        double v[kGatherRows];
        i64 c0[kGatherRows], c1[kGatherRows];
#pragma unroll
        for (int k = 0; k < kGatherRows; ++k) {
          const size_t q = q0 + k * gthreads;
          int src = -1;
          c0[k] = c1[k] = 0;
          if (q < hi) { src = S.gsrc[q]; c0[k] = S.cptr[q]; c1[k] = S.cptr[q + 1]; }
          v[k] = src >= 0 ? __ldg(S.b + src) : 0.0;
        }
        for (int j = 0;; ++j) {
          bool any = false;
#pragma unroll
          for (int k = 0; k < kGatherRows; ++k)
            if (c0[k] + j < c1[k]) { v[k] += __ldcg(S.upd + S.cidx[c0[k] + j]); any = true; }
          if (!any) break;
        }
#pragma unroll
        for (int k = 0; k < kGatherRows; ++k)
          if (q0 + k * gthreads < hi) S.vb[q0 + k * gthreads] = v[k];
      }
    } else if (kind == PH_GB) {
      // w = [D z_c ; -x_off], 4 rows per thread interleaved
      const size_t lo = PH.y, hi = PH.z;
      for (size_t q0 = lo + gtid; q0 < hi; q0 += kGatherRows * gthreads) {
        i64 w[kGatherRows];
#pragma unroll
        for (int k = 0; k < kGatherRows; ++k) w[k] = q0 + k * gthreads < hi ? S.wsrc[q0 + k * gthreads] : 0;
        double v[kGatherRows], d[kGatherRows];
#pragma unroll
        for (int k = 0; k < kGatherRows; ++k) {
          if (w[k] < 0) { v[k] = -__ldcg(S.xb + (-w[k] - 1)); d[k] = 0.0; }
          else { v[k] = __ldcg(S.xf + w[k]); d[k] = __ldg(S.dinv + w[k]); }
        }
#pragma unroll
        for (int k = 0; k < kGatherRows; ++k)
          if (q0 + k * gthreads < hi) S.vb[q0 + k * gthreads] = w[k] < 0 ? v[k] : d[k] != 0.0 ? v[k] / d[k] : 0.0;
      }
    } else if (kind == PH_CF || kind == PH_CB) {
      // the partial sums of the level's 2-D row blocks (forward) / column blocks
      // (backward): one warp per block, each lane two outputs (o, o + 32) with four
      // partial chains each (sixteen loads in flight, two rounds of the four chains per trip); fixed order, grid-independent:
      // sum = (a0 + a1) + (a2 + a3), a_k = the partials q = k mod 4 in index order
      const bool cf = kind == PH_CF, fz = (PH.w & 1) != 0;
      const int lane = tid & 31;
      const size_t nw = (size_t)gridDim.x * kWarps;
      if ((PH.w & 2) && !(S.flags & SWF_NO_CTA_COMBINE)) {
        // few items with long partial chains (the upper levels' big supernodes):
        // one CTA per item, warp w sums the partials [w ntl / 8, (w+1) ntl / 8)
        // (four chains, as below), then the eight warp sums are added in warp
        // order -- fixed, grid-independent
        const int warp = tid >> 5;
        double* const wred = sm;  // the tile ring is idle in a C phase
        for (size_t it = (size_t)PH.y + blockIdx.x; it < (size_t)PH.z; it += gridDim.x) {
          const CombDesc C = S.cmb[it];
          const double* pb = (cf ? S.fpart : S.bpart) + C.comb;
          const int q0 = (warp * C.ntl) / kWarps, q1 = ((warp + 1) * C.ntl) / kWarps;
          for (int o = lane; o < C.m; o += 64) {
            const bool two = o + 32 < C.m;
            double a[4] = {0.0, 0.0, 0.0, 0.0}, e[4] = {0.0, 0.0, 0.0, 0.0};
            int q = q0;
            // sixteen loads in flight per lane (the chains are dependent-latency
            // bound: ~1 us per round); the same four chains in the same order
            for (; q + 8 <= q1; q += 8) {
              double t[8], u[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                t[k] = __ldcg(pb + (i64)(q + k) * C.ld + o);
                u[k] = two ? __ldcg(pb + (i64)(q + k) * C.ld + o + 32) : 0.0;
              }
#pragma unroll
              for (int k = 0; k < 4; ++k) { a[k] += t[k]; e[k] += u[k]; }
#pragma unroll
              for (int k = 0; k < 4; ++k) { a[k] += t[k + 4]; e[k] += u[k + 4]; }
            }
            for (; q + 4 <= q1; q += 4) {
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                a[k] += __ldcg(pb + (i64)(q + k) * C.ld + o);
                if (two) e[k] += __ldcg(pb + (i64)(q + k) * C.ld + o + 32);
              }
            }
#pragma unroll
            for (int k = 0; k < 3; ++k)
              if (q + k < q1) {
                a[k] += __ldcg(pb + (i64)(q + k) * C.ld + o);
                if (two) e[k] += __ldcg(pb + (i64)(q + k) * C.ld + o + 32);
              }
            wred[warp * 2 * kVecMax / 4 + o] = (a[0] + a[1]) + (a[2] + a[3]);
            if (two) wred[warp * 2 * kVecMax / 4 + o + 32] = (e[0] + e[1]) + (e[2] + e[3]);
          }
          __syncthreads();
          for (int o = tid; o < C.m; o += kSweepThreads) {
            double sum = 0.0;
            for (int w = 0; w < kWarps; ++w) sum += wred[w * 2 * kVecMax / 4 + o];
            const int r = C.first + o;
            if (!cf) S.xb[C.col0 + r] = sum;
            else if (r < C.nc) S.xf[C.col0 + r] = sum;
            else S.upd[C.uptr + (r - C.nc)] = (fz ? gather_t(S, C.vo + r) : __ldcg(S.vb + C.vo + r)) - sum;
          }
          __syncthreads();
        }
      } else
      for (size_t it = (size_t)PH.y + (size_t)blockIdx.x * kWarps + (tid >> 5); it < (size_t)PH.z; it += nw) {
        const CombDesc C = S.cmb[it];
        const double* pb = (cf ? S.fpart : S.bpart) + C.comb;
        for (int o = lane; o < C.m; o += 64) {
          const bool two = o + 32 < C.m;
          double a[4] = {0.0, 0.0, 0.0, 0.0}, e[4] = {0.0, 0.0, 0.0, 0.0};
          int q = 0;
          for (; q + 8 <= C.ntl; q += 8) {  // sixteen loads in flight, the same chains and order
            double t[8], u[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              t[k] = __ldcg(pb + (i64)(q + k) * C.ld + o);
              u[k] = two ? __ldcg(pb + (i64)(q + k) * C.ld + o + 32) : 0.0;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) { a[k] += t[k]; e[k] += u[k]; }
#pragma unroll
            for (int k = 0; k < 4; ++k) { a[k] += t[k + 4]; e[k] += u[k + 4]; }
          }
          for (; q + 4 <= C.ntl; q += 4) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              a[k] += __ldcg(pb + (i64)(q + k) * C.ld + o);
              if (two) e[k] += __ldcg(pb + (i64)(q + k) * C.ld + o + 32);
            }
          }
#pragma unroll
          for (int k = 0; k < 3; ++k)
            if (q + k < C.ntl) {
              a[k] += __ldcg(pb + (i64)(q + k) * C.ld + o);
              if (two) e[k] += __ldcg(pb + (i64)(q + k) * C.ld + o + 32);
            }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h == 1 && !two) break;
            const double sum = h ? (e[0] + e[1]) + (e[2] + e[3]) : (a[0] + a[1]) + (a[2] + a[3]);
            const int r = C.first + o + 32 * h;
            if (!cf) S.xb[C.col0 + r] = sum;
            else if (r < C.nc) S.xf[C.col0 + r] = sum;
            else S.upd[C.uptr + (r - C.nc)] = (fz ? gather_t(S, C.vo + r) : __ldcg(S.vb + C.vo + r)) - sum;
          }
        }
      }
    } else if (kind == PH_PR) {
      for (size_t e = gtid; e < (size_t)S.n_out; e += gthreads) {
        double s = 0.0;
        for (i64 k = S.pro_ptr[e]; k < S.pro_ptr[e + 1]; ++k) s += __ldcg(S.xb + S.pro_pos[k]);
        S.out[e] = s;
      }
    } else if (!s_abort) {
      // ---------------------------------------------- M phase: tiles.  Tasks are
      // sorted largest first and dealt to the CTAs in snake order (no atomics);
      // every per-task quantity comes from one packed descriptor.
      const bool fwd = kind == PH_MF;
      const bool fused = PH.w != 0;  // task vectors gathered by the task itself
      const MTaskDesc* const MT = (fwd ? S.mtf : S.mtb) + PH.y;
      const int ntk = PH.z - PH.y;
      const int b = blockIdx.x, G = gridDim.x;
      auto task_of = [&](int i) -> int {
        const int k = (i & 1) ? i * G + (G - 1 - b) : i * G + b;
        return k < ntk ? k : -1;
      };
      // thread 0: stream the tile of descriptor d into ring slot `bf`, plus (vbytes > 0) the task
      // vector into vector slot `vs`
      auto prefetch = [&](const int4 d, int bf, long long vlo2, int vbytes, int vs) {
        s_tinfo[bf] = d.x;  // read by the consumer after at least one __syncthreads
        const int64_t off = (int64_t)(((uint64_t)(uint32_t)d.w << 32) | (uint32_t)d.z);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar[bf])),
                     "r"((uint32_t)d.y + (uint32_t)vbytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(sm + bf * kTileMax)),
            "l"(S.Lt + off), "r"((uint32_t)d.y), "r"(smem_u32(&mbar[bf]))
            : "memory");
        if (vbytes > 0)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(vbase + vs * (kVecMax + 2))),
              "l"(S.vb + vlo2), "r"((uint32_t)vbytes), "r"(smem_u32(&mbar[bf]))
              : "memory");
      };
      // this CTA's task descriptors stream into a 4-slot shared-memory ring with
      // cp.async, three tasks ahead (no descriptor load on any critical path)
      constexpr int kDW = (int)(sizeof(MTaskDesc) / 16);  // 16-byte words per descriptor
      auto desc_fetch = [&](int i) {  // threads < kDW: one commit group per call
        if (tid < kDW) {
          const int kt = task_of(i);
          if (kt >= 0)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(
                             reinterpret_cast<const int4*>(&s_desc[i % kDescRing]) + tid)),
                         "l"(reinterpret_cast<const int4*>(MT + kt) + tid)
                         : "memory");
          asm volatile("cp.async.commit_group;" ::: "memory");
        }
      };
      for (int q = 0; q < kDescAhead; ++q) desc_fetch(q);
      if (tid < kDW) asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();
      // thread 0's prefetch cursor over this CTA's tile stream (task pi, tile pk);
      // it runs at most kStages tiles ahead, i.e. <= 2 tasks past the current one.
      // It only moves to a task whose descriptor is known to be resident (task
      // index <= avail = current + kDescAhead - 1 after the wait below); a ring slot freed
      // before that is owed and refilled at the next task's start.
      int pi = -1, pk = 0, pk1 = 0, ps = 0, avail = kDescAhead - 1, owed = 0;
      auto issue_next = [&]() {  // thread 0: one ring slot is free
        while (pk >= pk1) {
          if (task_of(pi + 1) < 0) return;        // stream exhausted
          if (pi + 1 > avail) { ++owed; return; }  // descriptor not resident yet
          ++pi;
          pk = s_desc[pi % kDescRing].k0;
          pk1 = s_desc[pi % kDescRing].k1;
        }
        const MTaskDesc& Dp = s_desc[pi % kDescRing];
        const bool first = pk == Dp.k0;
        const int j = pk - Dp.k0;
        prefetch(j < kTdInline ? Dp.td[j] : S.tdesc[pk], ps % kStages, Dp.vlo2, first && !fused ? Dp.vbytes : 0,
                 pi % kVecSlots);
        ++ps;
        ++pk;
      };
      if (tid == 0)
        for (int q = 0; q < kStages; ++q) issue_next();
      int cs = 0;  // tiles consumed in this phase
      for (int i = 0;; ++i) {
        const int k = task_of(i);
        if (k < 0) break;
        const unsigned long long s0 = trc ? globaltimer() : 0ull;
        if (trc) ++t_tasks;
        // descriptors i+1, i+2 must be resident before the cursor reaches them;
        // task i+3's starts streaming now
        desc_fetch(i + kDescAhead);
        if (tid < kDW) asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
          avail = i + kDescAhead - 1;
          for (int q = owed; q > 0; --q) {
            owed = 0;
            issue_next();
            if (owed) { owed = q; break; }
          }
        }
        const MTaskDesc D = s_desc[i % kDescRing];
        double* const vvw = vbase + (i % kVecSlots) * (kVecMax + 2) + D.voff;
        const double* const vv = vvw;  // this task's vector
        if (fused) {
          // the gathers overlap the task's first tile, already in flight
          const long long lo = D.vlo2 + D.voff;
          for (int q = tid; q < D.vn; q += kSweepThreads) vvw[q] = fwd ? gather_t(S, lo + q) : gather_w(S, lo + q);
          __syncthreads();
        }
        int buf = 0;
        if (trc) t_start += globaltimer() - s0;
        unsigned long long b0 = 0;
        // wait for the next tile of the stream (its ring slot becomes `buf`)
        auto next_tile_and_wait = [&](int) {
          buf = cs % kStages;
          const unsigned long long w0 = trc ? globaltimer() : 0ull;
          mbar_wait(&mbar[buf], (parbits >> buf) & 1u);
          if (trc) { b0 = globaltimer(); t_wait += b0 - w0; ++t_tiles; }
          parbits ^= 1u << buf;
        };
        // after the tile's last read (callers __syncthreads first): refill its slot
        auto tile_done = [&]() {
          if (tid == 0) issue_next();
          if (trc) t_body += globaltimer() - b0;
          ++cs;
        };
#ifdef MDD_DEBUG_NOCOMPUTE
        if (g_nocompute) {  // timing experiment: stream the tiles, skip the arithmetic
          for (int kk = D.k0; kk < D.k1; ++kk) {
            next_tile_and_wait(kk);
            __syncthreads();
            tile_done();
          }
        } else
#endif
        if (D.big == 2) {
          // ---------------- strip of a wide supernode (nr <= kVecMax): fwd = rows
          // [r0, r0+rows) x columns [0, cols), bwd = rows [c0, nr) x columns
          // [c0, c0+cols) (the lower trapezoid it touches); the task vector is the
          // whole t (fwd) / w (bwd): no partial sums
          next_tile_and_wait(D.k0);
          const double* T = sm + buf * kTileMax;
          if (fwd) {
            double* const upd = S.upd + D.uptr;
            tile_matvec(T, D.rows, D.cols, vv, red, [&](int i2, double y) {
              const int r = D.rb + i2;
              if (r < D.nc) S.xf[D.col0 + r] = y;
              else upd[r - D.nc] = vv[r] - y;
            });
          } else {
            double* const xb = S.xb + D.col0 + D.cb;
            tile_matvec_t(T, D.nr - D.cb, D.cols, vv + D.cb, red, [&](int j, double y) { xb[j] = y; });
          }
          __syncthreads();
          tile_done();
        } else if (!D.big) {
          // ---------------- small supernode: all column tiles, one CTA
          // packed column tiles: tdesc.x = first column | columns << 16
          for (int kk = D.k0; kk < D.k1; ++kk) {
            next_tile_and_wait(kk);
            const int cx = s_tinfo[buf];  // written by thread 0 with the tile's bulk copy
            const int c0 = cx & 0xffff, cols = cx >> 16;
            const double* T = sm + buf * kTileMax;
            if (fwd) {
              if (c0 == 0)
                tile_matvec_packed(T, D.nr, 0, cols, vv, red, [&](int r, double y) { vec2[r] = y; });
              else
                tile_matvec_packed(T, D.nr, c0, cols, vv + c0, red, [&](int r, double y) { vec2[r] += y; });
            } else {
              double* const xb = S.xb + D.col0 + c0;
              tile_matvec_t_packed(T, D.nr, c0, cols, vv, red, [&](int j, double y) { xb[j] = y; });
            }
            __syncthreads();
            tile_done();
          }
          if (fwd) {
            double* const upd = S.upd + D.uptr;
            for (int r = tid; r < D.nr; r += kSweepThreads) {
              if (r < D.nc) S.xf[D.col0 + r] = vec2[r];
              else upd[r - D.nc] = vv[r] - vec2[r];
            }
          }
        } else {
          // ---------------- a group of <= 4 tiles of a 2-D supernode: one row block and
          // consecutive column blocks (fwd) / one column block and consecutive row
          // blocks (bwd), accumulated in shared memory into one partial sum
          double acc0 = 0.0, acc1 = 0.0;  // forward: this lane's rows (tile_rows8)
          for (int kk = D.k0; kk < D.k1; ++kk) {
            const int j = kk - D.k0;
            next_tile_and_wait(kk);
            const double* T = sm + buf * kTileMax;
            if (fwd) {
              const int cols = min(D.CB, D.nc - (D.cb + j) * D.CB);
              tile_rows8(T, D.rows, cols, vv + j * D.CB, acc0, acc1);
            } else {
              const int rows = min(D.RB, D.nr - (D.rb + j) * D.RB);
              if (j == 0) tile_matvec_t(T, rows, D.cols, vv, red, [&](int c, double y) { vec2[c] = y; });
              else tile_matvec_t(T, rows, D.cols, vv + j * D.RB, red, [&](int c, double y) { vec2[c] += y; });
            }
            __syncthreads();
            tile_done();
          }
          // this group's partial sums; the level's combine phase adds them
          if (fwd) {
            double* const part = S.fpart + D.part;
            const int lane = tid & 31, r = 8 * (tid >> 5) + (lane >> 2);
            if ((lane & 3) == 0) {
              if (r < D.rows) part[r] = acc0;
              if (r + 64 < D.rows) part[r + 64] = acc1;
            }
          } else {
            double* const part = S.bpart + D.part;
            for (int q = tid; q < D.cols; q += kSweepThreads) part[q] = vec2[q];
          }
        }
        __syncthreads();
      }
    }
    // the next phases read vb / upd / xf / xb with TMA bulk copies (async proxy):
    // order this thread's generic-proxy global writes before them
    asm volatile("fence.proxy.async.global;" ::: "memory");
    if (trc) {
      unsigned long long* tr = S.trace + kTraceWords * ((size_t)ph * gridDim.x + blockIdx.x);
      tr[0] = t_ph;
      tr[1] = globaltimer();
      tr[2] = t_wait;
      tr[3] = t_tiles;
      tr[4] = 0;  // (was: deferred-combine flushes)
      tr[5] = t_start;
      tr[6] = t_body;
      tr[7] = t_tasks;
    }
    if (ph + 1 < S.ph1) grid_barrier(S.ctl, (base + (unsigned long long)(ph - S.ph0) + 1) * grid, &s_abort);
  }
  if (blockIdx.x == 0 && tid == 0) {
    // every CTA read the epoch before the first barrier
    S.ctl[SW_TSUM] += globaltimer() - S.ctl[SW_T0];
    S.ctl[SW_TCNT] += 1;
    S.ctl[SW_T0] = ~0ull;
    S.ctl[SW_EPOCH] = base + (unsigned long long)(S.ph1 - S.ph0 - 1);
    __threadfence();
  }
}

// relayout of the column-major panels into contiguous tiles (setup).  tiles[k] =
// {g, a, b, kind}: 0 2-D (rb, cb), 1 forward row strip (first row a, b rows,
// columns [0, min(nc, a + b))), 2 backward column strip (a columns from b, rows
// [b, nr)), 3 small packed column tile
// (a = columns, b = first column)
__global__ void k_tile_relayout(SweepDev S, int ntiles, const double* __restrict__ L,
                                const int64_t* __restrict__ lptr) {
  const int k = blockIdx.x;
  if (k >= ntiles) return;
  const int4 tl = S.tiles[k];
  const int g = tl.x, kind = tl.w;
  const int nc = S.P.sn_ncol[g], nr = nc + S.P.sn_noff[g];
  const int RB = S.sn_RB[g], CB = S.sn_CB[g];
  int r0 = 0, c0 = 0, rows = nr, cols = nc;
  if (kind == 0) {
    r0 = tl.y * RB; c0 = tl.z * CB;
    rows = min(RB, nr - r0); cols = min(CB, nc - c0);
  } else if (kind == 1) {
    r0 = tl.y; rows = tl.z; cols = min(nc, r0 + rows);
  } else {
    c0 = tl.z; cols = tl.y; r0 = c0; rows = nr - c0;
  }
  double* dst = const_cast<double*>(S.Lt) + S.tile_off[k];
  if (kind == 3) {
    // packed: column jj of the tile (panel column c0 + jj) keeps rows c0 + jj .. nr-1
    c0 = tl.z;
    cols = tl.y;
    const int R = nr - c0;
    int off = 0;
    for (int jj = 0; jj < cols; ++jj) {
      const int len = R - jj;
      const double* src = L + lptr[g] + (i64)(c0 + jj) * nr + (c0 + jj);
      for (int q = threadIdx.x; q < len; q += blockDim.x) dst[off + q] = src[q];
      off += len;
    }
    if (threadIdx.x == 0 && (off & 1)) dst[off] = 0.0;
    return;
  }
  const double* src = L + lptr[g] + (i64)c0 * nr + r0;
  for (int q = threadIdx.x; q < rows * cols; q += blockDim.x) {
    const int j = q / rows, i = q % rows;
    dst[q] = src[(i64)j * nr + i];
  }
  if (threadIdx.x == 0 && ((rows * cols) & 1)) dst[rows * cols] = 0.0;
}

}  // namespace dev
}  // namespace mdd

#ifdef MDD_DEBUG_NOCOMPUTE
extern "C" int mdd_debug_set_nocompute(int on) {
  return (int)cudaMemcpyToSymbol(mdd::dev::g_nocompute, &on, sizeof(int));
}
#endif
