// Persistent, dependency-driven supernodal triangular sweep (sm_100a, FP64).
//
// One launch applies A_i^{-1} for ALL subdomains at once (north_star: "local
// solves A_i^{-1} as supernodal sparse LDL^T factors applied by hand-written
// level-scheduled triangular-solve kernels, with dense supernode blocks as
// warp-tiled TRSV"), fusing the restriction R_i (gather in the leaves), the
// forward sweep L y = b, the diagonal D^{-1}, the backward sweep L^T x = z and
// the prolongation sum_i R_i^T x_i (PAPER.md eq. AS, M_AS = sum R_i^T A_i^{-1} R_i).
// The same kernel applies E^{-1} for the coarse correction.
//
// Panels are in "partitioned-inverse" form P = [L11^{-1}; L21 L11^{-1}], so
//   forward :  z_c = D^{-1} (L11^{-1} t_c),     u = t_off - (L21 L11^{-1}) t_c
//   backward:  x_c = L11^{-T} z_c - (L21 L11^{-1})^T x_off
// are plain dense mat-vecs.  Every panel is cut into tiles of <= kTileMax
// doubles stored contiguously (factor_driver.cu), so each task streams ONE
// contiguous block from HBM with a single TMA bulk copy (cp.async.bulk +
// mbarrier) into shared memory.  The copy for the next task is issued before the
// current task waits for its dependencies, so HBM latency, ticket latency and
// dependency latency overlap.
//
// A small supernode (nr <= kVecMax, nr*nc <= kTileMax) is one tile and one task
// per direction.  A big one has an assemble task (its right-hand side t = b +
// children updates, to global memory) and RB x CB tiles whose partial sums are
// combined, in a fixed order (bit-reproducible), by the last tile to arrive in
// each row block (forward) or column block (backward).
//
// Scheduling: tasks (forward work in level order, backward work in reverse level
// order, prolongation chunks) are handed out by an atomic ticket; a task only
// waits for tasks with smaller tickets, so the schedule is deadlock-free for any
// grid size (also with one ticket of look-ahead).  Counters are cumulative
// across launches (epoch = launches so far); the last CTA to exit advances the
// epoch.  A wait that exceeds kSpinTimeoutNs raises an abort flag (reported by
// the host) instead of hanging the device.
#include "kernels.cuh"

namespace mdd {
namespace dev {

namespace {
constexpr unsigned long long kSpinTimeoutNs = 4000000000ull;  // 4 s
constexpr int kWarps = kSweepThreads / 32;

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
// one thread: arm the barrier for `bytes` and start the bulk copy global -> shared
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(m))
      : "memory");
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

// one thread: spin until *p >= target; false on abort / timeout
__device__ bool wait_ge(const unsigned long long* p, unsigned long long target, unsigned long long* ctl) {
  if (ld_acquire(p) >= target) return true;
  const unsigned long long t0 = globaltimer();
  unsigned int ns = 32;
  for (int it = 0;; ++it) {
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
    if (ld_acquire(p) >= target) return true;
    if ((it & 63) == 63) {
      if (*(volatile unsigned long long*)&ctl[SW_ABORT]) return false;
      if (globaltimer() - t0 > kSpinTimeoutNs) {
        atomicExch(&ctl[SW_ABORT], 1ull);
        return false;
      }
    }
  }
}

// warp 0: wait until every child of g finished its forward work (lanes check the
// children in parallel); the verdict is returned to all threads
__device__ bool wait_children(const SweepDev& S, int g, unsigned long long cur, int* s_flag) {
  const int tid = threadIdx.x;
  if (tid < 32) {
    bool ok = *(volatile unsigned long long*)&S.ctl[SW_ABORT] == 0;
    const i64 c0 = S.P.child_ptr[g], c1 = S.P.child_ptr[g + 1];
    for (i64 ci = c0 + tid; ok && ci < c1; ci += 32) {
      const int c = S.P.child_list[ci];
      ok = wait_ge(&S.fwd_cnt[c], cur * (unsigned long long)S.sn_nrb[c], S.ctl);
    }
    ok = __all_sync(0xffffffffu, ok);
    if (tid == 0) {
      __threadfence();
      *s_flag = ok;
    }
  }
  __syncthreads();
  return *s_flag != 0;
}

__device__ bool wait_one(const unsigned long long* p, unsigned long long target,
                         unsigned long long* ctl, int* s_flag) {
  if (threadIdx.x == 0) {
    bool ok = *(volatile unsigned long long*)&ctl[SW_ABORT] == 0;
    if (ok) ok = wait_ge(p, target, ctl);
    __threadfence();
    *s_flag = ok;
  }
  __syncthreads();
  return *s_flag != 0;
}

__device__ __forceinline__ void signal_add(unsigned long long* p) {
  __threadfence();
  atomicAdd(p, 1ull);
}

struct TileGeo {
  int nr, nc, RB, CB, nrb, ncb, rows, cols;
};
__device__ __forceinline__ TileGeo geo(const SweepDev& S, int g, int rb, int cb) {
  TileGeo t;
  t.nc = S.P.sn_ncol[g];
  t.nr = t.nc + S.P.sn_noff[g];
  t.RB = S.sn_RB[g];
  t.CB = S.sn_CB[g];
  t.nrb = S.sn_nrb[g];
  t.ncb = S.sn_ncb[g];
  t.rows = min(t.RB, t.nr - rb * t.RB);
  t.cols = min(t.CB, t.nc - cb * t.CB);
  return t;
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
  const int Rp = (R + 31) & ~31;
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
}

// y_j = sum_i T[j*R + i] w[i] (warp per column, lanes down the rows); fin(j, y_j)
template <class Fin>
__device__ __forceinline__ void tile_matvec_t(const double* T, int R, int C, const double* w, Fin fin) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < C; j += kWarps) {
    const double* col = T + j * R;
    double s0 = 0.0, s1 = 0.0;
    int i = lane;
    for (; i + 32 < R; i += 64) {
      s0 += col[i] * w[i];
      s1 += col[i + 32] * w[i + 32];
    }
    if (i < R) s0 += col[i] * w[i];
    const double s = warp_sum(s0 + s1);
    if (lane == 0) fin(j, s);
  }
}
}  // namespace

__global__ void __launch_bounds__(kSweepThreads, 3) k_sweep(SweepDev S) {
  extern __shared__ __align__(128) double sm[];
  double* const vec = sm + 2 * kTileMax;   // kVecMax
  double* const vec2 = vec + kVecMax;      // kVecMax
  double* const red = vec2 + kVecMax;      // kSweepThreads
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ int s_next[2];
  __shared__ int s_flag;
  const int tid = threadIdx.x;
  const PlanDev& P = S.P;
  if (S.stop && *S.stop) return;  // PCG already stopped: the whole sweep is a no-op
  const unsigned long long cur = S.ctl[SW_EPOCH] + 1;
  if (tid == 0) {
    atomicMin(&S.ctl[SW_T0], globaltimer());
    mbar_init(&mbar[0]);
    mbar_init(&mbar[1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  long long st_acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long c_prev = clock64();
#define STAT_MARK(slot) \
  if (S.stats && tid == 0) { long long c_ = clock64(); st_acc[(slot)] += c_ - c_prev; c_prev = c_; } \
  if (S.trace && tid == 0 && ((slot) == 0 || (slot) == 2 || (slot) == 4 || (slot) == 6)) \
    S.trace[4 * (size_t)t + 1] = globaltimer();

  // thread 0 helpers: start streaming a tile into a stage buffer.  tdesc[k] =
  // {tile, bytes, offset lo, offset hi} in task order: one load per prefetch
  auto prefetch_k = [&](int k, int b) {
    const int4 d = S.tdesc[k];
    const int64_t off = (int64_t)(((uint64_t)(uint32_t)d.w << 32) | (uint32_t)d.z);
    bulk_load(sm + b * kTileMax, S.Lt + off, (uint32_t)d.y, &mbar[b]);
  };
  auto first_k = [&](int t) -> int {
    if (t >= S.ntasks) return -1;
    const int a = S.tt_ptr[t];
    return a < S.tt_ptr[t + 1] ? a : -1;
  };
  int tn = 0;  // thread 0: the look-ahead ticket
  if (tid == 0) {
    const int t0 = (int)atomicAdd(&S.ctl[SW_TICKET], 1ull);
    s_next[0] = t0;
    const int fk = first_k(t0);
    if (fk >= 0) prefetch_k(fk, 0);
  }
  __syncthreads();
  uint32_t par[2] = {0u, 0u};
  int it = 0, buf = 0;
  // wait for the tile in `buf` and issue the next one of the stream into buf ^ 1
  auto next_tile_and_wait = [&](int k, int kend) {
    if (tid == 0) {
      const int nk = k + 1 < kend ? k + 1 : first_k(tn);
      if (nk >= 0) prefetch_k(nk, buf ^ 1);
    }
    mbar_wait(&mbar[buf], par[buf]);
    par[buf] ^= 1u;
  };
  for (;;) {
    const int t = s_next[it & 1];
    if (t >= S.ntasks) break;
    const int4 tk = S.tasks[t];
    const int type = tk.x;
    const int ka = S.tt_ptr[t], kb = S.tt_ptr[t + 1];
    if (tid == 0) {
      tn = (int)atomicAdd(&S.ctl[SW_TICKET], 1ull);
      s_next[(it + 1) & 1] = tn;
      if (ka == kb) {  // no tile of ours in flight: the next task's first tile goes to buf
        const int fk = first_k(tn);
        if (fk >= 0) prefetch_k(fk, buf);
      }
    }
    STAT_MARK(8);
    if (S.trace && tid == 0) {
      S.trace[4 * (size_t)t] = globaltimer();
      S.trace[4 * (size_t)t + 3] = ((unsigned long long)blockIdx.x << 8) | (unsigned long long)type;
    }
    double* const T = sm + buf * kTileMax;

    if (type == 0) {
      // ============================================ forward tile of a big supernode
      const int4 tl = S.tiles[tk.y];
      const int g = tl.x, rb = tl.y, cb = tl.z;
      const TileGeo G = geo(S, g, rb, cb);
      const i64 col0 = P.sn_col0[g];
      const bool ok = wait_one(&S.asm_cnt[g], cur, S.ctl, &s_flag);
      STAT_MARK(0);
      if (ok) {
        const double* tg = S.tg + S.sn_tg[g] + cb * G.CB;
        for (int k = tid; k < G.cols; k += kSweepThreads) vec[k] = __ldcg(tg + k);
        __syncthreads();
      }
      next_tile_and_wait(ka, kb);
      if (ok) {
        double* fp = S.fpart + S.sn_fpart[g] + (i64)cb * G.nr + (i64)rb * G.RB;
        tile_matvec(T, G.rows, G.cols, vec, red, [&](int i, double y) { fp[i] = y; });
        __syncthreads();
        const int rend = min(G.nr, (rb + 1) * G.RB);
        const int ntl = min(G.ncb, (rend + G.CB - 1) / G.CB);
        if (tid == 0) {
          __threadfence();
          const unsigned long long old = atomicAdd(&S.rb_cnt[S.sn_rbc[g] + rb], 1ull);
          s_flag = (old + 1 == cur * (unsigned long long)ntl);
          __threadfence();
        }
        __syncthreads();
        if (s_flag) {
          // last tile of the row block: combine partial sums in column-block order
          const double* fb = S.fpart + S.sn_fpart[g] + (i64)rb * G.RB;
          const double* tg = S.tg + S.sn_tg[g] + (i64)rb * G.RB;
          for (int i = tid; i < G.rows; i += kSweepThreads) {
            double s = 0.0;
            for (int q = 0; q < ntl; ++q) s += __ldcg(fb + (i64)q * G.nr + i);
            const int r = rb * G.RB + i;
            if (r < G.nc) S.xf[col0 + r] = __ldg(S.dinv + col0 + r) * s;
            else S.upd[P.sn_uptr[g] + (r - G.nc)] = __ldcg(tg + i) - s;
          }
          __syncthreads();
          if (tid == 0) signal_add(&S.fwd_cnt[g]);
        }
      }
      buf ^= 1;
      STAT_MARK(1);
    } else if (type == 1) {
      // ============================================ backward tile of a big supernode
      const int4 tl = S.tiles[tk.y];
      const int g = tl.x, rb = tl.y, cb = tl.z;
      const TileGeo G = geo(S, g, rb, cb);
      const i64 col0 = P.sn_col0[g];
      const int p = S.parent[g];
      const bool ok = p >= 0 ? wait_one(&S.bwd_cnt[p], cur * (unsigned long long)S.sn_ncb[p], S.ctl, &s_flag)
                             : wait_one(&S.fwd_cnt[g], cur * (unsigned long long)G.nrb, S.ctl, &s_flag);
      STAT_MARK(2);
      if (ok) {
        const i64* rows = P.offrows + P.sn_rowptr[g];
        for (int i = tid; i < G.rows; i += kSweepThreads) {
          const int r = rb * G.RB + i;
          vec[i] = r < G.nc ? __ldcg(S.xf + col0 + r) : -__ldcg(S.xb + rows[r - G.nc]);
        }
        __syncthreads();
      }
      next_tile_and_wait(ka, kb);
      if (ok) {
        double* bp = S.bpart + S.sn_bpart[g] + (i64)rb * G.nc + (i64)cb * G.CB;
        tile_matvec_t(T, G.rows, G.cols, vec, [&](int j, double y) { bp[j] = y; });
        __syncthreads();
        const int rb0 = (cb * G.CB) / G.RB;
        if (tid == 0) {
          __threadfence();
          const unsigned long long old = atomicAdd(&S.cb_cnt[S.sn_cbc[g] + cb], 1ull);
          s_flag = (old + 1 == cur * (unsigned long long)(G.nrb - rb0));
          __threadfence();
        }
        __syncthreads();
        if (s_flag) {
          // last tile of the column block: combine partial sums in row-block order
          const double* bb = S.bpart + S.sn_bpart[g] + (i64)cb * G.CB;
          for (int j = tid; j < G.cols; j += kSweepThreads) {
            double s = 0.0;
            for (int q = rb0; q < G.nrb; ++q) s += __ldcg(bb + (i64)q * G.nc + j);
            S.xb[col0 + cb * G.CB + j] = s;
          }
          __syncthreads();
          if (tid == 0) {
            signal_add(&S.bwd_cnt[g]);
            atomicAdd(&S.ctl[SW_BWD_DONE], 1ull);
          }
        }
      }
      buf ^= 1;
      STAT_MARK(3);
    } else if (type == 4) {
      // ============================================ forward of a cluster of small
      // supernodes (a subtree, or one supernode whose children were waited for),
      // postorder, one CTA: no inter-CTA synchronisation inside the cluster
      bool ok = true;
      if (tk.z) ok = wait_children(S, tk.y, cur, &s_flag);
      else if (tid == 0 && *(volatile unsigned long long*)&S.ctl[SW_ABORT]) ok = false;
      STAT_MARK(0);
      for (int k = ka; k < kb; ++k) {
        const int4 tl = S.tiles[S.tdesc[k].x];
        const int g = tl.x, cb = tl.z;
        const TileGeo G = geo(S, g, 0, cb);
        const i64 col0 = P.sn_col0[g];
        if (cb == 0 && ok) {
          // t = [b_c ; 0] + extend-add of the children's update vectors; acc = 0
          for (int q = tid; q < G.nr; q += kSweepThreads) {
            vec[q] = q < G.nc ? (S.gmap ? __ldg(S.b + __ldg(S.gmap + col0 + q)) : __ldg(S.b + col0 + q)) : 0.0;
            vec2[q] = 0.0;
          }
          __syncthreads();
          for (i64 ci = P.child_ptr[g]; ci < P.child_ptr[g + 1]; ++ci) {
            const int c = P.child_list[ci];
            const int noc = P.sn_noff[c];
            const double* u = S.upd + P.sn_uptr[c];
            const int* rm = P.relmap + P.sn_rowptr[c];
            for (int a = tid; a < noc; a += kSweepThreads) vec[rm[a]] += __ldcg(u + a);
            __syncthreads();
          }
        }
        next_tile_and_wait(k, kb);
        if (ok) {
          const double* v = vec + cb * G.CB;
          tile_matvec(sm + buf * kTileMax, G.rows, G.cols, v, red,
                      [&](int i, double y) { vec2[i] += y; });
          __syncthreads();
          if (cb == G.ncb - 1) {
            double* const xf = S.xf + col0;
            double* const upd = S.upd + P.sn_uptr[g];
            for (int i = tid; i < G.nr; i += kSweepThreads) {
              if (i < G.nc) xf[i] = __ldg(S.dinv + col0 + i) * vec2[i];
              else upd[i - G.nc] = vec[i] - vec2[i];
            }
            __syncthreads();
            // only the cluster root is waited for from outside the cluster
            if (tid == 0 && g == tk.y) signal_add(&S.fwd_cnt[g]);
          }
        }
        buf ^= 1;
      }
      STAT_MARK(1);
    } else if (type == 5) {
      // ============================================ backward of a cluster (reverse
      // postorder: every ancestor inside the cluster is done before its children)
      const int g0 = tk.y;
      const int p0 = S.parent[g0];
      const bool ok = p0 >= 0 ? wait_one(&S.bwd_cnt[p0], cur * (unsigned long long)S.sn_ncb[p0], S.ctl, &s_flag)
                              : wait_one(&S.fwd_cnt[g0], cur * (unsigned long long)S.sn_nrb[g0], S.ctl, &s_flag);
      STAT_MARK(2);
      for (int k = ka; k < kb; ++k) {
        const int4 tl = S.tiles[S.tdesc[k].x];
        const int g = tl.x, cb = tl.z;
        const TileGeo G = geo(S, g, 0, cb);
        const i64 col0 = P.sn_col0[g];
        if (cb == 0 && ok) {
          const i64* rows = P.offrows + P.sn_rowptr[g];
          for (int i = tid; i < G.nr; i += kSweepThreads)
            vec[i] = i < G.nc ? __ldcg(S.xf + col0 + i) : -__ldcg(S.xb + rows[i - G.nc]);
          __syncthreads();
        }
        next_tile_and_wait(k, kb);
        if (ok) {
          double* const xb = S.xb + col0 + cb * G.CB;
          tile_matvec_t(sm + buf * kTileMax, G.rows, G.cols, vec, [&](int j, double y) { xb[j] = y; });
          __syncthreads();
          // children outside the cluster exist only for a single-supernode cluster
          if (cb == G.ncb - 1 && tid == 0 && tk.z) {
            __threadfence();
            atomicAdd(&S.bwd_cnt[g], (unsigned long long)G.ncb);
          }
        }
        buf ^= 1;
      }
      if (tid == 0 && ok) {
        __threadfence();
        atomicAdd(&S.ctl[SW_BWD_DONE], (unsigned long long)tk.w);  // column blocks of the cluster
      }
      STAT_MARK(3);
    } else if (type == 3) {
      // ============================================ assemble t of a big supernode
      const int g = tk.y;
      const bool ok = wait_children(S, g, cur, &s_flag);
      STAT_MARK(6);
      if (ok) {
        const int nc = P.sn_ncol[g], nr = nc + P.sn_noff[g];
        const i64 col0 = P.sn_col0[g];
        double* tg = S.tg + S.sn_tg[g];
        for (int k = tid; k < nr; k += kSweepThreads)
          tg[k] = k < nc ? (S.gmap ? __ldg(S.b + __ldg(S.gmap + col0 + k)) : __ldg(S.b + col0 + k)) : 0.0;
        __syncthreads();
        for (i64 ci = P.child_ptr[g]; ci < P.child_ptr[g + 1]; ++ci) {
          const int c = P.child_list[ci];
          const int noc = P.sn_noff[c];
          const double* u = S.upd + P.sn_uptr[c];
          const int* rm = P.relmap + P.sn_rowptr[c];
          for (int a = tid; a < noc; a += kSweepThreads) {
            const int pos = rm[a];
            tg[pos] = __ldcg(tg + pos) + __ldcg(u + a);
          }
          __syncthreads();
        }
        if (tid == 0) signal_add(&S.asm_cnt[g]);
      }
      STAT_MARK(7);
    } else {
      // ============================================ prolongation chunk
      const bool ok = wait_one(&S.ctl[SW_BWD_DONE], cur * (unsigned long long)S.total_bwd, S.ctl, &s_flag);
      STAT_MARK(4);
      if (ok) {
        for (int e = tk.z + tid; e < tk.w; e += kSweepThreads) {
          double s = 0.0;
          for (i64 k = S.pro_ptr[e]; k < S.pro_ptr[e + 1]; ++k) s += __ldcg(S.xb + S.pro_pos[k]);
          S.out[e] = s;
        }
      }
      STAT_MARK(5);
    }
    if (S.stats && tid == 0) st_acc[9] += 1;
    if (S.trace && tid == 0) S.trace[4 * (size_t)t + 2] = globaltimer();
    __syncthreads();
    ++it;
  }
#undef STAT_MARK
  if (S.stats && tid == 0)
    for (int q = 0; q < 10; ++q) atomicAdd(&S.stats[q], (unsigned long long)st_acc[q]);
  // exit protocol: the last CTA resets the ticket and advances the epoch
  if (tid == 0) {
    __threadfence();
    const unsigned long long prev = atomicAdd(&S.ctl[SW_EXIT], 1ull);
    if (prev == (unsigned long long)gridDim.x - 1) {
      S.ctl[SW_TSUM] += globaltimer() - S.ctl[SW_T0];
      S.ctl[SW_TCNT] += 1;
      S.ctl[SW_T0] = ~0ull;
      S.ctl[SW_TICKET] = 0;
      S.ctl[SW_EXIT] = 0;
      S.ctl[SW_EPOCH] = cur;
      __threadfence();
    }
  }
}

// relayout of the column-major panels into contiguous tiles (setup)
__global__ void k_tile_relayout(SweepDev S, int ntiles, const double* __restrict__ L,
                                const int64_t* __restrict__ lptr) {
  const int k = blockIdx.x;
  if (k >= ntiles) return;
  const int4 tl = S.tiles[k];
  const int g = tl.x, rb = tl.y, cb = tl.z;
  const TileGeo G = geo(S, g, rb, cb);
  const double* src = L + lptr[g] + (i64)(cb * G.CB) * G.nr + rb * G.RB;
  double* dst = const_cast<double*>(S.Lt) + S.tile_off[k];
  for (int q = threadIdx.x; q < G.rows * G.cols; q += blockDim.x) {
    const int j = q / G.rows, i = q % G.rows;
    dst[q] = src[(i64)j * G.nr + i];
  }
  if (threadIdx.x == 0 && ((G.rows * G.cols) & 1)) dst[G.rows * G.cols] = 0.0;
}

}  // namespace dev
}  // namespace mdd
