// Persistent, dependency-driven supernodal triangular sweep (sm_100a, FP64).
//
// One launch applies A_i^{-1} for ALL subdomains at once (north_star: "local
// solves A_i^{-1} as supernodal sparse LDL^T factors applied by hand-written
// level-scheduled triangular-solve kernels, with dense supernode blocks as
// warp-tiled TRSV"), fusing the restriction R_i (gather in the leaves), the
// forward sweep L y = b, the diagonal D^{-1}, the backward sweep L^T x = z and
// the prolongation sum_i R_i^T x_i (PAPER.md eq. AS, M_AS = sum R_i^T A_i^{-1} R_i).
//
// Panels are stored in "partitioned-inverse" form P = [L11^{-1}; L21 L11^{-1}]
// (column-major nr x nc), so every row of the forward product and every column
// of the backward product of a supernode is independent:
//   forward :  z_c = D^{-1} (L11^{-1} t_c),     u = t_off - (L21 L11^{-1}) t_c
//   backward:  x_c = L11^{-T} z_c - (L21 L11^{-1})^T x_off
// which lets large (top-of-tree) supernodes be split over several CTAs.
//
// Scheduling: tasks (fwd row-blocks in level order, bwd column-blocks in reverse
// level order, prolongation chunks) are handed out by an atomic ticket; a task
// only waits for tasks with smaller tickets, which are held by running CTAs, so
// the schedule is deadlock-free for any grid size.  Completion counters are
// cumulative per launch epoch (no reset), the last CTA to exit advances the epoch.
// A wait that exceeds kSpinTimeoutNs raises an abort flag (reported by the host)
// instead of hanging the device.
#include "kernels.cuh"

namespace mdd {
namespace dev {

namespace {
constexpr unsigned long long kSpinTimeoutNs = 4000000000ull;  // 4 s
constexpr int kNarrow = 64;      // panels with nc <= kNarrow: one thread per row
constexpr int kColChunk = 16;    // backward: columns per register-blocked chunk

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

// thread 0 only: spin until *p >= target; false on abort / timeout
__device__ bool wait_ge(const unsigned long long* p, unsigned long long target,
                        unsigned long long* ctl) {
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

__device__ __forceinline__ void signal_add(unsigned long long* p) {
  __threadfence();
  atomicAdd(p, 1ull);
}
}  // namespace

__global__ void __launch_bounds__(kSweepThreads) k_sweep(SweepDev S) {
  extern __shared__ double sm[];
  __shared__ int s_task;
  __shared__ int s_ok;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  const PlanDev& P = S.P;
  if (S.stop && *S.stop) return;  // PCG already stopped: the whole sweep is a no-op
  const unsigned long long cur = S.ctl[SW_EPOCH] + 1;
  if (tid == 0) atomicMin(&S.ctl[SW_T0], globaltimer());
  // optional per-CTA cycle accounting (S.stats != NULL): [type*2] wait, [type*2+1] work,
  // [6] ticket, [7] tasks
  long long st_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long c_prev = clock64();

  for (;;) {
    if (tid == 0) s_task = (int)atomicAdd(&S.ctl[SW_TICKET], 1ull);
    __syncthreads();
    const int t = s_task;
    if (S.stats && tid == 0) { long long c = clock64(); st_acc[6] += c - c_prev; c_prev = c; }
    if (t >= S.ntasks) break;
    const int4 tk = S.tasks[t];
    const int type = tk.x, g = tk.y, lo = tk.z, hi = tk.w;
#define STAT_MARK(slot) \
  if (S.stats && tid == 0) { long long c = clock64(); st_acc[(slot)] += c - c_prev; c_prev = c; }

    if (type == 0) {
      // ------------------------------------------------ forward row block
      if (tid == 0) {
        bool ok = !S.ctl[SW_ABORT];
        for (i64 ci = P.child_ptr[g]; ok && ci < P.child_ptr[g + 1]; ++ci) {
          const int c = P.child_list[ci];
          ok = wait_ge(&S.fwd_cnt[c], cur * (unsigned long long)S.nbf[c], S.ctl);
        }
        if (ok) __threadfence();
        s_ok = ok;
      }
      __syncthreads();
      STAT_MARK(0);
      if (s_ok) {
        const int nc = P.sn_ncol[g], no = P.sn_noff[g], nr = nc + no;
        const i64 col0 = P.sn_col0[g];
        const double* __restrict__ Lp = S.L + P.sn_lptr[g];
        double* tc = sm;        // nc: right-hand side of the column block
        double* to = sm + nc;   // hi - max(lo, nc): off rows of this task
        const int olo = lo > nc ? lo : nc;
        for (int k = tid; k < nc; k += nt)
          tc[k] = S.gmap ? S.b[S.gmap[col0 + k]] : S.b[col0 + k];
        for (int k = tid; k < hi - olo; k += nt) to[k] = 0.0;
        __syncthreads();
        for (i64 ci = P.child_ptr[g]; ci < P.child_ptr[g + 1]; ++ci) {
          const int c = P.child_list[ci];
          const int noc = P.sn_noff[c];
          const double* u = S.upd + P.sn_uptr[c];
          const int* rm = P.relmap + P.sn_rowptr[c];
          for (int a = tid; a < noc; a += nt) {
            const int pos = rm[a];
            if (pos < nc) tc[pos] += __ldcg(u + a);
            else if (pos >= olo && pos < hi) to[pos - olo] += __ldcg(u + a);
          }
          __syncthreads();
        }
        if (nc <= kNarrow) {
          // narrow panel: one thread per row, all columns
          for (int i = lo + tid; i < hi; i += nt) {
            const int jn = i < nc ? i + 1 : nc;
            const double* row = Lp + i;
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int j = 0;
            for (; j + 4 <= jn; j += 4) {
              s0 += __ldg(row + (i64)j * nr) * tc[j];
              s1 += __ldg(row + (i64)(j + 1) * nr) * tc[j + 1];
              s2 += __ldg(row + (i64)(j + 2) * nr) * tc[j + 2];
              s3 += __ldg(row + (i64)(j + 3) * nr) * tc[j + 3];
            }
            for (; j < jn; ++j) s0 += __ldg(row + (i64)j * nr) * tc[j];
            const double v = (s0 + s1) + (s2 + s3);
            if (i < nc) S.xf[col0 + i] = __ldg(S.dinv + col0 + i) * v;
            else S.upd[P.sn_uptr[g] + (i - nc)] = to[i - olo] - v;
          }
        } else {
          // wide panel: 32-row groups, the 8 warps split the columns, fixed-order
          // reduction through shared memory
          double* red = sm + nc + (hi - olo);  // [nw][32]
          const int cs = (nc + nw - 1) / nw;
          const int ja = warp * cs, jb = min(nc, ja + cs);
          for (int r0 = lo; r0 < hi; r0 += 32) {
            const int i = r0 + lane;
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            if (i < hi) {
              const int je = min(jb, i < nc ? i + 1 : nc);
              const double* row = Lp + i;
              int j = ja;
              for (; j + 4 <= je; j += 4) {
                s0 += __ldg(row + (i64)j * nr) * tc[j];
                s1 += __ldg(row + (i64)(j + 1) * nr) * tc[j + 1];
                s2 += __ldg(row + (i64)(j + 2) * nr) * tc[j + 2];
                s3 += __ldg(row + (i64)(j + 3) * nr) * tc[j + 3];
              }
              for (; j < je; ++j) s0 += __ldg(row + (i64)j * nr) * tc[j];
            }
            red[warp * 32 + lane] = (s0 + s1) + (s2 + s3);
            __syncthreads();
            if (warp == 0 && i < hi) {
              double v = 0.0;
              for (int q = 0; q < nw; ++q) v += red[q * 32 + lane];
              if (i < nc) S.xf[col0 + i] = __ldg(S.dinv + col0 + i) * v;
              else S.upd[P.sn_uptr[g] + (i - nc)] = to[i - olo] - v;
            }
            __syncthreads();
          }
        }
        __syncthreads();
        if (tid == 0) signal_add(&S.fwd_cnt[g]);
      }
      STAT_MARK(1);
    } else if (type == 1) {
      // ------------------------------------------------ backward column block
      if (tid == 0) {
        bool ok = !S.ctl[SW_ABORT];
        const int p = S.parent[g];
        if (ok) ok = p >= 0 ? wait_ge(&S.bwd_cnt[p], cur * (unsigned long long)S.nbb[p], S.ctl)
                            : wait_ge(&S.fwd_cnt[g], cur * (unsigned long long)S.nbf[g], S.ctl);
        if (ok) __threadfence();
        s_ok = ok;
      }
      __syncthreads();
      STAT_MARK(2);
      if (s_ok) {
        const int nc = P.sn_ncol[g], no = P.sn_noff[g], nr = nc + no;
        const i64 col0 = P.sn_col0[g];
        const double* __restrict__ Lp = S.L + P.sn_lptr[g];
        const i64* rows = P.offrows + P.sn_rowptr[g];
        double* w = sm;  // [z_c ; -x_off]
        for (int k = lo + tid; k < nc; k += nt) w[k] = __ldcg(S.xf + col0 + k);  // rows >= lo only
        for (int k = tid; k < no; k += nt) w[nc + k] = -__ldcg(S.xb + rows[k]);
        __syncthreads();
        // column chunks of kColChunk: every thread walks rows (coalesced down each
        // column), per-column partial sums reduced warp-wise then across warps in
        // a fixed order
        double* red = sm + nr;  // [nw][kColChunk]
        for (int c0 = lo; c0 < hi; c0 += kColChunk) {
          const int nb = min(kColChunk, hi - c0);
          double acc[kColChunk];
#pragma unroll
          for (int q = 0; q < kColChunk; ++q) acc[q] = 0.0;
          for (int i = c0 + tid; i < nr; i += nt) {
            const double wi = w[i];
            const double* base = Lp + (i64)c0 * nr + i;
#pragma unroll
            for (int q = 0; q < kColChunk; ++q)
              if (q < nb) acc[q] += __ldg(base + (i64)q * nr) * wi;
          }
#pragma unroll
          for (int q = 0; q < kColChunk; ++q) {
            const double v = warp_sum(acc[q]);
            if (lane == 0) red[warp * kColChunk + q] = v;
          }
          __syncthreads();
          if (tid < nb) {
            double v = 0.0;
            for (int q = 0; q < nw; ++q) v += red[q * kColChunk + tid];
            S.xb[col0 + c0 + tid] = v;
          }
          __syncthreads();
        }
        __syncthreads();
        if (tid == 0) {
          signal_add(&S.bwd_cnt[g]);
          atomicAdd(&S.ctl[SW_BWD_DONE], 1ull);
        }
      }
      STAT_MARK(3);
    } else {
      // ------------------------------------------------ prolongation chunk
      if (tid == 0) {
        bool ok = !S.ctl[SW_ABORT];
        if (ok) ok = wait_ge(&S.ctl[SW_BWD_DONE], cur * (unsigned long long)S.total_bwd, S.ctl);
        if (ok) __threadfence();
        s_ok = ok;
      }
      __syncthreads();
      STAT_MARK(4);
      if (s_ok) {
        for (int e = lo + tid; e < hi; e += nt) {
          double s = 0.0;
          for (i64 k = S.pro_ptr[e]; k < S.pro_ptr[e + 1]; ++k) s += __ldcg(S.xb + S.pro_pos[k]);
          S.out[e] = s;
        }
      }
      __syncthreads();
      STAT_MARK(5);
    }
    if (S.stats && tid == 0) st_acc[7] += 1;
    __syncthreads();
  }
#undef STAT_MARK
  if (S.stats && tid == 0)
    for (int q = 0; q < 8; ++q) atomicAdd(&S.stats[q], (unsigned long long)st_acc[q]);
  // exit protocol: the last CTA resets the ticket and advances the epoch
  if (tid == 0) {
    __threadfence();
    const unsigned long long prev = atomicAdd(&S.ctl[SW_EXIT], 1ull);
    if (prev == (unsigned long long)gridDim.x - 1) {
      // device-side duration of this launch (first CTA start -> last CTA exit)
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

}  // namespace dev
}  // namespace mdd
