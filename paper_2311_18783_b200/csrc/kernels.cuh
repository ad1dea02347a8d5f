// Device kernels of the maxwell_dd library (sm_100a, FP64).
//
// Everything on the solve path is memory-bound sparse work, so no tensor cores:
// coalesced FP64 loads of the supernodal panels, shared-memory staging of the
// per-supernode vectors, warp-shuffle reductions, deterministic two-stage
// reductions for every dot product (bit-reproducible iteration counts).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mdd {
namespace dev {

typedef long long i64;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ----------------------------------------------------------- assembly
// Whitney element matrices of the Kuhn tets.  PAPER.md eq. (2.2):
//   K^e_mn = mu^{-1} |T| (2 gl_a x gl_b).(2 gl_c x gl_d)
//   M^e_mn = eps |T|/20 [(1+d_ac) gl_b.gl_d - (1+d_ad) gl_b.gl_c
//                        - (1+d_bc) gl_a.gl_d + (1+d_bd) gl_a.gl_c]
// for local edges m = (a,b), n = (c,d); gl = barycentric gradients.
__global__ void k_element_matrices(int64_t ntet, const int64_t* __restrict__ tet_id,
                                   const int64_t* __restrict__ tet_nodes, int nx, int ny,
                                   double h, const double* __restrict__ mu_inv,
                                   const double* __restrict__ eps, double* __restrict__ Ke,
                                   double* __restrict__ Me);

// A-slot sums in fixed contribution order (deterministic assembly):
//   K[s] = sum_c Ke[contrib[c]], M[s] likewise; A = K + gamma M
__global__ void k_assemble_slots(int64_t nslot, const int64_t* __restrict__ ptr,
                                 const int32_t* __restrict__ contrib,
                                 const double* __restrict__ Ke, const double* __restrict__ Me,
                                 double gamma, double* __restrict__ A, double* __restrict__ K,
                                 double* __restrict__ M);

__global__ void k_gather(int64_t n, const int64_t* __restrict__ idx, const double* __restrict__ src,
                         double* __restrict__ dst);
// dst[di[k]] = src[si[k]]
__global__ void k_scatter_gather(int64_t n, const int64_t* __restrict__ di, const int64_t* __restrict__ si,
                                 const double* __restrict__ src, double* __restrict__ dst);
// dense helpers for the GEVP pipeline (column-major)
__global__ void k_dense_scatter(int64_t n, const int64_t* __restrict__ pos, const double* __restrict__ v,
                                double* __restrict__ D);
__global__ void k_set_identity_minus(int64_t n, double* __restrict__ P);
__global__ void k_scale_rows(int64_t n, int64_t cols, const double* __restrict__ d, double* __restrict__ P);
__global__ void k_symmetrize(int64_t n, double* __restrict__ L);
__global__ void k_slot_sums(int64_t nslot, const int64_t* __restrict__ ptr, const int32_t* __restrict__ contrib,
                            const double* __restrict__ Ke, const double* __restrict__ Me, double gamma,
                            double* __restrict__ out);

__global__ void k_inv_sqrt_diag(int n, const int* __restrict__ ptr, const int* __restrict__ idx,
                                const double* __restrict__ val, double* __restrict__ s);
__global__ void k_scale_csr(int n, const int* __restrict__ ptr, const int* __restrict__ idx,
                            double* __restrict__ val, const double* __restrict__ rs,
                            const double* __restrict__ cs);

// --------------------------------------------------- multifrontal LDL^T
struct PlanDev {
  const i64* sn_col0;
  const int* sn_ncol;
  const int* sn_noff;
  const i64* sn_rowptr;
  const i64* offrows;
  const i64* sn_lptr;
  const i64* sn_uptr;
  const i64* sn_fptr;
  const i64* sn_umptr;
  const i64* child_ptr;
  const int* child_list;
  const int* relmap;
  const i64* asm_ptr;
  const i64* asm_src;
  const int* asm_pos;
  const int* level_sn;
};

// mode 0: SPD (pivot <= 0 flags an error); mode 1: rank-revealing (pivot <= tol is
// a dependent column: D^{-1} = 0, L column = 0, flagged in `dropped`); mode 2:
// static pivoting (pivot <= tol replaced by tol, counted in *err)
__global__ void k_mf_factor_level(PlanDev P, const int* __restrict__ list, const double* __restrict__ src,
                                  double* __restrict__ fronts, double* __restrict__ L,
                                  double* __restrict__ dinv, double* __restrict__ umat, int mode,
                                  double tol, uint8_t* __restrict__ dropped, int* __restrict__ err);

// -------------------------------------------- supernodal triangular sweeps
// (sweep.cu) control words of a persistent sweep and its phase kinds
enum { SW_EPOCH = 0 /* grid barriers completed by earlier launches */, SW_BAR, SW_ABORT, SW_T0, SW_TSUM, SW_TCNT, SW_COUNT };
enum { PH_GF = 0, PH_MF, PH_GB, PH_MB, PH_PR, PH_CF, PH_CB };
// SweepDev::flags (experiments, env MDD_SWEEP_FLAGS read per launch; 0 = default;
// measured on c4: one CTA per combine item, coarse sweep 3.78 -> 3.65 ms)
enum { SWF_NO_CTA_COMBINE = 2 };
constexpr int kSweepThreads = 256;
// (MDD_TILE_MAX / MDD_SWEEP_CTAS: experiment builds through MDD_NVCC_FLAGS; measured on
// c4's local sweep: 2304-double tiles with 4 CTAs per SM and 64 registers)
#ifndef MDD_TILE_MAX
#define MDD_TILE_MAX 3328
#endif
#ifndef MDD_SWEEP_CTAS
#define MDD_SWEEP_CTAS 3
#endif
constexpr int kTileMax = MDD_TILE_MAX;   // doubles per tile (26 KB, one TMA bulk copy)
constexpr int kSweepCtasPerSm = MDD_SWEEP_CTAS;  // resident persistent CTAs per SM (registers: launch bounds)
constexpr int kVecMax = 512;     // rows of a small supernode / of a tile
constexpr int64_t kSingleMax = 8192;    // stored entries of a supernode one CTA sweeps alone (measured: 32768 -> 8192 is -3 % per local sweep)
#ifndef MDD_STAGES
#define MDD_STAGES 2
#endif
constexpr int kStages = MDD_STAGES;       // tile ring slots per CTA (one tile streams while one computes)
constexpr int kVecSlots = kStages + 1;    // task-vector slots (> the tasks the ring can span)
constexpr int kDescAhead = 4;    // M-task descriptors streamed ahead of the current task
constexpr int kDescRing = 8;     // descriptor ring slots (> kDescAhead)
// MDD_SWEEP_TRACE words per (phase, CTA), thread 0's view (%globaltimer ns): start,
// end, time waiting on tile mbarriers, tiles consumed, 0, time from a task's top to its first tile wait (descriptor ring + fused
// gather), time from a tile's arrival to its slot refill (compute + barrier), tasks
constexpr int kTraceWords = 8;
constexpr int kSweepSmemDoubles = kStages * kTileMax + kVecSlots * (kVecMax + 2) + kVecMax + kSweepThreads;

// one task of an M phase (factor_driver.cu builds them, forward and backward)
struct __align__(16) MTaskDesc {
  long long col0;   // position of the supernode's first column
  long long vo;     // vb offset of the supernode's rows
  long long vlo2;   // even-aligned start of the task vector's bulk copy (vb index)
  long long uptr;   // offset of the supernode's update vector
  long long part;   // big: offset of this tile's partial sums (fpart / bpart)
  long long comb;   // big: first partial of its row block / column block
  long long cnt;    // unused
  int big, k0, k1;  // 0 small / 1 big 2-D tile / 2 strip (rb, cb = first row / column); tdesc range
  int nr, nc, rows, cols, rb, cb, RB, CB;
  int ntl;          // big: partial sums of its row block / column block
  int voff;         // offset of the vector inside its shared-memory buffer
  int vbytes;       // bytes of the vector bulk copy
  int vn;           // rows of the task vector (vb rows [vlo2 + voff, + vn))
  int pad_[3];
  // the task's first kTdInline tile descriptors (tdesc[k0 ..]): the producer thread
  // issues their bulk copies from shared memory, with no dependent global load on
  // the CTA's critical path (every task has <= 4 tiles at the default knobs)
  int4 td[4];
};
constexpr int kTdInline = 4;
static_assert(sizeof(MTaskDesc) == 192, "MTaskDesc layout");

// one row block (forward) / column block (backward) of a 2-D supernode whose
// partial sums a combine phase (PH_CF / PH_CB) adds, in a fixed order, after the
// level's tile phase: rows first .. first+m-1 of the panel (forward) / columns
// (backward); partial q of output o at comb + q * ld + o
struct __align__(16) CombDesc {
  long long comb, col0, uptr, vo;
  int ld, ntl, m, first, nc, pad_[3];
};
static_assert(sizeof(CombDesc) == 64, "CombDesc layout");

struct SweepDev {
  PlanDev P;
  const double* dinv;
  const MTaskDesc* mtf;          // M tasks, forward / backward descriptors
  const MTaskDesc* mtb;
  // phases {kind, a, b, w}: G: rows [a, b) of vb; M: mtask [a, b), w = 1 when the
  // level's gather is fused into its tasks (no G phase before it); C: combine
  // items [a, b), w bit 0 when the level's t rows are not in vb (fused), bit 1
  // one CTA per item (few items, long partial chains); PR
  const int4* phases;
  const CombDesc* cmb;
  int nphases;
  int ph0, ph1;                  // this launch runs phases [ph0, ph1) (a segment of a sharded coarse sweep)
  int flags;                     // SWF_* (experiments)
  const int4* tdesc;             // {tile, bytes, offset lo, offset hi}
  const int4* tiles;             // {supernode, row block, column block, 0}
  const int64_t* tile_off;       // into Lt
  const double* Lt;              // tiled P-form panels
  const int* sn_RB;              // tile rows / columns / counts per supernode
  const int* sn_CB;
  const int* sn_nrb;
  const int* sn_ncb;
  const int64_t* sn_fpart;       // big supernodes: partial-sum offsets
  const int64_t* sn_bpart;
  double* fpart;
  double* bpart;
  // per-supernode row vectors (t forward, w backward): rows of g at vb_off[g]
  double* vb;
  const int64_t* vb_off;
  const int32_t* gsrc;           // row -> index into b (column rows) or -1
  const int64_t* cptr;           // row -> children update entries (into upd)
  const int64_t* cidx;
  const int64_t* wsrc;           // row -> xf index (>= 0) or -(xb index) - 1
  unsigned long long* ctl;       // SW_* words
  double* upd;                   // update vectors (noff per supernode)
  double* xf;                    // forward result z (positions)
  double* xb;                    // solution (positions)
  const double* b;               // right-hand side (global index space of gsrc)
  const int64_t* pro_ptr;        // prolongation (global dof -> positions)
  const int32_t* pro_pos;
  double* out;                   // prolongation target (global)
  int n_out;
  const int* stop;               // PCG stop flag (nullable): set -> no-op launch
  unsigned long long* trace;     // optional per-phase timeline (MDD_SWEEP_TRACE=dir)
};
__global__ void k_sweep(SweepDev S);
__global__ void k_tile_relayout(SweepDev S, int ntiles, const double* __restrict__ L,
                                const int64_t* __restrict__ lptr);


// big fronts: assembly, blocked panel factorisation (trailing updates by cuBLAS),
// finishing copies and the D^{-1} fold (the triangular inverse and M21 by cuSOLVER /
// cuBLAS, factor_driver.cu)
__global__ void k_front_assemble(PlanDev P, int g, const double* __restrict__ src, double* __restrict__ fronts,
                                 const double* __restrict__ umat);
__global__ void k_front_assemble2(PlanDev P, int g, const double* __restrict__ src, double* __restrict__ fronts,
                                  const double* __restrict__ umat);
__global__ void k_panel_factor(PlanDev P, int g, int j0, int nb, double* __restrict__ fronts,
                               double* __restrict__ dinv, double* __restrict__ W, int mode, double tol,
                               uint8_t* __restrict__ dropped, int* __restrict__ err);
__global__ void k_front_finish_copy(PlanDev P, int g, const double* __restrict__ fronts, double* __restrict__ L,
                                    double* __restrict__ umat);
__global__ void k_front_fold_d(PlanDev P, int g, double* __restrict__ L, const double* __restrict__ dinv);


// ---------------------------------------------------------- PCG pieces
// optional tail of a kernel that leaves one partial sum per block: the last block
// to finish adds the partials in the order of k_reduce_step (same bits), stores
// S[slot], runs the CG scalar step `op` and re-arms the counter (counter == null:
// no tail)
struct RedStep {
  double* S;
  int* state;
  unsigned int* counter;
  int slot, op;
};
// y = M x (or y = sub - M x), 8 / 16 / 32 lanes per row on an SM-sized grid,
// optional fused dot partials of dotw . y
#define MDD_SPMV_G_DECL(NAME)                                                                    \
  __global__ void NAME(int nrows, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx, \
                       const double* __restrict__ val, const double* __restrict__ x,                \
                       const double* __restrict__ sub, double* __restrict__ y,                      \
                       const double* __restrict__ dotw, double* __restrict__ part,                  \
                       const int* __restrict__ stop, RedStep rs);
MDD_SPMV_G_DECL(k_spmv4)
MDD_SPMV_G_DECL(k_spmv8)
MDD_SPMV_G_DECL(k_spmv16)
MDD_SPMV_G_DECL(k_spmv32)
#undef MDD_SPMV_G_DECL
constexpr int kGeneoRows = 1024;  // rows per block of the Z_e^T v reduction (2048: slower)
constexpr int kGeneoZRows = 512;  // rows per block of W_i y_i (2 per thread: one wave on c1)
__global__ void k_geneo_zt(const int4* __restrict__ blk, const int64_t* __restrict__ woff,
                           const int64_t* __restrict__ poff, const int* __restrict__ nsz,
                           const int* __restrict__ gcol0, const int32_t* __restrict__ gpos,
                           const double* __restrict__ W, const int32_t* __restrict__ gmap,
                           const double* __restrict__ v, double* __restrict__ part, const int* __restrict__ stop);
__global__ void k_geneo_zt2(int ncols, const int* __restrict__ cblk, const int* __restrict__ cnch,
                            const int32_t* __restrict__ gpos, const double* __restrict__ part,
                            double* __restrict__ y, const int* __restrict__ stop);
__global__ void k_geneo_z(const int4* __restrict__ blk, const int64_t* __restrict__ woff,
                          const int64_t* __restrict__ poff, const int* __restrict__ nsz,
                          const int* __restrict__ kcnt, const int* __restrict__ gcol0,
                          const int32_t* __restrict__ gpos, const double* __restrict__ W,
                          const double* __restrict__ xc, double* __restrict__ u, const int* __restrict__ stop);
__global__ void k_z_apply(int n, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                          const double* __restrict__ val, const double* __restrict__ xc,
                          const int64_t* __restrict__ pptr, const int32_t* __restrict__ ppos,
                          const double* __restrict__ u, const double* __restrict__ addw,
                          double* __restrict__ out, const double* __restrict__ dotw,
                          double* __restrict__ part, const int* __restrict__ stop, RedStep rs);
__global__ void k_dot_part(int n, const double* __restrict__ a, const double* __restrict__ b,
                           double* __restrict__ part, const int* __restrict__ stop, RedStep rs);
__global__ void k_reduce(int nparts, const double* __restrict__ part, double* __restrict__ out,
                         const int* __restrict__ stop);
__global__ void k_scalar_step(int op, double* __restrict__ S, int* __restrict__ state);
__global__ void k_loop_cond(cudaGraphConditionalHandle h, const int* __restrict__ state);
__global__ void k_update_xr(int n, double* __restrict__ x, double* __restrict__ r,
                            const double* __restrict__ p, const double* __restrict__ q,
                            const double* __restrict__ S, double* __restrict__ part,
                            const int* __restrict__ stop, RedStep rs);
__global__ void k_update_p(int n, double* __restrict__ p, const double* __restrict__ z,
                           const double* __restrict__ S, const int* __restrict__ stop);
__global__ void k_axpby(int n, double a, const double* __restrict__ x, double b,
                        const double* __restrict__ y, double* __restrict__ out,
                        const int* __restrict__ stop);
__global__ void k_combine3(int n, const double* __restrict__ a, const double* __restrict__ b,
                           const double* __restrict__ c, double* __restrict__ out,
                           const int* __restrict__ stop);
__global__ void k_copy(int n, const double* __restrict__ a, double* __restrict__ out,
                       const int* __restrict__ stop);

// scalar slots of the PCG state
enum { S_RZ = 0, S_PQ, S_ALPHA, S_RR, S_NF, S_BETA, S_RZNEW, S_REL, S_TOL, S_TMP, S_COUNT };
// device state words of a solve
enum { ST_STOP = 0, ST_ITERS, ST_BREAKDOWN, ST_MAXIT, ST_CONVERGED, ST_COUNT };
}  // namespace dev
}  // namespace mdd
