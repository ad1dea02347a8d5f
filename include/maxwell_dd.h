/* maxwell_dd.h -- C ABI of the B200-native two-level Schwarz / GenEO PCG solver
 * for the lowest-order Nédélec discretisation of the positive Maxwell problem
 *
 *     curl(mu^{-1} curl E) + gamma eps E = f  in Omega,   E x n = 0 on the Dirichlet part
 *
 * (eq. 1.1; discrete system A U := (K + gamma M) U = f, eq. 1.5).
 *
 * The library owns its device memory; every pointer argument is either a HOST
 * pointer or a DEVICE pointer as stated per argument.  All functions return 0 on
 * success and a nonzero MDD_ERR_* code on failure; the message is then available
 * from mdd_last_error() (thread-local, valid until the next call).  No function
 * ever falls back to a CPU computation: a missing device or a CUDA error is an
 * error.  Indices are 0-based.
 *
 * Numbering contract (shared with any checker):
 *   node id     = i + (nx+1)*(j + (ny+1)*k),       0 <= i <= nx, ...
 *   cube id     = ci + nx*(cj + ny*ck);  tet id = 6*cube + s, s indexing the Kuhn
 *                 paths v -> v+e_a -> v+e_a+e_b -> v+(1,1,1) for
 *                 (a,b) in (x,y) (x,z) (y,x) (y,z) (z,x) (z,y)
 *   edges       = pairs (tail, head) of node ids, tail < head, numbered in
 *                 lexicographic (tail, head) order; orientation tail -> head
 *   free dofs   = non-Dirichlet edges, same order; free nodes likewise
 *   Dirichlet   = edges / nodes of boundary triangles on the box faces
 *                 (MDD_DIRICHLET_OUTER), on every boundary incl. hole walls
 *                 (MDD_DIRICHLET_ALL) or none (MDD_DIRICHLET_NONE)
 *   subdomain s = si + px*(sj + py*sk); it owns the cube box
 *                 [si*nx/px, (si+1)*nx/px) x ... and Omega_s adds `overlap`
 *                 cube layers around it (§4 "One layer of elements is
 *                 added in each direction"); N_s = free edges of its tets, increasing.
 */
#ifndef MAXWELL_DD_H
#define MAXWELL_DD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MDD_OK 0
#define MDD_ERR_CUDA 1      /* CUDA / cuSOLVER / cuBLAS failure or no device       */
#define MDD_ERR_ARG 2       /* invalid argument (sizes, modes, divisibility)        */
#define MDD_ERR_NOTPD 3     /* a matrix that must be SPD had a nonpositive pivot    */
#define MDD_ERR_NOCONV 4    /* PCG hit maxit (the result is still returned)          */
#define MDD_ERR_INTERNAL 5  /* broken internal invariant                             */
#define MDD_ERR_BREAKDOWN 6 /* PCG breakdown (p^T A p <= 0)                          */

#define MDD_DIRICHLET_OUTER 0
#define MDD_DIRICHLET_ALL 1
#define MDD_DIRICHLET_NONE 2

#define MDD_COARSE_NONE 0   /* one-level AS, eq. (2.3)                              */
#define MDD_COARSE_SNK 1    /* split near-kernel, Def. 2.3 (+ GenEO, GEVP 3.5)      */
#define MDD_COARSE_NK 2     /* global near-kernel G = C (§4 "AS-NK") (+ GenEO)      */

#define MDD_VARIANT_AS2 0       /* M_AS,2 = Q + (I - QA) M_AS (I - AQ), eq. (2.4)   */
#define MDD_VARIANT_ADDITIVE 1  /* M_AS + Q (north_star's written sum, D_i dropped) */
#define MDD_VARIANT_AS1 2       /* M_AS only                                        */
/* M_AS,2 again, PCG started from the coarse Galerkin solution x0 = Q f (DESIGN.md
 * reading R13).  Then Z^T r_k = 0 for all k and eq. (2.4) equals
 * M_AS r + Q (r - A M_AS r): the PCG loop applies that form (one coarse solve
 * and one A product per iteration instead of two each).  Same PCG iterates as
 * MDD_VARIANT_AS2 from x0 = Q f in exact arithmetic; mdd_apply_preconditioner
 * still applies the full eq. (2.4) operator. */
#define MDD_VARIANT_AS2_COARSE_START 3

typedef struct mdd_solver* mdd_handle;

typedef struct {
  int nx, ny, nz;              /* cube grid                                           */
  double h;                    /* cube edge length                                    */
  const uint8_t* cube_mask;    /* HOST, nx*ny*nz (1 = cube present) or NULL = all     */
  int dirichlet;               /* MDD_DIRICHLET_*                                     */
  const double* mu_inv;        /* HOST, 6*nx*ny*nz per tet (indexed by tet id), > 0   */
  const double* eps;           /* HOST, 6*nx*ny*nz per tet, > 0                       */
  double gamma;                /* > 0                                                 */
  int px, py, pz;              /* subdomain boxes per axis; must divide nx, ny, nz    */
  int overlap;                 /* cube layers added around each box, >= 0            */
  double coarse_threshold;     /* GenEO keeps eigenpairs of GEVP 3.5 with
                                  lambda > tau = 1/coarse_threshold; <= 0: no GenEO   */
  int coarse_kind;             /* MDD_COARSE_*                                        */
  int variant;                 /* MDD_VARIANT_*                                       */
  int device;                  /* CUDA device ordinal                                 */
  int reserved[8];             /* must be zero                                        */
} mdd_setup_desc;

/* Build everything the solve phase needs (§2-§3): mesh + numbering,
 * assembly of K, M, A (device), overlapping decomposition, R_i, D_i, local
 * supernodal LDL^T factors of A_i = R_i A R_i^T (device), the coarse space Z
 * (SNK Def. 2.3 or NK, plus GenEO columns of GEVP 3.5 solved on the device) and
 * the LDL^T factor of E = Z^T A Z.  Inputs are host pointers, copied; the caller
 * keeps ownership.  *out receives a handle owned by the caller (mdd_destroy). */
int mdd_setup(const mdd_setup_desc* desc, mdd_handle* out);

void mdd_destroy(mdd_handle h);

/* Preconditioned CG on A x = f with the configured preconditioner (x0 = 0, or
 * x0 = Q f for MDD_VARIANT_AS2_COARSE_START),
 * stopping at ||r_k||_2 <= tol ||f||_2 or maxit.  f, x: DEVICE pointers to n
 * doubles (n = free dofs, MDD_INFO_N).  *iters, *relres: HOST outputs.  Runs on
 * the handle's stream and synchronises it before returning. */
int mdd_solve(mdd_handle h, const double* f, double* x, double tol, int maxit, int* iters,
              double* relres);

/* Same, with HOST f and x; the host<->device copies are part of the call. */
int mdd_solve_host(mdd_handle h, const double* f, double* x, double tol, int maxit,
                   int* iters, double* relres);

/* Run all later device work of the handle on `stream` (a cudaStream_t of the
 * handle's device, owned by the caller, which must outlive the handle or be
 * replaced); NULL restores a private non-blocking stream.  Synchronises the
 * previous stream first. */
int mdd_set_stream(mdd_handle h, void* stream);
/* Switch the preconditioner variant (MDD_VARIANT_*) of an existing handle; the
 * setup data is shared by all variants.  Variants other than MDD_VARIANT_AS1
 * need a coarse space (MDD_ERR_ARG otherwise / for an unknown value). */
int mdd_set_variant(mdd_handle h, int variant);

/* z = M^{-1} r for the configured variant (eq. 2.3 / 2.4).  DEVICE pointers. */
int mdd_apply_preconditioner(mdd_handle h, const double* r, double* z);
/* y = A x (CSR SpMV).  DEVICE pointers. */
int mdd_apply_operator(mdd_handle h, const double* x, double* y);
/* z = sum_i R_i^T A_i^{-1} R_i r (eq. 2.3).  DEVICE pointers. */
int mdd_apply_local(mdd_handle h, const double* r, double* z);
/* y = Z E^{-1} Z^T v (coarse correction Q).  DEVICE pointers. */
int mdd_apply_coarse(mdd_handle h, const double* v, double* y);

/* Parity diagnostics (test infrastructure of the backward-error checks; not
 * on the solve path).
 * mdd_apply_local_parts: the local solutions x_i = A_i^{-1} R_i r of eq. (2.3)
 * BEFORE the prolongation sum.  r: DEVICE, n doubles; xloc: DEVICE, MDD_INFO_NLOC
 * doubles, subdomain-major, each block in N_i order (MDD_ARR_SUB_DOFS).
 * mdd_apply_coarse_inverse: y = E^{-1} v for the factorised coarse matrix E
 * (MDD_ARR_E_* / MDD_DARR_E_VAL, coarse-position order).  v, y: DEVICE,
 * MDD_INFO_N0 doubles.  MDD_ERR_ARG without a coarse space. */
int mdd_apply_local_parts(mdd_handle h, const double* r, double* xloc);
int mdd_apply_coarse_inverse(mdd_handle h, const double* v, double* y);

/* Integer / scalar facts about the handle (HOST array out[0..MDD_INFO_COUNT)). */
enum {
  MDD_INFO_N = 0,           /* free edge dofs n                        */
  MDD_INFO_NEDGES,          /* all edges                               */
  MDD_INFO_NFREE_NODES,     /* free nodes (columns of C)               */
  MDD_INFO_NSUB,            /* subdomains                              */
  MDD_INFO_NNZ_A,           /* nonzeros of A                           */
  MDD_INFO_NLOC,            /* sum_i n_i                               */
  MDD_INFO_GRAD_CANDIDATES, /* gradient candidate columns (SNK family) */
  MDD_INFO_GRAD_RANK,       /* dim V_G kept                            */
  MDD_INFO_NGENEO,          /* GenEO columns                           */
  MDD_INFO_N0,              /* coarse dimension                        */
  MDD_INFO_LOCAL_FACTOR_NNZ,/* stored entries of the local factors     */
  MDD_INFO_COARSE_FACTOR_NNZ,
  MDD_INFO_LOCAL_SUPERNODES,
  MDD_INFO_LOCAL_LEVELS,
  MDD_INFO_COARSE_SUPERNODES,
  MDD_INFO_COARSE_LEVELS,
  MDD_INFO_NNZ_Z,
  MDD_INFO_KERNELS_PER_ITER, /* kernel launches per PCG iteration       */
  MDD_INFO_LAST_LAUNCHES,   /* kernels launched by the last solve/apply call */
  MDD_INFO_COARSE_PERTURBED,/* pivots of the Jacobi-scaled E at or below 1e-14: numerically
                               dependent coarse directions, dropped (D^{-1} = 0); 0 =
                               exact LDL^T (reading R11)                    */
  MDD_INFO_NNZ_ZG,          /* entries of the gradient (SNK / NK) part of Z        */
  MDD_INFO_NNZ_W,           /* entries of the dense GenEO blocks of Z              */
  /* plan statistics: supernodes swept as packed small tasks / strips / 2-D tile
   * groups, and fronts factorised by the blocked path (> 1024 rows; cuBLAS
   * trailing updates), for the local factors and for E */
  MDD_INFO_LOCAL_SN_PACKED,
  MDD_INFO_LOCAL_SN_STRIP,
  MDD_INFO_LOCAL_SN_2D,
  MDD_INFO_LOCAL_BLOCKED_FRONTS,
  MDD_INFO_COARSE_SN_PACKED,
  MDD_INFO_COARSE_SN_STRIP,
  MDD_INFO_COARSE_SN_2D,
  MDD_INFO_COARSE_BLOCKED_FRONTS,
  MDD_INFO_GENEO_LANCZOS,   /* 1: the GenEO GEVPs were solved by block Lanczos (large
                               subdomains), 0: dense sygvdx per subdomain           */
  MDD_INFO_COUNT
};
int mdd_info(mdd_handle h, int64_t* out, int count);

/* Copy an internal integer array to HOST memory (int64 elements).  *len gets the
 * full length; at most cap elements are written (out may be NULL to query). */
enum {
  MDD_ARR_EDGE_TAIL = 0,    /* all edges                                 */
  MDD_ARR_EDGE_HEAD,
  MDD_ARR_FREE_EDGES,       /* free dof -> edge index                    */
  MDD_ARR_FREE_NODES,       /* free node -> node id                      */
  MDD_ARR_A_PTR,            /* CSR of A (free dofs), n+1                 */
  MDD_ARR_A_IDX,
  MDD_ARR_SUB_PTR,          /* nsub+1 offsets into MDD_ARR_SUB_DOFS       */
  MDD_ARR_SUB_DOFS,         /* concatenated N_i                           */
  MDD_ARR_GRAD_NODES_PTR,   /* nsub+1 offsets into MDD_ARR_GRAD_NODES     */
  MDD_ARR_GRAD_NODES,       /* per subdomain: free-node columns of G_i    */
  MDD_ARR_GENEO_COUNT,      /* nsub: GenEO vectors kept per subdomain     */
  MDD_ARR_E_PTR,            /* CSR of the factorised coarse matrix E (the  */
  MDD_ARR_E_IDX,            /* Jacobi-scaled S Z^T A Z S), rows/cols in coarse-position
                               order (the order of mdd_apply_coarse_inverse) */
  MDD_ARR_COUNT
};
int mdd_get_int_array(mdd_handle h, int which, int64_t* out, int64_t cap, int64_t* len);

/* Host-only topology query (no device needed): builds the mesh numbering, the
 * pattern of A, the decomposition and the G_i columns for `desc` (coefficients
 * are ignored and may be NULL) and copies array `which` (MDD_ARR_*, except
 * MDD_ARR_GENEO_COUNT) to HOST memory as for mdd_get_int_array. */
int mdd_topology_int_array(const mdd_setup_desc* desc, int which, int64_t* out, int64_t cap,
                           int64_t* len);

/* Host-only plan of the sharded solve (no device needed): for `rank` of `nranks`
 * ranks, the rank's subdomains (slabs along x), owned dofs, halo dofs and the
 * per-peer exchange lists in the rank's local numbering (owned dofs first, then
 * the halo), plus every dof's owner.  Arrays as for mdd_get_int_array. */
enum {
  MDD_SHARD_SUBS = 0,       /* this rank's subdomains (ascending)                       */
  MDD_SHARD_OWNED,          /* global dofs owned (ascending) = local 0 .. n_own-1       */
  MDD_SHARD_HALO,           /* global dofs read from other ranks = local n_own ..       */
  MDD_SHARD_SEND_PTR,       /* nranks+1 offsets into MDD_SHARD_SEND_IDX                 */
  MDD_SHARD_SEND_IDX,       /* per peer: local indices of owned dofs in its halo        */
  MDD_SHARD_RECV_PTR,       /* nranks+1 offsets into MDD_SHARD_RECV_IDX                 */
  MDD_SHARD_RECV_IDX,       /* per peer: local indices of halo dofs it owns             */
  MDD_SHARD_DOF_OWNER,      /* per global dof: owning rank                              */
  MDD_SHARD_COUNT
};
int mdd_shard_int_array(const mdd_setup_desc* desc, int rank, int nranks, int which, int64_t* out,
                        int64_t cap, int64_t* len);

/* Host-only subtree-to-rank mapping of a supernode (elimination) tree, the one
 * the sharded coarse solve applies to E's factor: nsn supernodes,
 * parent[g] (< 0: a root), cost[g] (factor entries of supernode g); on return
 * owner[g] = -1 for the replicated top supernodes (swept by every rank), else
 * the rank in [0, nranks) that sweeps g together with its whole subtree.  All
 * arrays HOST, caller-owned, nsn entries.  MDD_ERR_ARG on null arrays, bad
 * parents or nranks < 1; nranks > 1 needs at least nranks leaf subtrees. */
int mdd_tree_split(int nsn, const int32_t* parent, const int64_t* cost, int nranks, int32_t* owner);

/* Sharded solve.  After mdd_setup of the whole problem on every
 * rank (the setup is replicated), mdd_shard_setup(h, rank, nranks) builds this
 * rank's hot-path data: its owned rows of A, the supernodal factor of its
 * subdomains (prolongation onto its owned + halo dofs), its owned rows of Z and
 * the halo exchange lists of mdd_shard_int_array.  The PCG vectors of a rank
 * are its owned dofs (MDD_SHARD_OWNED order, n_own of mdd_shard_info).  Only
 * MDD_VARIANT_AS2_COARSE_START (the coarse correction z = w + Q(r - A w) with
 * one n0-allreduce per iteration) and MDD_VARIANT_AS1 are sharded.  With
 * nranks > 1, E^{-1} is applied distributed: the rank sweeps the subtrees of E's
 * supernode tree that mdd_tree_split gives it plus the replicated top, with an
 * allreduce of the frontier roots' update vectors between the two forward
 * segments and an n0-allreduce of the solution (env
 * MDD_SHARD_COARSE_REPLICATED=1: every rank sweeps the whole factor).
 * mdd_shard_info: out[0] n_own, [1] n_own + halo, [2] subdomains, [3] their
 *   factor entries, [4] 1 if the coarse solve is distributed, [5] coarse factor
 *   entries this rank sweeps, [6] of which replicated top, [7] update entries
 *   exchanged between the forward segments.
 * mdd_shard_nccl_init: NCCL communicator of the ranks (unique_id: the 128-byte
 *   ncclUniqueId of rank 0, broadcast by the caller, e.g. torch.distributed).
 * mdd_shard_solve: one rank's part of the sharded PCG; f_own / x_own: n_own
 *   doubles, DEVICE pointers (host = 0) or HOST pointers (host = 1, copies
 *   inside); every rank calls it collectively.
 * mdd_shard_solve_group: `count` handles of ONE process on one device, handle k
 *   set up as rank k of count, exchanging through device copies (DEVICE
 *   pointers); the sequence of kernels is the NCCL path's, rank by rank. */
int mdd_shard_setup(mdd_handle h, int rank, int nranks);
int mdd_shard_info(mdd_handle h, int64_t* out, int count);
int mdd_shard_nccl_init(mdd_handle h, const void* unique_id, int rank, int nranks);
int mdd_shard_solve(mdd_handle h, const double* f_own, double* x_own, double tol, int maxit, int host,
                    int* iters, double* relres);
int mdd_shard_solve_group(mdd_handle* hs, int count, const double* const* f_own, double* const* x_own,
                          double tol, int maxit, int* iters, double* relres);

/* Copy an internal double array to HOST memory. */
enum {
  MDD_DARR_A_VAL = 0,       /* values of A in MDD_ARR_A_IDX order         */
  MDD_DARR_K_VAL,           /* K in the same pattern                      */
  MDD_DARR_M_VAL,           /* M in the same pattern                      */
  MDD_DARR_GENEO_LAMBDA,    /* kept eigenvalues, subdomain-major          */
  MDD_DARR_SETUP_TIMES,     /* seconds per setup phase (see mdd_phase_name)*/
  MDD_DARR_E_VAL,           /* values of E in MDD_ARR_E_IDX order          */
  MDD_DARR_COUNT
};
int mdd_get_double_array(mdd_handle h, int which, double* out, int64_t cap, int64_t* len);
const char* mdd_phase_name(int phase);

/* Per-phase device time of the last mdd_solve with profiling enabled, in ms
 * (HOST out[0..MDD_PROF_COUNT)), and the number of launches of each phase. */
enum {
  MDD_PROF_SPMV = 0,        /* A p (+ dot) of the PCG iteration          */
  MDD_PROF_LOCAL,           /* local solves M_AS (the k_sweep launch)    */
  MDD_PROF_PREC_OTHER,      /* A products + vector ops inside M_AS,2     */
  MDD_PROF_COARSE,          /* Z^T, coarse solves E^{-1}, Z              */
  MDD_PROF_VECTOR,          /* PCG vector updates, reductions            */
  MDD_PROF_TOTAL,
  MDD_PROF_COUNT
};
int mdd_set_profiling(mdd_handle h, int enable);
/* Device time accumulated inside the persistent sweep kernel (first CTA start to
 * last CTA end, %globaltimer) over all its launches so far, and the launch count:
 * which = 0 local solves (M_AS), 1 coarse solves (E^{-1}).  HOST outputs. */
int mdd_sweep_timing(mdd_handle h, int which, double* ms_total, int64_t* launches);
int mdd_profile(mdd_handle h, double* ms, int64_t* launches, int count);

const char* mdd_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* MAXWELL_DD_H */
