// Device kernels of the maxwell_dd library (sm_100a, FP64).  See kernels.cuh.
#include "kernels.cuh"

namespace mdd {
namespace dev {

// ----------------------------------------------------------- assembly
__constant__ int c_kuhn[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
__constant__ int c_ledge[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

__global__ void k_element_matrices(int64_t ntet, const int64_t* __restrict__ tet_id,
                                   const int64_t* __restrict__ tet_nodes, int nx, int ny,
                                   double h, const double* __restrict__ mu_inv,
                                   const double* __restrict__ eps, double* __restrict__ Ke,
                                   double* __restrict__ Me) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntet) return;
  double x[4][3];
  for (int v = 0; v < 4; ++v) {
    int64_t id = tet_nodes[4 * t + v];
    int64_t i = id % (nx + 1), j = (id / (nx + 1)) % (ny + 1), k = id / ((int64_t)(nx + 1) * (ny + 1));
    x[v][0] = h * (double)i; x[v][1] = h * (double)j; x[v][2] = h * (double)k;
  }
  // J = [x1-x0, x2-x0, x3-x0] (columns); rows of J^{-1} are grad lambda_1..3
  double J[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) J[r][c] = x[c + 1][r] - x[0][r];
  double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
               J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
               J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
  double inv[3][3];
  inv[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
  inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
  inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
  inv[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
  inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
  inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
  inv[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
  inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
  inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
  double g[4][3];
  for (int c = 0; c < 3; ++c) {
    g[1][c] = inv[0][c]; g[2][c] = inv[1][c]; g[3][c] = inv[2][c];
    g[0][c] = -(inv[0][c] + inv[1][c] + inv[2][c]);
  }
  double vol = fabs(det) / 6.0;
  int64_t tid = tet_id[t];
  double mi = mu_inv[tid], ep = eps[tid];
  double cu[6][3];
  for (int e = 0; e < 6; ++e) {
    const double* a = g[c_ledge[e][0]];
    const double* b = g[c_ledge[e][1]];
    cu[e][0] = 2.0 * (a[1] * b[2] - a[2] * b[1]);
    cu[e][1] = 2.0 * (a[2] * b[0] - a[0] * b[2]);
    cu[e][2] = 2.0 * (a[0] * b[1] - a[1] * b[0]);
  }
  double G[4][4];
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) G[a][b] = g[a][0] * g[b][0] + g[a][1] * g[b][1] + g[a][2] * g[b][2];
  double kf = mi * vol, mf = ep * vol / 20.0;
  for (int m = 0; m < 6; ++m) {
    int a = c_ledge[m][0], b = c_ledge[m][1];
    for (int n = 0; n < 6; ++n) {
      int c = c_ledge[n][0], d = c_ledge[n][1];
      Ke[t * 36 + m * 6 + n] = kf * (cu[m][0] * cu[n][0] + cu[m][1] * cu[n][1] + cu[m][2] * cu[n][2]);
      Me[t * 36 + m * 6 + n] = mf * ((1 + (a == c)) * G[b][d] - (1 + (a == d)) * G[b][c] -
                                     (1 + (b == c)) * G[a][d] + (1 + (b == d)) * G[a][c]);
    }
  }
}

__global__ void k_assemble_slots(int64_t nslot, const int64_t* __restrict__ ptr,
                                 const int32_t* __restrict__ contrib,
                                 const double* __restrict__ Ke, const double* __restrict__ Me,
                                 double gamma, double* __restrict__ A, double* __restrict__ K,
                                 double* __restrict__ M) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nslot) return;
  double k = 0.0, m = 0.0;
  for (int64_t c = ptr[s]; c < ptr[s + 1]; ++c) {
    int32_t q = contrib[c];
    k += Ke[q];
    m += Me[q];
  }
  if (K) K[s] = k;
  if (M) M[s] = m;
  A[s] = k + gamma * m;
}

__global__ void k_gather(int64_t n, const int64_t* __restrict__ idx, const double* __restrict__ src,
                         double* __restrict__ dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

__global__ void k_scatter_gather(int64_t n, const int64_t* __restrict__ di, const int64_t* __restrict__ si,
                                 const double* __restrict__ src, double* __restrict__ dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[di[i]] = src[si[i]];
}

__global__ void k_dense_scatter(int64_t n, const int64_t* __restrict__ pos, const double* __restrict__ v,
                                double* __restrict__ D) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) D[pos[i]] = v[i];
}

// P = I (n x n); used before P -= G X
__global__ void k_set_identity_minus(int64_t n, double* __restrict__ P) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n * n) P[i] = (i % n == i / n) ? 1.0 : 0.0;
}

__global__ void k_scale_rows(int64_t n, int64_t cols, const double* __restrict__ d, double* __restrict__ P) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n * cols) P[i] *= d[i % n];
}

// L = (L + L^T) / 2 on the lower triangle (the GEVP reads the lower part)
__global__ void k_symmetrize(int64_t n, double* __restrict__ L) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * n) return;
  int64_t r = i % n, c = i / n;
  if (r > c) {
    double v = 0.5 * (L[r + c * n] + L[c + r * n]);
    L[r + c * n] = v;
  }
}

__global__ void k_slot_sums(int64_t nslot, const int64_t* __restrict__ ptr, const int32_t* __restrict__ contrib,
                            const double* __restrict__ Ke, const double* __restrict__ Me, double gamma,
                            double* __restrict__ out) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nslot) return;
  double k = 0.0, m = 0.0;
  for (int64_t c = ptr[s]; c < ptr[s + 1]; ++c) {
    k += Ke[contrib[c]];
    m += Me[contrib[c]];
  }
  out[s] = k + gamma * m;
}

// s[r] = 1/sqrt(E_rr) for a CSR matrix with int32 pointers
__global__ void k_inv_sqrt_diag(int n, const int* __restrict__ ptr, const int* __restrict__ idx,
                                const double* __restrict__ val, double* __restrict__ s) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double d = 0.0;
  for (int k = ptr[r]; k < ptr[r + 1]; ++k)
    if (idx[k] == r) d = val[k];
  s[r] = d > 0.0 ? 1.0 / sqrt(d) : -1.0;  // -1 flags a missing / nonpositive diagonal
}

// val[k] *= (rs ? rs[row] : 1) * (cs ? cs[idx[k]] : 1)
__global__ void k_scale_csr(int n, const int* __restrict__ ptr, const int* __restrict__ idx,
                            double* __restrict__ val, const double* __restrict__ rs,
                            const double* __restrict__ cs) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const double a = rs ? rs[r] : 1.0;
  for (int k = ptr[r]; k < ptr[r + 1]; ++k) val[k] *= a * (cs ? cs[idx[k]] : 1.0);
}

// --------------------------------------------------- multifrontal LDL^T
__global__ void k_mf_factor_level(PlanDev P, const int* __restrict__ list, const double* __restrict__ src,
                                  double* __restrict__ fronts, double* __restrict__ L,
                                  double* __restrict__ dinv, double* __restrict__ umat, int mode,
                                  double tol, uint8_t* __restrict__ dropped, int* __restrict__ err) {
  const int g = list[blockIdx.x];
  const int nc = P.sn_ncol[g], no = P.sn_noff[g], nr = nc + no;
  const i64 col0 = P.sn_col0[g];
  double* F = fronts + P.sn_fptr[g];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  for (i64 k = tid; k < (i64)nr * nr; k += nt) F[k] = 0.0;
  __syncthreads();
  for (i64 a = P.asm_ptr[g] + tid; a < P.asm_ptr[g + 1]; a += nt) F[P.asm_pos[a]] += src[P.asm_src[a]];
  __syncthreads();
  for (i64 ci = P.child_ptr[g]; ci < P.child_ptr[g + 1]; ++ci) {
    const int c = P.child_list[ci];
    const int noc = P.sn_noff[c];
    const double* U = umat + P.sn_umptr[c];
    const int* rm = P.relmap + P.sn_rowptr[c];
    for (i64 k = tid; k < (i64)noc * noc; k += nt) {
      int b = (int)(k / noc), a = (int)(k % noc);
      if (a >= b) F[(i64)rm[b] * nr + rm[a]] += U[k];
    }
    __syncthreads();
  }
  for (int j = 0; j < nc; ++j) {
    double* Fj = F + (i64)j * nr;
    const double d = Fj[j];
    bool drop = false;
    if (mode == 1) drop = !(d > tol);
    else if (mode == 2) {
      // static pivoting: a pivot at or below tol (relative to the unit diagonal of
      // the Jacobi-scaled matrix) is a rounding casualty of an SPD matrix with
      // kappa ~ 1/eps; it is replaced by tol and counted
      if (!(d > tol)) {
        if (tid == 0) atomicAdd(err, 1);
        __syncthreads();
        if (tid == 0) Fj[j] = tol;
        __syncthreads();
      }
    } else if (!(d > 0.0)) {
      if (tid == 0) atomicExch(err, 1);
      drop = true;
    }
    if (drop) {
      for (int i = j + 1 + tid; i < nr; i += nt) Fj[i] = 0.0;
      if (tid == 0) {
        dinv[col0 + j] = 0.0;
        if (dropped) dropped[col0 + j] = 1;
      }
      __syncthreads();
      continue;
    }
    const double dd = Fj[j];
    const double rd = 1.0 / dd;
    for (int i = j + 1 + tid; i < nr; i += nt) Fj[i] *= rd;
    __syncthreads();
    for (int k = j + 1 + warp; k < nr; k += nw) {
      const double lkd = Fj[k] * dd;
      double* Fk = F + (i64)k * nr;
      for (int i = k + lane; i < nr; i += 32) Fk[i] -= Fj[i] * lkd;
    }
    if (tid == 0) {
      dinv[col0 + j] = rd;
      if (dropped) dropped[col0 + j] = 0;
    }
    __syncthreads();
  }
  // L21 and the update matrix
  double* Lp = L + P.sn_lptr[g];
  for (i64 k = tid; k < (i64)nc * no; k += nt) {
    int j = (int)(k / no), i = nc + (int)(k % no);
    Lp[(i64)j * nr + i] = F[(i64)j * nr + i];
  }
  double* U = umat + P.sn_umptr[g];
  for (i64 k = tid; k < (i64)no * no; k += nt) {
    int b = (int)(k / no), a = (int)(k % no);
    U[k] = (a >= b) ? F[(i64)(nc + b) * nr + nc + a] : 0.0;
  }
  // explicit inverse of the unit-lower diagonal block, row by row:
  // X[i][j] = -sum_{k=j}^{i-1} L[i][k] X[k][j]
  for (int j = tid; j < nc; j += nt) Lp[(i64)j * nr + j] = 1.0;
  __syncthreads();
  for (int i = 1; i < nc; ++i) {
    for (int j = tid; j < i; j += nt) {
      double s = 0.0;
      for (int k = j; k < i; ++k) s -= F[(i64)k * nr + i] * Lp[(i64)j * nr + k];
      Lp[(i64)j * nr + i] = s;
    }
    __syncthreads();
  }
  // partitioned-inverse off block: M21 = L21 L11^{-1} (sweep.cu), from F's L21
  for (i64 k = tid; k < (i64)nc * no; k += nt) {
    const int j = (int)(k / no), i = nc + (int)(k % no);
    double s = 0.0;
    for (int q = j; q < nc; ++q) s += F[(i64)q * nr + i] * Lp[(i64)j * nr + q];
    Lp[(i64)j * nr + i] = s;
  }
  __syncthreads();
  // fold D^{-1} into the rows of the diagonal block: the forward sweep then yields
  // z_c = D^{-1} L11^{-1} t_c directly; the backward sweep divides z_c by D^{-1}
  // again in its gather (sweep.cu, G_b)
  for (i64 k = tid; k < (i64)nc * nc; k += nt) {
    const int j = (int)(k / nc), i = (int)(k % nc);
    if (i >= j) Lp[(i64)j * nr + i] *= dinv[col0 + i];
  }
}


// ---------------------------------------------- big fronts (blocked, cuBLAS updates)
// assemble one front: zero, original entries, children's update matrices
__global__ void k_front_assemble(PlanDev P, int g, const double* __restrict__ src, double* __restrict__ fronts,
                                 const double* __restrict__ umat) {
  const int nc = P.sn_ncol[g], no = P.sn_noff[g], nr = nc + no;
  double* F = fronts + P.sn_fptr[g];
  const int tid = threadIdx.x + blockIdx.x * blockDim.x, nt = blockDim.x * gridDim.x;
  for (i64 k = tid; k < (i64)nr * nr; k += nt) F[k] = 0.0;
}
__global__ void k_front_assemble2(PlanDev P, int g, const double* __restrict__ src, double* __restrict__ fronts,
                                  const double* __restrict__ umat) {
  const int nc = P.sn_ncol[g], no = P.sn_noff[g], nr = nc + no;
  double* F = fronts + P.sn_fptr[g];
  const int tid = threadIdx.x, nt = blockDim.x;
  for (i64 a = P.asm_ptr[g] + tid; a < P.asm_ptr[g + 1]; a += nt) F[P.asm_pos[a]] += src[P.asm_src[a]];
  __syncthreads();
  for (i64 ci = P.child_ptr[g]; ci < P.child_ptr[g + 1]; ++ci) {
    const int c = P.child_list[ci];
    const int noc = P.sn_noff[c];
    const double* U = umat + P.sn_umptr[c];
    const int* rm = P.relmap + P.sn_rowptr[c];
    for (i64 k = tid; k < (i64)noc * noc; k += nt) {
      int b = (int)(k / noc), a = (int)(k % noc);
      if (a >= b) F[(i64)rm[b] * nr + rm[a]] += U[k];
    }
    __syncthreads();
  }
}

// factor panel columns [j0, j0+nb) of a front (right-looking inside the panel, same
// pivot rules as k_mf_factor_level), then W = L_panel D_panel for the rows below
// the panel (n_rest x nb, ld n_rest) for the trailing update F22 -= W L_panel^T
__global__ void k_panel_factor(PlanDev P, int g, int j0, int nb, double* __restrict__ fronts,
                               double* __restrict__ dinv, double* __restrict__ W, int mode, double tol,
                               uint8_t* __restrict__ dropped, int* __restrict__ err) {
  const int nc = P.sn_ncol[g], no = P.sn_noff[g], nr = nc + no;
  const i64 col0 = P.sn_col0[g];
  double* F = fronts + P.sn_fptr[g];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  __shared__ double s_d[64];
  for (int jj = 0; jj < nb; ++jj) {
    const int j = j0 + jj;
    double* Fj = F + (i64)j * nr;
    const double d = Fj[j];
    bool drop = false;
    if (mode == 1) drop = !(d > tol);
    else if (mode == 2) {
      if (!(d > tol)) {
        if (tid == 0) { atomicAdd(err, 1); Fj[j] = tol; }
        __syncthreads();
      }
    } else if (!(d > 0.0)) {
      if (tid == 0) atomicExch(err, 1);
      drop = true;
    }
    if (drop) {
      for (int i = j + 1 + tid; i < nr; i += nt) Fj[i] = 0.0;
      if (tid == 0) {
        dinv[col0 + j] = 0.0;
        s_d[jj] = 0.0;
        if (dropped) dropped[col0 + j] = 1;
      }
      __syncthreads();
      continue;
    }
    const double dd = Fj[j];
    const double rd = 1.0 / dd;
    for (int i = j + 1 + tid; i < nr; i += nt) Fj[i] *= rd;
    __syncthreads();
    for (int k = j + 1 + warp; k < j0 + nb; k += nw) {  // the panel's own columns only
      const double lkd = Fj[k] * dd;
      double* Fk = F + (i64)k * nr;
      for (int i = k + lane; i < nr; i += 32) Fk[i] -= Fj[i] * lkd;
    }
    if (tid == 0) {
      dinv[col0 + j] = rd;
      s_d[jj] = dd;
      if (dropped) dropped[col0 + j] = 0;
    }
    __syncthreads();
  }
  const int r0 = j0 + nb, nrest = nr - r0;
  for (i64 k = tid; k < (i64)nrest * nb; k += nt) {
    const int jj = (int)(k / nrest), i = (int)(k % nrest);
    W[k] = F[(i64)(j0 + jj) * nr + r0 + i] * s_d[jj];
  }
}

// after the eliminations: L21 into the panel, the update matrix, the unit-lower
// L11 (strict part from F) into the panel's diagonal block for the in-place
// triangular inverse
__global__ void k_front_finish_copy(PlanDev P, int g, const double* __restrict__ fronts, double* __restrict__ L,
                                    double* __restrict__ umat) {
  const int nc = P.sn_ncol[g], no = P.sn_noff[g], nr = nc + no;
  const double* F = fronts + P.sn_fptr[g];
  double* Lp = L + P.sn_lptr[g];
  double* U = umat + P.sn_umptr[g];
  const int tid = threadIdx.x + blockIdx.x * blockDim.x, nt = blockDim.x * gridDim.x;
  for (i64 k = tid; k < (i64)nc * nr; k += nt) {
    const int j = (int)(k / nr), i = (int)(k % nr);
    Lp[k] = i > j ? F[(i64)j * nr + i] : (i == j ? 1.0 : 0.0);
  }
  for (i64 k = tid; k < (i64)no * no; k += nt) {
    const int b = (int)(k / no), a = (int)(k % no);
    U[k] = (a >= b) ? F[(i64)(nc + b) * nr + nc + a] : 0.0;
  }
}

// D^{-1} folded into the rows of the (inverted) diagonal block
__global__ void k_front_fold_d(PlanDev P, int g, double* __restrict__ L, const double* __restrict__ dinv) {
  const int nc = P.sn_ncol[g], nr = nc + P.sn_noff[g];
  const i64 col0 = P.sn_col0[g];
  double* Lp = L + P.sn_lptr[g];
  const int tid = threadIdx.x + blockIdx.x * blockDim.x, nt = blockDim.x * gridDim.x;
  for (i64 k = tid; k < (i64)nc * nc; k += nt) {
    const int j = (int)(k / nc), i = (int)(k % nc);
    if (i >= j) Lp[(i64)j * nr + i] *= dinv[col0 + i];
  }
}

// ---------------------------------------------------------- PCG pieces
#define STOPPED (stop != nullptr && stop[0] != 0)

// block-level sum of one value per thread -> part[blockIdx.x]; blockDim = 256
// block-level sum of one value per thread -> *dst (thread 0); blockDim = 256
__device__ __forceinline__ void block_sum_to(double v, double* dst) {
  __shared__ double ws[32];
  v = warp_sum(v);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) ws[w] = v;
  __syncthreads();
  if (w == 0) {
    int nw = blockDim.x >> 5;
    double s = lane < nw ? ws[lane] : 0.0;
    s = warp_sum(s);
    if (lane == 0) *dst = s;
  }
}
__device__ __forceinline__ void block_sum_store(double v, double* part) { block_sum_to(v, part + blockIdx.x); }

__device__ void scalar_op(int op, double* __restrict__ S, int* __restrict__ state);

// RedStep tail (see kernels.cuh): call after block_sum_store(..., part)
__device__ void reduce_step_tail(const double* part, const RedStep& rs) {
  if (!rs.counter) return;
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(rs.counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double s = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) s += __ldcg(part + i);
  __shared__ double tmp[1];
  block_sum_to(s, tmp);  // (not block_sum_store: this block's index is not 0)
  __syncthreads();
  if (threadIdx.x == 0) {
    rs.S[rs.slot] = tmp[0];
    scalar_op(rs.op, rs.S, rs.state);
    *rs.counter = 0u;
  }
}

// y = M x with TPR lanes per row (rows grid-strided over a fixed, SM-sized grid);
// optional fused partial dot(dotw, y) per block into part[blockIdx.x]
template <int TPR>
__device__ __forceinline__ void spmv_g_body(int nrows, const int64_t* __restrict__ ptr,
                                                const int32_t* __restrict__ idx,
                                                const double* __restrict__ val,
                                                const double* __restrict__ x,
                                                const double* __restrict__ sub, double* __restrict__ y,
                                                const double* __restrict__ dotw, double* __restrict__ part,
                                                const int* __restrict__ stop, const RedStep& rs) {
  if (STOPPED) return;
  const int g = (blockIdx.x * blockDim.x + threadIdx.x) / TPR;
  const int lane = threadIdx.x & (TPR - 1);
  const int ngroups = gridDim.x * blockDim.x / TPR;
  double dsum = 0.0;
  // the trip count is uniform per warp (the shuffles need every lane of the warp)
  for (int row = g;; row += ngroups) {
    const bool active = row < nrows;
    if (!__any_sync(0xffffffffu, active)) break;
    double s0 = 0.0, s1 = 0.0;
    if (active) {
      const int64_t a = ptr[row], b = ptr[row + 1];
      int64_t k = a + lane;
      for (; k + TPR < b; k += 2 * TPR) {
        s0 += val[k] * x[idx[k]];
        s1 += val[k + TPR] * x[idx[k + TPR]];
      }
      if (k < b) s0 += val[k] * x[idx[k]];
    }
    double s = s0 + s1;
#pragma unroll
    for (int o = TPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, TPR);
    if (active && lane == 0) {
      if (sub) s = sub[row] - s;
      y[row] = s;
      if (dotw) dsum += dotw[row] * s;
    }
  }
  if (part) {
    block_sum_store(dsum, part);
    reduce_step_tail(part, rs);
  }
}
#define MDD_SPMV_G(NAME, TPR)                                                                      \
  __global__ void __launch_bounds__(256)                                                           \
      NAME(int nrows, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,          \
           const double* __restrict__ val, const double* __restrict__ x,                          \
           const double* __restrict__ sub, double* __restrict__ y, const double* __restrict__ dotw, \
           double* __restrict__ part, const int* __restrict__ stop, RedStep rs) {                  \
    spmv_g_body<TPR>(nrows, ptr, idx, val, x, sub, y, dotw, part, stop, rs);                      \
  }
MDD_SPMV_G(k_spmv4, 4)
MDD_SPMV_G(k_spmv8, 8)
MDD_SPMV_G(k_spmv16, 16)
MDD_SPMV_G(k_spmv32, 32)
#undef MDD_SPMV_G

// ---------------------------------------------------------- GenEO blocks
// Z_e^T v, stage 1: for block b = (subdomain i, columns [k0, k0+kc), rows
// [r0, r0+rc)): part[b][q] = sum_{p in rows} W_i[p + (k0+q) n_i] v[gmap[off_i + p]]
// (per thread a strided row range, then warp shuffles, then the warps in order:
// a fixed reduction order, the stage-2 kernel adds the row chunks in order)
__global__ void __launch_bounds__(256) k_geneo_zt(const int4* __restrict__ blk, const int64_t* __restrict__ woff,
                                                  const int64_t* __restrict__ poff, const int* __restrict__ nsz,
                                                  const int* __restrict__ gcol0, const int32_t* __restrict__ gpos,
                                                  const double* __restrict__ W, const int32_t* __restrict__ gmap,
                                                  const double* __restrict__ v, double* __restrict__ part,
                                                  const int* __restrict__ stop) {
  if (STOPPED) return;
  constexpr int KC = 8;
  __shared__ double red[8][KC];
  const int4 b = blk[blockIdx.x];  // {subdomain, first column, columns, first row}
  const int i = b.x, k0 = b.y, kc = b.z, r0 = b.w;
  const int ni = nsz[i];
  const int r1 = min(ni, r0 + kGeneoRows);
  const double* Wi = W + woff[i] + (int64_t)k0 * ni;
  const int32_t* gm = gmap + poff[i];
  double acc[KC];
#pragma unroll
  for (int q = 0; q < KC; ++q) acc[q] = 0.0;
  // kGeneoRows / 256 rows per thread: every gather and W load of the chunk is
  // issued before the first multiply (memory-level parallelism)
  constexpr int RPT = kGeneoRows / 256;
  double vp[RPT];
#pragma unroll
  for (int t = 0; t < RPT; ++t) {
    const int p = r0 + t * 256 + (int)threadIdx.x;
    vp[t] = p < r1 ? __ldg(v + __ldg(gm + p)) : 0.0;
  }
#pragma unroll
  for (int q = 0; q < KC; ++q) {
    if (q < kc) {
      double w[RPT];
#pragma unroll
      for (int t = 0; t < RPT; ++t) {
        const int p = r0 + t * 256 + (int)threadIdx.x;
        w[t] = p < r1 ? __ldcs(Wi + (int64_t)q * ni + p) : 0.0;
      }
#pragma unroll
      for (int t = 0; t < RPT; ++t) acc[q] += w[t] * vp[t];
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < KC; ++q) {
    const double t = warp_sum(acc[q]);
    if (lane == 0) red[w][q] = t;
  }
  __syncthreads();
  if (threadIdx.x < kc) {
    double t = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q][threadIdx.x];
    part[(int64_t)blockIdx.x * KC + threadIdx.x] = t;
  }
}

// Z_e^T v, stage 2: y[gpos[c]] = sum of the row-chunk partials of column c, in order
// (cpart[c] = first block of column c's column chunk, cstride = blocks per row chunk)
__global__ void k_geneo_zt2(int ncols, const int* __restrict__ cblk, const int* __restrict__ cnch,
                            const int32_t* __restrict__ gpos, const double* __restrict__ part,
                            double* __restrict__ y, const int* __restrict__ stop) {
  if (STOPPED) return;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  // cblk[c] = (first block of the column's chunk) * 8 + lane within the chunk
  const int b0 = cblk[c] >> 3, q = cblk[c] & 7;
  double t = 0.0;
  for (int r = 0; r < cnch[c]; ++r) t += part[(int64_t)(b0 + r) * 8 + q];
  y[gpos[c]] = t;
}

// u[off_i + p] = sum_k W_i[p + k n_i] xc[gpos[gcol0_i + k]]  (rows of subdomain i);
// the block's k_i coarse values are staged in shared memory (64 at a time); each
// thread owns kGeneoZRows / 256 rows (all their loads of a column chunk in flight)
__global__ void __launch_bounds__(256) k_geneo_z(const int4* __restrict__ blk, const int64_t* __restrict__ woff,
                                                 const int64_t* __restrict__ poff, const int* __restrict__ nsz,
                                                 const int* __restrict__ kcnt, const int* __restrict__ gcol0,
                                                 const int32_t* __restrict__ gpos, const double* __restrict__ W,
                                                 const double* __restrict__ xc, double* __restrict__ u,
                                                 const int* __restrict__ stop) {
  if (STOPPED) return;
  constexpr int RPT = kGeneoZRows / 256;
  __shared__ double xs[64];
  const int4 b = blk[blockIdx.x];  // {subdomain, first row, -, -}
  const int i = b.x;
  const int ni = nsz[i], ki = kcnt[i];
  const double* Wi = W + woff[i];
  const int32_t* gp = gpos + gcol0[i];
  // per row: eight column streams; column k goes to s[t][k % 8]
  double s[RPT][8];
#pragma unroll
  for (int t = 0; t < RPT; ++t)
#pragma unroll
    for (int j = 0; j < 8; ++j) s[t][j] = 0.0;
  for (int kb = 0; kb < ki; kb += 64) {
    const int kn = min(64, ki - kb);
    __syncthreads();
    if (threadIdx.x < kn) xs[threadIdx.x] = __ldg(xc + __ldg(gp + kb + threadIdx.x));
    __syncthreads();
    int k = 0;
    for (; k + 8 <= kn; k += 8) {
      double w[RPT][8];
#pragma unroll
      for (int t = 0; t < RPT; ++t) {
        const int p = b.y + t * 256 + (int)threadIdx.x;
#pragma unroll
        for (int j = 0; j < 8; ++j) w[t][j] = p < ni ? __ldcs(Wi + (int64_t)(kb + k + j) * ni + p) : 0.0;
      }
#pragma unroll
      for (int t = 0; t < RPT; ++t)
#pragma unroll
        for (int j = 0; j < 8; ++j) s[t][j] += w[t][j] * xs[k + j];
    }
    for (int j = 0; k < kn; ++k, ++j)
#pragma unroll
      for (int t = 0; t < RPT; ++t) {
        const int p = b.y + t * 256 + (int)threadIdx.x;
        if (p < ni) s[t][j] += __ldcs(Wi + (int64_t)(kb + k) * ni + p) * xs[k];
      }
  }
#pragma unroll
  for (int t = 0; t < RPT; ++t) {
    const int p = b.y + t * 256 + (int)threadIdx.x;
    if (p < ni)
      u[poff[i] + p] = ((s[t][0] + s[t][1]) + (s[t][2] + s[t][3])) + ((s[t][4] + s[t][5]) + (s[t][6] + s[t][7]));
  }
}

// out[e] = Z_g(e, :) xc + sum of the GenEO contributions u at the copies of e
__global__ void __launch_bounds__(256) k_z_apply(int n, const int64_t* __restrict__ ptr,
                                                 const int32_t* __restrict__ idx, const double* __restrict__ val,
                                                 const double* __restrict__ xc, const int64_t* __restrict__ pptr,
                                                 const int32_t* __restrict__ ppos, const double* __restrict__ u,
                                                 const double* __restrict__ addw, double* __restrict__ out,
                                                 const double* __restrict__ dotw, double* __restrict__ part,
                                                 const int* __restrict__ stop, RedStep rs) {
  if (STOPPED) return;
  double d = 0.0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t k = ptr[e]; k < ptr[e + 1]; ++k) s += val[k] * xc[idx[k]];
    if (u)
      for (int64_t k = pptr[e]; k < pptr[e + 1]; ++k) s += u[ppos[k]];
    if (addw) s = addw[e] + s;
    out[e] = s;
    if (dotw) d += dotw[e] * s;  // the same per-thread order as k_dot_part
  }
  if (part) {
    block_sum_store(d, part);
    reduce_step_tail(part, rs);
  }
}

__global__ void k_dot_part(int n, const double* __restrict__ a, const double* __restrict__ b,
                           double* __restrict__ part, const int* __restrict__ stop, RedStep rs) {
  if (STOPPED) return;
  double s = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    s += a[i] * b[i];
  block_sum_store(s, part);
  reduce_step_tail(part, rs);
}

__global__ void k_reduce(int nparts, const double* __restrict__ part, double* __restrict__ out,
                         const int* __restrict__ stop) {
  if (STOPPED) return;
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += part[i];
  __shared__ double tmp[1];
  block_sum_to(s, tmp);
  __syncthreads();
  if (threadIdx.x == 0) *out = tmp[0];
}

// scalar recurrences of PCG (single thread).  state[ST_STOP] makes every later
// kernel of the iteration a no-op; state[ST_ITERS] counts iterations on the device
__device__ void scalar_op(int op, double* __restrict__ S, int* __restrict__ state) {
  switch (op) {
    case 0:  // after q = A p:  alpha = rz / pq
      if (!(S[S_PQ] > 0.0)) { state[ST_BREAKDOWN] = 1; state[ST_STOP] = 1; return; }
      S[S_ALPHA] = S[S_RZ] / S[S_PQ];
      break;
    case 1: {  // after the r update: convergence / iteration limit
      const int it = state[ST_ITERS] + 1;
      state[ST_ITERS] = it;
      S[S_REL] = sqrt(S[S_RR]) / S[S_NF];
      if (S[S_REL] <= S[S_TOL]) { state[ST_CONVERGED] = 1; state[ST_STOP] = 1; }
      else if (it >= state[ST_MAXIT]) state[ST_STOP] = 1;
      break;
    }
    case 2:  // after z = M r: beta
      S[S_BETA] = S[S_RZNEW] / S[S_RZ];
      S[S_RZ] = S[S_RZNEW];
      break;
    case 3:  // prologue: ||f||; f = 0 -> x = 0 converged in 0 iterations
      S[S_NF] = sqrt(S[S_RR]);
      S[S_REL] = S[S_NF] > 0.0 ? 1.0 : 0.0;
      if (!(S[S_NF] > 0.0)) { state[ST_CONVERGED] = 1; state[ST_STOP] = 1; }
      else if (state[ST_MAXIT] <= 0) state[ST_STOP] = 1;
      break;
  }
}

__global__ void k_scalar_step(int op, double* __restrict__ S, int* __restrict__ state) {
  if (state[ST_STOP]) return;
  scalar_op(op, S, state);
}

// device-side loop condition of the CUDA-graph WHILE node
__global__ void k_loop_cond(cudaGraphConditionalHandle h, const int* __restrict__ state) {
  cudaGraphSetConditional(h, state[ST_STOP] ? 0u : 1u);
}

__global__ void k_update_xr(int n, double* __restrict__ x, double* __restrict__ r,
                            const double* __restrict__ p, const double* __restrict__ q,
                            const double* __restrict__ S, double* __restrict__ part,
                            const int* __restrict__ stop, RedStep rs) {
  if (STOPPED) return;
  const double alpha = S[S_ALPHA];
  double s = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    double ri = r[i] - alpha * q[i];
    r[i] = ri;
    s += ri * ri;
  }
  block_sum_store(s, part);
  reduce_step_tail(part, rs);
}

__global__ void k_update_p(int n, double* __restrict__ p, const double* __restrict__ z,
                           const double* __restrict__ S, const int* __restrict__ stop) {
  if (STOPPED) return;
  const double beta = S[S_BETA];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}

__global__ void k_axpby(int n, double a, const double* __restrict__ x, double b,
                        const double* __restrict__ y, double* __restrict__ out,
                        const int* __restrict__ stop) {
  if (STOPPED) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = a * x[i] + b * y[i];
}

// out = a + b - c
__global__ void k_combine3(int n, const double* __restrict__ a, const double* __restrict__ b,
                           const double* __restrict__ c, double* __restrict__ out,
                           const int* __restrict__ stop) {
  if (STOPPED) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = a[i] + b[i] - c[i];
}

__global__ void k_copy(int n, const double* __restrict__ a, double* __restrict__ out,
                       const int* __restrict__ stop) {
  if (STOPPED) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = a[i];
}

}  // namespace dev
}  // namespace mdd
