// GenEO GEVPs of all subdomains at once by block Lanczos on the device (setup
// phase), for subdomains too large for the dense sygvdx path (c3 / c4: 29k-44k
// local dofs, where one dense pencil is 7-15 GB and O(n^3)).
//
// PAPER.md GEVP 3.5 (eq. 3.1), per subdomain j:
//   L_j V = lambda B_j V,   L_j = (I - xi_0j^T) D_j A_j D_j (I - xi_0j),  B_j = A_j^Neu,
//   xi_0j = G_j (G_j^T A_j G_j)^{-1} G_j^T A_j (Def. 2.4); keep lambda > tau and the
//   columns W = D_j (I - xi_0j) V.
// B_j^{-1} L_j is self-adjoint in the B_j inner product and its wanted eigenvalues
// are the largest ones, well above the bulk of the spectrum, so block Lanczos
// (Golub-Underwood) on B^{-1} L in the B inner product finds them; full
// B-reorthogonalisation (two classical Gram-Schmidt passes) keeps the basis
// orthonormal, and the block size (8) covers eigenvalue multiplicities of the
// symmetric recipes.  Operators, all subdomains in lockstep:
//   A_j, B_j   -- block-diagonal CSR SpMV over a padded index space (rows j*n_pad + i,
//                 i in N_j order)
//   G_j, G_j^T -- +-1 edge-node incidences (two per edge)
//   S_j^{-1}   -- S_j = G_j^T A_j G_j dense (g_j <= ~7k), Cholesky by cuSOLVER,
//                 solves by batched cuBLAS TRSM
//   B_j^{-1}   -- the supernodal LDL^T of all A_j^Neu (the same multifrontal
//                 factorisation and persistent sweep kernel as the local solves)
// Dense b x b / m x b pieces are strided-batched cuBLAS; the block-tridiagonal T is
// diagonalised by cuSOLVER syevd at a few checkpoints, where the host reads only
// the Ritz values and the residual bounds ||R_k s_i(last block)|| to decide
// convergence (a Ritz pair is converged at residual <= 1e-10 max(theta, tau),
// floored at 1e-14 theta_max;
// a subdomain is done when every Ritz value above tau and the largest one below
// it are converged and the count above tau did not change since the previous
// checkpoint).
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "geneo.h"

namespace mdd {

#define LZ_CUBLAS(x)                                                                           \
  do {                                                                                         \
    cublasStatus_t s__ = (x);                                                                  \
    if (s__ != CUBLAS_STATUS_SUCCESS)                                                          \
      throw Error(1, std::string(#x) + ": cublas status " + std::to_string((int)s__));         \
  } while (0)
#define LZ_CUSOLVER(x)                                                                         \
  do {                                                                                         \
    cusolverStatus_t s__ = (x);                                                                \
    if (s__ != CUSOLVER_STATUS_SUCCESS)                                                        \
      throw Error(1, std::string(#x) + ": cusolver status " + std::to_string((int)s__));       \
  } while (0)

namespace {

inline int nbk(int64_t n, int t) { return (int)std::max<int64_t>(1, (n + t - 1) / t); }

// Y[j][c][i] = sum_p val[p] X[j][c][idx[p] - j*cpad]  (block-diagonal CSR, rows
// r = j*rpad + i; X and Y in [nsub][ncols][pad] layout)
__global__ void k_bd_spmv(int64_t nrows, int rpad, int cpad, int ncols, const int64_t* __restrict__ ptr,
                          const int32_t* __restrict__ idx, const double* __restrict__ val,
                          const double* __restrict__ X, double* __restrict__ Y) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const int64_t j = r / rpad, i = r - j * rpad;
  const double* x = X + j * (int64_t)ncols * cpad - j * (int64_t)cpad;
  double* y = Y + j * (int64_t)ncols * rpad + i;
  const int64_t p0 = ptr[r], p1 = ptr[r + 1];
  for (int c = 0; c < ncols; ++c) {
    double s = 0.0;
    for (int64_t p = p0; p < p1; ++p) s += val[p] * x[(int64_t)c * cpad + idx[p]];
    y[(int64_t)c * rpad] = s;
  }
}

// node space: T[j][c][v] = sum_{k in edges(v)} sign * X[j][c][k]   (G_j^T X)
__global__ void k_gt(int64_t nnodes, int gpad, int npad, int ncols, const int64_t* __restrict__ ptr,
                     const int32_t* __restrict__ edge, const double* __restrict__ sgn,
                     const double* __restrict__ X, double* __restrict__ T) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nnodes) return;
  const int64_t j = r / gpad, v = r - j * gpad;
  const double* x = X + j * (int64_t)ncols * npad;
  double* t = T + j * (int64_t)ncols * gpad + v;
  for (int c = 0; c < ncols; ++c) {
    double s = 0.0;
    for (int64_t p = ptr[r]; p < ptr[r + 1]; ++p) s += sgn[p] * x[(int64_t)c * npad + edge[p]];
    t[(int64_t)c * gpad] = s;
  }
}

// edge space: Y[j][c][k] = D[j][k] * (X[j][c][k] - sum_t s_t S[j][c][col_t(k)])  when D != null,
// else Y = sum_t s_t S[...] (G_j s)
__global__ void k_g_apply(int64_t nedges, int npad, int gpad, int ncols, const int2* __restrict__ ecol,
                          const double* __restrict__ Sn, const double* __restrict__ X,
                          const double* __restrict__ D, double* __restrict__ Y) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nedges) return;
  const int64_t j = r / npad, k = r - j * npad;
  const int2 ec = ecol[r];  // tail column (sign -1), head column (sign +1); -1 = none
  const double* s = Sn + j * (int64_t)ncols * gpad;
  const double d = D ? D[r] : 1.0;
  for (int c = 0; c < ncols; ++c) {
    double g = 0.0;
    if (ec.x >= 0) g -= s[(int64_t)c * gpad + ec.x];
    if (ec.y >= 0) g += s[(int64_t)c * gpad + ec.y];
    const int64_t o = j * (int64_t)ncols * npad + (int64_t)c * npad + k;
    Y[o] = D ? d * (X[o] - g) : g;
  }
}

// Y[j][c][k] = D[j][k] * X[j][c][k]
__global__ void k_dscale(int64_t n, int npad, int ncols, const double* __restrict__ D, const double* __restrict__ X,
                         double* __restrict__ Y) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int64_t j = q / ((int64_t)ncols * npad), k = q % npad;
  Y[q] = D[j * npad + k] * X[q];
}

__global__ void k_sub(int64_t n, const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ y) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) y[q] = a[q] - b[q];
}

// deterministic start block: hashed uniform(-1, 1) on the live rows, 0 on padding
__global__ void k_lz_random(int64_t n, int npad, int ncols, const int* __restrict__ nj, double* __restrict__ X) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int64_t j = q / ((int64_t)ncols * npad), k = q % npad;
  uint64_t h = (uint64_t)q * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
  h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 27; h *= 0x94D049BB133111EBull; h ^= h >> 31;
  X[q] = k < nj[j] ? ((double)(h >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0 : 0.0;
}

// U[map[p] + off] = x[p]   (sweep positions -> padded block column)
__global__ void k_pos_scatter(int64_t n, const int32_t* __restrict__ map, const double* __restrict__ x,
                              double* __restrict__ U) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) U[map[p]] = x[p];
}

// T_j(r0 + a, c0 + c) = Blk_j(a, c) (b x b, col-major), and (sym) T_j(c0 + c, r0 + a)
// too; upper: only the upper triangle of Blk is read (a <= c), lower entries 0
__global__ void k_put_block(int nsub, int b, int mmax, double* __restrict__ T, int r0, int c0,
                            const double* __restrict__ Blk, int sym, int upper, int symmetrize) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nsub * b * b) return;
  const int j = q / (b * b), e = q % (b * b), a = e % b, c = e / b;
  const double* B = Blk + (int64_t)j * b * b;
  double v = B[c * b + a];
  if (upper && a > c) v = 0.0;
  if (symmetrize) v = 0.5 * (v + B[a * b + c]);
  double* Tj = T + (int64_t)j * mmax * mmax;
  Tj[(int64_t)(c0 + c) * mmax + (r0 + a)] = v;
  if (sym) Tj[(int64_t)(r0 + a) * mmax + (c0 + c)] = v;
}

// dense S_j = G_j^T A_j G_j, one thread per node row v (fixed summation order, no
// atomics): S[v][w] = sum_{k in edges(v)} s_kv sum_{(k, k2) in A_j} A s_{k2 w};
// padding diagonal = 1.  S is [nsub][gpad][gpad] col-major, zeroed on entry.
__global__ void k_gtag(int64_t nnodes, int gpad, int npad, const int* __restrict__ gj, const int64_t* __restrict__ nptr,
                       const int32_t* __restrict__ nedge, const double* __restrict__ nsgn,
                       const int64_t* __restrict__ aptr, const int32_t* __restrict__ aidx,
                       const double* __restrict__ aval, const int2* __restrict__ ecol, double* __restrict__ S) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nnodes) return;
  const int64_t j = r / gpad, v = r - j * gpad;
  double* Sj = S + j * (int64_t)gpad * gpad;
  if (v >= gj[j]) {
    Sj[v * gpad + v] = 1.0;
    return;
  }
  for (int64_t p = nptr[r]; p < nptr[r + 1]; ++p) {
    const int64_t k = j * (int64_t)npad + nedge[p];  // global padded edge row
    const double sv = nsgn[p];
    for (int64_t q = aptr[k]; q < aptr[k + 1]; ++q) {
      const int2 ec = ecol[aidx[q]];
      const double a = sv * aval[q];
      if (ec.x >= 0) Sj[(int64_t)ec.x * gpad + v] -= a;
      if (ec.y >= 0) Sj[(int64_t)ec.y * gpad + v] += a;
    }
  }
}

struct Ptrs {
  DBuf<double*> d;
  void set(double* base, int64_t stride, int n) {
    std::vector<double*> h(n);
    for (int j = 0; j < n; ++j) h[j] = base + (int64_t)j * stride;
    d.upload(h);
  }
};

}  // namespace

void geneo_lanczos(const GeneoInputs& in, double tau, std::vector<GeneoBlock>& out, cudaStream_t s) {
  const HostMesh& m = *in.mesh;
  const Decomp& dec = *in.dec;
  const int nsub = dec.nsub;
  MDD_REQUIRE(in.lxyz != nullptr, 5, "geneo_lanczos needs the local coordinates");
  out.clear();
  out.resize(nsub);
  const int b = std::max(2, std::min(16, getenv("MDD_LANCZOS_BLOCK") ? atoi(getenv("MDD_LANCZOS_BLOCK")) : 8));
  // ---------------------------------------------------------------- sizes
  std::vector<int> nj(nsub), gj(nsub);
  int nmax = 0, gmax = 1, nmin = INT32_MAX;
  for (int j = 0; j < nsub; ++j) {
    nj[j] = (int)dec.sub_dofs[j].size();
    gj[j] = (int)(*in.grad_nodes)[j].size();
    nmax = std::max(nmax, nj[j]);
    nmin = std::min(nmin, nj[j]);
    gmax = std::max(gmax, gj[j]);
  }
  const int npad = (nmax + 1) & ~1, gpad = gmax;
  const int64_t NR = (int64_t)nsub * npad, NG = (int64_t)nsub * gpad;
  int mmax = getenv("MDD_LANCZOS_MMAX") ? atoi(getenv("MDD_LANCZOS_MMAX")) : 1536;
  mmax = std::min(mmax, (nmin / b - 1) * b);
  mmax = (mmax / b) * b;
  MDD_REQUIRE(mmax >= 2 * b, 2, "subdomains too small for block Lanczos");

  // ------------------------------------------- host structures (padded space)
  std::vector<int64_t> aptr(NR + 1, 0), aslot, ncnt(1, 0);
  std::vector<int32_t> aidx, nctb;
  std::vector<int64_t> gptr(NG + 1, 0);
  std::vector<int32_t> gedge;
  std::vector<double> gsgn, dvec(NR, 0.0);
  std::vector<int2> ecol(NR, make_int2(-1, -1));
  std::vector<int32_t> g2l(m.n(), -1), colof(m.free_node.size() ? m.free_node.size() : 1, -1);
  std::vector<int32_t> grow, gcol;
  std::vector<double> gval;
  std::vector<int64_t> sys_val_off(nsub + 1, 0);
  for (int j = 0; j < nsub; ++j) {
    const Csr& lp = (*in.lpat)[j];
    const auto& D = dec.sub_dofs[j];
    sys_val_off[j] = (int64_t)aidx.size();
    for (int i = 0; i < nj[j]; ++i) {
      for (int64_t p = lp.ptr[i]; p < lp.ptr[i + 1]; ++p) {
        aidx.push_back(j * npad + lp.idx[p]);
        aslot.push_back((*in.lslot)[j][p]);
      }
      aptr[(int64_t)j * npad + i + 1] = lp.ptr[i + 1] - lp.ptr[i];
      dvec[(int64_t)j * npad + i] = 1.0 / (double)dec.mult[D[i]];
    }
    std::vector<int64_t> cnt;
    std::vector<int32_t> ctb;
    neumann_slots(m, dec, lp, j, g2l, cnt, ctb);
    const int64_t base = ncnt.back();
    for (int64_t p = 0; p < lp.nnz(); ++p) ncnt.push_back(base + cnt[p + 1]);
    nctb.insert(nctb.end(), ctb.begin(), ctb.end());
    gradient_entries(m, D, (*in.grad_nodes)[j], colof, grow, gcol, gval);
    std::vector<std::vector<std::pair<int32_t, double>>> byn(gj[j]);
    for (size_t q = 0; q < grow.size(); ++q) {
      int2& e = ecol[(int64_t)j * npad + grow[q]];
      if (gval[q] < 0) e.x = gcol[q]; else e.y = gcol[q];
      byn[gcol[q]].push_back({grow[q], gval[q]});
    }
    for (int v = 0; v < gj[j]; ++v) {
      for (auto& pr : byn[v]) { gedge.push_back(pr.first); gsgn.push_back(pr.second); }
      gptr[(int64_t)j * gpad + v + 1] = (int64_t)byn[v].size();
    }
  }
  sys_val_off[nsub] = (int64_t)aidx.size();
  for (int64_t r = 0; r < NR; ++r) aptr[r + 1] += aptr[r];
  for (int64_t r = 0; r < NG; ++r) gptr[r + 1] += gptr[r];
  // ecol holds LOCAL node columns; k_gtag / k_g_apply add the subdomain's offset
  // implicitly through their per-subdomain base pointers

  DBuf<int64_t> d_aptr, d_aslot, d_ncnt, d_gptr;
  DBuf<int32_t> d_aidx, d_nctb, d_gedge;
  DBuf<double> d_aval, d_bval, d_gsgn, d_dvec;
  DBuf<int2> d_ecol;
  DBuf<int> d_nj, d_gj;
  d_aptr.upload(aptr); d_aidx.upload(aidx); d_aslot.upload(aslot);
  d_ncnt.upload(ncnt); d_nctb.upload(nctb.empty() ? std::vector<int32_t>{0} : nctb);
  d_gptr.upload(gptr); d_gedge.upload(gedge.empty() ? std::vector<int32_t>{0} : gedge);
  d_gsgn.upload(gsgn.empty() ? std::vector<double>{0.0} : gsgn);
  d_dvec.upload(dvec); d_ecol.upload(ecol); d_nj.upload(nj); d_gj.upload(gj);
  const int64_t annz = (int64_t)aidx.size();
  d_aval.alloc(annz); d_bval.alloc(annz);
  dev::k_gather<<<nbk(annz, 256), 256, 0, s>>>(annz, d_aslot.p, in.A_val, d_aval.p);
  dev::k_slot_sums<<<nbk(annz, 256), 256, 0, s>>>(annz, d_ncnt.p, d_nctb.p, in.Ke, in.Me, in.gamma, d_bval.p);
  CUDA_CHECK(cudaGetLastError());
  d_aslot.release(); d_ncnt.release(); d_nctb.release();

  cublasHandle_t cb;
  cusolverDnHandle_t cs;
  LZ_CUBLAS(cublasCreate(&cb));
  LZ_CUSOLVER(cusolverDnCreate(&cs));
  struct Guard {
    cublasHandle_t cb; cusolverDnHandle_t cs;
    ~Guard() { cublasDestroy(cb); cusolverDnDestroy(cs); }
  } guard{cb, cs};
  LZ_CUBLAS(cublasSetStream(cb, s));
  LZ_CUSOLVER(cusolverDnSetStream(cs, s));

  // ---- S_j = G^T A G (for xi_0j) and S^B_j = G^T B G (the B-orthogonal deflation
  // of range(G_j), reading R15), dense Cholesky factors
  const bool deflate = !(getenv("MDD_GENEO_DEFLATE") && atoi(getenv("MDD_GENEO_DEFLATE")) == 0);
  DBuf<double> Sd, SdB;
  auto gram = [&](DBuf<double>& Sx, const double* vals, const char* what) {
    Sx.alloc((size_t)nsub * gpad * gpad);
    Sx.zero(s);
    k_gtag<<<nbk(NG, 128), 128, 0, s>>>(NG, gpad, npad, d_gj.p, d_gptr.p, d_gedge.p, d_gsgn.p, d_aptr.p, d_aidx.p,
                                        vals, d_ecol.p, Sx.p);
    CUDA_CHECK(cudaGetLastError());
    int lw = 0;
    LZ_CUSOLVER(cusolverDnDpotrf_bufferSize(cs, CUBLAS_FILL_MODE_LOWER, gpad, Sx.p, gpad, &lw));
    DBuf<double> work;
    work.alloc(std::max(lw, 1));
    DBuf<int> info;
    info.alloc(nsub);
    info.zero(s);
    for (int j = 0; j < nsub; ++j)
      LZ_CUSOLVER(cusolverDnDpotrf(cs, CUBLAS_FILL_MODE_LOWER, gpad, Sx.p + (int64_t)j * gpad * gpad, gpad, work.p,
                                   lw, info.p + j));
    std::vector<int> hi = info.download();
    for (int j = 0; j < nsub; ++j)
      MDD_REQUIRE(hi[j] == 0, 3, std::string(what) + " is not SPD in subdomain " + std::to_string(j));
  };
  gram(Sd, d_aval.p, "G_j^T A_j G_j");
  if (deflate) gram(SdB, d_bval.p, "G_j^T A_j^Neu G_j");

  // ------------------------------------------- B_j^{-1}: supernodal LDL^T of A^Neu
  DevFactor neu;
  {
    std::vector<std::vector<int64_t>> vslot(nsub);
    std::vector<SymSystem> sys(nsub);
    for (int j = 0; j < nsub; ++j) {
      const Csr& lp = (*in.lpat)[j];
      vslot[j].resize(lp.nnz());
      for (int64_t p = 0; p < lp.nnz(); ++p) vslot[j][p] = sys_val_off[j] + p;
      sys[j] = SymSystem{&lp, (*in.lxyz)[j].data(), vslot[j].data()};
    }
    build_factor_plan(neu.fp, sys, getenv("MDD_ND_LEAF") ? atoi(getenv("MDD_ND_LEAF")) : 64);
    neu.name = "neumann";
    std::vector<int32_t> gm(neu.fp.ntot);
    for (int j = 0; j < nsub; ++j)
      for (int64_t k = neu.fp.sys_off[j]; k < neu.fp.sys_off[j + 1]; ++k)
        gm[k] = (int32_t)((int64_t)j * b * npad + neu.fp.perm[k]);
    neu.upload(0, nullptr, nullptr, &gm);
    neu.factor(d_bval.p, 0, 0.0, nullptr, s);
  }
  DBuf<int32_t> d_pmap;  // sweep position -> padded block index (column 0)
  {
    std::vector<int32_t> gm(neu.fp.ntot);
    for (int j = 0; j < nsub; ++j)
      for (int64_t k = neu.fp.sys_off[j]; k < neu.fp.sys_off[j + 1]; ++k)
        gm[k] = (int32_t)((int64_t)j * b * npad + neu.fp.perm[k]);
    d_pmap.upload(gm);
  }
  const int64_t ntot = neu.fp.ntot;

  // ------------------------------------------------------------ operators
  const int64_t BLK = (int64_t)nsub * b * npad;  // one block of b columns
  DBuf<double> T1, T2, T3, Y, U, BU, Sn;
  T1.alloc(BLK); T2.alloc(BLK); T3.alloc(BLK); Y.alloc(BLK); U.alloc(BLK); BU.alloc(BLK);
  Sn.alloc((size_t)nsub * b * gpad);
  Ptrs pSd, pSn, pSdB;
  pSd.set(Sd.p, (int64_t)gpad * gpad, nsub);
  pSn.set(Sn.p, (int64_t)b * gpad, nsub);
  if (deflate) pSdB.set(SdB.p, (int64_t)gpad * gpad, nsub);
  DBuf<double> ones;
  ones.upload(std::vector<double>(NR, 1.0));
  const double one = 1.0, zero = 0.0, mone = -1.0;
  auto bd = [&](const double* val, const double* X, double* Yo, int nc) {
    k_bd_spmv<<<nbk(NR, 128), 128, 0, s>>>(NR, npad, npad, nc, d_aptr.p, d_aidx.p, val, X, Yo);
  };
  auto ssolve = [&](double* const* sn_ptrs, int nc) {
    LZ_CUBLAS(cublasDtrsmBatched(cb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT,
                                 gpad, nc, &one, pSd.d.p, gpad, sn_ptrs, gpad, nsub));
    LZ_CUBLAS(cublasDtrsmBatched(cb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT,
                                 gpad, nc, &one, pSd.d.p, gpad, sn_ptrs, gpad, nsub));
  };
  // (I - xi) X scaled by D: Out = D (X - G S^{-1} G^T A X)   (t1, sn: scratch)
  auto dproj = [&](const double* X, double* Out, double* t1, double* sn, double* const* snp, int nc) {
    bd(d_aval.p, X, t1, nc);
    k_gt<<<nbk(NG, 128), 128, 0, s>>>(NG, gpad, npad, nc, d_gptr.p, d_gedge.p, d_gsgn.p, t1, sn);
    ssolve(snp, nc);
    k_g_apply<<<nbk(NR, 128), 128, 0, s>>>(NR, npad, gpad, nc, d_ecol.p, sn, X, d_dvec.p, Out);
  };
  // Yo = L X = (I - xi^T) D A D (I - xi) X
  auto applyL = [&](const double* X, double* Yo) {
    dproj(X, T1.p, T2.p, Sn.p, pSn.d.p, b);           // q = D (I - xi) X
    bd(d_aval.p, T1.p, T2.p, b);                      // v = A q
    const int64_t n = BLK;
    k_dscale<<<nbk(n, 256), 256, 0, s>>>(n, npad, b, d_dvec.p, T2.p, T2.p);  // dv = D v
    k_gt<<<nbk(NG, 128), 128, 0, s>>>(NG, gpad, npad, b, d_gptr.p, d_gedge.p, d_gsgn.p, T2.p, Sn.p);
    ssolve(pSn.d.p, b);
    k_g_apply<<<nbk(NR, 128), 128, 0, s>>>(NR, npad, gpad, b, d_ecol.p, Sn.p, nullptr, nullptr, T1.p);  // G s
    bd(d_aval.p, T1.p, T3.p, b);                      // A G s
    k_sub<<<nbk(n, 256), 256, 0, s>>>(n, T2.p, T3.p, Yo);
  };
  // U <- U - G (G^T B G)^{-1} G^T B U: the B-orthogonal projection off range(G_j),
  // where the wanted eigenvectors have no component and B^{-1} amplifies rounding
  auto project = [&](double* Uo) {
    if (!deflate) return;
    bd(d_bval.p, Uo, T1.p, b);
    k_gt<<<nbk(NG, 128), 128, 0, s>>>(NG, gpad, npad, b, d_gptr.p, d_gedge.p, d_gsgn.p, T1.p, Sn.p);
    LZ_CUBLAS(cublasDtrsmBatched(cb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT,
                                 gpad, b, &one, pSdB.d.p, gpad, pSn.d.p, gpad, nsub));
    LZ_CUBLAS(cublasDtrsmBatched(cb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT,
                                 gpad, b, &one, pSdB.d.p, gpad, pSn.d.p, gpad, nsub));
    k_g_apply<<<nbk(NR, 128), 128, 0, s>>>(NR, npad, gpad, b, d_ecol.p, Sn.p, Uo, ones.p, Uo);
  };
  auto applyBinv = [&](const double* Yi, double* Uo) {
    for (int c = 0; c < b; ++c) {
      neu.sweep(Yi + (int64_t)c * npad, nullptr, s, nullptr);
      k_pos_scatter<<<nbk(ntot, 256), 256, 0, s>>>(ntot, d_pmap.p, neu.xb.p, Uo + (int64_t)c * npad);
    }
    project(Uo);
  };

  // ------------------------------------------------------------ Lanczos
  DBuf<double> Q, T, H, Cb, Tw, w;
  Q.alloc((size_t)nsub * mmax * npad);
  T.alloc((size_t)nsub * mmax * mmax);
  T.zero(s);
  H.alloc((size_t)nsub * mmax * b);
  Cb.alloc((size_t)nsub * b * b);
  Ptrs pCb, pU;
  pCb.set(Cb.p, (int64_t)b * b, nsub);
  pU.set(U.p, (int64_t)b * npad, nsub);
  DBuf<int> binfo;
  binfo.alloc(nsub);
  const int64_t sQ = (int64_t)mmax * npad, sB = (int64_t)b * npad;
  // B-orthonormalise U in place (U = Qn R, C = U^T B U = R^T R); R left in Cb
  auto borth = [&](const char* where) {
    bd(d_bval.p, U.p, BU.p, b);
    LZ_CUBLAS(cublasDgemmStridedBatched(cb, CUBLAS_OP_T, CUBLAS_OP_N, b, b, npad, &one, U.p, npad, sB, BU.p, npad, sB,
                                        &zero, Cb.p, b, (int64_t)b * b, nsub));
    LZ_CUSOLVER(cusolverDnDpotrfBatched(cs, CUBLAS_FILL_MODE_UPPER, b, pCb.d.p, b, binfo.p, nsub));
    std::vector<int> hi = binfo.download();
    for (int j = 0; j < nsub; ++j)
      MDD_REQUIRE(hi[j] == 0, 5, std::string("block Lanczos breakdown (") + where + ") in subdomain " +
                                     std::to_string(j));
    LZ_CUBLAS(cublasDtrsmBatched(cb, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT,
                                 npad, b, &one, pCb.d.p, b, pU.d.p, npad, nsub));
  };
  auto store_block = [&](int k) {  // U -> basis block k
    CUDA_CHECK(cudaMemcpy2DAsync(Q.p + (int64_t)k * b * npad, sQ * sizeof(double), U.p, sB * sizeof(double),
                                 sB * sizeof(double), nsub, cudaMemcpyDeviceToDevice, s));
  };
  k_lz_random<<<nbk(BLK, 256), 256, 0, s>>>(BLK, npad, b, d_nj.p, U.p);
  project(U.p);
  borth("start");
  store_block(0);

  const double rtol = 1e-10;
  std::vector<int> prev_cnt(nsub, -1), done(nsub, 0), kcnt(nsub, 0);
  std::vector<std::vector<double>> lam(nsub);
  int next_check = std::min(mmax, std::max(16 * b, 128));
  int mfinal = 0;
  DBuf<double> work;
  int lwork_max = 0;
  DBuf<int> einfo;
  einfo.alloc(nsub);
  Tw.alloc((size_t)nsub * mmax * mmax);
  w.alloc((size_t)nsub * mmax);
  for (int k = 0;; ++k) {
    const int m = (k + 1) * b;           // basis size after this step's block k
    const double* Qk = Q.p + (int64_t)k * b * npad;
    // U = B^{-1} L Q_k
    CUDA_CHECK(cudaMemcpy2DAsync(T3.p, sB * sizeof(double), Qk, sQ * sizeof(double), sB * sizeof(double), nsub,
                                 cudaMemcpyDeviceToDevice, s));
    applyL(T3.p, Y.p);
    // A_k = Q_k^T L Q_k (b x b), symmetrised into T(k, k)
    LZ_CUBLAS(cublasDgemmStridedBatched(cb, CUBLAS_OP_T, CUBLAS_OP_N, b, b, npad, &one, Qk, npad, sQ, Y.p, npad, sB,
                                        &zero, Cb.p, b, (int64_t)b * b, nsub));
    k_put_block<<<nbk(nsub * b * b, 128), 128, 0, s>>>(nsub, b, mmax, T.p, k * b, k * b, Cb.p, 0, 0, 1);
    applyBinv(Y.p, U.p);
    if (m >= mmax) {
      mfinal = m;
      break;
    }
    // full B-reorthogonalisation against blocks 0..k, two passes
    for (int pass = 0; pass < 2; ++pass) {
      bd(d_bval.p, U.p, BU.p, b);
      LZ_CUBLAS(cublasDgemmStridedBatched(cb, CUBLAS_OP_T, CUBLAS_OP_N, m, b, npad, &one, Q.p, npad, sQ, BU.p, npad,
                                          sB, &zero, H.p, mmax, (int64_t)mmax * b, nsub));
      LZ_CUBLAS(cublasDgemmStridedBatched(cb, CUBLAS_OP_N, CUBLAS_OP_N, npad, b, m, &mone, Q.p, npad, sQ, H.p, mmax,
                                          (int64_t)mmax * b, &one, U.p, npad, sB, nsub));
    }
    borth("step");
    store_block(k + 1);
    // T(k+1, k) = R (upper triangular), T(k, k+1) = R^T
    k_put_block<<<nbk(nsub * b * b, 128), 128, 0, s>>>(nsub, b, mmax, T.p, (k + 1) * b, k * b, Cb.p, 1, 1, 0);
    if (m < next_check && m + b < mmax) continue;
    next_check = std::min(mmax, std::max(next_check + 2 * b, (next_check * 3) / 2) / b * b);
    // ---- checkpoint: Ritz values and residual bounds ||R s_i(last block)||
    int lw = 0;
    LZ_CUSOLVER(cusolverDnDsyevd_bufferSize(cs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, Tw.p, m, w.p, &lw));
    if (lw > lwork_max) { lwork_max = lw; work.alloc(lw); }
    for (int j = 0; j < nsub; ++j) {
      if (done[j]) continue;
      double* Twj = Tw.p + (int64_t)j * mmax * mmax;
      CUDA_CHECK(cudaMemcpy2DAsync(Twj, m * sizeof(double), T.p + (int64_t)j * mmax * mmax, mmax * sizeof(double),
                                   m * sizeof(double), m, cudaMemcpyDeviceToDevice, s));
      LZ_CUSOLVER(cusolverDnDsyevd(cs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, Twj, m,
                                   w.p + (int64_t)j * mmax, work.p, lw, einfo.p + j));
    }
    std::vector<double> hw((size_t)nsub * mmax), hlast((size_t)nsub * b * m), hR((size_t)nsub * b * b);
    CUDA_CHECK(cudaStreamSynchronize(s));
    CUDA_CHECK(cudaMemcpy(hw.data(), w.p, hw.size() * sizeof(double), cudaMemcpyDeviceToHost));
    CUDA_CHECK(cudaMemcpy(hR.data(), Cb.p, hR.size() * sizeof(double), cudaMemcpyDeviceToHost));
    for (int j = 0; j < nsub; ++j)
      if (!done[j])
        CUDA_CHECK(cudaMemcpy2D(hlast.data() + (size_t)j * b * m, b * sizeof(double),
                                Tw.p + (int64_t)j * mmax * mmax + (m - b), m * sizeof(double), b * sizeof(double), m,
                                cudaMemcpyDeviceToHost));
    {
      std::vector<int> ei = einfo.download();
      for (int j = 0; j < nsub; ++j) MDD_REQUIRE(done[j] || ei[j] == 0, 1, "syevd of the Lanczos matrix failed");
    }
    int ndone = 0;
    for (int j = 0; j < nsub; ++j) {
      if (done[j]) { ++ndone; continue; }
      const double* wj = hw.data() + (size_t)j * mmax;
      const double* R = hR.data() + (size_t)j * b * b;     // upper triangle valid
      const double* last = hlast.data() + (size_t)j * b * m;  // row a of eigenvector i at last[i*b + a]
      const double tmax = std::max(1.0, std::fabs(wj[m - 1]));
      int cnt = 0;
      for (int i = 0; i < m; ++i) cnt += wj[i] > tau;
      bool conv = cnt < m;
      for (int i = m - 1; i >= 0 && conv; --i) {
        double r2 = 0.0;
        for (int a = 0; a < b; ++a) {
          double t = 0.0;
          for (int c = a; c < b; ++c) t += R[c * b + a] * last[(size_t)i * b + c];
          r2 += t * t;
        }
        // Ritz value error <= residual: relative to the eigenvalue itself (the kept
        // ones span many decades on high-contrast recipes), floored at what fp64
        // Lanczos can reach (~eps * theta_max)
        const double lim = std::max(rtol * std::max(std::fabs(wj[i]), tau), 1e-14 * tmax);
        if (std::sqrt(r2) > lim) conv = false;
        if (wj[i] <= tau) break;  // the largest Ritz value below tau was checked too
      }
      if (conv && cnt == prev_cnt[j]) {
        done[j] = 1;
        kcnt[j] = cnt;
        lam[j].assign(wj + (m - cnt), wj + m);
        ++ndone;
      }
      prev_cnt[j] = cnt;
    }
    if (getenv("MDD_LANCZOS_TRACE"))
      fprintf(stderr, "[lanczos] m %d done %d/%d\n", m, ndone, nsub);
    if (ndone == nsub) {
      mfinal = m;
      break;
    }
  }
  MDD_REQUIRE(mfinal > 0, 5, "block Lanczos: no checkpoint");
  for (int j = 0; j < nsub; ++j)
    MDD_REQUIRE(done[j], 5, "block Lanczos did not converge within " + std::to_string(mmax) +
                                " vectors in subdomain " + std::to_string(j) + " (raise MDD_LANCZOS_MMAX)");
  // Subdomains converged at earlier checkpoints: their Tw holds the decomposition at
  // that checkpoint's m, which is no longer known here -- recompute every
  // subdomain's decomposition at mfinal (the basis only grew; Ritz values above
  // tau only move up towards the eigenvalues, so re-take the count there too).
  {
    const int m = mfinal;
    int lw = 0;
    LZ_CUSOLVER(cusolverDnDsyevd_bufferSize(cs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, Tw.p, m, w.p, &lw));
    if (lw > lwork_max) { lwork_max = lw; work.alloc(lw); }
    for (int j = 0; j < nsub; ++j) {
      double* Twj = Tw.p + (int64_t)j * mmax * mmax;
      CUDA_CHECK(cudaMemcpy2DAsync(Twj, m * sizeof(double), T.p + (int64_t)j * mmax * mmax, mmax * sizeof(double),
                                   m * sizeof(double), m, cudaMemcpyDeviceToDevice, s));
      LZ_CUSOLVER(cusolverDnDsyevd(cs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, Twj, m,
                                   w.p + (int64_t)j * mmax, work.p, lw, einfo.p + j));
    }
    std::vector<double> hw((size_t)nsub * mmax);
    CUDA_CHECK(cudaStreamSynchronize(s));
    CUDA_CHECK(cudaMemcpy(hw.data(), w.p, hw.size() * sizeof(double), cudaMemcpyDeviceToHost));
    std::vector<int> ei = einfo.download();
    for (int j = 0; j < nsub; ++j) {
      MDD_REQUIRE(ei[j] == 0, 1, "syevd of the Lanczos matrix failed");
      const double* wj = hw.data() + (size_t)j * mmax;
      int cnt = 0;
      for (int i = 0; i < m; ++i) cnt += wj[i] > tau;
      kcnt[j] = cnt;
      lam[j].assign(wj + (m - cnt), wj + m);
    }
  }
  const int mf = mfinal;
  int kmax = 0;
  for (int j = 0; j < nsub; ++j) kmax = std::max(kmax, kcnt[j]);
  for (int j = 0; j < nsub; ++j) {
    out[j].k = kcnt[j];
    out[j].lambda = lam[j];
  }
  if (kmax == 0) return;
  // ---- Ritz vectors V_j = Q_j S_j(:, m-kmax : m), then W = D (I - xi) V
  T1.release(); T2.release(); T3.release(); Y.release(); U.release(); BU.release(); Sn.release();
  const int64_t BK = (int64_t)nsub * kmax * npad;
  DBuf<double> V, Wk, t1k, snk;
  V.alloc(BK); Wk.alloc(BK); t1k.alloc(BK); snk.alloc((size_t)nsub * kmax * gpad);
  Ptrs psnk;
  psnk.set(snk.p, (int64_t)kmax * gpad, nsub);
  LZ_CUBLAS(cublasDgemmStridedBatched(cb, CUBLAS_OP_N, CUBLAS_OP_N, npad, kmax, mf, &one, Q.p, npad, sQ,
                                      Tw.p + (int64_t)(mf - kmax) * mf, mf, (int64_t)mmax * mmax, &zero, V.p, npad,
                                      (int64_t)kmax * npad, nsub));
  Q.release();
  dproj(V.p, Wk.p, t1k.p, snk.p, psnk.d.p, kmax);
  for (int j = 0; j < nsub; ++j) {
    GeneoBlock& B = out[j];
    if (!B.k) continue;
    B.W.alloc((size_t)nj[j] * B.k);
    CUDA_CHECK(cudaMemcpy2DAsync(B.W.p, nj[j] * sizeof(double),
                                 Wk.p + (int64_t)j * kmax * npad + (int64_t)(kmax - B.k) * npad, npad * sizeof(double),
                                 nj[j] * sizeof(double), B.k, cudaMemcpyDeviceToDevice, s));
  }
  CUDA_CHECK(cudaStreamSynchronize(s));
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace mdd
