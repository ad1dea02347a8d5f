// E = Z^T A Z by blocks (setup phase).  Z = [Z_g | W_1 .. W_N]: the SNK gradient
// columns (Def. 2.3; <= 14 entries each) and the GenEO columns of each
// subdomain (GEVP 3.5; dense on N_i, k_i of them).  A single sparse product
// Z^T (A Z) multiplies through the dense GenEO columns entry by entry (c4: ~1e11
// intermediate products); instead
//   E_gg = Z_g^T (A Z_g)                         sparse x sparse (cuSPARSE, row-chunked)
//   E_gi = (A Z_g)[N_i, :]^T W_i                 one sparse x dense product per subdomain
//   E_ij = W_i[S, :]^T (A_{R_j, N_j} W_j)[S, :]  S = N_i cap R_j, R_j the dofs coupled to N_j:
//                                                a sparse x dense product per subdomain and
//                                                a dense GEMM per neighbouring pair i <= j
// and the blocks are placed into one CSR of E (columns sorted, both triangles;
// E_ji = E_ij^T and E_ig = E_gi^T from the same numbers, so E is exactly symmetric
// off the E_gg block).  Every sum runs in a fixed order (deterministic).
#include <cublas_v2.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <numeric>

#include "coarse_e.h"

namespace mdd {

// ---------------------------------------------------------- cuSPARSE helpers
namespace {

// non-owning view of a device CSR (row-chunk slices of a DevCsr)
struct CsrView {
  int64_t rows = 0, cols = 0, nnz = 0;
  int* ptr = nullptr;
  int* idx = nullptr;
  double* val = nullptr;
};
CsrView view(const DevCsr& A) { return CsrView{A.rows, A.cols, A.nnz, A.ptr.p, A.idx.p, A.val.p}; }

// C = A B with cuSPARSE SpGEMM.  ALG1 (the default) needs workspace that grows
// with the intermediate products and reports INSUFFICIENT_RESOURCES on the large
// coarse products; then ALG2 and finally the chunked ALG3 are used.
void spgemm(cusparseHandle_t H, const CsrView& A, const DevCsr& B, DevCsr& C, cudaStream_t s,
            const char* what) {
  CUSPARSE_CHECK(cusparseSetStream(H, s));
  const cusparseSpGEMMAlg_t algs[3] = {CUSPARSE_SPGEMM_DEFAULT, CUSPARSE_SPGEMM_ALG2,
                                       CUSPARSE_SPGEMM_ALG3};
  std::string errs;
  for (int ai = 0; ai < 3; ++ai) {
    const cusparseSpGEMMAlg_t alg = algs[ai];
    cusparseSpMatDescr_t a, b, c;
    CUSPARSE_CHECK(cusparseCreateCsr(&a, A.rows, A.cols, A.nnz, A.ptr, A.idx, A.val,
                                     CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I, CUSPARSE_INDEX_BASE_ZERO, CUDA_R_64F));
    CUSPARSE_CHECK(cusparseCreateCsr(&b, B.rows, B.cols, B.nnz, B.ptr.p, B.idx.p, B.val.p,
                                     CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I, CUSPARSE_INDEX_BASE_ZERO, CUDA_R_64F));
    C.rows = A.rows; C.cols = B.cols;
    C.ptr.alloc(C.rows + 1);
    CUSPARSE_CHECK(cusparseCreateCsr(&c, C.rows, C.cols, 0, C.ptr.p, nullptr, nullptr,
                                     CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I, CUSPARSE_INDEX_BASE_ZERO, CUDA_R_64F));
    cusparseSpGEMMDescr_t d;
    CUSPARSE_CHECK(cusparseSpGEMM_createDescr(&d));
    double one = 1.0, zero = 0.0;
    auto op = CUSPARSE_OPERATION_NON_TRANSPOSE;
    size_t b1 = 0, b2 = 0, b3 = 0;
    DBuf<char> w1, w2, w3;
    cusparseStatus_t st = cusparseSpGEMM_workEstimation(H, op, op, &one, a, b, &zero, c, CUDA_R_64F,
                                                        alg, d, &b1, nullptr);
    if (st == CUSPARSE_STATUS_SUCCESS) {
      w1.alloc(std::max<size_t>(b1, 1));
      st = cusparseSpGEMM_workEstimation(H, op, op, &one, a, b, &zero, c, CUDA_R_64F, alg, d, &b1, w1.p);
    }
    if (st == CUSPARSE_STATUS_SUCCESS && alg != CUSPARSE_SPGEMM_DEFAULT) {
      // ALG2 / ALG3: the compute buffer size comes from estimateMemory; buffer 1
      // stays alive until the copy
      int64_t nprod = 0;
      st = cusparseSpGEMM_getNumProducts(d, &nprod);
      if (st == CUSPARSE_STATUS_SUCCESS)
        st = cusparseSpGEMM_estimateMemory(H, op, op, &one, a, b, &zero, c, CUDA_R_64F, alg, d, 0.2f,
                                           &b3, nullptr, nullptr);
      if (st == CUSPARSE_STATUS_SUCCESS) {
        w3.alloc(std::max<size_t>(b3, 1));
        st = cusparseSpGEMM_estimateMemory(H, op, op, &one, a, b, &zero, c, CUDA_R_64F, alg, d, 0.2f,
                                           &b3, w3.p, &b2);
        w3.release();
      }
    } else if (st == CUSPARSE_STATUS_SUCCESS) {
      st = cusparseSpGEMM_compute(H, op, op, &one, a, b, &zero, c, CUDA_R_64F, alg, d, &b2, nullptr);
    }
    if (st == CUSPARSE_STATUS_SUCCESS) {
      w2.alloc(std::max<size_t>(b2, 1));
      st = cusparseSpGEMM_compute(H, op, op, &one, a, b, &zero, c, CUDA_R_64F, alg, d, &b2, w2.p);
    }
    int64_t r_ = 0, c_ = 0, nnz = 0;
    if (st == CUSPARSE_STATUS_SUCCESS) st = cusparseSpMatGetSize(c, &r_, &c_, &nnz);
    if (st == CUSPARSE_STATUS_SUCCESS) {
      C.nnz = nnz;
      C.idx.alloc(std::max<int64_t>(nnz, 1));
      C.val.alloc(std::max<int64_t>(nnz, 1));
      st = cusparseCsrSetPointers(c, C.ptr.p, C.idx.p, C.val.p);
    }
    if (st == CUSPARSE_STATUS_SUCCESS)
      st = cusparseSpGEMM_copy(H, op, op, &one, a, b, &zero, c, CUDA_R_64F, alg, d);
    CUDA_CHECK(cudaStreamSynchronize(s));
    cusparseSpGEMM_destroyDescr(d);
    cusparseDestroySpMat(a); cusparseDestroySpMat(b); cusparseDestroySpMat(c);
    if (st == CUSPARSE_STATUS_SUCCESS) return;
    errs += " alg" + std::to_string(ai) + ":status " + std::to_string((int)st);
    if (st != CUSPARSE_STATUS_INSUFFICIENT_RESOURCES && st != CUSPARSE_STATUS_NOT_SUPPORTED) break;
  }
  throw Error(1, std::string("cuSPARSE SpGEMM failed for ") + what + " (" + std::to_string(A.rows) +
                     "x" + std::to_string(A.cols) + " nnz " + std::to_string(A.nnz) + " times " +
                     std::to_string(B.rows) + "x" + std::to_string(B.cols) + " nnz " +
                     std::to_string(B.nnz) + "):" + errs);
}

}  // namespace

// C = A B by row chunks of A.  A chunk holds at most max_prod intermediate
// products (sum over its entries a_ik of nnz(B row k)), which bounds cuSPARSE's
// workspace (the single product of the c2 coarse matrix ran out of it); the
// chunks' CSR pieces are concatenated in row order (same entries, same values
// as the unchunked product: each output row is computed by one call).
void spgemm_rows(cusparseHandle_t H, const DevCsr& A, const DevCsr& B, DevCsr& C, cudaStream_t s,
                 const char* what) {
  // MDD_SPGEMM_MAX_PROD: test knob (forces chunking on small problems)
  const char* mp = getenv("MDD_SPGEMM_MAX_PROD");
  const int64_t max_prod = mp ? atoll(mp) : ((int64_t)48 << 20);
  std::vector<int> ap(A.rows + 1), bp(B.rows + 1), ai(A.nnz);
  CUDA_CHECK(cudaStreamSynchronize(s));
  CUDA_CHECK(cudaMemcpy(ap.data(), A.ptr.p, ap.size() * sizeof(int), cudaMemcpyDeviceToHost));
  CUDA_CHECK(cudaMemcpy(bp.data(), B.ptr.p, bp.size() * sizeof(int), cudaMemcpyDeviceToHost));
  if (A.nnz) CUDA_CHECK(cudaMemcpy(ai.data(), A.idx.p, ai.size() * sizeof(int), cudaMemcpyDeviceToHost));
  std::vector<int64_t> cut{0};
  int64_t acc = 0;
  for (int64_t r = 0; r < A.rows; ++r) {
    int64_t pr = 0;
    for (int k = ap[r]; k < ap[r + 1]; ++k) pr += bp[ai[k] + 1] - bp[ai[k]];
    if (acc + pr > max_prod && r > cut.back()) { cut.push_back(r); acc = 0; }
    acc += pr;
  }
  cut.push_back(A.rows);
  if (cut.size() == 2) {
    spgemm(H, view(A), B, C, s, what);
    return;
  }
  std::vector<DevCsr> parts(cut.size() - 1);
  std::vector<int64_t> pnnz(parts.size());
  int64_t tot = 0;
  for (size_t c = 0; c + 1 < cut.size(); ++c) {
    const int64_t r0 = cut[c], r1 = cut[c + 1];
    std::vector<int> rp(r1 - r0 + 1);
    for (int64_t r = r0; r <= r1; ++r) rp[r - r0] = ap[r] - ap[r0];
    DBuf<int> dptr;
    dptr.upload(rp);
    CsrView Ac{r1 - r0, A.cols, (int64_t)(ap[r1] - ap[r0]), dptr.p, A.idx.p + ap[r0], A.val.p + ap[r0]};
    spgemm(H, Ac, B, parts[c], s, what);
    pnnz[c] = parts[c].nnz;
    tot += parts[c].nnz;
  }
  MDD_REQUIRE(tot < INT32_MAX, 5, std::string(what) + ": product too large for 32-bit CSR offsets");
  C.rows = A.rows; C.cols = B.cols; C.nnz = tot;
  std::vector<int> cp(A.rows + 1, 0);
  int64_t off = 0;
  for (size_t c = 0; c < parts.size(); ++c) {
    std::vector<int> pp(parts[c].rows + 1);
    CUDA_CHECK(cudaMemcpy(pp.data(), parts[c].ptr.p, pp.size() * sizeof(int), cudaMemcpyDeviceToHost));
    for (int64_t r = 0; r < parts[c].rows; ++r) cp[cut[c] + r + 1] = (int)(off + pp[r + 1]);
    off += pnnz[c];
  }
  C.ptr.upload(cp);
  C.idx.alloc(std::max<int64_t>(tot, 1));
  C.val.alloc(std::max<int64_t>(tot, 1));
  off = 0;
  for (size_t c = 0; c < parts.size(); ++c) {
    if (pnnz[c]) {
      CUDA_CHECK(cudaMemcpyAsync(C.idx.p + off, parts[c].idx.p, pnnz[c] * sizeof(int), cudaMemcpyDeviceToDevice, s));
      CUDA_CHECK(cudaMemcpyAsync(C.val.p + off, parts[c].val.p, pnnz[c] * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    off += pnnz[c];
    CUDA_CHECK(cudaStreamSynchronize(s));
    parts[c] = DevCsr();
  }
}

void transpose(cusparseHandle_t H, const DevCsr& A, DevCsr& T, cudaStream_t s) {
  CUSPARSE_CHECK(cusparseSetStream(H, s));
  T.rows = A.cols; T.cols = A.rows; T.nnz = A.nnz;
  T.ptr.alloc(T.rows + 1);
  T.idx.alloc(std::max<int64_t>(A.nnz, 1));
  T.val.alloc(std::max<int64_t>(A.nnz, 1));
  size_t bs = 0;
  CUSPARSE_CHECK(cusparseCsr2cscEx2_bufferSize(H, A.rows, A.cols, A.nnz, A.val.p, A.ptr.p, A.idx.p,
                                               T.val.p, T.ptr.p, T.idx.p, CUDA_R_64F,
                                               CUSPARSE_ACTION_NUMERIC, CUSPARSE_INDEX_BASE_ZERO,
                                               CUSPARSE_CSR2CSC_ALG1, &bs));
  DBuf<char> w; w.alloc(std::max<size_t>(bs, 1));
  CUSPARSE_CHECK(cusparseCsr2cscEx2(H, A.rows, A.cols, A.nnz, A.val.p, A.ptr.p, A.idx.p, T.val.p,
                                    T.ptr.p, T.idx.p, CUDA_R_64F, CUSPARSE_ACTION_NUMERIC,
                                    CUSPARSE_INDEX_BASE_ZERO, CUSPARSE_CSR2CSC_ALG1, w.p));
  CUDA_CHECK(cudaStreamSynchronize(s));
}

// CSR (int32 pointers) download + sort each row; returns pattern and value slot
void download_sorted(const DevCsr& C, Csr& pat, std::vector<int64_t>& slot) {
  std::vector<int> ptr(C.rows + 1), idx(C.nnz);
  CUDA_CHECK(cudaMemcpy(ptr.data(), C.ptr.p, ptr.size() * sizeof(int), cudaMemcpyDeviceToHost));
  if (C.nnz) CUDA_CHECK(cudaMemcpy(idx.data(), C.idx.p, idx.size() * sizeof(int), cudaMemcpyDeviceToHost));
  pat.nrows = (int)C.rows; pat.ncols = (int)C.cols;
  pat.ptr.assign(C.rows + 1, 0);
  pat.idx.resize(C.nnz);
  slot.resize(C.nnz);
  for (int64_t r = 0; r < C.rows; ++r) {
    std::vector<std::pair<int, int64_t>> row;
    for (int64_t k = ptr[r]; k < ptr[r + 1]; ++k) row.push_back({idx[k], k});
    std::sort(row.begin(), row.end());
    for (size_t j = 0; j < row.size(); ++j) {
      pat.idx[ptr[r] + j] = row[j].first;
      slot[ptr[r] + j] = row[j].second;
    }
    pat.ptr[r + 1] = ptr[r + 1];
  }
}

namespace {

#define CE_CUBLAS(x)                                                                           \
  do {                                                                                         \
    cublasStatus_t s__ = (x);                                                                  \
    if (s__ != CUBLAS_STATUS_SUCCESS)                                                          \
      throw Error(1, std::string(#x) + ": cublas status " + std::to_string((int)s__));         \
  } while (0)

// C (m x k, col-major, ld m) = M (CSR m x n) B (n x k, col-major, ld ldb); values of M
// gathered through slot from vsrc; one thread per row, columns in order
__global__ void k_csr_dense(int m, int k, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                            const int64_t* __restrict__ slot, const double* __restrict__ vsrc,
                            const double* __restrict__ B, int64_t ldb, double* __restrict__ C) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  for (int c = 0; c < k; ++c) {
    double s = 0.0;
    for (int64_t p = ptr[r]; p < ptr[r + 1]; ++p) s += vsrc[slot[p]] * B[(int64_t)c * ldb + idx[p]];
    C[(int64_t)c * m + r] = s;
  }
}
// D (n x k, ld n) = rows idx of S (ld lds)
__global__ void k_gather_rows(int n, int k, const int32_t* __restrict__ idx, const double* __restrict__ S,
                              int64_t lds, double* __restrict__ D) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (int64_t)n * k) return;
  const int c = (int)(q / n), r = (int)(q % n);
  D[q] = S[(int64_t)c * lds + idx[r]];
}

inline int nb_(int64_t n, int t) { return (int)std::max<int64_t>(1, (n + t - 1) / t); }

}  // namespace

void coarse_E_blocks(cusparseHandle_t sp, const DevCsr& Ad, const Csr& Apat, const DevCsr& Zg, const DevCsr& Zgt,
                     const std::vector<std::vector<int32_t>>& sub_dofs, const std::vector<GeneoBlock>& geneo,
                     const std::vector<int32_t>& sub_nbr_ptr, const std::vector<int32_t>& sub_nbr,
                     cudaStream_t s, DevCsr& E) {
  const int nsub = (int)sub_dofs.size();
  const int64_t n = Ad.rows, ng = Zg.cols;
  // ---- E_gg and A Z_g
  DevCsr AZg, Egg;
  spgemm_rows(sp, Ad, Zg, AZg, s, "A Z_g");
  spgemm_rows(sp, Zgt, AZg, Egg, s, "Z_g^T (A Z_g)");
  Csr gpat;
  std::vector<int64_t> gslot;
  download_sorted(Egg, gpat, gslot);
  std::vector<int> azp(n + 1), azi(AZg.nnz);
  CUDA_CHECK(cudaMemcpy(azp.data(), AZg.ptr.p, (n + 1) * sizeof(int), cudaMemcpyDeviceToHost));
  if (AZg.nnz) CUDA_CHECK(cudaMemcpy(azi.data(), AZg.idx.p, AZg.nnz * sizeof(int), cudaMemcpyDeviceToHost));
  // ---- GenEO numbering and the value pool [E_gg | E_gi blocks | E_ij blocks]
  std::vector<int64_t> gc0(nsub + 1, ng);
  for (int i = 0; i < nsub; ++i) gc0[i + 1] = gc0[i] + geneo[i].k;
  const int64_t n0 = gc0[nsub];
  struct GBlk { std::vector<int32_t> cols; int64_t off; };      // E_gi: grad columns touching N_i
  std::vector<GBlk> gb(nsub);
  struct PBlk { int i, j; int64_t off; };                          // E_ij, i <= j
  std::vector<PBlk> pb;
  int64_t pool = Egg.nnz;
  std::vector<int32_t> gmark(ng, -1), dmark(n, -1);
  cublasHandle_t cb;
  CE_CUBLAS(cublasCreate(&cb));
  struct G_ { cublasHandle_t h; ~G_() { cublasDestroy(h); } } guard_{cb};
  CE_CUBLAS(cublasSetStream(cb, s));
  // sizes first (pool layout), then the device work
  for (int i = 0; i < nsub; ++i) {
    if (!geneo[i].k) continue;
    std::vector<int32_t>& cols = gb[i].cols;
    for (int32_t e : sub_dofs[i])
      for (int p = azp[e]; p < azp[e + 1]; ++p)
        if (gmark[azi[p]] != i) { gmark[azi[p]] = i; cols.push_back(azi[p]); }
    std::sort(cols.begin(), cols.end());
    gb[i].off = pool;
    pool += (int64_t)cols.size() * geneo[i].k;
  }
  for (int j = 0; j < nsub; ++j) {
    if (!geneo[j].k) continue;
    for (int q = sub_nbr_ptr[j]; q < sub_nbr_ptr[j + 1]; ++q) {
      const int i = sub_nbr[q];
      if (i > j || !geneo[i].k) continue;
      pb.push_back(PBlk{i, j, pool});
      pool += (int64_t)geneo[i].k * geneo[j].k;
    }
  }
  DBuf<double> P;
  P.alloc(std::max<int64_t>(pool, 1));
  CUDA_CHECK(cudaMemcpyAsync(P.p, Egg.val.p, Egg.nnz * sizeof(double), cudaMemcpyDeviceToDevice, s));
  std::vector<int32_t> cmap(ng, -1);
  // ---- E_gi = (A Z_g)[N_i, cols]^T W_i : rows of the transposed slice, cols local in N_i
  for (int i = 0; i < nsub; ++i) {
    if (!geneo[i].k) continue;
    const auto& D = sub_dofs[i];
    const auto& cols = gb[i].cols;
    for (size_t c = 0; c < cols.size(); ++c) cmap[cols[c]] = (int32_t)c;
    std::vector<int64_t> tp(cols.size() + 1, 0), tslot;
    std::vector<int32_t> ti;
    for (size_t l = 0; l < D.size(); ++l)
      for (int p = azp[D[l]]; p < azp[D[l] + 1]; ++p) tp[cmap[azi[p]] + 1]++;
    for (size_t c = 0; c < cols.size(); ++c) tp[c + 1] += tp[c];
    ti.resize(tp.back());
    tslot.resize(tp.back());
    std::vector<int64_t> cur(tp.begin(), tp.end() - 1);
    for (size_t l = 0; l < D.size(); ++l)
      for (int p = azp[D[l]]; p < azp[D[l] + 1]; ++p) {
        const int64_t d = cur[cmap[azi[p]]]++;
        ti[d] = (int32_t)l;
        tslot[d] = p;
      }
    for (int32_t c : cols) cmap[c] = -1;
    DBuf<int64_t> dp, ds;
    DBuf<int32_t> di;
    dp.upload(tp); di.upload(ti); ds.upload(tslot);
    k_csr_dense<<<nb_((int64_t)cols.size(), 128), 128, 0, s>>>((int)cols.size(), geneo[i].k, dp.p, di.p, ds.p,
                                                              AZg.val.p, geneo[i].W.p, (int64_t)D.size(),
                                                              P.p + gb[i].off);
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  AZg = DevCsr();
  // ---- E_ij: Y_j = A_{R_j, N_j} W_j, then W_i[S]^T Y_j[S] for the neighbours i <= j
  size_t next_pb = 0;
  for (int j = 0; j < nsub; ++j) {
    if (!geneo[j].k) continue;
    const auto& Dj = sub_dofs[j];
    const int kj = geneo[j].k;
    std::vector<int32_t> R;
    for (int32_t e : Dj)
      for (int64_t p = Apat.ptr[e]; p < Apat.ptr[e + 1]; ++p)
        if (dmark[Apat.idx[p]] != j) { dmark[Apat.idx[p]] = j; R.push_back(Apat.idx[p]); }
    std::sort(R.begin(), R.end());
    for (size_t r = 0; r < R.size(); ++r) dmark[R[r]] = -2 - (int32_t)r;
    // A_{R, N_j}: rows R, columns local in N_j (A symmetric: from A's rows N_j)
    std::vector<int64_t> rp(R.size() + 1, 0), rslot;
    std::vector<int32_t> ri;
    for (size_t l = 0; l < Dj.size(); ++l)
      for (int64_t p = Apat.ptr[Dj[l]]; p < Apat.ptr[Dj[l] + 1]; ++p) rp[-2 - dmark[Apat.idx[p]] + 1]++;
    for (size_t r = 0; r < R.size(); ++r) rp[r + 1] += rp[r];
    ri.resize(rp.back());
    rslot.resize(rp.back());
    {
      std::vector<int64_t> cur(rp.begin(), rp.end() - 1);
      for (size_t l = 0; l < Dj.size(); ++l)
        for (int64_t p = Apat.ptr[Dj[l]]; p < Apat.ptr[Dj[l] + 1]; ++p) {
          const int64_t d = cur[-2 - dmark[Apat.idx[p]]]++;
          ri[d] = (int32_t)l;
          rslot[d] = p;   // A symmetric: the value of (row, l) is A[Dj[l], row]
        }
    }
    DBuf<int64_t> dp, ds;
    DBuf<int32_t> di;
    dp.upload(rp); di.upload(ri); ds.upload(rslot);
    DBuf<double> Y;
    Y.alloc((size_t)R.size() * kj);
    k_csr_dense<<<nb_((int64_t)R.size(), 128), 128, 0, s>>>((int)R.size(), kj, dp.p, di.p, ds.p, Ad.val.p,
                                                           geneo[j].W.p, (int64_t)Dj.size(), Y.p);
    for (; next_pb < pb.size() && pb[next_pb].j == j; ++next_pb) {
      const PBlk& B = pb[next_pb];
      const int i = B.i, ki = geneo[i].k;
      std::vector<int32_t> si, sr;   // rows of S: local index in N_i, row of R
      const auto& Di = sub_dofs[i];
      for (size_t l = 0; l < Di.size(); ++l)
        if (dmark[Di[l]] <= -2) { si.push_back((int32_t)l); sr.push_back(-2 - dmark[Di[l]]); }
      if (si.empty()) {
        CUDA_CHECK(cudaMemsetAsync(P.p + B.off, 0, (size_t)ki * kj * sizeof(double), s));
        continue;
      }
      const int ns = (int)si.size();
      DBuf<int32_t> dsi, dsr;
      dsi.upload(si); dsr.upload(sr);
      DBuf<double> WS, YS;
      WS.alloc((size_t)ns * ki); YS.alloc((size_t)ns * kj);
      k_gather_rows<<<nb_((int64_t)ns * ki, 256), 256, 0, s>>>(ns, ki, dsi.p, geneo[i].W.p, (int64_t)Di.size(), WS.p);
      k_gather_rows<<<nb_((int64_t)ns * kj, 256), 256, 0, s>>>(ns, kj, dsr.p, Y.p, (int64_t)R.size(), YS.p);
      const double one = 1.0, zero = 0.0;
      CE_CUBLAS(cublasDgemm(cb, CUBLAS_OP_T, CUBLAS_OP_N, ki, kj, ns, &one, WS.p, ns, YS.p, ns, &zero, P.p + B.off,
                            ki));
      CUDA_CHECK(cudaStreamSynchronize(s));
    }
    for (int32_t e : R) dmark[e] = -1;
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  // ---- the CSR of E (sorted columns, both triangles) and its value slots into the pool
  std::vector<std::vector<std::pair<int32_t, int32_t>>> gin(ng);   // grad column -> (subdomain, row in E_gi)
  for (int i = 0; i < nsub; ++i)
    for (size_t c = 0; c < gb[i].cols.size(); ++c) gin[gb[i].cols[c]].push_back({i, (int32_t)c});
  std::vector<int64_t> pbi(nsub * (int64_t)nsub, -1);   // pool offset of block (i, j), i <= j
  for (const PBlk& B : pb) pbi[(int64_t)B.i * nsub + B.j] = B.off;
  std::vector<int> ep(n0 + 1, 0);
  std::vector<int32_t> ei;
  std::vector<int64_t> es;
  for (int64_t a = 0; a < ng; ++a) {
    for (int64_t p = gpat.ptr[a]; p < gpat.ptr[a + 1]; ++p) { ei.push_back(gpat.idx[p]); es.push_back(gslot[p]); }
    for (auto& pr : gin[a]) {
      const int i = pr.first;
      const int64_t m = (int64_t)gb[i].cols.size();
      for (int q = 0; q < geneo[i].k; ++q) {
        ei.push_back((int32_t)(gc0[i] + q));
        es.push_back(gb[i].off + (int64_t)q * m + pr.second);
      }
    }
    MDD_REQUIRE(ei.size() < (size_t)INT32_MAX, 5, "coarse matrix too large for 32-bit CSR offsets");
    ep[a + 1] = (int)ei.size();
  }
  for (int i = 0; i < nsub; ++i) {
    const int ki = geneo[i].k;
    const int64_t m = (int64_t)gb[i].cols.size();
    for (int q = 0; q < ki; ++q) {
      for (int64_t c = 0; c < m; ++c) { ei.push_back(gb[i].cols[c]); es.push_back(gb[i].off + (int64_t)q * m + c); }
      for (int j = 0; j < nsub; ++j) {
        const int kj = geneo[j].k;
        if (!kj) continue;
        if (i <= j) {
          const int64_t off = pbi[(int64_t)i * nsub + j];
          if (off < 0) continue;
          for (int t = 0; t < kj; ++t) { ei.push_back((int32_t)(gc0[j] + t)); es.push_back(off + (int64_t)t * ki + q); }
        } else {
          const int64_t off = pbi[(int64_t)j * nsub + i];
          if (off < 0) continue;
          for (int t = 0; t < kj; ++t) { ei.push_back((int32_t)(gc0[j] + t)); es.push_back(off + (int64_t)q * kj + t); }
        }
      }
      MDD_REQUIRE(ei.size() < (size_t)INT32_MAX, 5, "coarse matrix too large for 32-bit CSR offsets");
      ep[gc0[i] + q + 1] = (int)ei.size();
    }
  }
  E.rows = E.cols = n0;
  E.nnz = (int64_t)ei.size();
  E.ptr.upload(ep);
  E.idx.upload(ei);
  E.val.alloc(std::max<int64_t>(E.nnz, 1));
  DBuf<int64_t> dslot;
  dslot.upload(es);
  dev::k_gather<<<nb_(E.nnz, 256), 256, 0, s>>>(E.nnz, dslot.p, P.p, E.val.p);
  CUDA_CHECK(cudaStreamSynchronize(s));
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace mdd
