// Device sparse-matrix helpers of the setup phase (cuSPARSE products,
// transposes, downloads) and the block-wise assembly of the coarse matrix E.
#pragma once
#include <cusparse.h>

#include "device.h"
#include "geneo.h"

namespace mdd {

struct DevCsr {
  int64_t rows = 0, cols = 0, nnz = 0;
  DBuf<int> ptr, idx;
  DBuf<double> val;
};

// C = A B (cuSPARSE SpGEMM) by row chunks of A with bounded intermediate products
void spgemm_rows(cusparseHandle_t H, const DevCsr& A, const DevCsr& B, DevCsr& C, cudaStream_t s, const char* what);
// T = A^T (cuSPARSE csr2csc)
void transpose(cusparseHandle_t H, const DevCsr& A, DevCsr& T, cudaStream_t s);
// CSR (int32 pointers) download + sort each row; returns pattern and value slot
void download_sorted(const DevCsr& C, Csr& pat, std::vector<int64_t>& slot);

// E = Z^T A Z for Z = [Z_g | GenEO blocks] by blocks (coarse_e.cu).  Ad: A (n x n);
// Zg / Zgt: the gradient columns and their transpose; sub_nbr: per subdomain the
// subdomains whose N_j can couple to its N_i through A (itself included).
// E: n0 x n0 CSR, columns sorted, both triangles.
void coarse_E_blocks(cusparseHandle_t sp, const DevCsr& Ad, const Csr& Apat, const DevCsr& Zg, const DevCsr& Zgt,
                     const std::vector<std::vector<int32_t>>& sub_dofs, const std::vector<GeneoBlock>& geneo,
                     const std::vector<int32_t>& sub_nbr_ptr, const std::vector<int32_t>& sub_nbr,
                     cudaStream_t s, DevCsr& E);

}  // namespace mdd
