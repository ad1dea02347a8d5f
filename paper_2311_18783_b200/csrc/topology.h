// Host integer work of the setup (see topology.cpp).
#pragma once
#include "common.h"

namespace mdd {

struct Decomp {
  int nsub = 0;
  std::vector<std::vector<int32_t>> sub_tets;  // indices into the present-tet arrays
  std::vector<std::vector<int32_t>> sub_dofs;  // N_i, increasing
  std::vector<int32_t> mult;                   // #{i : e in N_i}
};

void build_A_pattern(const HostMesh& m, Csr& A, std::vector<i64>& slot_ptr,
                     std::vector<int32_t>& contrib);
void build_subdomains(const HostMesh& m, int px, int py, int pz, int overlap, Decomp& d);
// local pattern of A restricted to `dofs`; slot[k] = global A slot of local entry k.
// g2l must be an n-array of -1 (restored on exit).
void local_pattern(const Csr& A, const std::vector<int32_t>& dofs, std::vector<int32_t>& g2l,
                   Csr& loc, std::vector<i64>& slot);
void edge_xyz2(const HostMesh& m, int e_free, int32_t* out);
void gradient_nodes(const HostMesh& m, const std::vector<int32_t>& dofs, std::vector<int32_t>& cols);

}  // namespace mdd
