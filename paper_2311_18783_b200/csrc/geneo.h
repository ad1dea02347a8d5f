// GenEO enrichment on the device (PAPER.md GEVP 3.5, eq. 3.1).
#pragma once
#include "../../include/maxwell_dd.h"
#include "device.h"
#include "topology.h"

namespace mdd {

struct GeneoBlock {
  int k = 0;                      // eigenpairs kept (lambda > tau)
  std::vector<double> lambda;     // kept eigenvalues, ascending
  DBuf<double> W;                 // n_i x k, column-major: D_i (I - xi_0i) V (local coordinates)
};

struct GeneoInputs {
  const HostMesh* mesh;
  const Decomp* dec;
  const std::vector<Csr>* lpat;                 // local patterns of A_i (local indices)
  const std::vector<std::vector<int64_t>>* lslot;  // their global A slots
  const double* A_val;                          // device, global A values
  const double* Ke;                             // device, element curl-curl matrices (36 per tet)
  const double* Me;                             // device, element mass matrices
  double gamma;
  const std::vector<std::vector<int32_t>>* grad_nodes;  // G_i columns (free-node indices)
  const std::vector<std::vector<int32_t>>* lxyz = nullptr;  // doubled edge-midpoint coordinates (N_i order)
};

// dense GEVP per subdomain (cuSOLVER sygvdx): subdomains up to a few thousand dofs
void geneo_all(const GeneoInputs& in, double tau, std::vector<GeneoBlock>& out, cudaStream_t s);
// the same GEVP for all subdomains at once by block Lanczos (geneo_lanczos.cu)
void geneo_lanczos(const GeneoInputs& in, double tau, std::vector<GeneoBlock>& out, cudaStream_t s);

// per local slot of A_j's pattern, the element contributions (tet*36 + a*6 + b) of
// the tets of Omega_j in fixed order: A_j^Neu[slot] = sum K_e + gamma M_e (g2l:
// scratch of n entries, all -1 on entry and exit)
void neumann_slots(const HostMesh& m, const Decomp& dec, const Csr& lp, int j, std::vector<int32_t>& g2l,
                   std::vector<int64_t>& cnt, std::vector<int32_t>& ctb);
// entries (local row, column, +-1) of G_j = R_j C[:, grad nodes] (colof: scratch
// over free nodes, all -1 on entry and exit)
void gradient_entries(const HostMesh& m, const std::vector<int32_t>& D, const std::vector<int32_t>& gn,
                      std::vector<int32_t>& colof, std::vector<int32_t>& row, std::vector<int32_t>& col,
                      std::vector<double>& val);

}  // namespace mdd
