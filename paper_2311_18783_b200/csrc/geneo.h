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
};

void geneo_all(const GeneoInputs& in, double tau, std::vector<GeneoBlock>& out, cudaStream_t s);

}  // namespace mdd
