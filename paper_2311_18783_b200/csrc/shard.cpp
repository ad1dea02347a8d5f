// Sharded solve: the ownership and halo plan (host, integer work).
//
// north_star: "Subdomains are sharded across the GPUs of one 8xB200 box, with
// overlap-halo exchange and the coarse-space and dot-product allreduces".  Each
// rank owns a slab of subdomains and the dofs whose midpoint lies in their owned
// boxes; it keeps its owned dofs plus a halo (the rest of its subdomains' N_i and
// of its SpMV columns).  PCG vectors are distributed by owned dof; the forward
// halo exchange fills a rank's halo from the owners, the reverse one adds a
// rank's halo contributions (the prolongation sum_i R_i^T x_i of eq. 2.3 over
// subdomains of several ranks) into the owners.
#include "shard.h"

#include <algorithm>

namespace mdd {

void build_shard_plan(const HostMesh& m, const Decomp& dec, const Csr& Apat, int px, int py, int pz,
                      int rank, int nranks, ShardPlan& sp) {
  MDD_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, 2, "bad rank / nranks");
  MDD_REQUIRE(px >= nranks, 2, "a sharded solve needs at least one subdomain slab per rank (px >= nranks)");
  sp = ShardPlan();
  sp.rank = rank;
  sp.nranks = nranks;
  const int nsub = dec.nsub, n = m.n();
  sp.sub_rank.resize(nsub);
  for (int s = 0; s < nsub; ++s) sp.sub_rank[s] = (int)(((int64_t)(s % px) * nranks) / px);
  // dof owner: the owned box containing the edge midpoint
  const int sx = m.nx / px, sy = m.ny / py, sz = m.nz / pz;
  sp.dof_owner.resize(n);
  for (int e = 0; e < n; ++e) {
    const int ee = m.free_edge[e];
    int a[3], b[3];
    m.node_ijk(m.edge_tail[ee], a[0], a[1], a[2]);
    m.node_ijk(m.edge_head[ee], b[0], b[1], b[2]);
    // cube index of the midpoint along each axis: floor((a + b) / 2), the last box closed
    int c[3];
    const int nn[3] = {m.nx, m.ny, m.nz};
    for (int d = 0; d < 3; ++d) c[d] = std::min((a[d] + b[d]) / 2, nn[d] - 1);
    const int si = c[0] / sx, sj = c[1] / sy, sk = c[2] / sz;
    sp.dof_owner[e] = sp.sub_rank[si + px * (sj + py * sk)];
  }
  // every rank's needed set (own subdomains' N_i + columns of owned rows)
  std::vector<std::vector<int32_t>> halo_of(nranks);
  std::vector<std::vector<int32_t>> owned_of(nranks);
  for (int e = 0; e < n; ++e) owned_of[sp.dof_owner[e]].push_back(e);
  {
    std::vector<int32_t> mark(n, -1);
    for (int q = 0; q < nranks; ++q) {
      std::vector<int32_t>& h = halo_of[q];
      auto need = [&](int32_t e) {
        if (sp.dof_owner[e] != q && mark[e] != q) { mark[e] = q; h.push_back(e); }
      };
      for (int s = 0; s < nsub; ++s)
        if (sp.sub_rank[s] == q)
          for (int32_t e : dec.sub_dofs[s]) need(e);
      for (int32_t e : owned_of[q])
        for (int64_t p = Apat.ptr[e]; p < Apat.ptr[e + 1]; ++p) need(Apat.idx[p]);
      std::sort(h.begin(), h.end());
    }
  }
  for (int s = 0; s < nsub; ++s)
    if (sp.sub_rank[s] == rank) sp.subs.push_back(s);
  sp.owned = owned_of[rank];
  sp.halo = halo_of[rank];
  std::vector<int32_t> g2l(n, -1);
  for (int k = 0; k < sp.n_own(); ++k) g2l[sp.owned[k]] = k;
  for (size_t k = 0; k < sp.halo.size(); ++k) g2l[sp.halo[k]] = sp.n_own() + (int)k;
  sp.send_ptr.assign(nranks + 1, 0);
  sp.recv_ptr.assign(nranks + 1, 0);
  for (int q = 0; q < nranks; ++q) {
    if (q != rank) {
      for (int32_t e : halo_of[q])          // q's halo in q's order: the ones this rank owns
        if (sp.dof_owner[e] == rank) sp.send_idx.push_back(g2l[e]);
      for (int32_t e : sp.halo)
        if (sp.dof_owner[e] == q) sp.recv_idx.push_back(g2l[e]);
    }
    sp.send_ptr[q + 1] = (int64_t)sp.send_idx.size();
    sp.recv_ptr[q + 1] = (int64_t)sp.recv_idx.size();
  }
}

}  // namespace mdd
