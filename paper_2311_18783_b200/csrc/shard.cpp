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

namespace mdd {

// Subtree-to-rank mapping of the coarse factor's supernode tree:
// grow a replicated top from the roots, splitting the costliest frontier subtree,
// and deal the frontier subtrees to the ranks largest first (LPT); keep the
// configuration with the smallest per-rank work max_bin + top.  Integer work,
// deterministic on every rank.
void split_tree(int nsn, const int32_t* parent, const int64_t* cost, int nranks, std::vector<int32_t>& owner) {
  MDD_REQUIRE(nranks >= 1, 2, "nranks must be >= 1");
  owner.assign(nsn, 0);
  if (nranks == 1 || nsn == 0) return;
  std::vector<std::vector<int32_t>> ch(nsn);
  std::vector<int32_t> roots;
  for (int g = 0; g < nsn; ++g) {
    MDD_REQUIRE(parent[g] < nsn && parent[g] != g, 2, "split_tree: bad parent");
    if (parent[g] < 0) roots.push_back(g); else ch[parent[g]].push_back(g);
  }
  {
    std::vector<int32_t> order(roots);
    for (size_t k = 0; k < order.size() && order.size() <= (size_t)nsn; ++k)
      for (int32_t c : ch[order[k]]) order.push_back(c);
    MDD_REQUIRE((int)order.size() == nsn, 2, "split_tree: parent array is not a forest");
  }
  // subtree costs, children before parents (iterative postorder)
  std::vector<int64_t> sc(nsn, 0);
  {
    std::vector<std::pair<int32_t, size_t>> st;
    for (int32_t r : roots) {
      st.push_back({r, 0});
      while (!st.empty()) {
        auto& [g, k] = st.back();
        if (k < ch[g].size()) {
          const int32_t c = ch[g][k++];
          st.push_back({c, 0});
        } else {
          sc[g] += cost[g];
          if (parent[g] >= 0) sc[parent[g]] += sc[g];
          st.pop_back();
        }
      }
    }
  }
  auto by_cost = [&](int32_t a, int32_t b) { return sc[a] != sc[b] ? sc[a] > sc[b] : a < b; };
  auto deal = [&](std::vector<int32_t> fr, std::vector<int32_t>& rk, int64_t& maxbin) {
    std::sort(fr.begin(), fr.end(), by_cost);
    std::vector<int64_t> bin(nranks, 0);
    rk.assign(nsn, -1);
    for (int32_t g : fr) {
      const int b = (int)(std::min_element(bin.begin(), bin.end()) - bin.begin());
      bin[b] += sc[g];
      rk[g] = b;
    }
    maxbin = *std::max_element(bin.begin(), bin.end());
  };
  std::vector<int32_t> frontier(roots), top;
  std::vector<char> is_top(nsn, 0), best_top;
  std::vector<int32_t> rk, best_rk;
  int64_t topcost = 0, best = INT64_MAX;
  for (int it = 0; it <= 8 * nranks + 64; ++it) {
    int64_t mb = 0;
    deal(frontier, rk, mb);
    if ((int)frontier.size() >= nranks && mb + topcost < best) {
      best = mb + topcost;
      best_rk = rk;
      best_top = is_top;
    }
    // split the costliest frontier subtree that has children
    int32_t s = -1;
    for (int32_t g : frontier)
      if (!ch[g].empty() && (s < 0 || by_cost(g, s))) s = g;
    if (s < 0) break;
    frontier.erase(std::find(frontier.begin(), frontier.end(), s));
    frontier.insert(frontier.end(), ch[s].begin(), ch[s].end());
    is_top[s] = 1;
    topcost += cost[s];
  }
  MDD_REQUIRE(!best_rk.empty(), 2, "split_tree: fewer leaf subtrees than ranks");
  // top supernodes -> -1; every other supernode -> the rank of its frontier ancestor
  std::vector<int32_t> order;  // parents before children
  for (int32_t r : roots) order.push_back(r);
  for (size_t k = 0; k < order.size(); ++k)
    for (int32_t c : ch[order[k]]) order.push_back(c);
  MDD_REQUIRE((int)order.size() == nsn, 2, "split_tree: parent array is not a forest");
  for (int32_t g : order) {
    if (best_top[g]) owner[g] = -1;
    else if (best_rk[g] >= 0) owner[g] = best_rk[g];
    else owner[g] = owner[parent[g]];
  }
}

}  // namespace mdd
