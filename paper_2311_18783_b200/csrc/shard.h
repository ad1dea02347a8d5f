// Partition of the subdomains, dofs and halos over the ranks of a sharded solve
// (host, integer work).  See shard.cpp.
#pragma once
#include "common.h"
#include "topology.h"

namespace mdd {

struct ShardPlan {
  int rank = 0, nranks = 1;
  std::vector<int32_t> sub_rank;   // per subdomain: its rank
  std::vector<int32_t> dof_owner;  // per global dof: the owning rank
  std::vector<int32_t> subs;       // this rank's subdomains (ascending)
  std::vector<int32_t> owned;      // global dofs owned by this rank (ascending): local 0 .. n_own-1
  std::vector<int32_t> halo;       // other ranks' dofs this rank reads (ascending): local n_own ..
  // exchange lists per peer q (local indices): send_idx[send_ptr[q] .. send_ptr[q+1])
  // are owned dofs in q's halo (in q's halo order), recv_idx the halo dofs owned by q
  std::vector<int64_t> send_ptr, recv_ptr;
  std::vector<int32_t> send_idx, recv_idx;
  int n_own() const { return (int)owned.size(); }
  int n_local() const { return (int)(owned.size() + halo.size()); }
};

// Subdomain s = (si, sj, sk) goes to rank floor(si * nranks / px) (slabs along x,
// the weak-scaling axis of BASELINE config 4).  Dof e is owned by the rank of the
// subdomain whose owned cube box contains the edge's midpoint (half-open boxes,
// the last box closed).  The halo of a rank = the dofs of its subdomains' N_i and
// of the columns of its owned rows of A that it does not own.
void build_shard_plan(const HostMesh& m, const Decomp& dec, const Csr& Apat, int px, int py, int pz,
                      int rank, int nranks, ShardPlan& sp);

// Sharded coarse solve: subtree-to-rank mapping of a supernode tree (parent[g] <
// 0: a root; cost[g]: the supernode's factor entries).  owner[g] = -1 for the
// replicated top supernodes every rank sweeps, else the rank that sweeps g with
// its whole subtree.  A top is grown from the roots by splitting the costliest
// frontier subtree; the frontier subtrees go to the ranks largest first (LPT);
// the configuration with the smallest max-rank subtree work + top work wins.
void split_tree(int nsn, const int32_t* parent, const int64_t* cost, int nranks, std::vector<int32_t>& owner);

}  // namespace mdd
