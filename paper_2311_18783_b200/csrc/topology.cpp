// Host integer work of the setup: sparsity pattern of A with its deterministic
// assembly lists, the overlapping box decomposition (§2, §4), local
// patterns, prolongation maps and the gradient (SNK / NK) candidate columns.
#include "topology.h"

#include <algorithm>
#include <functional>
#include <numeric>

namespace mdd {

static const int LE[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

void build_A_pattern(const HostMesh& m, Csr& A, std::vector<i64>& slot_ptr,
                     std::vector<int32_t>& contrib) {
  const int n = m.n();
  const i64 T = m.ntets();
  // rows: union of the free edges of the tets around each free edge
  std::vector<i64> cnt(n + 1, 0);
  for (i64 t = 0; t < T; ++t)
    for (int a = 0; a < 6; ++a) {
      int ea = m.edge_to_free[m.tet_edge[t * 6 + a]];
      if (ea >= 0) cnt[ea + 1] += 6;
    }
  for (int i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  std::vector<int32_t> tmp(cnt[n]);
  {
    std::vector<i64> cur(cnt.begin(), cnt.end() - 1);
    for (i64 t = 0; t < T; ++t)
      for (int a = 0; a < 6; ++a) {
        int ea = m.edge_to_free[m.tet_edge[t * 6 + a]];
        if (ea < 0) continue;
        for (int b = 0; b < 6; ++b) tmp[cur[ea]++] = m.edge_to_free[m.tet_edge[t * 6 + b]];
      }
  }
  A.nrows = A.ncols = n;
  A.ptr.assign(n + 1, 0);
  A.idx.clear();
  for (int i = 0; i < n; ++i) {
    std::vector<int32_t> r(tmp.begin() + cnt[i], tmp.begin() + cnt[i + 1]);
    std::sort(r.begin(), r.end());
    r.erase(std::unique(r.begin(), r.end()), r.end());
    for (int32_t c : r)
      if (c >= 0) A.idx.push_back(c);
    A.ptr[i + 1] = (i64)A.idx.size();
  }
  // contributions per slot, ordered by (tet, m, n)
  const i64 nnz = A.nnz();
  std::vector<i64> sc(nnz + 1, 0);
  auto slot_of = [&](int r, int c) -> i64 {
    const int32_t* b = A.idx.data() + A.ptr[r];
    const int32_t* e = A.idx.data() + A.ptr[r + 1];
    const int32_t* it = std::lower_bound(b, e, c);
    return (i64)(it - A.idx.data());
  };
  std::vector<i64> slots(T * 36, -1);
  for (i64 t = 0; t < T; ++t)
    for (int a = 0; a < 6; ++a) {
      int ea = m.edge_to_free[m.tet_edge[t * 6 + a]];
      if (ea < 0) continue;
      for (int b = 0; b < 6; ++b) {
        int eb = m.edge_to_free[m.tet_edge[t * 6 + b]];
        if (eb < 0) continue;
        i64 s = slot_of(ea, eb);
        slots[t * 36 + a * 6 + b] = s;
        sc[s + 1]++;
      }
    }
  for (i64 s = 0; s < nnz; ++s) sc[s + 1] += sc[s];
  contrib.assign(sc[nnz], 0);
  std::vector<i64> cur(sc.begin(), sc.end() - 1);
  for (i64 q = 0; q < T * 36; ++q)
    if (slots[q] >= 0) contrib[cur[slots[q]]++] = (int32_t)q;
  slot_ptr.swap(sc);
}

void build_subdomains(const HostMesh& m, int px, int py, int pz, int overlap, Decomp& d) {
  MDD_REQUIRE(px >= 1 && py >= 1 && pz >= 1, 2, "subdomain counts must be >= 1");
  MDD_REQUIRE(m.nx % px == 0 && m.ny % py == 0 && m.nz % pz == 0, 2,
              "subdomain boxes must divide the cube grid");
  MDD_REQUIRE(overlap >= 0, 2, "overlap must be >= 0");
  const int sx = m.nx / px, sy = m.ny / py, sz = m.nz / pz;
  d.nsub = px * py * pz;
  d.sub_tets.assign(d.nsub, {});
  d.sub_dofs.assign(d.nsub, {});
  const i64 T = m.ntets();
  for (i64 t = 0; t < T; ++t) {
    i64 cube = m.tet_id[t] / 6;
    int ci = (int)(cube % m.nx), cj = (int)((cube / m.nx) % m.ny), ck = (int)(cube / ((i64)m.nx * m.ny));
    int lo[3], hi[3];
    int c3[3] = {ci, cj, ck}, s3[3] = {sx, sy, sz}, p3[3] = {px, py, pz};
    for (int a = 0; a < 3; ++a) {
      // subdomain b contains the cube iff b*s - ov <= c < (b+1)*s + ov (checked below)
      lo[a] = std::max(0, (c3[a] - overlap) / s3[a] - 1);
      hi[a] = std::min(p3[a] - 1, (c3[a] + overlap) / s3[a]);
    }
    for (int bk = lo[2]; bk <= hi[2]; ++bk)
      for (int bj = lo[1]; bj <= hi[1]; ++bj)
        for (int bi = lo[0]; bi <= hi[0]; ++bi) {
          if (!(bi * sx - overlap <= ci && ci < (bi + 1) * sx + overlap)) continue;
          if (!(bj * sy - overlap <= cj && cj < (bj + 1) * sy + overlap)) continue;
          if (!(bk * sz - overlap <= ck && ck < (bk + 1) * sz + overlap)) continue;
          d.sub_tets[bi + px * (bj + py * bk)].push_back((int32_t)t);
        }
  }
  const int n = m.n();
  d.mult.assign(n, 0);
  std::vector<int32_t> mark(n, -1);
  for (int s = 0; s < d.nsub; ++s) {
    auto& D = d.sub_dofs[s];
    for (int32_t t : d.sub_tets[s])
      for (int a = 0; a < 6; ++a) {
        int e = m.edge_to_free[m.tet_edge[(i64)t * 6 + a]];
        if (e >= 0 && mark[e] != s) { mark[e] = s; D.push_back(e); }
      }
    std::sort(D.begin(), D.end());
    for (int32_t e : D) d.mult[e]++;
  }
  for (int e = 0; e < n; ++e) MDD_REQUIRE(d.mult[e] > 0, 2, "a dof is covered by no subdomain");
}

void local_pattern(const Csr& A, const std::vector<int32_t>& dofs, std::vector<int32_t>& g2l,
                   Csr& loc, std::vector<i64>& slot) {
  const int ni = (int)dofs.size();
  for (int k = 0; k < ni; ++k) g2l[dofs[k]] = k;
  loc.nrows = loc.ncols = ni;
  loc.ptr.assign(ni + 1, 0);
  loc.idx.clear();
  slot.clear();
  for (int k = 0; k < ni; ++k) {
    int e = dofs[k];
    for (i64 p = A.ptr[e]; p < A.ptr[e + 1]; ++p) {
      int l = g2l[A.idx[p]];
      if (l >= 0) { loc.idx.push_back(l); slot.push_back(p); }
    }
    loc.ptr[k + 1] = (i64)loc.idx.size();
  }
  for (int k = 0; k < ni; ++k) g2l[dofs[k]] = -1;
}

void edge_xyz2(const HostMesh& m, int e_free, int32_t* out) {
  int e = m.free_edge[e_free];
  int ai, aj, ak, bi, bj, bk;
  m.node_ijk(m.edge_tail[e], ai, aj, ak);
  m.node_ijk(m.edge_head[e], bi, bj, bk);
  out[0] = ai + bi; out[1] = aj + bj; out[2] = ak + bk;
}

// G_i columns (reading R7): the free nodes of Omega_i; in each connected
// component of (free nodes, edges N_i) with no edge to a Dirichlet node, the
// largest node is dropped (its column is minus the sum of the others).
void gradient_nodes(const HostMesh& m, const std::vector<int32_t>& dofs, std::vector<int32_t>& cols) {
  std::vector<int32_t> nodes;
  for (int32_t e : dofs) {
    int ee = m.free_edge[e];
    int a = m.node_to_free[m.edge_tail[ee]], b = m.node_to_free[m.edge_head[ee]];
    if (a >= 0) nodes.push_back(a);
    if (b >= 0) nodes.push_back(b);
  }
  std::sort(nodes.begin(), nodes.end());
  nodes.erase(std::unique(nodes.begin(), nodes.end()), nodes.end());
  const int g = (int)nodes.size();
  auto loc = [&](int v) { return (int)(std::lower_bound(nodes.begin(), nodes.end(), v) - nodes.begin()); };
  std::vector<int32_t> par(g);
  std::iota(par.begin(), par.end(), 0);
  std::function<int(int)> find = [&](int a) {
    while (par[a] != a) { par[a] = par[par[a]]; a = par[a]; }
    return a;
  };
  std::vector<uint8_t> grounded_node(g, 0);
  for (int32_t e : dofs) {
    int ee = m.free_edge[e];
    int a = m.node_to_free[m.edge_tail[ee]], b = m.node_to_free[m.edge_head[ee]];
    if (a >= 0 && b >= 0) {
      int ra = find(loc(a)), rb = find(loc(b));
      if (ra != rb) par[std::max(ra, rb)] = std::min(ra, rb);
    } else if (a >= 0) grounded_node[loc(a)] = 1;
    else if (b >= 0) grounded_node[loc(b)] = 1;
  }
  std::vector<uint8_t> grounded(g, 0);
  std::vector<int32_t> maxnode(g, -1);
  for (int k = 0; k < g; ++k) {
    int r = find(k);
    if (grounded_node[k]) grounded[r] = 1;
    maxnode[r] = std::max(maxnode[r], k);
  }
  cols.clear();
  for (int k = 0; k < g; ++k) {
    int r = find(k);
    if (!grounded[r] && maxnode[r] == k) continue;
    cols.push_back(nodes[k]);
  }
}

}  // namespace mdd
