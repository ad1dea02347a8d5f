// Structured Kuhn-tetrahedral mesh and edge numbering (host, integer work).
//
// PAPER.md §4 ("Cartesian mesh ... Nédélec edge elements of lowest order"),
// BASELINE configs ("cubes, each cut into 6 tets").  Numbering contract in
// include/maxwell_dd.h.  The edge set is enumerated by lattice direction: every
// edge of a Kuhn cube is a translate of one of the 7 vectors
//   (1,0,0) (0,1,0) (1,1,0) (0,0,1) (1,0,1) (0,1,1) (1,1,1)
// listed by increasing node-id offset, so scanning tails ascending and types in
// this order yields the lexicographic (tail, head) numbering directly.
#include "common.h"

#include <algorithm>

namespace mdd {

static const int KUHN_PERM[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
static const int LOCAL_EDGE[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
static const int DIRV[7][3] = {{1, 0, 0}, {0, 1, 0}, {1, 1, 0}, {0, 0, 1}, {1, 0, 1}, {0, 1, 1}, {1, 1, 1}};

static int dir_type(int dx, int dy, int dz) {
  for (int t = 0; t < 7; ++t)
    if (DIRV[t][0] == dx && DIRV[t][1] == dy && DIRV[t][2] == dz) return t;
  return -1;
}

void build_mesh(HostMesh& m, int nx, int ny, int nz, double h, const uint8_t* cube_mask,
                int dirichlet_mode) {
  MDD_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1, 2, "grid dimensions must be >= 1");
  MDD_REQUIRE(dirichlet_mode >= 0 && dirichlet_mode <= 2, 2, "bad dirichlet mode");
  m = HostMesh();
  m.nx = nx; m.ny = ny; m.nz = nz; m.h = h; m.dirichlet_mode = dirichlet_mode;
  const i64 NX = nx + 1, NY = ny + 1, NZ = nz + 1;
  m.nnodes = NX * NY * NZ;
  const i64 ncubes = (i64)nx * ny * nz;
  auto nid = [&](i64 i, i64 j, i64 k) { return i + NX * (j + NY * k); };
  auto present = [&](i64 i, i64 j, i64 k) -> bool {
    if (i < 0 || j < 0 || k < 0 || i >= nx || j >= ny || k >= nz) return false;
    return cube_mask == nullptr || cube_mask[i + (i64)nx * (j + (i64)ny * k)] != 0;
  };
  // tets
  std::vector<uint8_t> has_edge((size_t)(m.nnodes * 7), 0);
  m.node_used.assign(m.nnodes, 0);
  for (i64 c = 0; c < ncubes; ++c) {
    if (cube_mask && !cube_mask[c]) continue;
    i64 ci = c % nx, cj = (c / nx) % ny, ck = c / ((i64)nx * ny);
    for (int s = 0; s < 6; ++s) {
      int p[4][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {1, 1, 1}};
      p[1][KUHN_PERM[s][0]] = 1;
      p[2][KUHN_PERM[s][0]] = 1; p[2][KUHN_PERM[s][1]] = 1;
      m.tet_id.push_back(6 * c + s);
      for (int v = 0; v < 4; ++v) {
        i64 id = nid(ci + p[v][0], cj + p[v][1], ck + p[v][2]);
        m.tet_nodes.push_back(id);
        m.node_used[id] = 1;
      }
      for (int e = 0; e < 6; ++e) {
        int a = LOCAL_EDGE[e][0], b = LOCAL_EDGE[e][1];
        int t = dir_type(p[b][0] - p[a][0], p[b][1] - p[a][1], p[b][2] - p[a][2]);
        i64 tail = nid(ci + p[a][0], cj + p[a][1], ck + p[a][2]);
        has_edge[tail * 7 + t] = 1;
      }
    }
  }
  // lexicographic numbering
  std::vector<int32_t> eidx((size_t)(m.nnodes * 7), -1);
  const i64 off[7] = {1, NX, NX + 1, NX * NY, NX * NY + 1, NX * NY + NX, NX * NY + NX + 1};
  for (i64 v = 0; v < m.nnodes; ++v)
    for (int t = 0; t < 7; ++t)
      if (has_edge[v * 7 + t]) {
        eidx[v * 7 + t] = (int32_t)m.edge_tail.size();
        m.edge_tail.push_back(v);
        m.edge_head.push_back(v + off[t]);
      }
  const i64 T = m.ntets();
  m.tet_edge.resize(T * 6);
  for (i64 t = 0; t < T; ++t) {
    const i64* tn = &m.tet_nodes[t * 4];
    for (int e = 0; e < 6; ++e) {
      i64 a = tn[LOCAL_EDGE[e][0]], b = tn[LOCAL_EDGE[e][1]];
      int ai, aj, ak, bi, bj, bk;
      m.node_ijk(a, ai, aj, ak);
      m.node_ijk(b, bi, bj, bk);
      int ty = dir_type(bi - ai, bj - aj, bk - ak);
      m.tet_edge[t * 6 + e] = eidx[a * 7 + ty];
    }
  }
  // Dirichlet: the 5 edges and 4 nodes of every cube side whose neighbour cube is
  // absent (mode all) or outside the box (mode outer).
  m.edge_dir.assign(m.nedges(), 0);
  m.node_dir.assign(m.nnodes, 0);
  if (dirichlet_mode != 2) {
    for (i64 c = 0; c < ncubes; ++c) {
      if (cube_mask && !cube_mask[c]) continue;
      i64 ci = c % nx, cj = (c / nx) % ny, ck = c / ((i64)nx * ny);
      i64 cc[3] = {ci, cj, ck};
      int ext[3] = {nx, ny, nz};
      for (int d = 0; d < 3; ++d)
        for (int side = 0; side < 2; ++side) {
          i64 nb[3] = {cc[0], cc[1], cc[2]};
          nb[d] += side ? 1 : -1;
          bool outside = nb[d] < 0 || nb[d] >= ext[d];
          bool boundary = dirichlet_mode == 0 ? outside : !present(nb[0], nb[1], nb[2]);
          if (!boundary) continue;
          int a = (d + 1) % 3, b = (d + 2) % 3;
          if (a > b) std::swap(a, b);
          i64 base[3] = {cc[0], cc[1], cc[2]};
          base[d] += side;
          i64 corner[4];
          for (int q = 0; q < 4; ++q) {
            i64 p[3] = {base[0], base[1], base[2]};
            p[a] += q & 1; p[b] += (q >> 1) & 1;
            corner[q] = nid(p[0], p[1], p[2]);
            m.node_dir[corner[q]] = 1;
          }
          int ta = -1, tb = -1, tab = -1;
          { int v[3] = {0, 0, 0}; v[a] = 1; ta = dir_type(v[0], v[1], v[2]); }
          { int v[3] = {0, 0, 0}; v[b] = 1; tb = dir_type(v[0], v[1], v[2]); }
          { int v[3] = {0, 0, 0}; v[a] = 1; v[b] = 1; tab = dir_type(v[0], v[1], v[2]); }
          m.edge_dir[eidx[corner[0] * 7 + ta]] = 1;  // low a-edge
          m.edge_dir[eidx[corner[2] * 7 + ta]] = 1;  // high a-edge (b = 1)
          m.edge_dir[eidx[corner[0] * 7 + tb]] = 1;
          m.edge_dir[eidx[corner[1] * 7 + tb]] = 1;
          m.edge_dir[eidx[corner[0] * 7 + tab]] = 1;
        }
    }
  }
  m.edge_to_free.assign(m.nedges(), -1);
  for (i64 e = 0; e < m.nedges(); ++e)
    if (!m.edge_dir[e]) {
      m.edge_to_free[e] = (int32_t)m.free_edge.size();
      m.free_edge.push_back((int32_t)e);
    }
  m.node_to_free.assign(m.nnodes, -1);
  for (i64 v = 0; v < m.nnodes; ++v)
    if (m.node_used[v] && !m.node_dir[v]) {
      m.node_to_free[v] = (int32_t)m.free_node.size();
      m.free_node.push_back((int32_t)v);
    }
}

}  // namespace mdd
