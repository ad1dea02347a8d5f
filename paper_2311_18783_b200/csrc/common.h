// Shared host-side types for the maxwell_dd library (product path; no oracle code).
#pragma once
#include <cstdint>
#include <string>
#include <vector>
#include <stdexcept>

namespace mdd {

typedef int64_t i64;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define MDD_REQUIRE(cond, code, msg)                                   \
  do {                                                                 \
    if (!(cond)) throw ::mdd::Error((code), std::string(msg));         \
  } while (0)

// ---------------------------------------------------------------- mesh
// Structured nx*ny*nz cube grid, each cube cut into the 6 Kuhn tets.  See
// include/maxwell_dd.h for the numbering contract.
struct HostMesh {
  int nx = 0, ny = 0, nz = 0;
  double h = 0.0;
  int dirichlet_mode = 0;               // 0 outer, 1 all boundary, 2 none
  i64 nnodes = 0;
  std::vector<i64> tet_id;              // present tets, ascending (6*cube + s)
  std::vector<i64> tet_nodes;           // 4 per tet, increasing
  std::vector<i64> edge_tail, edge_head;// all edges, lexicographic
  std::vector<int32_t> tet_edge;        // 6 per tet (edge index, LOCAL_EDGES order)
  std::vector<uint8_t> edge_dir, node_dir, node_used;
  std::vector<int32_t> free_edge;       // free dof -> edge index
  std::vector<int32_t> edge_to_free;    // edge -> free dof or -1
  std::vector<int32_t> free_node;       // free node index -> node id
  std::vector<int32_t> node_to_free;    // node id -> free node index or -1
  i64 nedges() const { return (i64)edge_tail.size(); }
  int n() const { return (int)free_edge.size(); }
  i64 ntets() const { return (i64)tet_id.size(); }
  void node_ijk(i64 v, int& i, int& j, int& k) const {
    i = (int)(v % (nx + 1));
    j = (int)((v / (nx + 1)) % (ny + 1));
    k = (int)(v / ((i64)(nx + 1) * (ny + 1)));
  }
};

void build_mesh(HostMesh& m, int nx, int ny, int nz, double h, const uint8_t* cube_mask,
                int dirichlet_mode);

// ------------------------------------------------------ sparse patterns
struct Csr {
  int nrows = 0, ncols = 0;
  std::vector<i64> ptr;
  std::vector<int32_t> idx;
  i64 nnz() const { return ptr.empty() ? 0 : ptr.back(); }
};

// ------------------------------------------------ supernodal factor plan
// A batch of independent symmetric systems, concatenated.  Unknown u of
// system s lives at "position" pos = sys_off[s] + permuted index.
struct FactorPlan {
  int nsys = 0;
  i64 ntot = 0;
  std::vector<i64> sys_off;             // nsys + 1
  std::vector<int32_t> perm;            // position -> original local index (within its system)
  std::vector<int32_t> iperm_global;    // (sys_off + local) -> position
  // supernodes (ordered: children before parents, systems interleaved by level)
  int nsn = 0;
  std::vector<i64> sn_col0;             // first position
  std::vector<int32_t> sn_ncol, sn_noff, sn_parent, sn_level;
  std::vector<i64> sn_rowptr;           // into offrows
  std::vector<i64> offrows;             // positions of off-diagonal rows
  std::vector<i64> sn_lptr;             // into L values: nrow*ncol panel, col-major
  std::vector<i64> sn_uptr;             // into update-vector buffer (noff)
  std::vector<i64> sn_fptr;             // into front workspace (nrow*nrow) for factorisation
  std::vector<i64> sn_umptr;            // into update-matrix buffer (noff*noff)
  std::vector<i64> child_ptr;           // nsn + 1
  std::vector<int32_t> child_list;
  std::vector<i64> relmap_ptr;          // per supernode: offsets into relmap of its noff rows
  std::vector<int32_t> relmap;          // position of each off row inside the parent's row list
  int nlevels = 0;
  std::vector<int32_t> level_ptr;       // nlevels + 1 into level_sn
  std::vector<int32_t> level_sn;
  i64 lsize = 0, usize = 0, fsize = 0, umsize = 0;
  // assembly map: matrix entry (source value slot) -> (supernode, front row, front col)
  std::vector<i64> asm_ptr;             // nsn + 1
  std::vector<i64> asm_src;             // source value index
  std::vector<int32_t> asm_pos;         // row*nrow + col inside the front (row >= col)
  i64 factor_nnz() const;
};

struct SymSystem {
  const Csr* pat;                       // full symmetric pattern (both triangles), local indices
  const int32_t* xyz2;                  // 3 ints per unknown: doubled lattice coordinates
  const i64* val_slot;                  // per pattern entry: index of its value in the source array
  const uint8_t* last = nullptr;        // optional: unknowns ordered after the nested dissection
  // optional, with `last`: per unknown 6 ints (lo xyz, hi xyz, doubled coordinates)
  // bounding its coupling region; a flagged unknown then closes the smallest
  // dissection subtree whose box contains that region instead of the whole order
  const int32_t* box = nullptr;
};

void build_factor_plan(FactorPlan& fp, const std::vector<SymSystem>& systems, int leaf_size);

}  // namespace mdd
