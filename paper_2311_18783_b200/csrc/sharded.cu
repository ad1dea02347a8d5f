// Sharded PCG over several GPUs (north_star: "Subdomains are sharded across the
// GPUs of one 8xB200 box, with overlap-halo exchange and the coarse-space and
// dot-product allreduces over NCCL/NVLink").
//
// A rank owns a slab of subdomains and the dofs of their owned boxes
// (shard.cpp); its PCG vectors live on its owned dofs plus a halo.  One
// iteration of the bench's loop (reading R13: x0 = Q f, z = w + Q (r - A w),
// w = M_AS r) on a rank:
//   halo(p) -> q = A p (owned rows)               | allreduce(p.q)  -> alpha
//   x, r update (owned)                            | allreduce(r.r)  -> stop?
//   halo(r) -> sweep of the rank's subdomains (R_i r, A_i^{-1}, R_i^T onto its
//     local dofs) -> reverse halo (owners add the overlap contributions)
//   halo(w) -> t = r - A w (owned rows)
//   Z^T t over the owned rows (partial per coarse column) | allreduce(n0)
//   E^{-1} (the coarse factor, every rank) -> z = w + Z y (owned rows)
//   allreduce(r.z) -> beta, p update
// The exchanges go through a Transport: NCCL point-to-point + allreduce between
// processes (one GPU each), or device copies between several handles of one
// process on one GPU (the group solve of the tests, which runs the same
// sequence of kernels rank by rank between the exchanges).  The coarse factor
// is set up on every rank, but E^{-1} is applied distributed:
// each rank sweeps the subtrees of E's supernode tree split_tree gave it plus
// the replicated top separators, with one allreduce of the frontier roots'
// update vectors between the forward sweeps and one of the solution after.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <memory>

#include "handle.h"
#include "shard.h"

namespace mdd {

namespace {

// ---------------------------------------------------------------- kernels
__global__ void k_pack(int n, const int32_t* __restrict__ idx, const double* __restrict__ v, double* __restrict__ b) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) b[k] = v[idx[k]];
}
__global__ void k_unpack(int n, const int32_t* __restrict__ idx, const double* __restrict__ b, double* __restrict__ v,
                         int add) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) v[idx[k]] = add ? v[idx[k]] + b[k] : b[k];
}
// dst[di[k]] (+)= src[si[k]] (two handles of one process, same device)
__global__ void k_halo_copy(int n, const int32_t* __restrict__ si, const double* __restrict__ src,
                            const int32_t* __restrict__ di, double* __restrict__ dst, int add) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) dst[di[k]] = add ? dst[di[k]] + src[si[k]] : src[si[k]];
}
// b[own[j]] = v[pos[own[j]]] (pos null: v[own[j]]): this rank's entries of an
// exchange buffer whose other entries are zero
__global__ void k_scatter_owned(int64_t nown, const int64_t* __restrict__ pos, const int32_t* __restrict__ own,
                                const double* __restrict__ v, double* __restrict__ b) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < nown) {
    const int32_t k = own[j];
    b[k] = v[pos ? pos[k] : k];
  }
}
// v[pos[k]] = b[k]
__global__ void k_unpack_all(int64_t n, const int64_t* __restrict__ pos, const double* __restrict__ b,
                             double* __restrict__ v) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) v[pos[k]] = b[k];
}
__global__ void k_vadd(int64_t n, const double* __restrict__ a, double* __restrict__ acc) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) acc[k] += a[k];
}

// ------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*ErrStr)(ncclResult_t) = nullptr;
};

// the process's libnccl (torch's, already loaded) when present, else the system one
const NcclApi& nccl() {
  static NcclApi api;
  if (api.lib) return api;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  MDD_REQUIRE(h != nullptr, 1, std::string("libnccl.so.2 not loadable: ") + dlerror());
  auto sym = [&](const char* n) {
    void* f = dlsym(h, n);
    MDD_REQUIRE(f != nullptr, 1, std::string("NCCL symbol missing: ") + n);
    return f;
  };
  api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
  api.Send = (decltype(api.Send))sym("ncclSend");
  api.Recv = (decltype(api.Recv))sym("ncclRecv");
  api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
  api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
  api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
  api.ErrStr = (decltype(api.ErrStr))sym("ncclGetErrorString");
  api.lib = h;
  return api;
}
#define NCCL_OK(x)                                                                           \
  do {                                                                                       \
    ncclResult_t r__ = (x);                                                                  \
    if (r__ != ncclSuccess) throw Error(1, std::string(#x) + ": " + nccl().ErrStr(r__));     \
  } while (0)

}  // namespace

// ----------------------------------------------------------- shard state
struct ShardState {
  ShardPlan plan;
  int n_own = 0, n_loc = 0;
  DBuf<int64_t> A_ptr;            // owned rows of A, columns in local numbering
  DBuf<int32_t> A_idx;
  DBuf<double> A_val;
  DevFactor loc;                  // the rank's subdomains; prolongation onto its local dofs
  DBuf<int64_t> lpro_ptr;
  DBuf<int32_t> lpro_pos;
  DBuf<int64_t> Z_ptr, Zt_ptr;    // owned rows of Z (columns: coarse positions) and their transpose
  DBuf<int32_t> Z_idx, Zt_idx;
  DBuf<double> Z_val, Zt_val;
  DBuf<int32_t> send_idx, recv_idx;
  DBuf<double> sbuf, rbuf, acc;
  DBuf<double> x, r, p, q, z, w, t, u;   // p, r, w: local layout (n_loc); the rest owned (n_loc for simplicity)
  // distributed coarse solve (nranks > 1): this rank's view of the replicated
  // coarse factor sweeping its subtrees (segment A) and the replicated top
  // (segment B); between the two, the update vectors of the frontier subtree
  // roots (ux_pos, the same list on every rank; this rank fills ux_own) are
  // summed over the ranks; after B, the coarse solution (y_own: the positions
  // this rank provides) likewise
  bool dist_coarse = false;
  DevFactor crs;
  DBuf<int64_t> ux_pos;
  DBuf<int32_t> ux_own, y_own;
  DBuf<double> ubuf, ybuf;
  int64_t n_ux = 0, n_ux_own = 0, n_y_own = 0, top_entries = 0;
  ncclComm_t comm = nullptr;
  ~ShardState() {
    if (comm) nccl().CommDestroy(comm);
  }
};

void shard_free(ShardState* s) { delete s; }

namespace {

void shard_setup(mdd_solver* H, int rank, int nranks) {
  CUDA_CHECK(cudaSetDevice(H->device));
  cudaStream_t s = H->stream;
  auto S = std::unique_ptr<ShardState>(new ShardState());
  ShardPlan& P = S->plan;
  build_shard_plan(H->mesh, H->dec, H->Apat, H->desc.px, H->desc.py, H->desc.pz, rank, nranks, P);
  const int n = H->n;
  S->n_own = P.n_own();
  S->n_loc = P.n_local();
  std::vector<int32_t> g2l(n, -1);
  for (int k = 0; k < S->n_own; ++k) g2l[P.owned[k]] = k;
  for (size_t k = 0; k < P.halo.size(); ++k) g2l[P.halo[k]] = S->n_own + (int)k;
  // ---- owned rows of A (values gathered from the assembled A by slot)
  {
    std::vector<int64_t> ptr(S->n_own + 1, 0), slot;
    std::vector<int32_t> idx;
    for (int k = 0; k < S->n_own; ++k) {
      const int e = P.owned[k];
      for (int64_t q = H->Apat.ptr[e]; q < H->Apat.ptr[e + 1]; ++q) {
        const int32_t c = g2l[H->Apat.idx[q]];
        MDD_REQUIRE(c >= 0, 5, "shard plan: an SpMV column is not local");
        idx.push_back(c);
        slot.push_back(q);
      }
      ptr[k + 1] = (int64_t)idx.size();
    }
    S->A_ptr.upload(ptr);
    S->A_idx.upload(idx);
    S->A_val.alloc(std::max<size_t>(slot.size(), 1));
    DBuf<int64_t> ds;
    ds.upload(slot);
    dev::k_gather<<<nblk((int64_t)slot.size(), 256), 256, 0, s>>>((int64_t)slot.size(), ds.p, H->A_val.p, S->A_val.p);
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  // ---- local factor of the rank's subdomains (same symbolic recipe as the global one)
  {
    const int ns = (int)P.subs.size();
    std::vector<Csr> lpat(ns);
    std::vector<std::vector<int64_t>> lslot(ns);
    std::vector<std::vector<int32_t>> lxyz(ns);
    std::vector<int32_t> scratch(n, -1);
    std::vector<SymSystem> sys(ns);
    for (int a = 0; a < ns; ++a) {
      const auto& D = H->dec.sub_dofs[P.subs[a]];
      local_pattern(H->Apat, D, scratch, lpat[a], lslot[a]);
      lxyz[a].resize(3 * D.size());
      for (size_t k = 0; k < D.size(); ++k) edge_xyz2(H->mesh, D[k], &lxyz[a][3 * k]);
      sys[a] = SymSystem{&lpat[a], lxyz[a].data(), lslot[a].data()};
    }
    build_factor_plan(S->loc.fp, sys, env_int("MDD_ND_LEAF", 64));
    S->loc.name = "local_shard";
    const FactorPlan& fp = S->loc.fp;
    std::vector<int32_t> gm(fp.ntot);
    std::vector<int64_t> pp(S->n_loc + 1, 0);
    for (int a = 0; a < ns; ++a) {
      const auto& D = H->dec.sub_dofs[P.subs[a]];
      for (int64_t k = fp.sys_off[a]; k < fp.sys_off[a + 1]; ++k) gm[k] = g2l[D[fp.perm[k]]];
      for (int32_t e : D) pp[g2l[e] + 1]++;
    }
    for (int k = 0; k < S->n_loc; ++k) pp[k + 1] += pp[k];
    std::vector<int32_t> pos(pp[S->n_loc]);
    std::vector<int64_t> cur(pp.begin(), pp.end() - 1);
    for (int a = 0; a < ns; ++a) {
      const auto& D = H->dec.sub_dofs[P.subs[a]];
      for (size_t k = 0; k < D.size(); ++k) pos[cur[g2l[D[k]]]++] = fp.iperm_global[fp.sys_off[a] + k];
    }
    S->lpro_ptr.upload(pp);
    S->lpro_pos.upload(pos);
    S->loc.upload(S->n_loc, S->lpro_ptr.p, S->lpro_pos.p, &gm);
    S->loc.factor(H->A_val.p, 0, 0.0, nullptr, s);
  }
  // ---- owned rows of Z and their transpose (coarse positions x owned rows)
  if (H->has_coarse) {
    std::vector<int64_t> zp = [&] {
      std::vector<int64_t> v(n + 1);
      CUDA_CHECK(cudaMemcpy(v.data(), H->Z_ptr.p, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));
      return v;
    }();
    std::vector<int32_t> zi(zp[n]);
    CUDA_CHECK(cudaMemcpy(zi.data(), H->Z_idx.p, zi.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
    std::vector<int64_t> ptr(S->n_own + 1, 0), slot;
    std::vector<int32_t> idx;
    for (int k = 0; k < S->n_own; ++k) {
      const int e = P.owned[k];
      for (int64_t q = zp[e]; q < zp[e + 1]; ++q) { idx.push_back(zi[q]); slot.push_back(q); }
      ptr[k + 1] = (int64_t)idx.size();
    }
    const int64_t nb = H->n0, nz = (int64_t)idx.size();
    std::vector<int64_t> tp(nb + 1, 0), tslot(nz);
    std::vector<int32_t> ti(nz);
    for (int32_t c : idx) tp[c + 1]++;
    for (int64_t c = 0; c < nb; ++c) tp[c + 1] += tp[c];
    std::vector<int64_t> tc(tp.begin(), tp.end() - 1);
    for (int k = 0; k < S->n_own; ++k)
      for (int64_t q = ptr[k]; q < ptr[k + 1]; ++q) {
        const int64_t d = tc[idx[q]]++;
        ti[d] = k;
        tslot[d] = slot[q];
      }
    S->Z_ptr.upload(ptr);
    S->Z_idx.upload(idx.empty() ? std::vector<int32_t>{0} : idx);
    S->Zt_ptr.upload(tp);
    S->Zt_idx.upload(ti.empty() ? std::vector<int32_t>{0} : ti);
    S->Z_val.alloc(std::max<int64_t>(nz, 1));
    S->Zt_val.alloc(std::max<int64_t>(nz, 1));
    DBuf<int64_t> d1, d2;
    d1.upload(slot.empty() ? std::vector<int64_t>{0} : slot);
    d2.upload(tslot.empty() ? std::vector<int64_t>{0} : tslot);
    if (nz) {
      dev::k_gather<<<nblk(nz, 256), 256, 0, s>>>(nz, d1.p, H->Z_val.p, S->Z_val.p);
      dev::k_gather<<<nblk(nz, 256), 256, 0, s>>>(nz, d2.p, H->Z_val.p, S->Zt_val.p);
    }
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  // ---- distributed coarse solve: subtree-to-rank split of E's supernode tree
  if (H->has_coarse && nranks > 1 && !getenv("MDD_SHARD_COARSE_REPLICATED")) {
    const FactorPlan& cf = H->crs.fp;
    std::vector<int64_t> cost(cf.nsn);
    for (int g = 0; g < cf.nsn; ++g) {
      const int64_t nc = cf.sn_ncol[g], no = cf.sn_noff[g];
      cost[g] = nc * (nc + 1) / 2 + nc * no;
    }
    std::vector<int32_t> owner;
    split_tree(cf.nsn, cf.sn_parent.data(), cost.data(), nranks, owner);
    S->crs.fp = cf;
    std::vector<int64_t>().swap(S->crs.fp.asm_src);  // assembly maps: factorisation only
    std::vector<int32_t>().swap(S->crs.fp.asm_pos);
    S->crs.base = &H->crs;
    S->crs.name = "coarse_shard" + std::to_string(rank);
    S->crs.role.assign(cf.nsn, 0);
    for (int g = 0; g < cf.nsn; ++g) S->crs.role[g] = owner[g] < 0 ? 2 : owner[g] == rank ? 1 : 0;
    S->crs.upload();
    // update vectors of the frontier subtree roots (a non-top supernode whose
    // parent is top): every rank's list, in supernode order; this rank's entries
    std::vector<int64_t> ux;
    std::vector<int32_t> uo, yo;
    for (int g = 0; g < cf.nsn; ++g) {
      const int pg = cf.sn_parent[g];
      if (owner[g] < 0 || pg < 0 || owner[pg] >= 0) continue;
      for (int a = 0; a < cf.sn_noff[g]; ++a) {
        if (owner[g] == rank) uo.push_back((int32_t)ux.size());
        ux.push_back(cf.sn_uptr[g] + a);
      }
    }
    // coarse positions this rank provides: its subtrees' columns; rank 0 also the top's
    for (int g = 0; g < cf.nsn; ++g)
      if (owner[g] == rank || (owner[g] < 0 && rank == 0))
        for (int c = 0; c < cf.sn_ncol[g]; ++c) yo.push_back((int32_t)(cf.sn_col0[g] + c));
    S->top_entries = 0;
    for (int g = 0; g < cf.nsn; ++g)
      if (owner[g] < 0) S->top_entries += cost[g];
    S->n_ux = (int64_t)ux.size();
    S->n_ux_own = (int64_t)uo.size();
    S->n_y_own = (int64_t)yo.size();
    S->ux_pos.upload(ux.empty() ? std::vector<int64_t>{0} : ux);
    S->ux_own.upload(uo.empty() ? std::vector<int32_t>{0} : uo);
    S->y_own.upload(yo.empty() ? std::vector<int32_t>{0} : yo);
    S->ubuf.alloc(std::max<int64_t>(S->n_ux, 1));
    S->ybuf.alloc(std::max<int64_t>(H->n0, 1));
    S->dist_coarse = true;
  }
  // ---- exchange lists and vectors
  S->send_idx.upload(P.send_idx.empty() ? std::vector<int32_t>{0} : P.send_idx);
  S->recv_idx.upload(P.recv_idx.empty() ? std::vector<int32_t>{0} : P.recv_idx);
  const size_t nbuf = std::max<size_t>(std::max(P.send_idx.size(), P.recv_idx.size()), 1);
  S->sbuf.alloc(nbuf);
  S->rbuf.alloc(nbuf);
  S->acc.alloc(std::max<int64_t>(std::max<int64_t>(H->n0, S->n_ux), 8) + 8);
  for (DBuf<double>* b : {&S->x, &S->r, &S->p, &S->q, &S->z, &S->w, &S->t, &S->u}) {
    b->alloc(std::max(S->n_loc, 1));
    b->zero(s);
  }
  CUDA_CHECK(cudaStreamSynchronize(s));
  shard_free(H->shard);
  H->shard = S.release();
}

// ------------------------------------------------------------- transports
struct Member {
  mdd_solver* h;
  ShardState* s;
};
using VecOf = std::function<double*(Member&)>;

struct Transport {
  virtual ~Transport() {}
  // forward: owners -> halos; reverse: halos added into the owners
  virtual void halo(std::vector<Member>& M, const VecOf& vec, bool reverse, cudaStream_t st) = 0;
  // buf[0..count) = sum over ranks
  virtual void allreduce(std::vector<Member>& M, const VecOf& buf, int64_t count, cudaStream_t st) = 0;
};

struct NcclTransport : Transport {
  void halo(std::vector<Member>& M, const VecOf& vec, bool reverse, cudaStream_t st) override {
    Member& m = M[0];
    ShardState& S = *m.s;
    const ShardPlan& P = S.plan;
    double* v = vec(m);
    // forward: send owned values at send_idx, receive into recv_idx; reverse: the
    // roles of the two lists swap and the receiver adds
    const int32_t* out_idx = reverse ? S.recv_idx.p : S.send_idx.p;
    const int32_t* in_idx = reverse ? S.send_idx.p : S.recv_idx.p;
    const std::vector<int64_t>& optr = reverse ? P.recv_ptr : P.send_ptr;
    const std::vector<int64_t>& iptr = reverse ? P.send_ptr : P.recv_ptr;
    const int nout = (int)optr[P.nranks], nin = (int)iptr[P.nranks];
    if (nout) k_pack<<<nblk(nout, 256), 256, 0, st>>>(nout, out_idx, v, S.sbuf.p);
    NCCL_OK(nccl().GroupStart());
    for (int q = 0; q < P.nranks; ++q) {
      if (q == P.rank) continue;
      const int64_t no = optr[q + 1] - optr[q], ni = iptr[q + 1] - iptr[q];
      if (no) NCCL_OK(nccl().Send(S.sbuf.p + optr[q], (size_t)no, ncclDouble, q, S.comm, st));
      if (ni) NCCL_OK(nccl().Recv(S.rbuf.p + iptr[q], (size_t)ni, ncclDouble, q, S.comm, st));
    }
    NCCL_OK(nccl().GroupEnd());
    if (nin) k_unpack<<<nblk(nin, 256), 256, 0, st>>>(nin, in_idx, S.rbuf.p, v, reverse ? 1 : 0);
  }
  void allreduce(std::vector<Member>& M, const VecOf& buf, int64_t count, cudaStream_t st) override {
    double* b = buf(M[0]);
    NCCL_OK(nccl().AllReduce(b, b, (size_t)count, ncclDouble, ncclSum, M[0].s->comm, st));
  }
};

// several handles of one process on one device: direct device copies between
// their buffers, rank by rank in a fixed order (deterministic sums)
struct GroupTransport : Transport {
  void halo(std::vector<Member>& M, const VecOf& vec, bool reverse, cudaStream_t st) override {
    const int R = (int)M.size();
    for (int dst = 0; dst < R; ++dst)
      for (int src = 0; src < R; ++src) {
        if (src == dst) continue;
        const ShardPlan& Ps = M[src].s->plan;
        const ShardPlan& Pd = M[dst].s->plan;
        if (!reverse) {   // src owner -> dst halo
          const int64_t n = Ps.send_ptr[dst + 1] - Ps.send_ptr[dst];
          if (n) k_halo_copy<<<nblk(n, 256), 256, 0, st>>>((int)n, M[src].s->send_idx.p + Ps.send_ptr[dst], vec(M[src]),
                                                          M[dst].s->recv_idx.p + Pd.recv_ptr[src], vec(M[dst]), 0);
        } else {          // src halo added into dst owner
          const int64_t n = Ps.recv_ptr[dst + 1] - Ps.recv_ptr[dst];
          if (n) k_halo_copy<<<nblk(n, 256), 256, 0, st>>>((int)n, M[src].s->recv_idx.p + Ps.recv_ptr[dst], vec(M[src]),
                                                          M[dst].s->send_idx.p + Pd.send_ptr[src], vec(M[dst]), 1);
        }
      }
  }
  void allreduce(std::vector<Member>& M, const VecOf& buf, int64_t count, cudaStream_t st) override {
    double* acc = M[0].s->acc.p;
    CUDA_CHECK(cudaMemcpyAsync(acc, buf(M[0]), count * sizeof(double), cudaMemcpyDeviceToDevice, st));
    for (size_t k = 1; k < M.size(); ++k) k_vadd<<<nblk(count, 256), 256, 0, st>>>(count, buf(M[k]), acc);
    for (auto& m : M) CUDA_CHECK(cudaMemcpyAsync(buf(m), acc, count * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
};

// ------------------------------------------------------------ sharded PCG
struct ShardSolve {
  std::vector<Member>& M;
  Transport& T;
  cudaStream_t st;
  bool coarse;
  int launches = 0;

  template <class F>
  void each(F f) {
    for (auto& m : M) f(m);
  }
  // y = A x over the owned rows (x: local layout, halo filled); sub: y = sub - A x
  void spmv_own(Member& m, const double* x, double* y, const double* sub = nullptr) {
    dev::k_spmv8<<<m.h->nparts, 256, 0, st>>>(m.s->n_own, m.s->A_ptr.p, m.s->A_idx.p, m.s->A_val.p, x, sub, y,
                                             nullptr, nullptr, m.h->state.p, mdd_solver::rnone());
    ++launches;
  }
  // S[slot] of every rank = global dot over the owned rows
  void dot(const VecOf& a, const VecOf& b, int slot) {
    each([&](Member& m) {
      dev::k_dot_part<<<m.h->nparts, 256, 0, st>>>(m.s->n_own, a(m), b(m), m.h->part.p, m.h->state.p,
                                                   mdd_solver::rnone());
      dev::k_reduce<<<1, 256, 0, st>>>(m.h->nparts, m.h->part.p, m.h->S.p + slot, m.h->state.p);
      launches += 2;
    });
    T.allreduce(M, [slot](Member& m) { return m.h->S.p + slot; }, 1, st);
  }
  void scalar(int op) {
    each([&](Member& m) { dev::k_scalar_step<<<1, 1, 0, st>>>(op, m.h->S.p, m.h->state.p); ++launches; });
  }
  // out = add + Z E^{-1} Z^T v over the owned rows (add may be null)
  void coarse_apply(const VecOf& v, const VecOf& out, const VecOf& add) {
    each([&](Member& m) {
      dev::k_spmv32<<<m.h->nparts, 256, 0, st>>>((int)m.h->n0, m.s->Zt_ptr.p, m.s->Zt_idx.p, m.s->Zt_val.p, v(m),
                                                nullptr, m.h->xc.p, nullptr, nullptr, m.h->state.p,
                                                mdd_solver::rnone());
      ++launches;
    });
    T.allreduce(M, [](Member& m) { return m.h->xc.p; }, M[0].h->n0, st);
    const bool dist = M[0].s->dist_coarse;
    if (dist) {
      // E^{-1} distributed: each rank sweeps its subtrees forward (segment A), the
      // frontier roots' update vectors are summed over the ranks, every rank sweeps
      // the top forward and backward and its subtrees backward (segment B), and
      // the ranks' parts of the solution are summed (zeros elsewhere: exact)
      each([&](Member& m) {
        m.s->crs.sweep(m.h->xc.p, nullptr, st, m.h->state.p, 0);
        CUDA_CHECK(cudaMemsetAsync(m.s->ubuf.p, 0, m.s->ubuf.n * sizeof(double), st));
        const int64_t no = m.s->n_ux_own;
        if (no) k_scatter_owned<<<nblk(no, 256), 256, 0, st>>>(no, m.s->ux_pos.p, m.s->ux_own.p, m.s->crs.upd.p,
                                                               m.s->ubuf.p);
        launches += 2;
      });
      if (M[0].s->n_ux) {
        T.allreduce(M, [](Member& m) { return m.s->ubuf.p; }, M[0].s->n_ux, st);
        each([&](Member& m) {
          k_unpack_all<<<nblk(m.s->n_ux, 256), 256, 0, st>>>(m.s->n_ux, m.s->ux_pos.p, m.s->ubuf.p, m.s->crs.upd.p);
          ++launches;
        });
      }
      each([&](Member& m) {
        m.s->crs.sweep(m.h->xc.p, nullptr, st, m.h->state.p, 1);
        CUDA_CHECK(cudaMemsetAsync(m.s->ybuf.p, 0, m.s->ybuf.n * sizeof(double), st));
        if (m.s->n_y_own)
          k_scatter_owned<<<nblk(m.s->n_y_own, 256), 256, 0, st>>>(m.s->n_y_own, nullptr, m.s->y_own.p,
                                                                  m.s->crs.xb.p, m.s->ybuf.p);
        launches += 2;
      });
      T.allreduce(M, [](Member& m) { return m.s->ybuf.p; }, M[0].h->n0, st);
    }
    each([&](Member& m) {
      if (!dist) m.h->crs.sweep(m.h->xc.p, nullptr, st, m.h->state.p);
      const double* y = dist ? m.s->ybuf.p : m.h->crs.xb.p;
      dev::k_spmv8<<<m.h->nparts, 256, 0, st>>>(m.s->n_own, m.s->Z_ptr.p, m.s->Z_idx.p, m.s->Z_val.p,
                                               y, nullptr, m.s->u.p, nullptr, nullptr, m.h->state.p,
                                               mdd_solver::rnone());
      double* o = out(m);
      const double* a = add ? add(m) : nullptr;
      dev::k_axpby<<<nblk(m.s->n_own, 256), 256, 0, st>>>(m.s->n_own, 1.0, m.s->u.p, a ? 1.0 : 0.0,
                                                          a ? a : m.s->u.p, o, m.h->state.p);
      launches += 3;
    });
  }
  // z = M^{-1} r (coarse start: w + Q (r - A w)); r must be owned-complete
  void precond() {
    T.halo(M, [](Member& m) { return m.s->r.p; }, false, st);
    each([&](Member& m) { m.s->loc.sweep(m.s->r.p, m.s->w.p, st, m.h->state.p); ++launches; });
    T.halo(M, [](Member& m) { return m.s->w.p; }, true, st);    // owners add the overlap parts
    if (!coarse) {
      each([&](Member& m) {
        dev::k_copy<<<nblk(m.s->n_own, 256), 256, 0, st>>>(m.s->n_own, m.s->w.p, m.s->z.p, m.h->state.p);
        ++launches;
      });
      return;
    }
    T.halo(M, [](Member& m) { return m.s->w.p; }, false, st);   // the owners' sums back into the halos
    each([&](Member& m) { spmv_own(m, m.s->w.p, m.s->t.p, m.s->r.p); });   // t = r - A w
    coarse_apply([](Member& m) { return m.s->t.p; }, [](Member& m) { return m.s->z.p; },
                 [](Member& m) { return m.s->w.p; });
  }

  void run(const std::vector<const double*>& f, const std::vector<double*>& x, double tol, int maxit, bool host,
           int* iters, double* relres) {
    using namespace dev;
    // stage: x = 0, r = f (owned), S = {tol}, state = {maxit}
    each([&](Member& m) {
      mdd_solver* h = m.h;
      for (int k = 0; k < S_COUNT; ++k) h->host_S[k] = 0.0;
      h->host_S[S_TOL] = tol;
      for (int k = 0; k < ST_COUNT; ++k) h->host_state[k] = 0;
      h->host_state[ST_MAXIT] = maxit;
      CUDA_CHECK(cudaMemcpyAsync(h->S.p, h->host_S, S_COUNT * sizeof(double), cudaMemcpyHostToDevice, st));
      CUDA_CHECK(cudaMemcpyAsync(h->state.p, h->host_state, ST_COUNT * sizeof(int), cudaMemcpyHostToDevice, st));
      CUDA_CHECK(cudaStreamSynchronize(st));  // the pinned staging is reused by the next member
      for (DBuf<double>* b : {&m.s->x, &m.s->r, &m.s->p, &m.s->w})
        CUDA_CHECK(cudaMemsetAsync(b->p, 0, m.s->n_loc * sizeof(double), st));
    });
    for (size_t k = 0; k < M.size(); ++k)
      CUDA_CHECK(cudaMemcpyAsync(M[k].s->r.p, f[k], M[k].s->n_own * sizeof(double),
                                 host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
    auto vr = [](Member& m) { return m.s->r.p; };
    auto vz = [](Member& m) { return m.s->z.p; };
    auto vp = [](Member& m) { return m.s->p.p; };
    auto vq = [](Member& m) { return m.s->q.p; };
    // prologue: ||f||, x0 = Q f, r0 = f - A x0, z0, p0, r0.z0
    dot(vr, vr, S_RR);
    scalar(3);
    if (coarse) {
      coarse_apply(vr, [](Member& m) { return m.s->x.p; }, nullptr);
      T.halo(M, [](Member& m) { return m.s->x.p; }, false, st);
      each([&](Member& m) {
        spmv_own(m, m.s->x.p, m.s->t.p, m.s->r.p);
        dev::k_copy<<<nblk(m.s->n_own, 256), 256, 0, st>>>(m.s->n_own, m.s->t.p, m.s->r.p, m.h->state.p);
        ++launches;
      });
    }
    precond();
    each([&](Member& m) {
      dev::k_copy<<<nblk(m.s->n_own, 256), 256, 0, st>>>(m.s->n_own, m.s->z.p, m.s->p.p, m.h->state.p);
      ++launches;
    });
    dot(vr, vz, S_RZ);
    int* hs = M[0].h->host_state;
    for (int it = 0; it <= maxit + 1; ++it) {
      CUDA_CHECK(cudaMemcpyAsync(hs, M[0].h->state.p, ST_COUNT * sizeof(int), cudaMemcpyDeviceToHost, st));
      CUDA_CHECK(cudaStreamSynchronize(st));
      if (hs[ST_STOP]) break;
      T.halo(M, vp, false, st);
      each([&](Member& m) { spmv_own(m, m.s->p.p, m.s->q.p); });
      dot(vp, vq, S_PQ);
      scalar(0);
      each([&](Member& m) {
        dev::k_update_xr<<<m.h->nparts, 256, 0, st>>>(m.s->n_own, m.s->x.p, m.s->r.p, m.s->p.p, m.s->q.p, m.h->S.p,
                                                     m.h->part.p, m.h->state.p, mdd_solver::rnone());
        dev::k_reduce<<<1, 256, 0, st>>>(m.h->nparts, m.h->part.p, m.h->S.p + S_RR, m.h->state.p);
        launches += 2;
      });
      T.allreduce(M, [](Member& m) { return m.h->S.p + S_RR; }, 1, st);
      scalar(1);
      precond();
      dot(vr, vz, S_RZNEW);
      scalar(2);
      each([&](Member& m) {
        dev::k_update_p<<<m.h->nparts, 256, 0, st>>>(m.s->n_own, m.s->p.p, m.s->z.p, m.h->S.p, m.h->state.p);
        ++launches;
      });
    }
    for (size_t k = 0; k < M.size(); ++k)
      CUDA_CHECK(cudaMemcpyAsync(x[k], M[k].s->x.p, M[k].s->n_own * sizeof(double),
                                 host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, st));
    CUDA_CHECK(cudaMemcpyAsync(M[0].h->host_S, M[0].h->S.p, S_COUNT * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaMemcpyAsync(hs, M[0].h->state.p, ST_COUNT * sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    CUDA_CHECK(cudaGetLastError());
    for (auto& m : M) {
      m.s->loc.check_abort(st);
      if (m.h->has_coarse) m.h->crs.check_abort(st);
      if (m.s->dist_coarse) m.s->crs.check_abort(st);
    }
    *iters = hs[ST_ITERS];
    *relres = M[0].h->host_S[S_REL];
    for (auto& m : M) m.h->launches = launches;
    if (hs[ST_BREAKDOWN]) throw Error(MDD_ERR_BREAKDOWN, "PCG breakdown: p^T A p <= 0");
    if (!hs[ST_CONVERGED]) throw Error(MDD_ERR_NOCONV, "PCG did not converge within maxit");
  }
};

bool shard_coarse(mdd_solver* h) {
  MDD_REQUIRE(h->desc.variant == MDD_VARIANT_AS2_COARSE_START || h->desc.variant == MDD_VARIANT_AS1, 2,
              "the sharded solve runs MDD_VARIANT_AS2_COARSE_START (or AS1)");
  return h->has_coarse && h->desc.variant == MDD_VARIANT_AS2_COARSE_START;
}

int sguard(const std::function<void()>& f) {
  try {
    f();
    return MDD_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return MDD_ERR_INTERNAL;
  }
}

}  // namespace

}  // namespace mdd

extern "C" {

int mdd_shard_setup(mdd_handle h, int rank, int nranks) {
  if (!h) { mdd::set_last_error("null argument"); return MDD_ERR_ARG; }
  return mdd::sguard([&] { mdd::shard_setup(h, rank, nranks); });
}

int mdd_shard_info(mdd_handle h, int64_t* out, int count) {
  if (!h || !out || !h->shard) { mdd::set_last_error("null argument or no shard"); return MDD_ERR_ARG; }
  const mdd::ShardState& S = *h->shard;
  const int64_t v[8] = {S.n_own, S.n_loc, (int64_t)S.plan.subs.size(), S.loc.fp.factor_nnz(),
                        S.dist_coarse ? 1 : 0,
                        S.dist_coarse ? S.crs.swept_entries : (h->has_coarse ? h->crs.fp.factor_nnz() : 0),
                        S.top_entries, S.n_ux};
  for (int k = 0; k < count && k < 8; ++k) out[k] = v[k];
  return MDD_OK;
}

int mdd_shard_nccl_init(mdd_handle h, const void* unique_id, int rank, int nranks) {
  if (!h || !unique_id || !h->shard) { mdd::set_last_error("null argument or no shard"); return MDD_ERR_ARG; }
  return mdd::sguard([&] {
    MDD_REQUIRE(h->shard->plan.rank == rank && h->shard->plan.nranks == nranks, 2,
                "mdd_shard_nccl_init: rank / nranks differ from mdd_shard_setup");
    CUDA_CHECK(cudaSetDevice(h->device));
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    NCCL_OK(mdd::nccl().CommInitRank(&h->shard->comm, nranks, id, rank));
  });
}

int mdd_shard_solve(mdd_handle h, const double* f_own, double* x_own, double tol, int maxit, int host, int* iters,
                    double* relres) {
  if (!h || !f_own || !x_own || !iters || !relres || !h->shard) {
    mdd::set_last_error("null argument or no shard");
    return MDD_ERR_ARG;
  }
  return mdd::sguard([&] {
    MDD_REQUIRE(h->shard->comm != nullptr || h->shard->plan.nranks == 1, 2, "NCCL communicator not initialised");
    MDD_REQUIRE(tol > 0 && maxit >= 0, 2, "tol must be > 0 and maxit >= 0");
    CUDA_CHECK(cudaSetDevice(h->device));
    std::vector<mdd::Member> M{mdd::Member{h, h->shard}};
    mdd::NcclTransport nt;
    mdd::GroupTransport gt;  // one rank: every exchange is empty
    // NCCL whenever a communicator exists (also for one rank: the allreduces then
    // run through NCCL); without one, a single rank's exchanges are empty
    mdd::Transport& T = h->shard->comm ? (mdd::Transport&)nt : (mdd::Transport&)gt;
    mdd::ShardSolve S{M, T, h->stream, mdd::shard_coarse(h)};
    S.run({f_own}, {x_own}, tol, maxit, host != 0, iters, relres);
  });
}

int mdd_shard_solve_group(mdd_handle* hs, int count, const double* const* f_own, double* const* x_own, double tol,
                          int maxit, int* iters, double* relres) {
  if (!hs || count <= 0 || !f_own || !x_own || !iters || !relres) {
    mdd::set_last_error("null argument");
    return MDD_ERR_ARG;
  }
  return mdd::sguard([&] {
    std::vector<mdd::Member> M;
    std::vector<const double*> f;
    std::vector<double*> x;
    for (int k = 0; k < count; ++k) {
      MDD_REQUIRE(hs[k] && hs[k]->shard, 2, "every handle needs mdd_shard_setup");
      MDD_REQUIRE(hs[k]->shard->plan.rank == k && hs[k]->shard->plan.nranks == count, 2,
                  "handle k must be rank k of `count` ranks");
      MDD_REQUIRE(hs[k]->device == hs[0]->device, 2, "a group solve runs on one device");
      M.push_back(mdd::Member{hs[k], hs[k]->shard});
      f.push_back(f_own[k]);
      x.push_back(x_own[k]);
    }
    CUDA_CHECK(cudaSetDevice(hs[0]->device));
    const bool coarse = mdd::shard_coarse(hs[0]);
    for (int k = 1; k < count; ++k) MDD_REQUIRE(mdd::shard_coarse(hs[k]) == coarse, 2, "mixed variants");
    mdd::GroupTransport T;
    // every member's kernels go to member 0's stream, in rank order between exchanges
    CUDA_CHECK(cudaDeviceSynchronize());
    mdd::ShardSolve S{M, T, hs[0]->stream, coarse};
    S.run(f, x, tol, maxit, false, iters, relres);
  });
}

}  // extern "C"
