// The handle of the C ABI (struct mdd_solver): setup data, hot-path buffers and
// the PCG orchestration shared by api.cu and sharded.cu.
#pragma once
#include <cuda_runtime.h>
#include <cusparse.h>

#include <algorithm>
#include <cstdlib>
#include <functional>
#include <string>
#include <vector>

#include "../../include/maxwell_dd.h"
#include "device.h"
#include "topology.h"

namespace mdd {
inline int env_int(const char* k, int d) {
  const char* v = getenv(k);
  return v ? atoi(v) : d;
}
inline int nblk(int64_t n, int t) { return (int)std::max<int64_t>(1, (n + t - 1) / t); }
struct ShardState;
void shard_free(ShardState* s);
void set_last_error(const std::string& msg);   // the text mdd_last_error() returns (api.cu)
}  // namespace mdd

using namespace mdd;

struct mdd_solver {
  mdd_setup_desc desc;
  int device = 0;
  cudaStream_t stream = nullptr;
  cusparseHandle_t sp = nullptr;
  HostMesh mesh;
  Csr Apat;
  Decomp dec;
  std::vector<std::vector<int32_t>> grad_nodes;
  int n = 0;
  // A
  DBuf<int64_t> A_ptr;
  DBuf<int32_t> A_idx;
  DBuf<double> A_val, K_val, M_val;
  DBuf<double> Ke, Me;          // element matrices, kept until the GEVPs are done
  // local solves
  DevFactor loc;
  DBuf<int32_t> gmap;          // local position -> global dof
  DBuf<int64_t> pro_ptr;       // global dof -> list of local positions
  DBuf<int32_t> pro_pos;
  // coarse
  bool has_coarse = false;
  DevFactor crs;
  DBuf<int64_t> Z_ptr, Zt_ptr;  // setup only: mixed Z (n x n0, cols = coarse positions), Z^T
  DBuf<int32_t> Z_idx, Zt_idx;
  DBuf<double> Z_val, Zt_val;
  // hot path: gradient part of Z (CSR by dof and by coarse position) + dense GenEO blocks
  DBuf<int64_t> Zg_ptr, Zgt_ptr, W_off, W_poff;
  DBuf<int32_t> Zg_idx, Zgt_idx, W_gpos;
  DBuf<double> Zg_val, Zgt_val, W_val, u_loc;
  DBuf<int> W_n, W_k, W_gc0, W_cblk, W_cnch;
  DBuf<double> W_part;
  DBuf<int4> W_bzt, W_bz;
  int nbzt = 0, nbz = 0;
  int spmv_tpr = env_int("MDD_SPMV_TPR", 8);  // lanes per row of the A product (4 / 8 / 16)
  int64_t nnzZg = 0, nnzW = 0;
  int64_t n0 = 0, grad_cand = 0, grad_rank = 0, ngeneo = 0, nnzZ = 0, coarse_perturbed = 0;
  std::vector<int64_t> geneo_count;
  std::vector<double> geneo_lambda;
  bool geneo_lanczos = false;   // GenEO GEVPs by block Lanczos (else dense sygvdx)
  // parity diagnostics: the factorised (Jacobi-scaled) E in its original column
  // order (sorted pattern + value slots into E_val) and, per subdomain-major local
  // dof (sys_off[i] + k, k in N_i order), its position in the local factor
  Csr E_pat;
  std::vector<int64_t> E_slot;
  DBuf<double> E_val;
  DBuf<int64_t> loc_pos;
  // PCG work
  DBuf<double> x, r, p, q, z, t1, t2, t3, t4, xloc, xc, S, part;
  DBuf<int> state;
  DBuf<unsigned int> red_counter;  // last-block counter of the fused reduction tails (re-armed by them)
  // a reduction tail: S[slot] = sum of the producing kernel's block partials, then
  // the CG scalar step op, by its last block
  dev::RedStep rstep(int slot, int op) { return dev::RedStep{S.p, state.p, red_counter.p, slot, op}; }
  static dev::RedStep rnone() { return dev::RedStep{nullptr, nullptr, nullptr, 0, 0}; }
  int* state_host = nullptr;
  int nparts = 0;
  std::vector<double> setup_times;
  int64_t kernels_per_iter = 0;
  int64_t launches = 0;         // kernels launched by the last solve / apply call
  bool own_stream = true;
  bool profiling = false;
  double prof_ms[MDD_PROF_COUNT] = {0};
  int64_t prof_launch[MDD_PROF_COUNT] = {0};
  cudaEvent_t ev[16];
  // eager profiling: event pairs around the local / coarse applications of one
  // iteration (ev[7..15]); nullptr outside the profiling path
  std::vector<std::pair<int, int>>* prof_pairs = nullptr;
  int prof_next = 7;
  void prof_begin(int phase) {
    if (!prof_pairs || prof_next + 1 >= 16) return;
    CUDA_CHECK(cudaEventRecord(ev[prof_next], stream));
    prof_pairs->push_back({phase, prof_next});
    prof_next += 2;
  }
  void prof_end() {
    if (!prof_pairs || prof_pairs->empty()) return;
    CUDA_CHECK(cudaEventRecord(ev[prof_pairs->back().second + 1], stream));
  }
  // CUDA graph of the whole solve: prologue + device-side WHILE loop over iterations
  cudaGraphExec_t graph_exec = nullptr;
  cudaStream_t graph_stream = nullptr;
  int64_t launches_prologue = 0, launches_body = 0;
  double* host_S = nullptr;     // pinned staging of S / state
  int* host_state = nullptr;

  void drop_graph() {
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    graph_exec = nullptr;
    graph_stream = nullptr;
  }

  // sharded solve (sharded.cu): this rank's owned rows, halo plan, local factor
  // over its subdomains and exchange buffers; null for a single-GPU handle
  mdd::ShardState* shard = nullptr;

  ~mdd_solver() {
    mdd::shard_free(shard);
    drop_graph();
    if (host_S) cudaFreeHost(host_S);
    if (host_state) cudaFreeHost(host_state);
    if (state_host) cudaFreeHost(state_host);
    if (sp) cusparseDestroy(sp);
    if (profiling)
      for (auto& e : ev) cudaEventDestroy(e);
    if (stream && own_stream) cudaStreamDestroy(stream);
  }

  // ------------------------------------------------------------ helpers
  // A x with 8 lanes per row on an SM-sized grid (nparts blocks: the fused dot's
  // partials are reduced by the kernel's last block when rs is given)
  void spmv(const int64_t* ptr, const int32_t* idx, const double* val, int rows, const double* in,
            double* out, const double* dotw = nullptr, double* part_ = nullptr, const double* sub = nullptr,
            dev::RedStep rs = rnone()) {
    if (spmv_tpr == 4)
      dev::k_spmv4<<<nparts, 256, 0, stream>>>(rows, ptr, idx, val, in, sub, out, dotw, part_, state.p, rs);
    else if (spmv_tpr == 16)
      dev::k_spmv16<<<nparts, 256, 0, stream>>>(rows, ptr, idx, val, in, sub, out, dotw, part_, state.p, rs);
    else
      dev::k_spmv8<<<nparts, 256, 0, stream>>>(rows, ptr, idx, val, in, sub, out, dotw, part_, state.p, rs);
    launches += 1;
  }
  void applyA(const double* in, double* out) {
    spmv(A_ptr.p, A_idx.p, A_val.p, n, in, out);
  }
  // z = sum_i R_i^T A_i^{-1} R_i r: one persistent launch (gather, fwd, D^{-1}, bwd,
  // prolongation)
  void apply_local(const double* rr, double* zz) {
    prof_begin(MDD_PROF_LOCAL);
    loc.sweep(rr, zz, stream, state.p);
    prof_end();
    launches += 1;
  }
  // y = Z E^{-1} Z^T v: Z_g^T v (CSR) and Z_e^T v (tall-skinny over the GenEO blocks),
  // the sweep on E, then Z_g xc + prolongation of the GenEO blocks' W_i xc_i
  // (addw, dotw: y = addw + Q v and dotw . y partials into part, fused into the
  // last kernel; used by the PCG loop's coarse-start form)
  void apply_coarse(const double* v, double* y, const double* addw = nullptr, const double* dotw = nullptr,
                    dev::RedStep rs = rnone()) {
    prof_begin(MDD_PROF_COARSE);
    dev::k_spmv32<<<nparts, 256, 0, stream>>>((int)n0, Zgt_ptr.p, Zgt_idx.p, Zgt_val.p, v, nullptr, xc.p,
                                              nullptr, nullptr, state.p, rnone());
    if (nbzt) {
      dev::k_geneo_zt<<<nbzt, 256, 0, stream>>>(W_bzt.p, W_off.p, W_poff.p, W_n.p, W_gc0.p, W_gpos.p, W_val.p,
                                                gmap.p, v, W_part.p, state.p);
      dev::k_geneo_zt2<<<nblk(ngeneo, 128), 128, 0, stream>>>((int)ngeneo, W_cblk.p, W_cnch.p, W_gpos.p,
                                                              W_part.p, xc.p, state.p);
    }
    crs.sweep(xc.p, nullptr, stream, state.p);
    if (nbz)
      dev::k_geneo_z<<<nbz, 256, 0, stream>>>(W_bz.p, W_off.p, W_poff.p, W_n.p, W_k.p, W_gc0.p, W_gpos.p,
                                              W_val.p, crs.xb.p, u_loc.p, state.p);
    dev::k_z_apply<<<nparts, 256, 0, stream>>>(n, Zg_ptr.p, Zg_idx.p, Zg_val.p, crs.xb.p, pro_ptr.p, pro_pos.p,
                                              nbz ? u_loc.p : nullptr, addw, y, dotw, dotw ? part.p : nullptr,
                                              state.p, rs);
    prof_end();
    launches += 3 + (nbzt ? 2 : 0) + (nbz ? 1 : 0);
  }
  void apply_prec(const double* rr, double* zz) {
    int v = desc.variant;
    if (!has_coarse || v == MDD_VARIANT_AS1) {
      apply_local(rr, zz);
      return;
    }
    if (v == MDD_VARIANT_ADDITIVE) {
      apply_local(rr, t4.p);
      apply_coarse(rr, t1.p);
      dev::k_axpby<<<nblk(n, 256), 256, 0, stream>>>(n, 1.0, t4.p, 1.0, t1.p, zz, state.p);
      launches += 1;
      return;
    }
    // eq. (2.4): z = Q r + (I - Q A) M_AS (I - A Q) r
    apply_coarse(rr, t1.p);                                        // t1 = Q r
    applyA(t1.p, t2.p);                                            // t2 = A Q r
    dev::k_axpby<<<nblk(n, 256), 256, 0, stream>>>(n, 1.0, rr, -1.0, t2.p, t3.p, state.p);  // t3 = r - A Q r
    apply_local(t3.p, t4.p);                                       // t4 = w
    applyA(t4.p, t2.p);                                            // t2 = A w
    apply_coarse(t2.p, t3.p);                                      // t3 = Q A w
    dev::k_combine3<<<nblk(n, 256), 256, 0, stream>>>(n, t1.p, t4.p, t3.p, zz, state.p);
    launches += 2;  // axpby + combine3
  }
  bool coarse_start() const { return has_coarse && desc.variant == MDD_VARIANT_AS2_COARSE_START; }
  // the preconditioner inside the PCG loop: for the coarse start (Z^T r = 0,
  // reading R13) eq. (2.4) is z = w + Q (r - A w), w = M_AS r
  // (rs: the r . z reduction tail the coarse-start form runs inside its last kernel)
  void apply_prec_loop(const double* rr, double* zz, dev::RedStep rs = rnone()) {
    if (!coarse_start()) {
      apply_prec(rr, zz);
      return;
    }
    apply_local(rr, t4.p);                                         // w = M_AS r
    spmv(A_ptr.p, A_idx.p, A_val.p, n, t4.p, t3.p, nullptr, nullptr, rr);  // r - A w
    apply_coarse(t3.p, zz, t4.p, rr, rs);   // z = w + Q (r - A w), with the r . z partials
  }
  // r . z after apply_prec_loop: the coarse-start form left its partials in part
  // (the coarse-start loop already reduced it inside apply_prec_loop)
  void dot_rz(int slot, int op) {
    if (coarse_start()) return;
    dev::k_dot_part<<<nparts, 256, 0, stream>>>(n, r.p, z.p, part.p, state.p, rstep(slot, op));
    launches += 1;
  }
  void check_aborts() {
    loc.check_abort(stream);
    if (has_coarse) crs.check_abort(stream);
  }
  void dot(const double* a, const double* b, int slot) {
    dev::k_dot_part<<<nparts, 256, 0, stream>>>(n, a, b, part.p, state.p, rnone());
    dev::k_reduce<<<1, 256, 0, stream>>>(nparts, part.p, S.p + slot, state.p);
    launches += 2;
  }
  // ---------------------------------------------------------------- PCG
  // prologue (x = 0 and r = f staged by the host): ||f||, z = M r, p = z, rz
  void enqueue_prologue() {
    dev::k_dot_part<<<nparts, 256, 0, stream>>>(n, r.p, r.p, part.p, state.p, rstep(dev::S_RR, 3));
    launches += 1;
    if (coarse_start()) {
      // x0 = Q f, r0 = f - A x0 (the staged x is 0; reading R13)
      apply_coarse(r.p, x.p);
      spmv(A_ptr.p, A_idx.p, A_val.p, n, x.p, t3.p, nullptr, nullptr, r.p);
      dev::k_copy<<<nblk(n, 256), 256, 0, stream>>>(n, t3.p, r.p, state.p);
      launches += 1;
    }
    apply_prec_loop(r.p, z.p);
    dev::k_copy<<<nblk(n, 256), 256, 0, stream>>>(n, z.p, p.p, state.p);
    launches += 1;
    dot(r.p, z.p, dev::S_RZ);
  }
  // one PCG iteration; every kernel is a no-op once state[ST_STOP] is set.
  // marks: optional event indices for the eager profiling path
  void enqueue_body(const std::function<void(int)>& mark) {
    if (mark) mark(2);
    spmv(A_ptr.p, A_idx.p, A_val.p, n, p.p, q.p, p.p, part.p, nullptr, rstep(dev::S_PQ, 0));
    if (mark) mark(3);
    dev::k_update_xr<<<nparts, 256, 0, stream>>>(n, x.p, r.p, p.p, q.p, S.p, part.p, state.p,
                                                 rstep(dev::S_RR, 1));
    launches += 1;
    if (mark) mark(4);
    apply_prec_loop(r.p, z.p, rstep(dev::S_RZNEW, 2));
    if (mark) mark(5);
    dot_rz(dev::S_RZNEW, 2);
    dev::k_update_p<<<nparts, 256, 0, stream>>>(n, p.p, z.p, S.p, state.p);
    launches += 1;
    if (mark) mark(6);
  }
  // graph: prologue -> WHILE(state not stopped) { body ; k_loop_cond }
  void build_graph() {
    drop_graph();
    cudaGraph_t g;
    CUDA_CHECK(cudaGraphCreate(&g, 0));
    launches = 0;
    CUDA_CHECK(cudaStreamBeginCaptureToGraph(stream, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    enqueue_prologue();
    CUDA_CHECK(cudaStreamEndCapture(stream, &g));
    launches_prologue = launches;
    // sinks of the prologue
    size_t nn = 0, ne = 0;
    CUDA_CHECK(cudaGraphGetNodes(g, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    CUDA_CHECK(cudaGraphGetNodes(g, nodes.data(), &nn));
    CUDA_CHECK(cudaGraphGetEdges(g, nullptr, nullptr, &ne));
    std::vector<cudaGraphNode_t> from(ne), to(ne);
    if (ne) CUDA_CHECK(cudaGraphGetEdges(g, from.data(), to.data(), &ne));
    std::vector<cudaGraphNode_t> sinks;
    for (auto nd : nodes)
      if (std::find(from.begin(), from.end(), nd) == from.end()) sinks.push_back(nd);
    cudaGraphConditionalHandle h;
    CUDA_CHECK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cn;
    CUDA_CHECK(cudaGraphAddNode(&cn, g, sinks.data(), sinks.size(), &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    launches = 0;
    CUDA_CHECK(cudaStreamBeginCaptureToGraph(stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    enqueue_body(nullptr);
    dev::k_loop_cond<<<1, 1, 0, stream>>>(h, state.p);
    launches += 1;
    CUDA_CHECK(cudaStreamEndCapture(stream, &body));
    launches_body = launches;
    CUDA_CHECK(cudaGraphInstantiate(&graph_exec, g, 0));
    CUDA_CHECK(cudaGraphDestroy(g));
    graph_stream = stream;
  }
};
