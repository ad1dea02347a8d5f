// Symbolic phase of the supernodal LDL^T (host, integer work): geometric
// nested-dissection ordering, elimination tree, postorder, column structures,
// fundamental + relaxed supernodes, the level schedule, the extend-add
// relative maps and the assembly map.  The numeric work (factorisation and the
// triangular solves of the hot path) runs in CUDA kernels (kernels.cu: the
// multifrontal factorisation, factor_driver.cu: its driver, sweep.cu: the sweeps).
//
// North star: "the local solves A_i^{-1} as supernodal sparse LDL^T factors
// applied by hand-written level-scheduled triangular-solve kernels".
#include "common.h"

#include <cstdlib>

#include <algorithm>
#include <map>
#include <numeric>

namespace mdd {

i64 FactorPlan::factor_nnz() const {
  i64 s = 0;
  for (int k = 0; k < nsn; ++k) {
    i64 nc = sn_ncol[k], no = sn_noff[k];
    s += nc * (nc + 1) / 2 + nc * no;
  }
  return s;
}

namespace {

struct NDWork {
  const Csr* pat;
  const int32_t* xyz2;
  const int32_t* box = nullptr;  // deferred unknowns' coupling boxes (SymSystem::box)
  int search_min = 0;            // > 0: sets this large search their cut plane (below)
  std::vector<int32_t> side;   // per vertex: -1 not in current set, 0 left, 1 right, 2 sep
  std::vector<int32_t> order;  // output: new -> old
  int leaf;
};

// V: unknowns to dissect; T: deferred unknowns whose coupling box lies inside
// this subtree's region (ordered after the subtree's separator)
void nd_rec(NDWork& w, std::vector<int32_t>& V, std::vector<int32_t>& T) {
  const size_t nv = V.size();
  auto close = [&]() {
    std::sort(T.begin(), T.end());
    w.order.insert(w.order.end(), T.begin(), T.end());
  };
  if (nv == 0) { close(); return; }
  if ((int)nv <= w.leaf) {
    std::sort(V.begin(), V.end());
    w.order.insert(w.order.end(), V.begin(), V.end());
    close();
    return;
  }
  int lo[3] = {INT32_MAX, INT32_MAX, INT32_MAX}, hi[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
  for (int32_t v : V)
    for (int d = 0; d < 3; ++d) {
      lo[d] = std::min(lo[d], w.xyz2[3 * v + d]);
      hi[d] = std::max(hi[d], w.xyz2[3 * v + d]);
    }
  int axis = 0;
  for (int d = 1; d < 3; ++d)
    if (hi[d] - lo[d] > hi[axis] - lo[axis]) axis = d;
  std::vector<int32_t> L, R, S;
  bool done = false;
  if (hi[axis] > lo[axis]) {
    std::vector<int32_t> cs(nv);
    for (size_t k = 0; k < nv; ++k) cs[k] = w.xyz2[3 * V[k] + axis];
    std::nth_element(cs.begin(), cs.begin() + nv / 2, cs.end());
    int med = cs[nv / 2];
    // prefer an even (node-plane) value: in-plane edges then form an exact separator
    int cand[3] = {med - (med & 1), med + (med & 1), med};
    if (w.search_min > 0 && (i64)nv >= w.search_min && w.box) {
      // the coarse system: the median plane of a box partition lies on subdomain
      // boundaries, where every node has a copy per overlapping subdomain and every
      // adjacent subdomain's GenEO columns cross the cut.  Take, among the node
      // planes of the middle half, the one with the smallest separator + crossing
      // deferred columns (the dense root and its ancestors grow with its square).
      for (int32_t v : V) w.side[v] = 0;
      std::vector<int32_t> maxc(nv);
      for (size_t k = 0; k < nv; ++k) {
        const int32_t v = V[k];
        int32_t m2 = w.xyz2[3 * v + axis];
        for (i64 p = w.pat->ptr[v]; p < w.pat->ptr[v + 1]; ++p) {
          const int32_t u = w.pat->idx[p];
          if (w.side[u] >= 0) m2 = std::max(m2, w.xyz2[3 * u + axis]);
        }
        maxc[k] = m2;
      }
      for (int32_t v : V) w.side[v] = -1;
      std::vector<int32_t> sc(cs);
      std::sort(sc.begin(), sc.end());
      const int32_t qlo = sc[nv / 4], qhi = sc[(3 * nv) / 4];
      i64 best = INT64_MAX;
      int bs = cand[0];
      for (int32_t sp = qlo + (qlo & 1); sp <= qhi; sp += 2) {
        i64 nl = 0, nr = 0, ns = 0;
        for (size_t k = 0; k < nv; ++k) {
          const int32_t c = w.xyz2[3 * V[k] + axis];
          if (c == sp) ++ns;
          else if (c > sp) ++nr;
          else if (maxc[k] > sp) ++ns;
          else ++nl;
        }
        if (4 * nl < (i64)nv || 4 * nr < (i64)nv) continue;
        i64 nts = 0;
        for (int32_t t : T) {
          const int32_t* b = w.box + 6 * t;
          if (!(b[3 + axis] < sp) && !(b[axis] > sp)) ++nts;
        }
        const i64 score = ns + nts;
        if (score < best || (score == best && std::abs(sp - med) < std::abs(bs - med))) { best = score; bs = sp; }
      }
      cand[0] = bs;
    }
    for (int ci = 0; ci < 3 && !done; ++ci) {
      int s = cand[ci];
      L.clear(); R.clear(); S.clear();
      for (int32_t v : V) {
        int c = w.xyz2[3 * v + axis];
        if (c < s) L.push_back(v); else if (c > s) R.push_back(v); else S.push_back(v);
      }
      if (L.empty() || R.empty()) continue;
      for (int32_t v : L) w.side[v] = 0;
      for (int32_t v : R) w.side[v] = 1;
      for (int32_t v : S) w.side[v] = 2;
      // vertices of L adjacent to R join the separator
      std::vector<int32_t> L2;
      for (int32_t v : L) {
        bool cross = false;
        for (i64 p = w.pat->ptr[v]; p < w.pat->ptr[v + 1]; ++p)
          if (w.side[w.pat->idx[p]] == 1) { cross = true; break; }
        if (cross) S.push_back(v); else L2.push_back(v);
      }
      L.swap(L2);
      for (int32_t v : V) w.side[v] = -1;
      if (S.size() < nv) done = true;
    }
  }
  if (!done) {  // cannot split geometrically: dense leaf
    std::sort(V.begin(), V.end());
    w.order.insert(w.order.end(), V.begin(), V.end());
    close();
    return;
  }
  // deferred unknowns strictly on one side of the cut plane go down with it
  std::vector<int32_t> TL, TR, TS;
  int plane = 0;
  if (!T.empty()) {
    // the cut value: the largest L coordinate + 1 .. smallest R coordinate - 1
    int lmax = INT32_MIN, rmin = INT32_MAX;
    for (int32_t v : L) lmax = std::max(lmax, w.xyz2[3 * v + axis]);
    for (int32_t v : R) rmin = std::min(rmin, w.xyz2[3 * v + axis]);
    plane = L.empty() ? rmin - 1 : lmax + 1;
    for (int32_t t : T) {
      const int32_t* b = w.box + 6 * t;
      if (b[3 + axis] < plane && !L.empty()) TL.push_back(t);
      else if (b[axis] > std::max(plane, rmin - 1) && !R.empty()) TR.push_back(t);
      else TS.push_back(t);
    }
    std::vector<int32_t>().swap(T);
  }
  std::vector<int32_t>().swap(V);
  nd_rec(w, L, TL);
  nd_rec(w, R, TR);
  std::sort(S.begin(), S.end());
  w.order.insert(w.order.end(), S.begin(), S.end());
  std::sort(TS.begin(), TS.end());
  w.order.insert(w.order.end(), TS.begin(), TS.end());
}

// elimination tree of the symmetric matrix P A P^T (Liu); pattern given in the new numbering
void etree(int n, const std::vector<i64>& ptr, const std::vector<int32_t>& idx, std::vector<int32_t>& parent) {
  parent.assign(n, -1);
  std::vector<int32_t> anc(n, -1);
  for (int k = 0; k < n; ++k) {
    for (i64 p = ptr[k]; p < ptr[k + 1]; ++p) {
      int i = idx[p];
      if (i >= k) continue;
      while (i != -1 && i < k) {
        int nxt = anc[i];
        anc[i] = k;
        if (nxt == -1) parent[i] = k;
        i = nxt;
      }
    }
  }
}

struct Sys1 {
  int n;
  std::vector<int32_t> perm;                 // new -> old
  std::vector<int32_t> parent;               // etree (new numbering)
  std::vector<std::vector<int32_t>> cstruct; // strictly-lower row structure per column
  // supernodes
  std::vector<int32_t> sfirst, slast;        // inclusive column ranges
  std::vector<std::vector<int32_t>> soff;    // off rows (local new numbering)
  std::vector<int32_t> sparent;
};

void analyse_one(Sys1& s, const SymSystem& sys, int leaf) {
  const Csr& A = *sys.pat;
  const int n = A.nrows;
  s.n = n;
  NDWork w;
  w.pat = &A; w.xyz2 = sys.xyz2; w.leaf = leaf; w.box = sys.box;
  w.search_min = getenv("MDD_ND_SEARCH") ? atoi(getenv("MDD_ND_SEARCH")) : 20000;
  w.side.assign(n, -1);
  std::vector<int32_t> V, tail, none;
  for (int v = 0; v < n; ++v) (sys.last && sys.last[v] ? tail : V).push_back(v);
  if (sys.box) {
    // flagged unknowns close the smallest subtree containing their coupling box
    nd_rec(w, V, tail);
  } else {
    // flagged unknowns (e.g. dense-support coarse columns) close the order, so
    // their coupling never creates a clique inside the dissection
    nd_rec(w, V, none);
    w.order.insert(w.order.end(), tail.begin(), tail.end());
  }
  MDD_REQUIRE((int)w.order.size() == n, 5, "nested dissection lost vertices");
  std::vector<int32_t> perm = w.order, iperm(n);
  // etree + postorder, twice (the second pass is a no-op relabel check)
  for (int pass = 0; pass < 2; ++pass) {
    for (int k = 0; k < n; ++k) iperm[perm[k]] = k;
    std::vector<i64> ptr(n + 1, 0);
    std::vector<int32_t> idx;
    idx.reserve(A.nnz());
    for (int k = 0; k < n; ++k) {
      int o = perm[k];
      for (i64 p = A.ptr[o]; p < A.ptr[o + 1]; ++p) idx.push_back(iperm[A.idx[p]]);
      ptr[k + 1] = (i64)idx.size();
    }
    std::vector<int32_t> parent;
    etree(n, ptr, idx, parent);
    // postorder (children visited in increasing order)
    std::vector<int32_t> head(n, -1), next(n, -1), post;
    post.reserve(n);
    for (int j = n - 1; j >= 0; --j)
      if (parent[j] != -1) { next[j] = head[parent[j]]; head[parent[j]] = j; }
    std::vector<int32_t> stack;
    for (int r = 0; r < n; ++r) {
      if (parent[r] != -1) continue;
      stack.push_back(r);
      while (!stack.empty()) {
        int t = stack.back();
        if (head[t] != -1) { int c = head[t]; head[t] = next[c]; stack.push_back(c); }
        else { stack.pop_back(); post.push_back(t); }
      }
    }
    std::vector<int32_t> np(n);
    for (int k = 0; k < n; ++k) np[k] = perm[post[k]];
    perm.swap(np);
    if (pass == 1) {
      for (int k = 0; k < n; ++k) iperm[perm[k]] = k;
      s.parent.assign(n, -1);
      // recompute on final labels
      std::vector<i64> ptr2(n + 1, 0);
      std::vector<int32_t> idx2;
      idx2.reserve(A.nnz());
      for (int k = 0; k < n; ++k) {
        int o = perm[k];
        for (i64 p = A.ptr[o]; p < A.ptr[o + 1]; ++p) idx2.push_back(iperm[A.idx[p]]);
        ptr2[k + 1] = (i64)idx2.size();
      }
      etree(n, ptr2, idx2, s.parent);
      for (int k = 0; k < n; ++k)
        MDD_REQUIRE(s.parent[k] == -1 || s.parent[k] > k, 5, "postorder violated");
      // column structures
      s.cstruct.assign(n, {});
      std::vector<std::vector<int32_t>> kids(n);
      for (int k = 0; k < n; ++k)
        if (s.parent[k] != -1) kids[s.parent[k]].push_back(k);
      std::vector<int32_t> mark(n, -1);
      for (int j = 0; j < n; ++j) {
        std::vector<int32_t>& st = s.cstruct[j];
        mark[j] = j;
        for (i64 p = ptr2[j]; p < ptr2[j + 1]; ++p) {
          int i = idx2[p];
          if (i > j && mark[i] != j) { mark[i] = j; st.push_back(i); }
        }
        for (int c : kids[j])
          for (int i : s.cstruct[c])
            if (i > j && mark[i] != j) { mark[i] = j; st.push_back(i); }
        std::sort(st.begin(), st.end());
      }
    }
  }
  s.perm = perm;
  // fundamental supernodes
  std::vector<int32_t> nkids(n, 0);
  for (int k = 0; k < n; ++k)
    if (s.parent[k] != -1) nkids[s.parent[k]]++;
  std::vector<int32_t> sn_of(n);
  for (int j = 0; j < n; ++j) {
    bool join = j > 0 && s.parent[j - 1] == j && nkids[j] == 1 &&
                s.cstruct[j - 1].size() == s.cstruct[j].size() + 1;
    if (join) { s.slast.back() = j; }
    else { s.sfirst.push_back(j); s.slast.push_back(j); }
    sn_of[j] = (int)s.sfirst.size() - 1;
  }
  int ns = (int)s.sfirst.size();
  auto off_of = [&](int k) {
    std::vector<int32_t> o;
    for (int i : s.cstruct[s.slast[k]]) o.push_back(i);
    return o;
  };
  std::vector<std::vector<int32_t>> off(ns);
  std::vector<int32_t> spar(ns, -1);
  for (int k = 0; k < ns; ++k) {
    off[k] = off_of(k);
    int pj = s.parent[s.slast[k]];
    spar[k] = pj == -1 ? -1 : sn_of[pj];
  }
  // relaxed amalgamation: merge a supernode into its parent when contiguous and
  // the explicit zeros added are few
  std::vector<int32_t> alive(ns, 1), first = s.sfirst, last = s.slast;
  std::vector<int32_t> rep(ns);
  std::iota(rep.begin(), rep.end(), 0);
  auto find = [&](int a) { while (rep[a] != a) { rep[a] = rep[rep[a]]; a = rep[a]; } return a; };
  for (int k = 0; k < ns; ++k) {
    if (spar[k] == -1) continue;
    int p = find(spar[k]);
    if (last[k] + 1 != first[p]) continue;
    i64 nck = last[k] - first[k] + 1, ncp = last[p] - first[p] + 1;
    i64 nok = (i64)off[k].size(), nop = (i64)off[p].size();
    i64 nc = nck + ncp;
    i64 merged = (nc * (nc + 1)) / 2 + nc * nop;
    i64 orig = (nck * (nck + 1)) / 2 + nck * nok + (ncp * (ncp + 1)) / 2 + ncp * nop;
    i64 z = merged - orig;
    // relaxed amalgamation (MDD_AMALG=1: more aggressive, fewer levels and supernodes
    // for the latency-bound sweep at the cost of explicit zeros)
    static const int aggressive = getenv("MDD_AMALG") ? atoi(getenv("MDD_AMALG")) : 0;
    bool ok = aggressive ? ((nc <= 16) || (nc <= 64 && z * 3 <= merged) || (z * 8 <= merged))
                         : ((nc <= 8) || (nc <= 32 && z * 5 <= merged) || (z * 20 <= merged));
    if (!ok) continue;
    first[p] = first[k];
    alive[k] = 0;
    rep[k] = p;
  }
  for (int k = 0; k < ns; ++k)
    if (alive[k]) {
      s.sfirst.push_back(0);  // placeholder, rebuilt below
    }
  s.sfirst.clear(); s.slast.clear(); s.soff.clear(); s.sparent.clear();
  std::vector<int32_t> newid(ns, -1);
  for (int k = 0; k < ns; ++k)
    if (alive[k]) {
      newid[k] = (int)s.sfirst.size();
      s.sfirst.push_back(first[k]);
      s.slast.push_back(last[k]);
      s.soff.push_back(off[k]);
    }
  for (int k = 0; k < ns; ++k)
    if (alive[k]) s.sparent.push_back(spar[k] == -1 ? -1 : newid[find(spar[k])]);
  // the surviving order is ascending in columns; parents come after children
  for (size_t k = 0; k < s.sparent.size(); ++k)
    MDD_REQUIRE(s.sparent[k] == -1 || s.sparent[k] > (int)k, 5, "supernode order violated");
  s.cstruct.clear();
  s.cstruct.shrink_to_fit();
}

}  // namespace

void build_factor_plan(FactorPlan& fp, const std::vector<SymSystem>& systems, int leaf_size) {
  fp = FactorPlan();
  fp.nsys = (int)systems.size();
  std::vector<Sys1> S(fp.nsys);
  fp.sys_off.assign(fp.nsys + 1, 0);
  for (int q = 0; q < fp.nsys; ++q) {
    analyse_one(S[q], systems[q], leaf_size);
    fp.sys_off[q + 1] = fp.sys_off[q] + S[q].n;
  }
  fp.ntot = fp.sys_off[fp.nsys];
  fp.perm.resize(fp.ntot);
  fp.iperm_global.resize(fp.ntot);
  for (int q = 0; q < fp.nsys; ++q)
    for (int k = 0; k < S[q].n; ++k) {
      fp.perm[fp.sys_off[q] + k] = S[q].perm[k];
      fp.iperm_global[fp.sys_off[q] + S[q].perm[k]] = (int32_t)(fp.sys_off[q] + k);
    }
  // supernodes, system by system
  std::vector<int> sn_base(fp.nsys + 1, 0);
  for (int q = 0; q < fp.nsys; ++q) sn_base[q + 1] = sn_base[q] + (int)S[q].sfirst.size();
  fp.nsn = sn_base[fp.nsys];
  fp.sn_col0.resize(fp.nsn); fp.sn_ncol.resize(fp.nsn); fp.sn_noff.resize(fp.nsn);
  fp.sn_parent.resize(fp.nsn); fp.sn_level.assign(fp.nsn, 0);
  fp.sn_rowptr.assign(fp.nsn + 1, 0);
  for (int q = 0; q < fp.nsys; ++q)
    for (size_t k = 0; k < S[q].sfirst.size(); ++k) {
      int g = sn_base[q] + (int)k;
      fp.sn_col0[g] = fp.sys_off[q] + S[q].sfirst[k];
      fp.sn_ncol[g] = S[q].slast[k] - S[q].sfirst[k] + 1;
      fp.sn_noff[g] = (int32_t)S[q].soff[k].size();
      fp.sn_parent[g] = S[q].sparent[k] == -1 ? -1 : sn_base[q] + S[q].sparent[k];
      fp.sn_rowptr[g + 1] = fp.sn_rowptr[g] + fp.sn_noff[g];
    }
  fp.offrows.resize(fp.sn_rowptr[fp.nsn]);
  for (int q = 0; q < fp.nsys; ++q)
    for (size_t k = 0; k < S[q].sfirst.size(); ++k) {
      int g = sn_base[q] + (int)k;
      i64 o = fp.sn_rowptr[g];
      for (int r : S[q].soff[k]) fp.offrows[o++] = fp.sys_off[q] + r;
    }
  // levels (leaves 0)
  for (int g = 0; g < fp.nsn; ++g)
    if (fp.sn_parent[g] != -1)
      fp.sn_level[fp.sn_parent[g]] = std::max(fp.sn_level[fp.sn_parent[g]], fp.sn_level[g] + 1);
  fp.nlevels = 0;
  for (int g = 0; g < fp.nsn; ++g) fp.nlevels = std::max(fp.nlevels, fp.sn_level[g] + 1);
  fp.level_ptr.assign(fp.nlevels + 1, 0);
  for (int g = 0; g < fp.nsn; ++g) fp.level_ptr[fp.sn_level[g] + 1]++;
  for (int l = 0; l < fp.nlevels; ++l) fp.level_ptr[l + 1] += fp.level_ptr[l];
  fp.level_sn.resize(fp.nsn);
  {
    std::vector<int32_t> cur(fp.level_ptr.begin(), fp.level_ptr.end() - 1);
    for (int g = 0; g < fp.nsn; ++g) fp.level_sn[cur[fp.sn_level[g]]++] = g;
  }
  // children, buffers
  fp.child_ptr.assign(fp.nsn + 1, 0);
  for (int g = 0; g < fp.nsn; ++g)
    if (fp.sn_parent[g] != -1) fp.child_ptr[fp.sn_parent[g] + 1]++;
  for (int g = 0; g < fp.nsn; ++g) fp.child_ptr[g + 1] += fp.child_ptr[g];
  fp.child_list.resize(fp.child_ptr[fp.nsn]);
  {
    std::vector<i64> cur(fp.child_ptr.begin(), fp.child_ptr.end() - 1);
    for (int g = 0; g < fp.nsn; ++g)
      if (fp.sn_parent[g] != -1) fp.child_list[cur[fp.sn_parent[g]]++] = g;
  }
  fp.sn_lptr.assign(fp.nsn + 1, 0);
  fp.sn_uptr.assign(fp.nsn + 1, 0);
  fp.sn_fptr.assign(fp.nsn + 1, 0);
  fp.sn_umptr.assign(fp.nsn + 1, 0);
  for (int g = 0; g < fp.nsn; ++g) {
    i64 nc = fp.sn_ncol[g], no = fp.sn_noff[g], nr = nc + no;
    fp.sn_lptr[g + 1] = fp.sn_lptr[g] + nr * nc;
    fp.sn_uptr[g + 1] = fp.sn_uptr[g] + no;
    fp.sn_fptr[g + 1] = fp.sn_fptr[g] + nr * nr;
    fp.sn_umptr[g + 1] = fp.sn_umptr[g] + no * no;
  }
  fp.lsize = fp.sn_lptr[fp.nsn];
  fp.usize = fp.sn_uptr[fp.nsn];
  // The numeric factorisation runs level by level, so a front is live during its
  // level only (level-local offsets; peak = the largest level), and an update
  // matrix from its supernode's level until its parent's level has assembled it
  // (first-fit offsets over those lifetimes; peak = the most live at one level).
  // Summing every front and update matrix instead ran out of the 180 GB on the
  // c4 coarse factor.
  {
    i64 fmax = 0;
    for (int l = 0; l < fp.nlevels; ++l) {
      i64 off = 0;
      for (int k = fp.level_ptr[l]; k < fp.level_ptr[l + 1]; ++k) {
        const int g = fp.level_sn[k];
        const i64 nr = (i64)fp.sn_ncol[g] + fp.sn_noff[g];
        fp.sn_fptr[g] = off;
        off += nr * nr;
      }
      fmax = std::max(fmax, off);
    }
    fp.sn_fptr[fp.nsn] = fmax;
    fp.fsize = fmax;
    std::map<i64, i64> freel;  // offset -> length of the free blocks
    i64 top = 0;
    std::vector<std::vector<int>> release(fp.nlevels + 2);
    auto give_back = [&](i64 off, i64 len) {
      auto it = freel.emplace(off, len).first;
      auto nx = std::next(it);
      if (nx != freel.end() && it->first + it->second == nx->first) { it->second += nx->second; freel.erase(nx); }
      if (it != freel.begin()) {
        auto pv = std::prev(it);
        if (pv->first + pv->second == it->first) { pv->second += it->second; freel.erase(it); }
      }
    };
    for (int l = 0; l < fp.nlevels; ++l) {
      for (int g : release[l]) give_back(fp.sn_umptr[g], (i64)fp.sn_noff[g] * fp.sn_noff[g]);
      for (int k = fp.level_ptr[l]; k < fp.level_ptr[l + 1]; ++k) {
        const int g = fp.level_sn[k];
        const i64 len = (i64)fp.sn_noff[g] * fp.sn_noff[g];
        if (len == 0) { fp.sn_umptr[g] = 0; continue; }
        auto it = freel.begin();
        while (it != freel.end() && it->second < len) ++it;
        if (it != freel.end()) {
          const i64 off = it->first, rest = it->second - len;
          freel.erase(it);
          if (rest > 0) freel.emplace(off + len, rest);
          fp.sn_umptr[g] = off;
        } else {
          fp.sn_umptr[g] = top;
          top += len;
        }
        const int lp = fp.sn_parent[g] == -1 ? l : fp.sn_level[fp.sn_parent[g]];
        release[lp + 1].push_back(g);
      }
    }
    fp.sn_umptr[fp.nsn] = top;
    fp.umsize = top;
  }
  // relative maps: position of each off row of g in its parent's row list
  fp.relmap_ptr = fp.sn_rowptr;
  fp.relmap.assign(fp.offrows.size(), -1);
  for (int g = 0; g < fp.nsn; ++g) {
    int p = fp.sn_parent[g];
    if (p == -1) { MDD_REQUIRE(fp.sn_noff[g] == 0, 5, "root supernode with off rows"); continue; }
    const i64* po = &fp.offrows[fp.sn_rowptr[p]];
    int nop = fp.sn_noff[p];
    for (i64 k = fp.sn_rowptr[g]; k < fp.sn_rowptr[g + 1]; ++k) {
      i64 r = fp.offrows[k];
      int pos;
      if (r >= fp.sn_col0[p] && r < fp.sn_col0[p] + fp.sn_ncol[p]) pos = (int)(r - fp.sn_col0[p]);
      else {
        const i64* it = std::lower_bound(po, po + nop, r);
        MDD_REQUIRE(it != po + nop && *it == r, 5, "child row missing from parent structure");
        pos = fp.sn_ncol[p] + (int)(it - po);
      }
      fp.relmap[k] = pos;
    }
  }
  // assembly map: lower entries (new row >= new col) of every system
  fp.asm_ptr.assign(fp.nsn + 1, 0);
  std::vector<int32_t> sn_of_pos(fp.ntot);
  for (int g = 0; g < fp.nsn; ++g)
    for (int c = 0; c < fp.sn_ncol[g]; ++c) sn_of_pos[fp.sn_col0[g] + c] = g;
  std::vector<std::vector<std::pair<i64, int32_t>>> per(fp.nsn);
  for (int q = 0; q < fp.nsys; ++q) {
    const Csr& A = *systems[q].pat;
    for (int o = 0; o < A.nrows; ++o) {
      i64 pr = fp.iperm_global[fp.sys_off[q] + o];
      for (i64 p = A.ptr[o]; p < A.ptr[o + 1]; ++p) {
        i64 pc = fp.iperm_global[fp.sys_off[q] + A.idx[p]];
        if (pr < pc) continue;  // keep lower (row >= col)
        int g = sn_of_pos[pc];
        int nr = fp.sn_ncol[g] + fp.sn_noff[g];
        int frow;
        if (pr < fp.sn_col0[g] + fp.sn_ncol[g]) frow = (int)(pr - fp.sn_col0[g]);
        else {
          const i64* po = &fp.offrows[fp.sn_rowptr[g]];
          const i64* it = std::lower_bound(po, po + fp.sn_noff[g], pr);
          MDD_REQUIRE(it != po + fp.sn_noff[g] && *it == pr, 5, "matrix entry outside structure");
          frow = fp.sn_ncol[g] + (int)(it - po);
        }
        int fcol = (int)(pc - fp.sn_col0[g]);
        per[g].push_back({systems[q].val_slot[p], (int32_t)(fcol * nr + frow)});
      }
    }
  }
  for (int g = 0; g < fp.nsn; ++g) fp.asm_ptr[g + 1] = fp.asm_ptr[g] + (i64)per[g].size();
  fp.asm_src.resize(fp.asm_ptr[fp.nsn]);
  fp.asm_pos.resize(fp.asm_ptr[fp.nsn]);
  for (int g = 0; g < fp.nsn; ++g) {
    i64 o = fp.asm_ptr[g];
    for (auto& pr : per[g]) { fp.asm_src[o] = pr.first; fp.asm_pos[o] = pr.second; ++o; }
  }
}

}  // namespace mdd
