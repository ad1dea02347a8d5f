"""CPU ORACLE — test infrastructure only.

A plain, slow, fp64 CPU implementation of what the solve path computes, written
from PAPER.md (arxiv 2311.18783) and the readings listed in DESIGN.md §2.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import it.  The product package
``paper_2311_18783_b200`` never imports it and shares no code with it; the only
shared module is ``workloads`` (seeded input draws, no method arithmetic).

Modules (each function cites the PAPER.md passage it follows):
  mesh      structured cube grid -> Kuhn tetrahedra, edge numbering, Dirichlet
  assembly  Whitney (lowest-order Nedelec) K, M, A = K + gamma M, gradient C
  dd        box subdomains, overlap, R_i, D_i (PoU), A_i, A_i^Neu, k0, k1
  coarse    G_i, xi_0i, GenEO GEVP, SNK / NK / GenEO columns, E = Z^T A Z
  solver    M_AS, M_AS,2 (eq. 2.8), PCG

Parity status of every function is in DESIGN.md §6 ("Oracle pins").
"""
