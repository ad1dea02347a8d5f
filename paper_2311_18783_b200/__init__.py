"""B200-native two-level additive Schwarz (SNK + GenEO) preconditioned CG for the
lowest-order Nédélec discretisation of the positive Maxwell problem
(arxiv 2311.18783).  The compute path is the CUDA library libmaxwell_dd.so
(include/maxwell_dd.h); this package is its thin Python binding."""
from .solver import MaxwellDD, topology_array  # noqa: F401
