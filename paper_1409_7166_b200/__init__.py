"""B200-native topology-based power-grid transient analysis (arxiv 1409.7166).

The hot path (RHS, red-black SOR / Jacobi / multi-colour CSR relaxation sweeps
with fused convergence reduction, inductor companion update, time-step driver)
lives in the sm_100a library ``lib/libpgb200.so`` behind the C ABI of
``include/pgrid.h``; this package is its thin Python binding.
"""
from ._lib import PgError, PgNoConvergence, load  # noqa: F401
from .api import Grid, TransientResult, release_memory  # noqa: F401
from .slab import SlabGroup, partition_rows, slab_spec  # noqa: F401

__all__ = ["Grid", "TransientResult", "release_memory", "PgError", "PgNoConvergence", "load", "SlabGroup",
           "partition_rows", "slab_spec"]
