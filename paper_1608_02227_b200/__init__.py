"""B200-native hot path of Aybat & Wang (arXiv 1608.02227): constant-step P-APG on the
Tikhonov-smoothed dual of the least-squares convex-regression QP, every pair dualized.

The product is libcr.so (C ABI, include/cr.h) built from ``csrc/``; ``binding`` is a thin
ctypes layer over it.  See DESIGN.md.
"""
from . import binding  # noqa: F401
from .binding import (  # noqa: F401
    CrError, LocalGroup, Solver, load, lipschitz_host, nccl_unique_id, selftest_p2p, selftest_p2p_allgather,
    workspace_size, EXPORTS,
)

__all__ = ["CrError", "LocalGroup", "Solver", "load", "lipschitz_host", "nccl_unique_id", "selftest_p2p",
           "selftest_p2p_allgather", "workspace_size", "EXPORTS"]
