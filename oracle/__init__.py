"""Oracle for the smoothed-dual P-APG hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/`` (including the numerics scripts under ``tests/numerics/``),
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference`` legs may
import this package.  The product path
(``paper_1608_02227_b200``) never imports it and shares no code with it; the
only common module is ``crdata`` (seeded input generators, no method
arithmetic).

Contents
--------
``papg_oracle.c`` (loaded here via ctypes)
    fp64 Fig. 2 iteration with K = N, plain loops + OpenMP over rows;
    the adaptive-step variant (Eq. (adaptive-check)) written out literally;
    the continuation over gamma_t (Section 2.4.1) in core.py on top of it.
``partition.py``
    Fig. 2 with a general partition K < N (Assumption 1): Step 1 = per-block exact
    G-norm projections through the NNLS dual of each block QP.
``ref.py``
    dense A1/A2/C (Def. A1A2), the exact regularized optimum via the
    NNLS form of the dual, the univariate sorted-slope convex fit
    (Lemma 1 pin), sigma_max(C)^2/gamma by ARPACK Lanczos (Eq.
    (lischitz)), closed-form dual value.

Parity status per function:
    oracle_papg, oracle_eta, oracle_stats, oracle_project_rows, oracle_papg_adaptive -- pinned
    (tests/test_oracle_pins.py); lipschitz(structured) -- pinned against the
    definition form and Lemma 4 closed forms.
"""
from .core import (  # noqa: F401
    build_oracle, lib, papg, papg_adaptive, continuation, eta, stats, project_rows, momentum_next, max_threads, extrapolate, state_after,
)
