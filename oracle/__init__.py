"""Plain, slow, obviously-correct fp64 CPU oracle for the FCG-NO hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.  The
product path (``paper_2402_05598_b200``) never imports, links or executes
anything here, and this package imports nothing from the product path; the two
share no code.  Inputs come from ``synthetic/`` (random numbers only).

Every function cites the PAPER.md passage (``P:line``) or the DESIGN.md reading
(``R#``) it follows.  Parity pins live in ``tests/test_oracle_*.py``.

Parity status: every function here is pinned by at least one
test against the paper or the mathematics, except the NO forward *inside* FCG
with random weights, which the paper prints no number for ("parity unpinned"
against the paper: pinned only by properties and closed forms).
"""
from .stencil import h_of, harmonic, faces, apply_A, dense_A
from .dots import two_product, dot, norm2
from .no import (K_MODES, mode_indices, analysis, synthesis, gelu, unpack_weights, no_forward,
                 param_count, cheb_basis, analysis_cheb, synthesis_cheb)
from .fcg import m_schedule, fcg, cg, CONVERGED, MAXIT, BREAKDOWN, NONFINITE, RUNNING
from .notay import a_norm, notay_ratio, notay_ratio_scaled, notay_curve
from .classical import diagonal, jacobi, sgs

__all__ = [
    "h_of", "harmonic", "faces", "apply_A", "dense_A", "two_product", "dot", "norm2",
    "K_MODES", "mode_indices", "analysis", "synthesis", "gelu", "unpack_weights", "no_forward",
    "cheb_basis", "analysis_cheb", "synthesis_cheb",
    "param_count", "m_schedule", "fcg", "cg", "CONVERGED", "MAXIT", "BREAKDOWN", "NONFINITE",
    "RUNNING", "a_norm", "notay_ratio", "notay_ratio_scaled", "notay_curve", "diagonal", "jacobi", "sgs",
]
