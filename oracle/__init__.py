"""CPU oracle for the single-pass randomized ID ingest path (arxiv 2405.16076).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import anything
in this package.  The product path (``paper_2405_16076_b200``) never imports it
and shares no code with it: the oracle re-implements the Philox stream, the
Gauss-16 sketch entries, the selection draws and every arithmetic step on its
own, in plain numpy fp64, following the paper step by step.

Citation tags: ``P:n`` = line n of the paper's LaTeX source;
readings R1..R14 are listed in DESIGN.md section 3.

Parity-pin status per function:
  philox4x32_10        pinned (Random123 / cuRAND known-answer vectors)
  gauss16 levels       pinned (symmetry, independent erfc bisection, moments)
  sketch / ingest      pinned (identity sketch, slab additivity, JL statistics)
  ridge scores         pinned (exact leverage at lambda=0, closed form at lambda>0,
                       hand case A=I2, Lemma 1 direction)
  selection            pinned (C1 block 1 forced admissions, MC frequencies)
  Alg 4 coefficients   pinned (exact recovery, self-representation, identity sketch)
  NA-Hutch++ estimate  pinned (P=0 case, exactness, unbiasedness over seeds)
  gradient variant     (oracle/gradient.py) pinned: exact simplex gradients of
                       linear fields, central / one-sided stencils, P(0) = Alg 4 and the
                       stacked normal equations, GCV(0) closed form, golden section on
                       known functions, constant fields = plain selection
  ridge scores at lambda>0 with Gaussian sketch / Bernoulli trajectories on
  C2-C5 are "parity unpinned" beyond the above.
"""

from .philox import philox4x32_10, uniform24
from .gauss16 import gauss16_magnitudes, gauss16_levels, gauss16_scale, omega_rows
from .oid import (OracleParams, OracleOID, ridge_scores, hutchpp_estimate, alg4_coefficients, alg5_coefficients,
                  alg6_coefficients, alg7_coefficients, extend_prev, sketch_pinv, pinv_psd)

__all__ = [
    "philox4x32_10", "uniform24", "gauss16_magnitudes", "gauss16_levels", "gauss16_scale", "omega_rows",
    "OracleParams", "OracleOID", "ridge_scores", "hutchpp_estimate", "alg4_coefficients", "alg5_coefficients",
    "alg6_coefficients", "alg7_coefficients", "extend_prev", "sketch_pinv", "pinv_psd",
]
