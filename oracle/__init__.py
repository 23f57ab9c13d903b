"""oracle — plain, slow, obviously-correct CPU (numpy, complex128) implementation
of the two-term power-series solve of PAPER.md §III (arXiv 2109.04129).

TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` leg may import or execute anything here. The
product path (paper_2109_04129_b200 / libps) never imports it, and this package
never imports the product path; the two share no code. The only shared module
is the input generator `hmgen` (operator assembly, no power-series arithmetic),
and the oracle does not even use that: it reads the `.hm` file with its own
parser (oracle/hmfile.py).

Modules
  hmfile  — independent reader of the versioned H-matrix file.
  scaling — Eqs. (14)-(23): sequential right scaling alpha_k with fill-in,
            D_k^{-1} = inverse of the scaled diagonal blocks.
  series  — Eqs. (24), (26), (30)-(36), (44)-(45): the two-term solve, and the
            n-term / adaptive series (R25).
  dense   — dense materialisation of Z_N, Z_F for the closed-form pin
            x2 = Z_N^{-1} b - Z_N^{-1} Z_F Z_N^{-1} b (Appendix B of
            SURVEY.md) and dense-LU reference solutions.

Parity pins: every function is pinned by tests/test_oracle_*.py against the
paper's textbook cases, closed forms and invariants.
"""
from .hmfile import HMatrix, read_hm  # noqa: F401
from .scaling import Scaling, compute_scaling  # noqa: F401
from .series import (apply_Rt, apply_R, apply_Dinv, apply_ZF, apply_U, series_solve,  # noqa: F401
                     solve, SolveResult, check_convergence, series_solve_adaptive,
                     series_diverged)
