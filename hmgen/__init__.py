"""hmgen — seeded, deterministic INPUT GENERATOR for the power-series solver.

This package is shared by both sides of the parity test (oracle and GPU path)
and holds none of the method's arithmetic (§III): it only builds the
H-matrix operator Z = Z_N + Z_F of PAPER.md Eq. (13) from a generated PEC
geometry (§II, Eqs. 1-3, 9-12) and writes it to the versioned `.hm`
file described in include/ps.h, plus plane-wave right-hand sides.
"""
from .build import (CONFIGS, build_config, make_mesh, rwg_basis, write_hm,  # noqa: F401
                    plane_wave_dirs, generate, load_or_generate, EfieLib)
