"""paper_2109_04129_b200 — B200-native two-term power-series solver (arXiv 2109.04129).

Thin Python binding over the C-ABI library libps (include/ps.h): argument
marshalling only; every step of the hot path runs in libps's sm_100a kernels.
There is no CPU fallback: if libps.so is missing or no CUDA device is present,
the calls raise.
"""
from .binding import (PsError, PsHandle, PS_OP_DINV, PS_OP_R, PS_OP_RT, PS_OP_U,  # noqa: F401
                      PS_OP_ZF, load_library, lib_path, INFO_KEYS, solve_group, nccl_unique_id,
                      partition, farfield)
