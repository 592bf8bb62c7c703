"""B200-native state-vector gate engine for arXiv quant-ph/0608239
("Massive Parallel Quantum Computer Simulator", De Raedt et al.).

The compute path is libqsim_b200.so (hand-written sm_100a CUDA + NCCL)
behind the C-ABI in include/qsim.h; this package is its thin binding.
"""
from .qsim import (QSim, QsimError, exchange_peers, get_loopback_id, get_unique_id, pack_gates, plan_json,  # noqa: F401
                   probe_peaks, run_loopback,
                   G_1Q, G_CTRL, G_PERM, G_SWAP)
from ._native import LIB_PATH, EXPORTS  # noqa: F401
from .program import Program, ProgramError, parse_program, run_program, serialize_program  # noqa: F401
from . import shor  # noqa: F401
