"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This package holds NO state-vector arithmetic: it only builds gate lists
(2x2 matrices, control/target qubit lists, permutation tables) and the
counter-based random numbers the workloads draw.  Both `oracle/` and the
product binding consume the same materialised inputs bit for bit
(SURVEY.md §8(c) readings 9-11).
"""
from .gates import (  # noqa: F401
    Gate, G_1Q, G_CTRL, G_PERM, G_SWAP,
    H, X, Y, XBAR, YBAR, R, PAULI_X, SplitMix64, sm64, haar_u2,
    one_q, ctrl, cnot, cphase, toffoli, perm_gate, swap,
)
from .circuits import (  # noqa: F401
    qft_ladder, inverse_qft_ladder, qft_adder, random_brickwork, random_chain,
    shor_order_finding, shor_base, qft_basis, config1_adder, config2_random,
    config3_shor, config4_qft, config5_random36, count_ops, multiplicative_order,
    paper_adder, h_on_all, PAPER_ADDERS, load_register_bits,
)
