"""Gate records, the paper's named 2x2 matrices, and the counter-based RNG.

Conventions:
  * qubit 0 is the least-significant bit of the amplitude index;
  * controls fire on |1>;
  * a 2x2 matrix is row-major [u00, u01, u10, u11] and maps
    (a0, a1) -> (u00 a0 + u01 a1, u10 a0 + u11 a1).

Only input construction lives here (no state-vector updates).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence, Tuple

import numpy as np

G_1Q, G_CTRL, G_PERM, G_SWAP = 0, 1, 2, 3
M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15

U2 = Tuple[complex, complex, complex, complex]


@dataclass
class Gate:
    kind: int
    target: int = -1
    controls: Tuple[int, ...] = ()
    targets: Tuple[int, ...] = ()
    u: U2 = (1, 0, 0, 1)
    perm: Optional[np.ndarray] = field(default=None, repr=False)

    def qubits(self) -> Tuple[int, ...]:
        if self.kind in (G_1Q, G_CTRL):
            return tuple(self.controls) + (self.target,)
        return tuple(self.controls) + tuple(self.targets)


S2 = 1.0 / math.sqrt(2.0)
# Eq. Hadamard
H: U2 = (S2, S2, S2, -S2)
# Eq. Xoperation: e^{i pi S^x/2}, NOT Pauli-X
X: U2 = (S2, 1j * S2, 1j * S2, S2)
# Eq. Yoperation: e^{i pi S^y/2}
Y: U2 = (S2, S2, -S2, S2)
# inverses X-bar, Y-bar: U^dagger
XBAR: U2 = (S2, -1j * S2, -1j * S2, S2)
YBAR: U2 = (S2, -S2, S2, S2)
# CNOT target action (Eq. CNOT2)
PAULI_X: U2 = (0, 1, 1, 0)


def R(phi: float) -> U2:
    """Eq. singlephase: diag(1, e^{i phi})."""
    return (1, 0, 0, complex(math.cos(phi), math.sin(phi)))


def V(phi: float) -> U2:
    """Target matrix of the controlled-V, Eq. COMM4."""
    e = complex(math.cos(phi), math.sin(phi))
    return ((1 + e) / 2, (1 - e) / 2, (1 - e) / 2, (1 + e) / 2)


def one_q(q: int, u: U2) -> Gate:
    return Gate(G_1Q, target=q, u=tuple(complex(x) for x in u))


def ctrl(controls: Sequence[int], t: int, u: U2) -> Gate:
    return Gate(G_CTRL, target=t, controls=tuple(controls), u=tuple(complex(x) for x in u))


def cnot(c: int, t: int) -> Gate:
    return ctrl((c,), t, PAULI_X)


def cphase(c: int, t: int, phi: float) -> Gate:
    """Controlled phase shift R_{tc}(phi), Eq. COMM5."""
    return ctrl((c,), t, R(phi))


def toffoli(c1: int, c2: int, t: int) -> Gate:
    """Eq. Toffoli."""
    return ctrl((c1, c2), t, PAULI_X)


def perm_gate(controls: Sequence[int], targets: Sequence[int], perm) -> Gate:
    p = np.ascontiguousarray(np.asarray(perm, dtype=np.uint32))
    assert p.size == 1 << len(targets)
    return Gate(G_PERM, controls=tuple(controls), targets=tuple(targets), perm=p)


def swap(a: int, b: int) -> Gate:
    return Gate(G_SWAP, targets=(a, b))


# --------------------------------------------------------------------------
# SplitMix64 (SURVEY.md §8(c) readings 9, 10, 14). Counter-based: the s-th
# draw of stream `seed` is sm64(seed + (s+1)*GOLDEN).
# --------------------------------------------------------------------------
def sm64(x: int) -> int:
    """SplitMix64 finaliser applied to x (already advanced by the caller)."""
    z = x & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


class SplitMix64:
    def __init__(self, seed: int):
        self.state = seed & M64

    def next(self) -> int:
        self.state = (self.state + GOLDEN) & M64
        return sm64(self.state)

    def uniform(self) -> float:
        """53-bit double in [0, 1)."""
        return (self.next() >> 11) * (1.0 / (1 << 53))


def haar_u2(rng: SplitMix64) -> U2:
    """Haar-random U(2) (reading 10): U = e^{ia}[[e^{ipsi}cos t, e^{ichi}sin t],
    [-e^{-ichi}sin t, e^{-ipsi}cos t]], a,psi,chi ~ U[0,2pi), t = asin(sqrt(xi))."""
    two_pi = 2.0 * math.pi
    a = two_pi * rng.uniform()
    psi = two_pi * rng.uniform()
    chi = two_pi * rng.uniform()
    t = math.asin(math.sqrt(rng.uniform()))
    ea = complex(math.cos(a), math.sin(a))
    ep = complex(math.cos(psi), math.sin(psi))
    ec = complex(math.cos(chi), math.sin(chi))
    c, s = math.cos(t), math.sin(t)
    return (ea * ep * c, ea * ec * s, -ea * ec.conjugate() * s, ea * ep.conjugate() * c)
