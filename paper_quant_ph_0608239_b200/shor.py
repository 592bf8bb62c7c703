"""Shor's algorithm end to end on the engine (§VI.B).

The quantum part runs in the engine's kernels: H on the X-qubit x-register,
f(x) = y^x mod G into the F-qubit f-register by controlled modular
multiplications (the paper's "conditional operation"; reading R7:
controlled multiplication by y^(2^j) mod G on the f-register initialised to 1,
as register permutations through qsim_apply_perm), the inverse QFT with swaps
on the x-register (reading R4), then sampling of the x-register.
The classical part is host code: the convergents of k / 2^X (Eq. Shor6,
P:1052-1060) give candidate periods, and for an even r with y^(r/2) != -1
mod G, gcd(y^(r/2) +- 1, G) are the factors.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .program import GateRecord

_G_1Q, _G_CTRL, _G_PERM, _G_SWAP = 0, 1, 2, 3
_S2 = 1.0 / math.sqrt(2.0)
_H = (_S2, _S2, _S2, -_S2)


def convergents(k: int, X: int) -> List[Tuple[int, int]]:
    """Convergents p/q of the continued fraction of k / 2^X, in order."""
    a, b = k, 1 << X
    out = []
    h0, h1, k0, k1 = 0, 1, 1, 0  # p_{-2}, p_{-1}, q_{-2}, q_{-1}
    while b:
        q = a // b
        a, b = b, a - q * b
        h0, h1 = h1, q * h1 + h0
        k0, k1 = k1, q * k1 + k0
        out.append((h1, k1))
    return out


def period_candidates(k: int, X: int, G: int) -> List[int]:
    """Denominators r < G of the convergents within 1 / 2^(X+1) of k / 2^X
    (Eq. Shor6)."""
    N = 1 << X
    out = []
    for p, q in convergents(k, X):
        if q >= G:
            break
        if q > 0 and 2 * abs(k * q - p * N) <= q:  # |k/N - p/q| <= 1/(2N)  <=>  2|kq - pN| <= q
            out.append(q)
    return out


def order_from_samples(samples: Sequence[int], X: int, G: int, y: int) -> Optional[int]:
    """Smallest r with y^r = 1 mod G built from the candidates of the samples:
    a convergent may give a divisor of r (when gcd(k', r) > 1), so the lcm of
    candidates is tried as well."""
    cands = set()
    for k in samples:
        cands.update(period_candidates(int(k), X, G))
    found = None
    lcm = 1
    for r in sorted(cands):
        if pow(y, r, G) == 1:
            found = r if found is None else min(found, r)
        lcm = lcm * r // math.gcd(lcm, r)
        if lcm < G and pow(y, lcm, G) == 1:
            found = lcm if found is None else min(found, lcm)
    return found


def factors_from_order(G: int, y: int, r: int) -> Optional[Tuple[int, int]]:
    """an even r with y^(r/2) != +-1 mod G gives gcd(y^(r/2) +- 1, G)."""
    if r % 2:
        return None
    h = pow(y, r // 2, G)
    if h in (1, G - 1):
        return None
    a, b = math.gcd(h - 1, G), math.gcd(h + 1, G)
    for f in (a, b):
        if 1 < f < G:
            return (min(f, G // f), max(f, G // f))
    return None


def modmul_table(c: int, G: int, F: int) -> np.ndarray:
    """Permutation of the f-register: w -> c w mod G for w < G, else w."""
    w = np.arange(1 << F, dtype=np.int64)
    t = w.copy()
    t[:G] = (c * w[:G]) % G
    return t.astype(np.uint32)


def circuit(G: int, y: int, X: int, F: int) -> List[GateRecord]:
    """x-register = qubits 0..X-1 (Table III lists <Q_i> for i < X), f-register
    X..X+F-1 initialised to |1> (initial index 1 << X)."""
    if G >= (1 << F) or math.gcd(y, G) != 1:
        raise ValueError("need G < 2^F and gcd(y, G) = 1")
    xs, fs = list(range(X)), tuple(range(X, X + F))
    gates = [GateRecord(_G_1Q, target=q, u=_H) for q in xs]
    c = y % G
    for j in range(X):
        gates.append(GateRecord(_G_PERM, controls=(xs[j],), targets=fs, perm=modmul_table(c, G, F)))
        c = (c * c) % G
    # inverse QFT with swaps (reading R4): the forward ladder is, for j = X-1 .. 0,
    # H(j) then CP(l -> j, 2 pi / 2^(j-l+1)) for l = j-1 .. 0, then the bit-reversal
    # swaps; its inverse is the swaps, then for j = 0 .. X-1 the negated phases
    # CP(l -> j), l = 0 .. j-1, then H(j)
    for i in reversed(range(X // 2)):
        gates.append(GateRecord(_G_SWAP, targets=(xs[i], xs[X - 1 - i])))
    for j in range(X):
        for l in range(j):
            phi = -2.0 * math.pi / (1 << (j - l + 1))
            gates.append(GateRecord(_G_CTRL, target=xs[j], controls=(xs[l],),
                                    u=(1, 0, 0, complex(math.cos(phi), math.sin(phi)))))
        gates.append(GateRecord(_G_1Q, target=xs[j], u=_H))
    return gates


@dataclass
class ShorResult:
    samples: np.ndarray
    r: Optional[int]
    factors: Optional[Tuple[int, int]]
    expectations: np.ndarray  # <Q_i>, i < X (Eq. Shor7)


def run(G: int, y: int, X: int, F: int, shots: int = 16, seed: int = 1, sim=None,
        full_register: bool = True) -> ShorResult:
    """full_register: draw basis states of the WHOLE (X + F)-qubit register
    (the two-level sampler when X + F > 24) and keep their
    x-register bits; else sample the x-register marginal directly."""
    from .qsim import QSim, pack_gates
    sim = sim or QSim(X + F)
    gates = circuit(G, y, X, F)
    sim.init_basis(1 << X)
    sim.run_circuit(gates, packed=pack_gates(gates))
    ex = sim.expectations()[:X]
    if full_register:
        full = sim.measure(list(range(X + F)), seed=seed, shots=shots)
        samples = full & np.uint64((1 << X) - 1)
    else:
        samples = sim.measure(list(range(X)), seed=seed, shots=shots)
    r = order_from_samples(samples, X, G, y)
    return ShorResult(samples, r, factors_from_order(G, y, r) if r else None, ex)
