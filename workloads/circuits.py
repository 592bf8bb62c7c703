"""Gate-list generators for the paper's workloads and BASELINE.json's configs.

Each generator returns a `Workload` (n qubits, initial basis index, gate
list, metadata).  Readings of the paper that fix the circuits are listed in
DESIGN.md §3 and SURVEY.md §8(c):
  * QFT ladder (reading 4/5, V5): for j = m-1..0: H(q_j), then for
    l = j-1..0: CP(q_l, q_j, +2 pi / 2^(j-l+1)); optional bit-reversal swaps.
  * adder (Fig. adder caption P:864-882; V4/V5): swap-free QFT on
    the accumulator, CP(a_i, b_j, 2 pi/2^(j-i+1)) for i <= j, inverse ladder.
  * Shor (Eqs. Shor0-Shor2; reading 7): H on the x-register,
    controlled multiplications by x^(2^j) mod N as permutations of the
    f-register, inverse QFT (with swaps) on the x-register.
  * random circuits (BASELINE.json configs 2/5; readings 10-12).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Sequence

import numpy as np

from .gates import (G_1Q, G_CTRL, G_PERM, G_SWAP, Gate, H, SplitMix64, cnot,
                    cphase, haar_u2, one_q, perm_gate, swap)


@dataclass
class Workload:
    name: str
    n: int
    init: int
    gates: List[Gate]
    meta: Dict = field(default_factory=dict)


def dagger(g: Gate) -> Gate:
    if g.kind in (G_1Q, G_CTRL):
        u00, u01, u10, u11 = g.u
        return Gate(g.kind, target=g.target, controls=g.controls,
                    u=(u00.conjugate(), u10.conjugate(), u01.conjugate(), u11.conjugate()))
    if g.kind == G_PERM:
        inv = np.empty_like(g.perm)
        inv[g.perm] = np.arange(g.perm.size, dtype=np.uint32)
        return Gate(G_PERM, controls=g.controls, targets=g.targets, perm=inv)
    return Gate(g.kind, targets=g.targets)


def inverse(gates: Sequence[Gate]) -> List[Gate]:
    return [dagger(g) for g in reversed(gates)]


def qft_ladder(qubits: Sequence[int], swaps: bool) -> List[Gate]:
    """QFT on register `qubits` (register bit i <-> qubits[i]); V5."""
    m = len(qubits)
    out: List[Gate] = []
    for j in range(m - 1, -1, -1):
        out.append(one_q(qubits[j], H))
        for l in range(j - 1, -1, -1):
            out.append(cphase(qubits[l], qubits[j], 2.0 * math.pi / (1 << (j - l + 1))))
    if swaps:
        for j in range(m // 2):
            out.append(swap(qubits[j], qubits[m - 1 - j]))
    return out


def inverse_qft_ladder(qubits: Sequence[int], swaps: bool) -> List[Gate]:
    return inverse(qft_ladder(qubits, swaps))


def add_phases(src: Sequence[int], acc: Sequence[int]) -> List[Gate]:
    """Controlled phases adding register `src` into the Fourier-space `acc`
    (m(m+1)/2 gates for equal widths, V4)."""
    out = []
    m = len(acc)
    for j in range(m - 1, -1, -1):
        for i in range(min(j, len(src) - 1), -1, -1):
            out.append(cphase(src[i], acc[j], 2.0 * math.pi / (1 << (j - i + 1))))
    return out


def qft_adder(regs: Sequence[Sequence[int]]) -> List[Gate]:
    """Add registers regs[0..-2] into regs[-1] modulo 2^m."""
    acc = regs[-1]
    out = qft_ladder(acc, swaps=False)
    for r in regs[:-1]:
        out += add_phases(r, acc)
    out += inverse_qft_ladder(acc, swaps=False)
    return out


def config1_adder(seed: int = 1, m: int = 6) -> Workload:
    rng = SplitMix64(seed)
    a = rng.next() % (1 << m)
    b = rng.next() % (1 << m)
    ra = list(range(m))
    rb = list(range(m, 2 * m))
    gates = qft_adder([ra, rb])
    expect = a + (1 << m) * ((a + b) % (1 << m))
    return Workload("qft_adder", 2 * m, a + (b << m), gates,
                    {"a": a, "b": b, "m": m, "expect_index": expect})


def random_brickwork(n: int, depth: int, seed: int) -> List[Gate]:
    """BASELINE.json config 2 family: each layer = Haar U2 on every qubit,
    then CNOT(lower -> higher) on brickwork pairs with offset (layer mod 2)."""
    rng = SplitMix64(seed)
    out: List[Gate] = []
    for layer in range(depth):
        for q in range(n):
            out.append(one_q(q, haar_u2(rng)))
        for c in range(layer % 2, n - 1, 2):
            out.append(cnot(c, c + 1))
    return out


def config2_random(seed: int = 2, n: int = 24, depth: int = 40) -> Workload:
    return Workload("random_brickwork", n, 0, random_brickwork(n, depth, seed),
                    {"depth": depth, "seed": seed})


def multiplicative_order(x: int, N: int) -> int:
    r, v = 1, x % N
    while v != 1:
        v = (v * x) % N
        r += 1
    return r


def shor_base(seed: int, N: int) -> int:
    """Reading 9: x = 2 + (splitmix64 mod (N-2)), redrawn until gcd(x,N)=1."""
    rng = SplitMix64(seed)
    while True:
        x = 2 + rng.next() % (N - 2)
        if math.gcd(x, N) == 1:
            return x


def modmul_perm(c: int, N: int, f: int) -> np.ndarray:
    """perm[w] = c*w mod N for w < N, w otherwise (reading 7)."""
    w = np.arange(1 << f, dtype=np.int64)
    p = np.where(w < N, (c * w) % N, w)
    return p.astype(np.uint32)


def shor_order_finding(N: int, x: int, t: int, f: int) -> Workload:
    """x-register q0..t-1, f-register q_t..q_{t+f-1} initialised to |1>."""
    assert N < (1 << f)
    ctrl_reg = list(range(t))
    work = list(range(t, t + f))
    gates = [one_q(q, H) for q in ctrl_reg]
    c = x % N
    for j in range(t):
        gates.append(perm_gate((ctrl_reg[j],), work, modmul_perm(c, N, f)))
        c = (c * c) % N
    gates += inverse_qft_ladder(ctrl_reg, swaps=True)
    r = multiplicative_order(x, N)
    return Workload("shor_order_finding", t + f, 1 << t, gates,
                    {"N": N, "x": x, "t": t, "f": f, "r": r})


def config3_shor(seed: int = 3, N: int = 899, t: int = 18, f: int = 10) -> Workload:
    return shor_order_finding(N, shor_base(seed, N), t, f)


def qft_basis(n: int, x0: int) -> Workload:
    return Workload("qft", n, x0, qft_ladder(list(range(n)), swaps=True), {"x0": x0})


def config4_qft(seed: int = 4, n: int = 32) -> Workload:
    x0 = SplitMix64(seed).next() % (1 << n)
    return qft_basis(n, x0)


def random_chain(n: int, layers: int, seed: int, sweep: bool) -> List[Gate]:
    """BASELINE.json config 5 family (reading 11/12): H on all; `layers` x
    (Haar U2 on every qubit + CNOT chain i->i+1, i ascending); then the
    per-position sweep H(p), U2(p) for p = 0..n-1."""
    rng = SplitMix64(seed)
    out = [one_q(q, H) for q in range(n)]
    for _ in range(layers):
        for q in range(n):
            out.append(one_q(q, haar_u2(rng)))
        for i in range(n - 1):
            out.append(cnot(i, i + 1))
    if sweep:
        for p in range(n):
            out.append(one_q(p, H))
            out.append(one_q(p, haar_u2(rng)))
    return out


def config5_random36(seed: int = 5, n: int = 36, layers: int = 10, sweep: bool = True) -> Workload:
    return Workload("random_chain", n, 0, random_chain(n, layers, seed, sweep),
                    {"layers": layers, "seed": seed})


def count_ops(gates: Sequence[Gate]) -> Dict[str, int]:
    c = {"1q": 0, "ctrl": 0, "perm": 0, "swap": 0}
    for g in gates:
        c[{G_1Q: "1q", G_CTRL: "ctrl", G_PERM: "perm", G_SWAP: "swap"}[g.kind]] += 1
    c["total"] = len(gates)
    return c


# ---------------------------------------------------------------------------
# The paper's own benchmark workloads (Tables IV-IX)
# ---------------------------------------------------------------------------
PAPER_ADDERS = {
    # name: (register width m, register values); N_O as printed (V4)
    "3-11QBA": (11, (292, 585, 1170), 286),    # 33 qubits
    "2-17QBA": (17, (26214, 104857), 493),     # 34 qubits
    "5-7QBA": (7, (7, 9, 19, 35, 65), 194),    # 35 qubits
    "3-12QBA": (12, (781, 1054, 3296), 342),   # 36 qubits
}


def load_register_bits(regs, values):
    """Put numbers in the registers with the doubled gates XX, YY, X-bar X-bar,
    Y-bar Y-bar: each loads |1> up to a phase and
    counts as 2 operations.  The four kinds are cycled over the one-bits."""
    from .gates import X, XBAR, Y, YBAR
    kinds = (X, Y, XBAR, YBAR)
    out, k = [], 0
    for reg, val in zip(regs, values):
        for b, q in enumerate(reg):
            if (val >> b) & 1:
                u = kinds[k % 4]
                out += [one_q(q, u), one_q(q, u)]
                k += 1
    return out


def paper_adder(name: str) -> Workload:
    """n-mQBA of the paper: load the registers from |0..0>, QFT the last
    register, add the others into it with controlled phases, inverse QFT
    (Fig. adder caption).  Expect the last register to hold
    sum mod 2^m with probability 1."""
    m, values, n_o = PAPER_ADDERS[name]
    regs = [list(range(i * m, (i + 1) * m)) for i in range(len(values))]
    gates = load_register_bits(regs, values) + qft_adder(regs)
    expect = sum(values) % (1 << m)
    return Workload(name, m * len(values), 0, gates,
                    {"m": m, "values": values, "expect_sum": expect, "n_o_paper": n_o, "sum_register": regs[-1]})


def h_on_all(L: int) -> Workload:
    """The scaling test: a Hadamard on every qubit ("H" rows of
    Tables IV-IX, N_O = L)."""
    from .gates import H as HD
    return Workload("H-all", L, 0, [one_q(q, HD) for q in range(L)], {})
