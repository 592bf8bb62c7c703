"""Independent references used to pin the oracle (and the GPU path).

None of these restate the oracle's index-loop update rules: they are
(a) dense Kronecker-product operators / tensor contractions, (b) closed forms
from the paper or from Fourier analysis, (c) exact-rounded sums.
"""
from __future__ import annotations

import math
from typing import Sequence

import numpy as np

I2 = np.eye(2, dtype=np.complex128)
P1 = np.array([[0, 0], [0, 1]], dtype=np.complex128)


def mat(u) -> np.ndarray:
    return np.array([[u[0], u[1]], [u[2], u[3]]], dtype=np.complex128)


def kron_list(factors_by_qubit: dict, n: int) -> np.ndarray:
    """kron with qubit n-1 leftmost, qubit 0 rightmost (qubit 0 = LSB)."""
    out = np.ones((1, 1), dtype=np.complex128)
    for q in range(n - 1, -1, -1):
        out = np.kron(out, factors_by_qubit.get(q, I2))
    return out


def dense_controlled(n: int, controls: Sequence[int], t: int, u) -> np.ndarray:
    """|1..1><1..1|_C (x) U_t + (I - |1..1><1..1|_C) (x) I_t  =  I + P1_C (x) (U - I)_t."""
    f = {c: P1 for c in controls}
    f[t] = mat(u) - I2
    return np.eye(1 << n, dtype=np.complex128) + kron_list(f, n)


def tensor_apply_perm(psi: np.ndarray, n: int, controls, targets, perm) -> np.ndarray:
    """Apply a controlled register permutation by tensor contraction: reshape
    psi to n axes (axis a <-> qubit n-1-a), contract the target axes with the
    2^t x 2^t permutation matrix P[perm[w], w] = 1, mix with the identity
    on the control = |1..1> slice."""
    t = len(targets)
    Pm = np.zeros((1 << t, 1 << t), dtype=np.complex128)
    for w in range(1 << t):
        Pm[perm[w], w] = 1
    # register index bit b <-> targets[b]; as a tensor (2,)*t in C order the
    # first axis is the most significant register bit b = t-1.
    Pt = Pm.reshape((2,) * (2 * t))
    T = psi.reshape((2,) * n)
    ax = lambda q: n - 1 - q  # noqa: E731
    tgt_axes = [ax(targets[b]) for b in range(t - 1, -1, -1)]
    out = np.tensordot(Pt, T, axes=(list(range(t, 2 * t)), tgt_axes))
    # tensordot puts the t new axes first, in order of tgt_axes; move them back
    rest = [a for a in range(n) if a not in tgt_axes]
    order = tgt_axes + rest
    inv = np.argsort(order)
    out = np.transpose(out, inv)
    if controls:
        sl = [slice(None)] * n
        for c in controls:
            sl[ax(c)] = 1
        res = T.copy()
        res[tuple(sl)] = out[tuple(sl)]
        out = res
    return np.ascontiguousarray(out).reshape(-1)


def tensor_swap(psi: np.ndarray, n: int, a: int, b: int) -> np.ndarray:
    T = psi.reshape((2,) * n)
    return np.ascontiguousarray(np.swapaxes(T, n - 1 - a, n - 1 - b)).reshape(-1)


def qft_closed_form(n: int, x0: int) -> np.ndarray:
    """QFT|x0> = 2^{-n/2} sum_k e^{+2 pi i x0 k / 2^n} |k> (V5), phase reduced
    in integers first: ((x0*k) mod 2^n)."""
    N = 1 << n
    k = np.arange(N, dtype=np.uint64)
    ph = (np.uint64(x0) * k) & np.uint64(N - 1)  # exact mod 2^n for n <= 32
    ang = 2.0 * np.pi * ph.astype(np.float64) / N
    return (np.cos(ang) + 1j * np.sin(ang)) / math.sqrt(N)


def shor_pk(r: int, X: int) -> np.ndarray:
    """Corrected Eq. Shor5 (reading 1, "+" sign):
    the x-register distribution after the inverse QFT of the periodic state,
    p_k = [(r-(N-rs)) |S_s(th)|^2 + (N-rs) |S_{s+1}(th)|^2] / N^2 with
    N = 2^X, s = floor(N/r), th = 2 pi ((k r) mod N)/N and
    |S_m(th)|^2 = sin^2(m th/2)/sin^2(th/2) (-> m^2 at th = 0)."""
    N = 1 << X
    s = N // r
    k = np.arange(N, dtype=np.int64)
    kr = (k * r) % N
    th = 2.0 * np.pi * kr.astype(np.float64) / N
    with np.errstate(divide="ignore", invalid="ignore"):
        den = np.sin(th / 2.0) ** 2
        Ss = np.where(kr == 0, float(s * s), np.sin(s * th / 2.0) ** 2 / den)
        Ss1 = np.where(kr == 0, float((s + 1) * (s + 1)), np.sin((s + 1) * th / 2.0) ** 2 / den)
    extra = N - r * s
    return ((r - extra) * Ss + extra * Ss1) / float(N) ** 2


def shor_pk_bruteforce(r: int, X: int) -> np.ndarray:
    """V2: |FFT|^2 of the periodic x-register state, summed over f-values."""
    N = 1 << X
    p = np.zeros(N)
    for x0 in range(r):
        v = np.zeros(N, dtype=np.complex128)
        v[x0::r] = 1.0
        v /= math.sqrt(N)
        F = np.fft.fft(v) / math.sqrt(N)
        p += np.abs(F) ** 2
    return p


def expectations_from_pk(p: np.ndarray, X: int) -> np.ndarray:
    """Eq. Shor7: <Q_i> = sum_k p_k k_i."""
    k = np.arange(p.size)
    return np.array([float(np.sum(p[((k >> i) & 1) == 1])) for i in range(X)])


def fsum_probs(amps: np.ndarray, n: int, qubits: Sequence[int]) -> np.ndarray:
    """Exact-rounded marginal via math.fsum."""
    k = len(qubits)
    pr = (amps.real ** 2 + amps.imag ** 2)
    idx = np.arange(1 << n)
    beta = np.zeros(1 << n, dtype=np.int64)
    for b, q in enumerate(qubits):
        beta |= ((idx >> q) & 1) << b
    return np.array([math.fsum(pr[beta == v]) for v in range(1 << k)])

