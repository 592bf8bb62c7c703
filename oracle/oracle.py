"""ctypes front-end of oracle/qsim_oracle.c (TEST INFRASTRUCTURE ONLY).

`Oracle(n)` holds one plain 2^n complex128 array and applies a gate list
from `workloads` gate by gate, in the given order, with the C routines that
restate the paper's update rules (see the C file's header for citations).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "qsim_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def oracle_lib_path() -> str:
    return _LIB


def build_oracle(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", _LIB + ".tmp", _SRC, "-lm"])
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build_oracle()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.POINTER
        d, i, u64 = ctypes.c_double, ctypes.c_int, ctypes.c_uint64
        lib.or_init_basis.argtypes = [P(d), i, u64]
        lib.or_apply_controlled.argtypes = [P(d), i, P(i), i, i, P(d)]
        lib.or_apply_1q.argtypes = [P(d), i, i, P(d)]
        lib.or_apply_perm.argtypes = [P(d), i, P(i), i, P(i), i, P(ctypes.c_uint32)]
        lib.or_apply_perm.restype = i
        lib.or_swap.argtypes = [P(d), i, i, i]
        lib.or_probabilities.argtypes = [P(d), i, P(i), i, P(d)]
        lib.or_expectations.argtypes = [P(d), i, P(d)]
        lib.or_sample.argtypes = [P(d), i, u64, u64, P(u64), P(ctypes.c_uint8)]
        lib.or_num_threads.restype = i
        _lib = lib
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(seq: Sequence[int]):
    arr = (ctypes.c_int * max(1, len(seq)))(*seq)
    return arr


def u_to_doubles(u) -> np.ndarray:
    return np.array([c for z in u for c in (complex(z).real, complex(z).imag)], dtype=np.float64)


class Oracle:
    """One plain 2^n complex128 state vector (qubit 0 = LSB)."""

    def __init__(self, n: int):
        assert 1 <= n <= 34
        self.n = n
        self.lib = _load()
        self.psi = np.zeros(2 << n, dtype=np.float64)

    @staticmethod
    def threads() -> int:
        return _load().or_num_threads()

    def init_basis(self, x: int) -> None:
        assert 0 <= x < (1 << self.n)
        self.lib.or_init_basis(_dp(self.psi), self.n, x)

    def set_state(self, amps: np.ndarray) -> None:
        a = np.asarray(amps, dtype=np.complex128)
        assert a.size == 1 << self.n
        self.psi[0::2] = a.real
        self.psi[1::2] = a.imag

    def amplitudes(self) -> np.ndarray:
        return self.psi.view(np.complex128).copy()

    def apply(self, g) -> None:
        from workloads.gates import G_1Q, G_CTRL, G_PERM, G_SWAP
        if g.kind == G_1Q:
            self.lib.or_apply_1q(_dp(self.psi), self.n, g.target, _dp(u_to_doubles(g.u)))
        elif g.kind == G_CTRL:
            c = list(g.controls)
            self.lib.or_apply_controlled(_dp(self.psi), self.n, _ip(c), len(c), g.target,
                                         _dp(u_to_doubles(g.u)))
        elif g.kind == G_PERM:
            c, t = list(g.controls), list(g.targets)
            perm = np.ascontiguousarray(g.perm, dtype=np.uint32)
            rc = self.lib.or_apply_perm(_dp(self.psi), self.n, _ip(c), len(c), _ip(t), len(t),
                                        perm.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)))
            if rc != 0:
                raise ValueError("permutation is not a bijection")
        elif g.kind == G_SWAP:
            self.lib.or_swap(_dp(self.psi), self.n, g.targets[0], g.targets[1])
        else:
            raise ValueError(g.kind)

    def run(self, gates) -> None:
        for g in gates:
            self.apply(g)

    def probabilities(self, qubits: Sequence[int]) -> np.ndarray:
        k = len(qubits)
        out = np.zeros(1 << k, dtype=np.float64)
        self.lib.or_probabilities(_dp(self.psi), self.n, _ip(list(qubits)), k, _dp(out))
        return out

    def norm(self) -> float:
        return float(self.probabilities([])[0])

    def expectations(self) -> np.ndarray:
        out = np.zeros(self.n, dtype=np.float64)
        self.lib.or_expectations(_dp(self.psi), self.n, _dp(out))
        return out

    def measure(self, qubits: Sequence[int], seed: int, shots: int,
                probs: Optional[np.ndarray] = None):
        """Returns (outcomes uint64[shots], tie flags uint8[shots])."""
        p = self.probabilities(qubits) if probs is None else np.ascontiguousarray(probs)
        return sample_from(p, len(qubits), seed, shots)


def sample_from(p: np.ndarray, k: int, seed: int, shots: int):
    lib = _load()
    p = np.ascontiguousarray(p, dtype=np.float64)
    out = np.zeros(shots, dtype=np.uint64)
    tie = np.zeros(shots, dtype=np.uint8)
    lib.or_sample(_dp(p), k, seed, shots, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                  tie.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)))
    return out, tie
