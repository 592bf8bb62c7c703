"""Shor end to end (§VI.B): classical post-processing pinned on CPU
against exact arithmetic and the closed-form distribution; the quantum part on
the GPU against the oracle and the closed form."""
import math

import numpy as np
import pytest

from paper_quant_ph_0608239_b200 import shor
from tests import pins
from workloads import circuits as C


def test_convergents_are_best_approximations():
    # 0.[1;2,2,2,...] style check: the convergents of k/2^X reproduce k/2^X at the end
    for k, X in [(3, 4), (1365, 12), (2**18 - 1, 18), (173, 9)]:
        cv = shor.convergents(k, X)
        p, q = cv[-1]
        assert p * (1 << X) == k * q and math.gcd(p, q) == 1
        for (p1, q1), (p2, q2) in zip(cv, cv[1:]):
            assert abs(p2 * q1 - p1 * q2) == 1  # consecutive convergents are unimodular


@pytest.mark.parametrize("G,y", [(15, 7), (21, 2), (35, 3), (247, 194), (899, 2)])
def test_order_from_closed_form_samples(G, y):
    """Samples drawn from the corrected closed form p_k(r) (reading R1) with X
    satisfying Eq. Shor0 recover the multiplicative order r."""
    r = C.multiplicative_order(y, G)
    X = (G * G - 1).bit_length()  # G^2 <= 2^X <= 2 G^2 (Eq. Shor0)
    p = pins.shor_pk(r, X)
    rng = np.random.default_rng(G)
    ks = rng.choice(p.size, size=24, p=p / p.sum())
    assert shor.order_from_samples(ks, X, G, y) == r


def test_factors_from_order():
    assert shor.factors_from_order(15, 7, 4) == (3, 5)
    assert shor.factors_from_order(247, 194, 18) == (13, 19)     # Table III L=24 row
    assert shor.factors_from_order(21, 2, 6) == (3, 7)
    assert shor.factors_from_order(15, 14, 2) is None             # y^(r/2) = -1 mod G


def test_circuit_matches_workload_generator():
    """The product's Shor circuit and the test generator agree gate for gate."""
    g1 = shor.circuit(35, 3, 8, 6)
    w = C.shor_order_finding(35, 3, 8, 6)
    assert len(g1) == len(w.gates)
    for a, b in zip(g1, w.gates):
        assert a.kind == b.kind and a.target == b.target and tuple(a.controls) == tuple(b.controls)
        assert tuple(a.targets) == tuple(b.targets)
        assert np.allclose(np.asarray(a.u, dtype=complex), np.asarray(b.u, dtype=complex), atol=1e-15)
        if a.perm is not None:
            assert np.array_equal(a.perm, b.perm)


@pytest.mark.gpu
@pytest.mark.parametrize("G,y,X,F", [(247, 194, 16, 8), (15, 7, 8, 4), (899, 2, 20, 10)])
def test_shor_end_to_end_gpu(G, y, X, F):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    res = shor.run(G, y, X, F, shots=32, seed=5)
    r = C.multiplicative_order(y, G)
    assert np.max(np.abs(res.expectations - pins.expectations_from_pk(pins.shor_pk(r, X), X))) <= 1e-10
    assert res.r == r
    want = shor.factors_from_order(G, y, r)
    assert res.factors == want
