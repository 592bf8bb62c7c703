"""Full-register sampling on the GPU (-m gpu).

qsim_measure with k > 24 listed qubits runs the two-level sampler: the draw
u_s and the outcome rule min{beta : C(beta) > u_s} are the one-level rule's
(reading R14), so the outcomes equal the oracle's sampler on the full 2^k
marginal exactly, except draws within 1e-12 of a CDF boundary (ties).
"""
import numpy as np
import pytest

from workloads import circuits as C

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_quant_ph_0608239_b200 as pkg
    return pkg


def _oracle(oracle_mod, n, init, gates):
    o = oracle_mod.Oracle(n)
    o.init_basis(init)
    o.run(gates)
    return o


def _check(shots, ref, tie, min_ok):
    ok = tie == 0
    assert ok.sum() >= min_ok
    assert np.array_equal(shots[ok], ref[ok])


@pytest.mark.parametrize("ranks", [1, 8])
def test_measure_whole_register_26q(P, oracle_mod, ranks):
    """All 26 qubits (k = n) of a random state, 1 shard and 8 virtual shards."""
    n = 26
    gates = C.random_brickwork(n, 3, seed=12)
    sim = P.QSim(n, n_ranks=ranks, transport="local" if ranks == 1 else "virtual")
    sim.init_basis(0)
    sim.run_circuit(gates)
    o = _oracle(oracle_mod, n, 0, gates)
    qs = list(range(n))
    shots = sim.measure(qs, seed=2024, shots=48)
    ref, tie = o.measure(qs, 2024, 48)
    _check(shots, ref, tie, 40)
    sim.close()


def test_measure_permuted_listed_subset(P, oracle_mod):
    """25 of 27 qubits listed in a shuffled order (unlisted qubits summed,
    beta bit b <-> qubits[b]), after a remapping circuit (sigma != identity)."""
    n = 27
    gates = C.random_chain(n, 2, seed=4, sweep=False) + C.qft_ladder(list(range(8)), swaps=True)
    sim = P.QSim(n, n_ranks=4, transport="virtual")
    sim.init_basis(5)
    sim.run_circuit(gates)
    o = _oracle(oracle_mod, n, 5, gates)
    qs = [int(q) for q in np.random.default_rng(3).permutation(n)[:25]]
    shots = sim.measure(qs, seed=99, shots=40)
    ref, tie = o.measure(qs, 99, 40)
    _check(shots, ref, tie, 32)
    sim.close()


def test_measure_two_level_batches(P, oracle_mod):
    """The second level built in many small batches of high bins (option
    sample_batch) gives the same outcomes as one batch."""
    n = 26
    gates = C.random_brickwork(n, 2, seed=31)
    sim = P.QSim(n, n_ranks=2, transport="virtual")
    sim.init_basis(0)
    sim.run_circuit(gates)
    qs = list(range(n))
    one = sim.measure(qs, seed=5, shots=64)
    sim.set_option("sample_batch", 3)
    many = sim.measure(qs, seed=5, shots=64)
    assert np.array_equal(one, many)
    o = _oracle(oracle_mod, n, 0, gates)
    ref, tie = o.measure(qs, 5, 64)
    _check(many, ref, tie, 56)
    sim.close()


def test_measure_whole_register_loopback(P, oracle_mod):
    """k = n = 25 on 4 SPMD loopback ranks (the NCCL-branch reductions), with
    enough shots and small batches that the rank-order reduction buffer is
    larger than the sampler's first buffers (they must not alias)."""
    n = 25
    gates = C.random_brickwork(n, 2, seed=21)
    o = _oracle(oracle_mod, n, 0, gates)
    ref, tie = o.measure(list(range(n)), 7, 40)
    qs = [int(q) for q in np.random.default_rng(5).permutation(n)]  # the whole register, permuted order
    ref2, tie2 = o.measure(qs[:25], 8, 40)

    def body(sim, r):
        sim.init_basis(0)
        sim.run_circuit(gates)
        a = sim.measure(list(range(n)), seed=7, shots=40)
        sim.set_option("sample_batch", 5)
        b = sim.measure(qs[:25], seed=8, shots=40)
        sim.set_option("sample_batch", 0)
        many = sim.measure(list(range(n)), seed=9, shots=20000)
        return a, b, many

    for a, b, many in P.run_loopback(n, 4, body):
        _check(a, ref, tie, 32)
        _check(b, ref2, tie2, 32)
        # 20000 shots of the whole register: the outcome frequencies follow |a|^2
        p = np.abs(o.amplitudes()) ** 2
        assert abs(float(np.mean(p[many.astype(np.int64)])) - float(np.sum(p * p))) < 0.2 * float(np.sum(p * p))


def test_measure_basis_state_and_limits(P):
    """A basis state samples to itself at every shot (k = n = 30)."""
    n = 30
    sim = P.QSim(n)
    x = 0x2ACE1234 & ((1 << n) - 1)
    sim.init_basis(x)
    sim.run_circuit([])
    got = sim.measure(list(range(n)), seed=1, shots=16)
    assert np.all(got == x)
    sim.close()
