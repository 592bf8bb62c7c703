"""The SPMD (one context per rank) exchange path on ONE GPU (-m gpu).

Each rank is a QSim on the loopback transport, driven by its own host
thread; a send/recv pair is a device copy.  This runs the unchanged code the
NCCL transport runs with P > 1 (runtime.cpp): the piece pipeline over two
streams, k_pack / unpack for non-contiguous exchange bits, k_pair_combine
for pairwise global gates, the all-gathered readouts (<Q_i>, marginals,
samples, amplitudes) and the communication timeout.  Every rank is checked
against the CPU oracle (P:759-779 exchange; P:1061-1076 readouts).
"""
import numpy as np
import pytest

from tests.test_gpu_parity import kitchen_sink, oracle_run
from workloads import circuits as C
from workloads import gates as G

pytestmark = pytest.mark.gpu
TOL = 1e-11


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_quant_ph_0608239_b200 as pkg
    return pkg


def spmd_run(P, n, ranks, init, gates, opts=None, scratch_bytes=None, readout=None):
    """Run `gates` on `ranks` loopback ranks; every rank returns its logical
    amplitudes (a collective readout), stats and readout(sim)."""
    def body(sim, r):
        for k, v in (opts or {}).items():
            sim.set_option(k, v)
        sim.init_basis(init)
        sim.run_circuit(gates)
        extra = readout(sim) if readout else None
        return sim.get_amplitudes(), sim.stats(), extra
    return P.run_loopback(n, ranks, body, scratch_bytes=scratch_bytes)


@pytest.mark.parametrize("ranks", [2, 4, 8])
@pytest.mark.parametrize("policy", [0, 1, 2])
def test_loopback_kitchen_sink(P, oracle_mod, ranks, policy):
    """Every gate kind on every position, remap / pairwise / auto policy,
    with a tiny scratch (so every exchange runs as many pipelined pieces)."""
    n = 14
    gates = kitchen_sink(n, seed=31 + ranks)
    o = oracle_run(oracle_mod, n, 3, gates)
    ref = o.amplitudes()
    res = spmd_run(P, n, ranks, 3, gates, {"global_policy": policy}, scratch_bytes=4096)
    for r, (amp, st, _) in enumerate(res):
        assert np.max(np.abs(amp - ref)) <= TOL, (r, np.max(np.abs(amp - ref)))
        assert st["exchanges"] >= 1
        assert st["link_gbs"] == 0  # 4-KB scratch: no link probe (nominal rate), on every rank alike
    assert all(np.array_equal(res[0][0], x[0]) for x in res)
    # the virtual transport (one context, device copies between its shards)
    # plans the same steps and does the same arithmetic: identical bits (with
    # the pass/exchange overlap on, as on the SPMD transports, the planner's
    # cost model and so its plan are the same)
    sim = P.QSim(n, n_ranks=ranks, transport="virtual")
    sim.set_option("overlap", 2)
    sim.set_option("global_policy", policy)
    sim.init_basis(3)
    sim.run_circuit(gates)
    assert np.array_equal(sim.get_amplitudes(), res[0][0])


@pytest.mark.parametrize("ranks", [2, 8])
def test_loopback_config5_family(P, oracle_mod, ranks):
    """The config-5 circuit family (H on all, Haar layers + CNOT chains
    through the global qubits, per-position sweep) at 20 qubits."""
    n = 20
    gates = C.random_chain(n, 4, seed=5, sweep=True)
    o = oracle_run(oracle_mod, n, 0, gates)
    ref = o.amplitudes()
    res = spmd_run(P, n, ranks, 0, gates, readout=lambda s: (s.expectations(), s.norm()))
    for amp, st, (ex, nrm) in res:
        assert np.max(np.abs(amp - ref)) <= TOL
        assert abs(1 - nrm) <= 1e-12
        assert np.max(np.abs(ex - o.expectations())) <= 1e-12
        assert st["exchanges"] >= 1
    # the link rate measured at creation is reduced to one value over the ranks
    assert res[0][1]["link_gbs"] > 0 and len({st["link_gbs"] for _, st, _ in res}) == 1


def test_loopback_noncontiguous_remap_and_readouts(P, oracle_mod):
    """Explicit SWAP-K remaps of LOW local qubits with the
    nonlocal ones: the exchanged blocks are strided (k_pack / unpack), and a
    round trip is bit-exact.  Marginals and samples are all-gathered."""
    n, ranks = 13, 4
    gates = C.random_brickwork(n, 3, seed=9)
    o = oracle_run(oracle_mod, n, 5, gates)

    def body(sim, r):
        sim.init_basis(5)
        sim.run_circuit(gates)
        before = sim.get_amplitudes()
        lay = sim.layout()
        glob = [q for q in range(n) if lay[q] >= n - 2]
        loc = sorted((q for q in range(n) if lay[q] < n - 2), key=lambda q: lay[q])[:2]  # lowest local bits
        sim.remap(loc, glob)
        lay2 = sim.layout()
        mid = sim.get_amplitudes()
        sim.remap(glob, loc)
        after = sim.get_amplitudes()
        probs = sim.probabilities([0, 5, n - 1])
        shots = sim.measure([1, 2, n - 2], seed=77, shots=500)
        return before, mid, after, lay, lay2, probs, shots, sim.stats()

    res = P.run_loopback(n, ranks, body, scratch_bytes=2048)
    ref = o.amplitudes()
    for before, mid, after, lay, lay2, probs, shots, st in res:
        assert np.max(np.abs(before - ref)) <= TOL
        assert np.array_equal(before, mid) and np.array_equal(before, after)
        assert lay2 != lay and all(lay2[q] >= n - 2 for q in range(n) if lay[q] < 2)
        assert np.max(np.abs(probs - o.probabilities([0, 5, n - 1]))) <= 1e-13
        ref_shots, tie = o.measure([1, 2, n - 2], 77, 500)
        assert np.array_equal(shots[tie == 0], ref_shots[tie == 0])
        assert st["exchanges"] >= 2


def test_loopback_timeout_on_spmd_mismatch(P):
    """An SPMD call mismatch (rank 0 exchanges, rank 1 does not) returns
    QSIM_ERR_COMM after the communication timeout instead of hanging."""
    n = 12

    def body(sim, r):
        sim.set_option("comm_timeout_ms", 1500)
        sim.init_basis(0)
        sim.run_circuit([G.one_q(q, G.H) for q in range(n)])
        sim.sync()
        if r == 0:
            lay = sim.layout()
            glob = [q for q in range(n) if lay[q] >= n - 1]
            loc = [q for q in range(n) if lay[q] == 0]
            try:
                sim.remap(loc, glob)
            except P.QsimError as e:
                return e.name
            return "no error"
        return "ok"

    res = P.run_loopback(n, 2, body)
    assert res == ["QSIM_ERR_COMM", "ok"]


@pytest.mark.parametrize("n,ranks", [(22, 2), (22, 4), (18, 8)])
def test_overlapped_pass_exchange(P, oracle_mod, n, ranks):
    """A pass followed by an exchange whose local bits are not tile bits of
    the pass runs block by block with each block's transfer overlapping the
    next block's compute (option "overlap"): identical amplitudes with the
    overlap on and off, on the loopback (NCCL-branch) and virtual transports,
    and equal to the oracle (config-5 family circuits where it applies)."""
    gates = C.random_chain(n, 6, seed=15, sweep=True)
    ref = oracle_run(oracle_mod, n, 0, gates).amplitudes()
    out = {}
    for ov in (1, 0):
        res = spmd_run(P, n, ranks, 0, gates, {"overlap": ov}, scratch_bytes=1 << 16)
        out[ov] = res
        for amp, st, _ in res:
            assert np.max(np.abs(amp - ref)) <= TOL
            assert (st["overlapped"] >= 1) == bool(ov)
    assert np.array_equal(out[0][0][0], out[1][0][0])
    sim = P.QSim(n, n_ranks=ranks, transport="virtual")
    sim.set_option("overlap", 2)  # virtual shards overlap only on request
    sim.init_basis(0)
    sim.run_circuit(gates)
    got = sim.get_amplitudes()
    assert sim.stats()["overlapped"] >= 1
    assert np.array_equal(got, out[1][0][0])
