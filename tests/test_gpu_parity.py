"""GPU parity: the CUDA path through the C-ABI vs the CPU oracle (-m gpu).

Bar (BASELINE.json north_star): max |delta amplitude| <= 1e-11,
|1 - ||psi||^2| <= 1e-12, measured basis states / integer outcomes exact
(sampling ties within 1e-12 of a CDF boundary excluded, reading R14).
"""
import math
import os

import numpy as np
import pytest

from tests import pins
from workloads import circuits as C
from workloads import gates as G

pytestmark = pytest.mark.gpu
TOL = 1e-11
NORM_TOL = 1e-12


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_quant_ph_0608239_b200 as pkg
    return pkg


def gpu_run(P, n, init, gates, ranks=1, fusion=True, transport=None, jit=1):
    tp = transport or ("local" if ranks == 1 else "virtual")
    sim = P.QSim(n, n_ranks=ranks, transport=tp)
    sim.set_option("fusion", int(fusion))
    sim.set_option("jit", int(jit))
    sim.init_basis(init)
    sim.run_circuit(gates)
    return sim


def oracle_run(oracle_mod, n, init, gates):
    o = oracle_mod.Oracle(n)
    o.init_basis(init)
    o.run(gates)
    return o


def assert_parity(sim, o, n):
    got = sim.get_amplitudes()
    ref = o.amplitudes()
    err = np.max(np.abs(got - ref))
    assert err <= TOL, err
    assert abs(1 - sim.norm()) <= NORM_TOL
    return got


def kitchen_sink(n, seed):
    """Every gate kind on every position: Haar layer, H/X/Y/Xbar/Ybar/R, CNOT,
    CP, controlled-V, Toffoli, 2-control U2, perms, swaps."""
    rng = G.SplitMix64(seed)
    r = np.random.default_rng(seed)
    gates = [G.one_q(q, G.haar_u2(rng)) for q in range(n)]
    named = [G.H, G.X, G.Y, G.XBAR, G.YBAR, G.R(0.37)]
    for q in range(n):
        gates.append(G.one_q(q, named[q % len(named)]))
        c = (q + 1 + q % 3) % n
        gates.append(G.cnot(c, q))
        gates.append(G.cphase((q + 5) % n, q, 0.1 * (q + 1)))
        gates.append(G.ctrl([(q + 2) % n], q, G.V(0.3 + q)))
        a, b = (q + 3) % n, (q + 7) % n
        if len({a, b, q}) == 3:
            gates.append(G.toffoli(a, b, q))
            gates.append(G.ctrl([a, b], q, G.haar_u2(rng)))
        gates.append(G.one_q(q, G.haar_u2(rng)))
    for t0 in range(0, n - 2, 3):
        tg = [t0, (t0 + 4) % n, (t0 + 9) % n]
        if len(set(tg)) == 3:
            ctl = [x for x in [(t0 + 1) % n] if x not in tg]
            gates.append(G.perm_gate(ctl, tg, r.permutation(8).astype(np.uint32)))
    gates.append(G.swap(0, n - 1))
    gates.append(G.one_q(0, G.haar_u2(rng)))
    gates.append(G.swap(2, 5))
    gates += [G.one_q(q, G.haar_u2(rng)) for q in range(n)]
    return gates


@pytest.mark.parametrize("n", [11, 12, 13, 16])
@pytest.mark.parametrize("fusion", [True, False])
def test_every_gate_every_position(P, oracle_mod, n, fusion):
    gates = kitchen_sink(n, seed=n)
    sim = gpu_run(P, n, 5, gates, fusion=fusion)
    assert_parity(sim, oracle_run(oracle_mod, n, 5, gates), n)


@pytest.mark.parametrize("n,ranks", [(13, 1), (16, 1), (15, 4)])
def test_jit_tier_matches_interpreter(P, oracle_mod, n, ranks):
    """The NVRTC pass-specialised kernels and the interpreter k_pass.  They
    round differently (the JIT tier applies general 2x2 and 4x4 blocks in the
    3M form, accumulates exact integer phase angles and applies Hadamards as
    sums/differences) and agree to 1e-13; both match the oracle."""
    plain = C.random_brickwork(n, 4, seed=n)
    s_int = gpu_run(P, n, 1, plain, ranks=ranks, jit=0)
    s_jit = gpu_run(P, n, 1, plain, ranks=ranks, jit=1)
    a_int, a_jit = s_int.get_amplitudes(), s_jit.get_amplitudes()
    assert s_jit.stats()["jit_launches"] > 0, s_jit.lib.qsim_last_error(s_jit.ctx).decode()[:3000]
    assert s_int.stats()["jit_launches"] == 0
    assert np.max(np.abs(a_int - a_jit)) <= 1e-13
    gates = kitchen_sink(n, seed=7 * n) + C.qft_ladder(list(range(n)), True) + plain
    s_int = gpu_run(P, n, 1, gates, ranks=ranks, jit=0)
    s_jit = gpu_run(P, n, 1, gates, ranks=ranks, jit=1)
    assert np.max(np.abs(s_int.get_amplitudes() - s_jit.get_amplitudes())) <= 1e-13
    o = oracle_run(oracle_mod, n, 1, gates)
    assert_parity(s_jit, o, n)
    assert_parity(s_int, o, n)


def mixed_blocks(n, seed):
    """Brickwork layers interleaved with gates that touch a block's pair from
    outside (controls, phases, Toffolis, swaps, one-qubit runs)."""
    rng = G.SplitMix64(seed)
    gates = []
    for layer in range(5):
        gates += [G.one_q(q, G.haar_u2(rng)) for q in range(n)]
        gates += [G.cnot(q, q + 1) for q in range(layer % 2, n - 1, 2)]
        gates += [G.cphase(1, 2, 0.3 + layer), G.ctrl([5], 3, G.haar_u2(rng)), G.one_q(4, G.H),
                  G.one_q(4, G.haar_u2(rng)), G.toffoli(0, 6, 7), G.ctrl([8], 9, G.haar_u2(rng)),
                  G.one_q(8, G.haar_u2(rng)), G.one_q(9, G.haar_u2(rng)), G.swap(10, n - 1),
                  G.ctrl([2], 1, G.PAULI_X), G.one_q(2, G.R(0.7)), G.ctrl([n - 1], 0, G.haar_u2(rng))]
    return gates


@pytest.mark.parametrize("n,ranks", [(13, 1), (16, 1), (16, 4)])
@pytest.mark.parametrize("jit", [0, 1])
def test_block_fusion_parity(P, oracle_mod, n, ranks, jit):
    """Fused two-qubit blocks (OPC_U4, plan.cpp fuse_ops) vs the oracle, with
    block fusion on and off, on both pass tiers."""
    gates = C.random_brickwork(n, 6, seed=n) + mixed_blocks(n, seed=n)
    o = oracle_run(oracle_mod, n, 9, gates)
    for bf in (1, 0):
        sim = P.QSim(n, n_ranks=ranks, transport="local" if ranks == 1 else "virtual")
        sim.set_option("jit", jit)
        sim.set_option("block_fusion", bf)
        sim.init_basis(9)
        sim.run_circuit(gates)
        assert_parity(sim, o, n)


@pytest.mark.parametrize("n,ranks", [(13, 1), (16, 1), (16, 4), (14, 2)])
def test_perm_run_parity(P, oracle_mod, n, ranks):
    """A run of permutations of one register with 0/1/2 controls in and out of
    the tile, on contiguous (low) and scattered targets (k_perm_run)."""
    r = np.random.default_rng(n + ranks)
    gates = [G.one_q(q, G.haar_u2(G.SplitMix64(q + 1))) for q in range(n)]
    for tg in [(0, 1, 2), (5, 1, n - 3, 8)]:
        for ctl in [(), (4,), (n - 1, 3), (n - 2,), (6,), (3, n - 1), ()]:
            if set(ctl) & set(tg):
                continue
            gates.append(G.perm_gate(ctl, tg, r.permutation(1 << len(tg)).astype(np.uint32)))
        gates.append(G.cnot(tg[0], n - 1))
    sim = gpu_run(P, n, 3, gates, ranks=ranks)
    assert_parity(sim, oracle_run(oracle_mod, n, 3, gates), n)


@pytest.mark.parametrize("ranks", [1, 4])
def test_expectations_async(P, oracle_mod, ranks):
    """qsim_expectations_async into pinned memory, several circuits enqueued
    back to back before one sync: each buffer holds its own circuit's <Q_i>,
    bitwise equal to the synchronous call, and equal to the oracle's."""
    import torch
    n = 14
    sim = P.QSim(n, n_ranks=ranks, transport="virtual" if ranks > 1 else "local")
    circuits = [C.random_brickwork(n, 3, seed=s) for s in range(3)]
    bufs = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in circuits]
    for g, b in zip(circuits, bufs):
        sim.init_basis(3)
        sim.run_circuit(g)
        sim.expectations_async(b)
    sim.sync()
    for g, b in zip(circuits, bufs):
        sim.init_basis(3)
        sim.run_circuit(g)
        ex = sim.expectations()
        assert np.array_equal(b.numpy(), ex)
        assert np.max(np.abs(ex - oracle_run(oracle_mod, n, 3, g).expectations())) <= 1e-12


@pytest.mark.parametrize("ranks", [1, 4])
def test_fused_readout(P, oracle_mod, ranks):
    """<Q_i> fused into the last pass (readout variant, option fuse_readout):
    equal to the separate reduction's and the oracle's to 1e-13, on circuits
    whose last pass ends with deferred predicated swaps, phase runs, a fresh
    single pass, and one whose last data step is a permutation run (no
    fusion: the separate reduction runs)."""
    w3 = C.shor_order_finding(35, 3, 8, 6)
    w1 = C.config1_adder()
    cases = [(14, 5, kitchen_sink(14, seed=4)), (w1.n, w1.init, w1.gates), (16, 0, C.random_brickwork(16, 5, seed=8)),
             (18, 77, C.qft_basis(18, 77).gates), (13, 1, [G.one_q(q, G.H) for q in range(13)]),
             (w3.n, w3.init, w3.gates[:1 + max(i for i, g in enumerate(w3.gates) if g.kind == G.G_PERM)])]
    for n, init, gates in cases:
        ref = oracle_run(oracle_mod, n, init, gates).expectations()
        got = {}
        for fuse in (1, 0):
            sim = P.QSim(n, n_ranks=ranks, transport="local" if ranks == 1 else "virtual")
            sim.set_option("fuse_readout", fuse)
            sim.init_basis(init)
            sim.run_circuit(gates)
            got[fuse] = sim.expectations()
            st = sim.stats()
            sim.close()
            assert np.max(np.abs(got[fuse] - ref)) <= 1e-13, (n, fuse)
            if not fuse:
                assert st["fused_readouts"] == 0
        assert np.max(np.abs(got[1] - got[0])) <= 1e-13


def test_fused_readout_loopback(P, oracle_mod):
    """The fused readout on 4 loopback ranks (SPMD: per-rank partials, all-
    gathered and combined in rank order)."""
    n, gates = 16, C.random_chain(16, 3, seed=21, sweep=True)

    def body(sim, r):
        sim.init_basis(9)
        sim.run_circuit(gates)
        return sim.expectations(), sim.stats()["fused_readouts"]

    ref = oracle_run(oracle_mod, n, 9, gates).expectations()
    for ex, nf in P.run_loopback(n, 4, body):
        assert np.max(np.abs(ex - ref)) <= 1e-13
        assert nf >= 1


def test_perm_run_max_shared_memory(P, oracle_mod):
    """12-qubit register, 20 controlled perms: runs of 12 and 8 whose tables
    and double-buffered tiles take up to 224 KB of shared memory per CTA."""
    r = np.random.default_rng(9)
    n, tg = 16, tuple(range(12))
    gates = [G.one_q(q, G.haar_u2(G.SplitMix64(q))) for q in range(n)]
    for j in range(20):
        gates.append(G.perm_gate((12 + j % 4,), tg, r.permutation(1 << 12).astype(np.uint32)))
    sim = gpu_run(P, n, 5, gates)
    assert_parity(sim, oracle_run(oracle_mod, n, 5, gates), n)
    assert sim.stats()["perm_launches"] == 2


@pytest.mark.parametrize("ranks", [1, 4])
def test_streamed_flush_parity(P, oracle_mod, ranks):
    """Steps launched while the planner still runs (runtime.cpp flush): with
    the JIT kernels cached and the plan cache off, the passes before the
    permutation stream, the rest goes the batch way (upload + launch); both
    runs, and a third through the plan cache, match the oracle."""
    n = 16
    gates = (C.random_brickwork(n, 6, seed=7) + [G.perm_gate((3,), (0, 1, 2), np.array([3, 0, 7, 1, 2, 6, 4, 5], np.uint32))]
             + C.qft_ladder(list(range(n)), swaps=True) + C.random_brickwork(n, 2, seed=8))
    ref = oracle_run(oracle_mod, n, 5, gates)
    sim = P.QSim(n, n_ranks=ranks, transport="virtual" if ranks > 1 else "local")
    sim.set_option("plan_cache", 0)
    for rep in range(2):
        sim.init_basis(5)
        sim.run_circuit(gates)
        assert_parity(sim, ref, n)
    st = sim.stats()
    assert st["streamed_steps"] > 0 and st["perm_launches"] > 0
    sim.set_option("plan_cache", 1)
    for rep in range(2):
        sim.init_basis(5)
        sim.run_circuit(gates)
        assert_parity(sim, ref, n)
    assert sim.stats()["plan_cache_hits"] >= 1


@pytest.mark.parametrize("ranks,n", [(2, 14), (4, 15), (8, 16), (8, 12), (4, 9)])
def test_every_gate_sharded_virtual(P, oracle_mod, ranks, n):
    gates = kitchen_sink(n, seed=100 + n)
    sim = gpu_run(P, n, 3, gates, ranks=ranks)
    assert_parity(sim, oracle_run(oracle_mod, n, 3, gates), n)
    st = sim.stats()
    assert st["exchanges"] > 0


@pytest.mark.parametrize("policy,ranks,n", [(1, 2, 14), (1, 8, 16), (1, 4, 9), (2, 8, 15)])
def test_global_policy_pairwise_virtual(P, oracle_mod, policy, ranks, n):
    """Pairwise combine of partner shards for gates on nonlocal qubits."""
    gates = kitchen_sink(n, seed=200 + n) + C.random_chain(n, 1, seed=n, sweep=True)
    sim = P.QSim(n, n_ranks=ranks, transport="virtual")
    sim.set_option("global_policy", policy)
    sim.init_basis(2)
    sim.run_circuit(gates)
    assert_parity(sim, oracle_run(oracle_mod, n, 2, gates), n)


def test_tiny_states(P, oracle_mod):
    for n, ranks in [(1, 1), (2, 1), (2, 2), (3, 4), (5, 1)]:
        gates = [G.one_q(q, G.haar_u2(G.SplitMix64(q))) for q in range(n)]
        if n >= 2:
            gates += [G.cnot(0, 1), G.cphase(1, 0, 0.5)]
        sim = gpu_run(P, n, (1 << n) - 1, gates, ranks=ranks)
        assert_parity(sim, oracle_run(oracle_mod, n, (1 << n) - 1, gates), n)


def test_config1_adder(P, oracle_mod):
    w = C.config1_adder()
    sim = gpu_run(P, w.n, w.init, w.gates)
    got = assert_parity(sim, oracle_run(oracle_mod, w.n, w.init, w.gates), w.n)
    p = np.abs(got) ** 2
    assert int(np.argmax(p)) == w.meta["expect_index"]
    assert p[w.meta["expect_index"]] >= 1 - 1e-12
    shots = sim.measure(list(range(w.n)), seed=7, shots=64)
    assert np.all(shots == w.meta["expect_index"])


def test_adder_all_inputs_m5(P):
    m = 5
    gates = C.qft_adder([list(range(m)), list(range(m, 2 * m))])
    for a in range(0, 32, 3):
        for b in range(0, 32, 5):
            sim = gpu_run(P, 2 * m, a + (b << m), gates)
            pb = sim.probabilities(list(range(m, 2 * m)))
            assert pb[(a + b) % 32] >= 1 - 1e-12


@pytest.mark.parametrize("ranks", [1, 2, 4, 8])
def test_random_brickwork_small(P, oracle_mod, ranks):
    n = 18
    gates = C.random_brickwork(n, 12, seed=2)
    sim = gpu_run(P, n, 0, gates, ranks=ranks)
    assert_parity(sim, oracle_run(oracle_mod, n, 0, gates), n)


def test_config2_full(P, oracle_mod):
    """BASELINE config 2 at full size (24 q, depth 40, 1420 gates): full state."""
    w = C.config2_random()
    sim = gpu_run(P, w.n, w.init, w.gates)
    o = oracle_run(oracle_mod, w.n, w.init, w.gates)
    assert_parity(sim, o, w.n)
    ex = sim.expectations()
    assert np.max(np.abs(ex - o.expectations())) <= 1e-12


def test_config2_echo_and_determinism(P):
    w = C.config2_random()
    sim = gpu_run(P, w.n, 0, w.gates)
    a1 = sim.get_amplitudes(0, 1 << 16)
    sim2 = gpu_run(P, w.n, 0, w.gates)
    a2 = sim2.get_amplitudes(0, 1 << 16)
    assert np.array_equal(a1, a2)  # bitwise deterministic
    sim.run_circuit(C.inverse(w.gates))
    amps = sim.get_amplitudes(0, 1 << 12)
    assert abs(amps[0] - 1) < 1e-11 and np.max(np.abs(amps[1:])) < 1e-11


def test_shor_small(P, oracle_mod):
    w = C.shor_order_finding(35, 3, 10, 6)
    sim = gpu_run(P, w.n, w.init, w.gates)
    o = oracle_run(oracle_mod, w.n, w.init, w.gates)
    assert_parity(sim, o, w.n)
    ctl = list(range(10))
    pg = sim.probabilities(ctl)
    assert np.max(np.abs(pg - pins.shor_pk(w.meta["r"], 10))) < 1e-12
    shots = sim.measure(ctl, seed=11, shots=500)
    ref, tie = o.measure(ctl, seed=11, shots=500)
    ok = tie == 0
    assert np.array_equal(shots[ok], ref[ok])


@pytest.mark.parametrize("ranks", [2, 4])
def test_shor_sharded(P, oracle_mod, ranks):
    w = C.shor_order_finding(21, 2, 9, 5)
    sim = gpu_run(P, w.n, w.init, w.gates, ranks=ranks)
    assert_parity(sim, oracle_run(oracle_mod, w.n, w.init, w.gates), w.n)


def test_config3_full(P, oracle_mod):
    """BASELINE config 3 (28 q, N=899): the control-register marginal equals
    the corrected closed form (reading 1/8) and samples match the oracle's
    sampler applied to that closed form with the same seed."""
    w = C.config3_shor()
    sim = gpu_run(P, w.n, w.init, w.gates)
    ctl = list(range(18))
    pg = sim.probabilities(ctl)
    pk = pins.shor_pk(w.meta["r"], 18)
    assert np.max(np.abs(pg - pk)) <= 1e-10
    assert abs(1 - sim.norm()) <= NORM_TOL
    from oracle.oracle import sample_from
    shots = sim.measure(ctl, seed=3, shots=2000)
    ref, tie = sample_from(pk, 18, 3, 2000)
    ok = tie == 0
    assert ok.sum() > 1900 and np.array_equal(shots[ok], ref[ok])


def phase_kinds_circuit(n, seed):
    """Long runs of diagonal phases whose terms take every form the JIT phase
    runs have (jit.cpp PhasePlan): unpredicated R (host-formed factors),
    controlled phases with far controls (CTA-uniform slots), with controls on
    lane/warp-range qubits (per-thread slots), mixed and sparse ones
    (accumulators), split into several flush epochs by interleaved H gates."""
    r = np.random.default_rng(seed)
    gates = [G.one_q(q, G.H) for q in range(n)]
    for rnd in range(6):
        for _ in range(3 * n):
            kind = r.integers(4)
            q = int(r.integers(n))
            phi = float(r.uniform(-math.pi, math.pi))
            if kind == 0:
                gates.append(G.one_q(q, G.R(phi)))
            elif kind == 1:
                c = int(r.integers(n))
                if c != q:
                    gates.append(G.cphase(c, q, phi))
            elif kind == 2:
                a, b = (int(x) for x in r.choice(n, 2, replace=False))
                if q not in (a, b):
                    gates.append(G.ctrl([a, b], q, G.R(phi)))
            else:
                c = n - 1 - int(r.integers(3))
                if c != q:
                    gates.append(G.cphase(c, q, phi))
        for q in r.choice(n, 3, replace=False):
            gates.append(G.one_q(int(q), G.H if rnd % 2 else G.haar_u2(G.SplitMix64(seed + rnd))))
    return gates


@pytest.mark.parametrize("n,ranks", [(14, 1), (18, 1), (21, 1), (18, 4)])
def test_phase_run_factor_kinds(P, oracle_mod, n, ranks):
    """Phase runs with host-formed, per-tile, per-launch and accumulated
    factors in the same passes vs the oracle (and the interpreter tier)."""
    gates = phase_kinds_circuit(n, 100 + n)
    o = oracle_run(oracle_mod, n, 5, gates)
    for jit in (1, 0):
        sim = gpu_run(P, n, 5, gates, ranks=ranks, jit=jit)
        assert_parity(sim, o, n)
        sim.close()


@pytest.mark.parametrize("ranks", [1, 2, 4, 8])
def test_qft_closed_form(P, ranks):
    n, x0 = 20, 0xABCDE
    w = C.qft_basis(n, x0)
    sim = gpu_run(P, n, x0, w.gates, ranks=ranks)
    got = sim.get_amplitudes()
    assert np.max(np.abs(got - pins.qft_closed_form(n, x0))) <= TOL


def test_config4_qft32_one_gpu(P):
    """BASELINE config 4 (32 q, 64 GiB) on one GPU: sampled blocks vs the
    closed form with integer phase reduction."""
    import torch
    free, _ = torch.cuda.mem_get_info()
    if free < (70 << 30):
        pytest.skip("needs ~70 GB free")
    w = C.config4_qft()
    sim = gpu_run(P, 32, w.init, w.gates)
    rng = np.random.default_rng(4)
    x0 = w.meta["x0"]
    for start in rng.integers(0, (1 << 32) - 4096, size=16):
        got = sim.get_amplitudes(int(start), 4096)
        k = np.arange(int(start), int(start) + 4096, dtype=np.uint64)
        ph = (np.uint64(x0) * k) & np.uint64((1 << 32) - 1)
        ref = np.exp(2j * np.pi * ph.astype(np.float64) / 2.0 ** 32) / 2.0 ** 16
        assert np.max(np.abs(got - ref)) <= TOL
    assert abs(1 - sim.norm()) <= NORM_TOL
    sim.close()


def test_config5_family_sharded(P, oracle_mod):
    """config 5's circuit family (H all, Haar layers + CNOT chain, sweep) on
    8 virtual shards (3 nonlocal qubits)."""
    n = 18
    gates = C.random_chain(n, 3, seed=5, sweep=True)
    sim = gpu_run(P, n, 0, gates, ranks=8)
    o = oracle_run(oracle_mod, n, 0, gates)
    assert_parity(sim, o, n)
    assert np.max(np.abs(sim.expectations() - o.expectations())) <= 1e-12


@pytest.mark.parametrize("ranks", [1, 4])
def test_readouts(P, oracle_mod, ranks):
    n = 16
    gates = C.random_brickwork(n, 5, seed=8)
    sim = gpu_run(P, n, 0, gates, ranks=ranks)
    o = oracle_run(oracle_mod, n, 0, gates)
    for qs in ([], [0], [15], [3, 14], [13, 0, 7], list(range(10)), [15, 14, 1, 2, 12, 8]):
        assert np.max(np.abs(sim.probabilities(qs) - o.probabilities(qs))) <= 1e-13
    assert np.max(np.abs(sim.expectations() - o.expectations())) <= 1e-13
    qs = [2, 9, 15, 0]
    shots = sim.measure(qs, seed=1234, shots=5000)
    ref, tie = o.measure(qs, seed=1234, shots=5000)
    assert np.array_equal(shots[tie == 0], ref[tie == 0])


def _table_blocks():
    blocks, cur = [], None
    for line in open(os.path.join(os.path.dirname(__file__), "golden", "tables_I_II.txt")):
        if line.startswith("#") or not line.strip():
            continue
        if line.startswith("TABLE"):
            parts = line.split()
            cur = {"table": parts[1], "remap": parts[-1], "rows": []}
            blocks.append(cur)
        else:
            cur["rows"].append([int(x, 2) for x in line.split()])
    return blocks


def test_paper_tables_I_II_placement(P):
    """Tables I and II: after the paper's local<->nonlocal
    interchanges (Eqs. onequbitchange, twoqubitchange0-5) rank R, address A
    holds exactly the printed a(x).  L=4, M=2, four virtual shards."""
    blocks = _table_blocks()
    for x in range(16):
        sim = None
        for b in blocks:
            if b["remap"] == "-":
                sim = P.QSim(4, n_ranks=4, transport="virtual")
                sim.init_basis(x)
                sim.sync()
            else:
                pairs = [p.split(":") for p in b["remap"].split(",")]
                sim.remap([int(a) for a, _ in pairs], [int(g) for _, g in pairs])
                sim.sync()
            shards = [t.cpu().numpy().view(np.complex128) for t in sim.shard_tensors()]
            where = [(r, a) for r in range(4) for a in range(4) if abs(shards[r][a]) > 0.5]
            assert len(where) == 1
            r, a = where[0]
            assert b["rows"][a][r] == x, (b["table"], b["remap"], x, where)
            assert abs(sim.get_amplitudes(x, 1)[0] - 1) == 0


def test_remap_roundtrip_exact(P, oracle_mod):
    n = 14
    gates = C.random_brickwork(n, 4, seed=1)
    sim = gpu_run(P, n, 0, gates, ranks=4)
    before = sim.get_amplitudes()
    lay = sim.layout()
    glob = [q for q in range(n) if lay[q] >= n - 2]
    loc = [q for q in range(n) if lay[q] < n - 2][:2]
    sim.remap(loc, glob)
    sim.remap(glob, loc)
    assert np.array_equal(sim.get_amplitudes(), before)


def test_errors_leave_state_untouched(P):
    from paper_quant_ph_0608239_b200 import QsimError
    n = 13
    sim = gpu_run(P, n, 0, C.random_brickwork(n, 2, seed=3))
    before = sim.get_amplitudes()
    bad = [([G.one_q(0, (1, 1, 0, 1))], 4), ([G.cnot(3, 3)], 3), ([G.one_q(13, G.H)], 2),
           ([G.perm_gate((), (0, 1), np.array([0, 0, 1, 2]))], 5)]
    for gates, code in bad:
        with pytest.raises(QsimError) as e:
            sim.run_circuit(gates)
        assert e.value.status == code
    with pytest.raises(QsimError):
        sim.probabilities([0, 0])
    assert np.array_equal(sim.get_amplitudes(), before)
    s2 = P.QSim(5)
    with pytest.raises(QsimError) as e:
        s2.norm()
    assert e.value.name == "QSIM_ERR_STATE"


def test_nccl_transport_single_rank(P, oracle_mod):
    """The NCCL transport end to end on one GPU (world size 1): unique id from
    qsim_get_unique_id broadcast over torch.distributed, ncclCommInitRank,
    then the usual parity.  (Multi-rank NCCL needs several GPUs; its host
    logic is covered by tests/test_dist_gloo.py.)"""
    import socket
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        n = 15
        gates = kitchen_sink(n, seed=5)
        sim = P.QSim.distributed(n)
        sim.init_basis(9)
        sim.run_circuit(gates)
        o = oracle_run(oracle_mod, n, 9, gates)
        assert_parity(sim, o, n)
        assert np.max(np.abs(sim.expectations() - o.expectations())) <= 1e-13
        sim.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seed", range(int(os.environ.get("QSIM_FUZZ_SEEDS", "8"))))
def test_gpu_fuzz(P, oracle_mod, seed):
    """Random circuits of every gate kind (tests/test_plan_fuzz.py) on the
    GPU with the planner options varied, against the oracle."""
    from tests.test_plan_fuzz import random_circuit
    rng = np.random.default_rng(5000 + seed)
    n = int(rng.integers(12, 17))
    ranks = int([1, 1, 2, 4, 8][rng.integers(0, 5)])
    gates = random_circuit(n, 80, 5000 + seed)
    init = int(rng.integers(0, 1 << n))
    sim = P.QSim(n, n_ranks=ranks, transport="local" if ranks == 1 else "virtual")
    sim.set_option("block_fusion", seed % 4 != 0)
    sim.set_option("low_remap", (seed // 2) % 2 == 0)
    sim.set_option("remap_lookahead", [0, 3, 6][seed % 3])
    sim.set_option("jit", seed % 5 != 4)
    if ranks > 1:
        sim.set_option("global_policy", seed % 3)
        sim.set_option("overlap", 2 * (seed % 2))  # the pass + exchange overlap on half the seeds
    sim.init_basis(init)
    sim.run_circuit(gates)
    o = oracle_run(oracle_mod, n, init, gates)
    assert_parity(sim, o, n)
    if n <= 16:  # full-register sampling (one level at k <= 24) vs the oracle's sampler
        qs = list(range(n))
        shots = sim.measure(qs, seed=seed, shots=64)
        ref, tie = o.measure(qs, seed, 64)
        assert np.array_equal(shots[tie == 0], ref[tie == 0])
    # again with the kernels cached: plan cache on (replay) or off (re-plan,
    # streamed launches)
    sim.set_option("plan_cache", seed % 2)
    sim.init_basis(init)
    sim.run_circuit(gates)
    assert_parity(sim, o, n)
    # <Q_i> straight after the circuit (fused into its last pass when that is
    # a JIT pass) vs the oracle
    sim.init_basis(init)
    sim.run_circuit(gates)
    assert np.max(np.abs(sim.expectations() - o.expectations())) <= 1e-13


@pytest.mark.parametrize("seed", range(int(os.environ.get("QSIM_FUZZ_LONG_SEEDS", "2"))))
def test_gpu_fuzz_long(P, oracle_mod, seed):
    """Long random circuits (600-1500 gates of every kind plus a QFT ladder):
    passes that hit the per-pass op and parameter budgets, long phase runs
    with lazy flushes and CTA-uniform terms, 1 or 4 shards."""
    from tests.test_plan_fuzz import random_circuit
    rng = np.random.default_rng(9000 + seed)
    n = int(rng.integers(16, 21))
    ranks = int([1, 4][seed % 2])
    gates = random_circuit(n, int(rng.integers(600, 1500)), 9000 + seed) + C.qft_ladder(list(range(n)), swaps=True)
    init = int(rng.integers(0, 1 << n))
    sim = P.QSim(n, n_ranks=ranks, transport="local" if ranks == 1 else "virtual")
    sim.init_basis(init)
    sim.run_circuit(gates)
    o = oracle_run(oracle_mod, n, init, gates)
    assert_parity(sim, o, n)
    sim.init_basis(init)
    sim.run_circuit(gates)
    assert np.max(np.abs(sim.expectations() - o.expectations())) <= 1e-13


@pytest.mark.parametrize("G,y,X,F", [(247, 194, 14, 8), (899, 2, 12, 10), (35, 3, 10, 6)])
def test_perm_run_repeat_bitwise(P, oracle_mod, G, y, X, F):
    """Race canary for the permutation run (bulk-copy staging on mbarriers,
    composed chain head; compute-sanitizer is unavailable on this pool):
    eight runs give bitwise-identical states equal to the oracle, for
    registers of 6, 8 and 10 qubits (in-tile controls, several instances per
    CTA)."""
    w = C.shor_order_finding(G, y, X, F)
    ref = oracle_run(oracle_mod, w.n, w.init, w.gates).amplitudes()
    first = None
    for _ in range(8):
        sim = gpu_run(P, w.n, w.init, w.gates)
        got = sim.get_amplitudes()
        sim.close()
        assert np.max(np.abs(got - ref)) <= TOL
        if first is None:
            first = got
        assert np.array_equal(got, first)
