"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names the passage it pins.  A plausible bug in the oracle (a
dropped term, a sign, a wrong index or control mask, a transposed operand,
a wrong register bit order in the permutation) fails at least one test.
"""
import math
import os

import numpy as np
import pytest

from tests import pins
from workloads import gates as G
from workloads import circuits as C

RNG = np.random.default_rng(12345)


def rand_state(n, rng=RNG):
    v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return v / np.linalg.norm(v)


def run_oracle(oracle_mod, n, psi0, gates):
    o = oracle_mod.Oracle(n)
    o.set_state(psi0)
    o.run(gates)
    return o.amplitudes()


# ---------------------------------------------------------------- Kronecker
@pytest.mark.parametrize("n", [3, 5])
def test_1q_every_position_vs_kron(oracle_mod, n):
    """Eqs. NUM2-NUM5 generalised to any U: equals U_q (x) I."""
    rng = G.SplitMix64(7)
    for q in range(n):
        for u in (G.H, G.X, G.Y, G.XBAR, G.YBAR, G.R(0.3), G.haar_u2(rng)):
            psi = rand_state(n)
            ref = pins.kron_list({q: pins.mat(u)}, n) @ psi
            got = run_oracle(oracle_mod, n, psi, [G.one_q(q, u)])
            assert np.max(np.abs(got - ref)) <= 1e-13


@pytest.mark.parametrize("n", [3, 5])
def test_controlled_every_position_vs_kron(oracle_mod, n):
    """CNOT/CP/controlled-V/Toffoli = I + P1_C (x) (U - I)_t."""
    rng = G.SplitMix64(8)
    for t in range(n):
        for c in range(n):
            if c == t:
                continue
            for u in (G.PAULI_X, G.R(1.1), G.V(0.7), G.haar_u2(rng)):
                psi = rand_state(n)
                ref = pins.dense_controlled(n, [c], t, u) @ psi
                got = run_oracle(oracle_mod, n, psi, [G.ctrl([c], t, u)])
                assert np.max(np.abs(got - ref)) <= 1e-13
        others = [q for q in range(n) if q != t]
        for i in range(len(others)):
            for j in range(i + 1, len(others)):
                cs = [others[i], others[j]]
                u = G.haar_u2(rng)
                psi = rand_state(n)
                ref = pins.dense_controlled(n, cs, t, u) @ psi
                got = run_oracle(oracle_mod, n, psi, [G.ctrl(cs, t, u)])
                assert np.max(np.abs(got - ref)) <= 1e-13


def test_perm_vs_tensor(oracle_mod):
    """Controlled register permutation vs a tensor contraction
    with the permutation matrix; non-contiguous, unsorted targets."""
    n = 6
    rng = np.random.default_rng(3)
    cases = [((), (0, 1, 2)), ((5,), (1, 3)), ((0, 4), (5, 2, 1)), ((2,), (4, 0, 5, 1))]
    for controls, targets in cases:
        perm = rng.permutation(1 << len(targets)).astype(np.uint32)
        psi = rand_state(n)
        ref = pins.tensor_apply_perm(psi, n, list(controls), list(targets), perm)
        got = run_oracle(oracle_mod, n, psi, [G.perm_gate(controls, targets, perm)])
        assert np.max(np.abs(got - ref)) == 0.0


def test_perm_rejects_non_bijection(oracle_mod):
    o = oracle_mod.Oracle(3)
    with pytest.raises(ValueError):
        o.apply(G.perm_gate((), (0, 1), np.array([0, 1, 1, 3], dtype=np.uint32)))


def test_swap_vs_tensor(oracle_mod):
    n = 5
    for a in range(n):
        for b in range(n):
            if a != b:
                psi = rand_state(n)
                ref = pins.tensor_swap(psi, n, a, b)
                got = run_oracle(oracle_mod, n, psi, [G.swap(a, b)])
                assert np.max(np.abs(got - ref)) == 0.0


# ------------------------------------------------------ paper worked examples
def test_paper_examples(oracle_mod):
    a = rand_state(2)
    s = 1 / math.sqrt(2)
    # Eq. CNOT2: CNOT_10 (a0,a1,a2,a3) -> (a0,a3,a2,a1)
    got = run_oracle(oracle_mod, 2, a, [G.cnot(0, 1)])
    assert np.allclose(got, [a[0], a[3], a[2], a[1]], atol=0, rtol=0)
    # Eq. COMM5: R_10(phi) multiplies a3 only
    phi = 0.77
    got = run_oracle(oracle_mod, 2, a, [G.cphase(0, 1, phi)])
    e = complex(math.cos(phi), math.sin(phi))
    assert np.max(np.abs(got - np.array([a[0], a[1], a[2], e * a[3]]))) < 1e-15
    # Eq. COMM4: controlled V_10(phi)
    got = run_oracle(oracle_mod, 2, a, [G.ctrl([0], 1, G.V(phi))])
    ref = [a[0], ((1 + e) * a[1] + (1 - e) * a[3]) / 2, a[2], ((1 - e) * a[1] + (1 + e) * a[3]) / 2]
    assert np.max(np.abs(got - np.array(ref))) < 1e-15
    # V(pi) is the CNOT
    got_v = run_oracle(oracle_mod, 2, a, [G.ctrl([0], 1, G.V(math.pi))])
    assert np.max(np.abs(got_v - np.array([a[0], a[3], a[2], a[1]]))) < 1e-15
    # Eq. Toffoli: T_210 swaps a3 <-> a7
    b = rand_state(3)
    got = run_oracle(oracle_mod, 3, b, [G.toffoli(0, 1, 2)])
    ref = b.copy()
    ref[3], ref[7] = b[7], b[3]
    assert np.array_equal(got, ref)
    # Eqs. Hadamard/Xoperation/Yoperation on (1,0) and general (a0,a1)
    c = rand_state(1)
    assert np.max(np.abs(run_oracle(oracle_mod, 1, c, [G.one_q(0, G.H)]) -
                         s * np.array([c[0] + c[1], c[0] - c[1]]))) < 1e-15
    assert np.max(np.abs(run_oracle(oracle_mod, 1, c, [G.one_q(0, G.X)]) -
                         s * np.array([c[0] + 1j * c[1], c[1] + 1j * c[0]]))) < 1e-15
    assert np.max(np.abs(run_oracle(oracle_mod, 1, c, [G.one_q(0, G.Y)]) -
                         s * np.array([c[0] + c[1], c[1] - c[0]]))) < 1e-15
    # Eq. singlephase R(pi) on qubit 1 of 2 negates a2, a3
    got = run_oracle(oracle_mod, 2, a, [G.one_q(1, G.R(math.pi))])
    assert np.max(np.abs(got - np.array([a[0], a[1], -a[2], -a[3]]))) < 1e-15
    # doubled gates load |1>: XX|0>=i|1>, YY|0>=-|1>, and the bars
    zero = np.array([1, 0], dtype=complex)
    for u, ph in ((G.X, 1j), (G.Y, -1), (G.XBAR, -1j), (G.YBAR, 1)):
        got = run_oracle(oracle_mod, 1, zero, [G.one_q(0, u), G.one_q(0, u)])
        assert np.max(np.abs(got - np.array([0, ph]))) < 1e-15


def test_init_basis_and_layout(oracle_mod):
    o = oracle_mod.Oracle(4)
    o.init_basis(6)
    amps = o.amplitudes()
    assert amps[6] == 1 and np.count_nonzero(amps) == 1


# ------------------------------------------------------------ whole programs
def test_h_on_all_uniform(oracle_mod):
    """H on every qubit: uniform 2^{-n/2}, every <Q_i> = 1/2."""
    n = 12
    o = oracle_mod.Oracle(n)
    o.init_basis(0)
    o.run([G.one_q(q, G.H) for q in range(n)])
    amps = o.amplitudes()
    assert np.max(np.abs(amps - 2 ** (-n / 2))) <= 1e-15 * 2 ** (-n / 2) * 4
    assert np.max(np.abs(o.expectations() - 0.5)) < 1e-14


@pytest.mark.parametrize("n", [1, 2, 5, 9])
def test_qft_closed_form(oracle_mod, n):
    """QFT ladder + swaps on |x0> equals the closed form (V5)."""
    rng = np.random.default_rng(n)
    for x0 in {0, (1 << n) - 1, int(rng.integers(0, 1 << n))}:
        w = C.qft_basis(n, x0)
        o = oracle_mod.Oracle(n)
        o.init_basis(w.init)
        o.run(w.gates)
        assert np.max(np.abs(o.amplitudes() - pins.qft_closed_form(n, x0))) <= 1e-13


def test_qft_inverse_identity(oracle_mod):
    n = 7
    psi = rand_state(n)
    q = list(range(n))
    got = run_oracle(oracle_mod, n, psi, C.qft_ladder(q, True) + C.inverse_qft_ladder(q, True))
    assert np.max(np.abs(got - psi)) < 1e-13


def test_adder_all_inputs_m4(oracle_mod):
    """QFT adder: |a,b> -> |a,(a+b) mod 2^m> with probability 1."""
    m = 4
    ra, rb = list(range(m)), list(range(m, 2 * m))
    gates = C.qft_adder([ra, rb])
    assert len(gates) == 3 * m * (m + 1) // 2  # N_O decomposition, V4
    for a in range(1 << m):
        for b in range(1 << m):
            o = oracle_mod.Oracle(2 * m)
            o.init_basis(a + (b << m))
            o.run(gates)
            p = np.abs(o.amplitudes()) ** 2
            assert p[a + (((a + b) % (1 << m)) << m)] >= 1 - 1e-12


def test_adder_config1(oracle_mod):
    w = C.config1_adder()
    assert len(w.gates) == 63
    o = oracle_mod.Oracle(w.n)
    o.init_basis(w.init)
    o.run(w.gates)
    p = np.abs(o.amplitudes()) ** 2
    assert p[w.meta["expect_index"]] >= 1 - 1e-12
    assert abs(o.norm() - 1) <= 1e-12


@pytest.mark.slow
def test_adder_paper_fig2(oracle_mod):
    """Fig. adder caption: 1365 + 682 on two 11-qubit registers
    gives 2047 (mod 2^11) with probability 1; 22 qubits."""
    m = 11
    ra, rb = list(range(m)), list(range(m, 2 * m))
    gates = C.qft_adder([ra, rb])
    assert len(gates) == 66 + 66 + 66  # QFT(11)=11+55, add 66, inverse 66 (V4)
    o = oracle_mod.Oracle(2 * m)
    o.init_basis(1365 + (682 << m))
    o.run(gates)
    pa = o.probabilities(ra)
    pb = o.probabilities(rb)
    assert pa[1365] >= 1 - 1e-12 and pb[2047] >= 1 - 1e-12


def test_three_register_adder_small(oracle_mod):
    """n-register adders of Tables IV-VIII (e.g. 3-11QBA): sum mod 2^m."""
    m = 3
    regs = [list(range(0, 3)), list(range(3, 6)), list(range(6, 9))]
    gates = C.qft_adder(regs)
    for (a, b, c) in [(1, 2, 3), (7, 7, 7), (5, 0, 6)]:
        o = oracle_mod.Oracle(9)
        o.init_basis(a + (b << 3) + (c << 6))
        o.run(gates)
        assert o.probabilities(regs[2])[(a + b + c) % 8] >= 1 - 1e-12


# ------------------------------------------------------------------- Shor
def test_table3_periods():
    """V1: the printed periods r of Table III."""
    rows = [l.split("|")[0].split() for l in open(os.path.join(os.path.dirname(__file__), "golden", "table3.txt"))
            if not l.startswith("#")]
    for L, X, Gn, y, r in rows:
        assert C.multiplicative_order(int(y), int(Gn)) == int(r)
        assert math.gcd(int(y), int(Gn)) == 1


def test_shor_closed_form_vs_fft():
    """Corrected Eq. Shor5 (reading 1) vs brute-force FFT (V2); sum p_k = 1;
    p_64(r=4, X=8) = 1/4."""
    for r, X in ((3, 8), (18, 10), (5, 9), (4, 8), (7, 6)):
        p = pins.shor_pk(r, X)
        assert np.max(np.abs(p - pins.shor_pk_bruteforce(r, X))) < 1e-13
        assert abs(p.sum() - 1) < 1e-12
    assert abs(pins.shor_pk(4, 8)[64] - 0.25) < 1e-15


def test_table3_closed_form():
    """Eq. Shor7 with corrected Eq. Shor5 reproduces every printed Table III
    column to 3 decimals (V3)."""
    for line in open(os.path.join(os.path.dirname(__file__), "golden", "table3.txt")):
        if line.startswith("#"):
            continue
        head, vals = line.split("|")
        L, X, Gn, y, r = map(int, head.split())
        printed = np.array([float(v) for v in vals.split()])
        q = pins.expectations_from_pk(pins.shor_pk(r, X), X)
        assert np.max(np.abs(q - printed)) <= 5e-4 + 1e-9, (L, Gn)


@pytest.mark.parametrize("N,x,t,f", [(15, 7, 8, 4), (21, 2, 9, 5), (21, 5, 8, 5), (35, 3, 10, 6)])
def test_shor_oracle_vs_closed_form(oracle_mod, N, x, t, f):
    """Oracle Shor run (controlled mod-mult permutations + inverse QFT with
    swaps) reproduces the closed-form x-register distribution (V6)."""
    w = C.shor_order_finding(N, x, t, f)
    o = oracle_mod.Oracle(w.n)
    o.init_basis(w.init)
    o.run(w.gates)
    p = o.probabilities(list(range(t)))
    assert np.max(np.abs(p - pins.shor_pk(w.meta["r"], t))) < 1e-12


@pytest.mark.slow
def test_shor_table3_L24_oracle(oracle_mod):
    """Table III L=24 column: G=247, y=194, X=16, F=8; the oracle's
    <Q_i> match the printed values to 3 decimals and the closed form to 1e-10."""
    w = C.shor_order_finding(247, 194, 16, 8)
    assert w.n == 24 and w.meta["r"] == 18
    o = oracle_mod.Oracle(24)
    o.init_basis(w.init)
    o.run(w.gates)
    q = o.expectations()[:16]
    line = [l for l in open(os.path.join(os.path.dirname(__file__), "golden", "table3.txt"))
            if l.startswith("24 ")][0]
    printed = np.array([float(v) for v in line.split("|")[1].split()])
    assert np.max(np.abs(q - printed)) <= 5e-4 + 1e-9
    closed = pins.expectations_from_pk(pins.shor_pk(18, 16), 16)
    assert np.max(np.abs(q - closed)) <= 1e-10


# ------------------------------------------------------ norms, sums, samples
def test_norm_and_echo(oracle_mod):
    n = 10
    gates = C.random_brickwork(n, 6, seed=9)
    o = oracle_mod.Oracle(n)
    o.init_basis(0)
    o.run(gates)
    assert abs(o.norm() - 1) <= 1e-12
    o.run(C.inverse(gates))
    amps = o.amplitudes()
    assert abs(amps[0] - 1) < 1e-12 and np.max(np.abs(amps[1:])) < 1e-12


def test_probabilities_vs_fsum(oracle_mod):
    n = 11
    psi = rand_state(n)
    o = oracle_mod.Oracle(n)
    o.set_state(psi)
    for qs in ([], [0], [10], [3, 7], [9, 0, 4], list(range(7))):
        got = o.probabilities(qs)
        ref = pins.fsum_probs(psi, n, qs)
        assert np.max(np.abs(got - ref)) <= 4e-16
    ex = o.expectations()
    for q in range(n):
        assert abs(ex[q] - pins.fsum_probs(psi, n, [q])[1]) <= 4e-16


def test_sampler_rule(oracle_mod):
    """Reading 14: u_s = (sm64(seed+(s+1)G) >> 11) 2^-53 C_tot, outcome =
    min{beta: C(beta) > u_s}; checked against thresholds computed here."""
    from oracle.oracle import sample_from
    p = np.array([0.25, 0.25, 0.5, 0.0])
    seed, shots = 99, 2000
    out, tie = sample_from(p, 2, seed, shots)
    for s in range(shots):
        u = (G.sm64((seed + (s + 1) * G.GOLDEN) & G.M64) >> 11) * 2.0 ** -53
        exp = 0 if u < 0.25 else (1 if u < 0.5 else 2)
        assert out[s] == exp
    assert np.all(out != 3)
    # point mass: every shot is the basis state, no ties
    p = np.zeros(16)
    p[11] = 1.0
    out, tie = sample_from(p, 4, 5, 100)
    assert np.all(out == 11) and not tie.any()
    # uniform: frequencies close to 1/8
    out, _ = sample_from(np.full(8, 1 / 8), 3, 1, 80000)
    freq = np.bincount(out.astype(np.int64), minlength=8) / 80000
    assert np.max(np.abs(freq - 1 / 8)) < 0.01


def test_paper_adder_op_counts():
    """N_O of the paper's adder benchmarks (Tables IV-VIII)
    decomposes as 2 x (one-bits) + QFT + adds + inverse QFT (V4)."""
    for name, (m, values, n_o) in C.PAPER_ADDERS.items():
        w = C.paper_adder(name)
        assert len(w.gates) == n_o, name
        assert w.n == m * len(values)
    assert C.paper_adder("3-11QBA").meta["expect_sum"] == 2047     # P:1293 caption values
    assert C.paper_adder("2-17QBA").meta["expect_sum"] == 131071


def test_paper_adder_small_instance(oracle_mod):
    """Same construction (doubled loading gates + QFT adder) on 3 x 4-qubit
    registers: the sum register holds the sum mod 16 with probability 1."""
    regs = [list(range(0, 4)), list(range(4, 8)), list(range(8, 12))]
    vals = (5, 9, 14)
    gates = C.load_register_bits(regs, vals) + C.qft_adder(regs)
    o = oracle_mod.Oracle(12)
    o.init_basis(0)
    o.run(gates)
    assert o.probabilities(regs[2])[sum(vals) % 16] >= 1 - 1e-12
    assert o.probabilities(regs[0])[5] >= 1 - 1e-12
