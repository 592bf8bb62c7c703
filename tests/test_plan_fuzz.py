"""Seeded random circuits of every gate kind through the host planner
(fusion, two-qubit blocks, permutation runs, low-qubit remap, exchanges,
pairwise, relabels), executed from the plan JSON on numpy and compared with
the oracle (-m "not gpu")."""
import numpy as np
import pytest

from tests.plan_exec import run_plan
from workloads import gates as G


def random_circuit(n, m, seed):
    rng = np.random.default_rng(seed)
    sm = G.SplitMix64(seed)
    out = []
    named = [G.H, G.X, G.Y, G.XBAR, G.YBAR, G.PAULI_X]
    for _ in range(m):
        k = rng.integers(0, 10)
        q = [int(x) for x in rng.permutation(n)[:4]]
        if k == 0:
            out.append(G.one_q(q[0], G.haar_u2(sm)))
        elif k == 1:
            out.append(G.one_q(q[0], named[rng.integers(0, len(named))]))
        elif k == 2:
            out.append(G.cnot(q[0], q[1]))
        elif k == 3:
            out.append(G.cphase(q[0], q[1], float(rng.uniform(-3, 3))))
        elif k == 4:
            out.append(G.ctrl([q[0]], q[1], G.haar_u2(sm)))
        elif k == 5:
            out.append(G.toffoli(q[0], q[1], q[2]))
        elif k == 6:
            out.append(G.one_q(q[0], G.R(float(rng.uniform(-3, 3)))))
        elif k == 7:
            out.append(G.swap(q[0], q[1]))
        elif k == 8:
            t = sorted(q[1:3]) if rng.integers(0, 2) else q[1:4]
            ctl = [q[0]] if rng.integers(0, 2) else []
            for _ in range(int(rng.integers(1, 4))):  # runs of perms of one register
                out.append(G.perm_gate(ctl, t, rng.permutation(1 << len(t)).astype(np.uint32)))
        else:  # a brickwork-like cluster (block fusion)
            a, b = q[0], q[1]
            out += [G.one_q(a, G.haar_u2(sm)), G.one_q(b, G.haar_u2(sm)), G.cnot(a, b),
                    G.one_q(a, G.haar_u2(sm)), G.one_q(b, G.haar_u2(sm))]
    return out


@pytest.fixture(scope="module")
def pkg():
    from paper_quant_ph_0608239_b200 import build
    build.build()
    import paper_quant_ph_0608239_b200 as P
    return P


@pytest.mark.parametrize("seed", range(12))
def test_planner_fuzz(pkg, oracle_mod, seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(12, 16))
    P = int([1, 1, 2, 4, 8][rng.integers(0, 5)])
    gates = random_circuit(n, 60, seed)
    init = int(rng.integers(0, 1 << n))
    policy = [None, "remap", "pairwise"][seed % 3]
    js = pkg.plan_json(n, P, gates, 1, policy, bool(seed % 4), bool((seed // 2) % 2), [0, 3, 6][seed % 3])
    got = run_plan(js, n, init, gates)
    o = oracle_mod.Oracle(n)
    o.init_basis(init)
    o.run(gates)
    assert np.max(np.abs(got - o.amplitudes())) <= 1e-12


def test_exchange_victims_prefer_off_tile_for_overlap():
    """Host planner: the exchange victims avoid the tile of the pass emitted
    just before (when the Belady pool allows), so that pass can run block by
    block under the exchange (runtime overlap).  On the config-5 family at 36
    qubits over 8 ranks every exchange is overlappable; each candidate's
    modelled time is reported."""
    import json
    from paper_quant_ph_0608239_b200 import plan_json
    from workloads import circuits as C
    d = json.loads(plan_json(36, 8, C.random_chain(36, 10, seed=5, sweep=True), overlap=True))
    st = d["plan"]["steps"]
    pairs = [(st[i], st[i + 1]) for i in range(len(st) - 1) if st[i + 1]["type"] == "exchange"]
    assert pairs and all(p["type"] == "pass" for p, _ in pairs)
    for p, x in pairs:
        assert not set(x["lpos"]) & (set(p["tp"]) | set(p["tp_out"]))
    assert len(d["candidates"]) >= 2 and all(c["model_s"] > 0 for c in d["candidates"])
