"""C-ABI library checks and host-side planner logic (-m "not gpu")."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

from tests.plan_exec import run_plan
from workloads import circuits as C
from workloads import gates as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pkg():
    from paper_quant_ph_0608239_b200 import build
    build.build()
    import paper_quant_ph_0608239_b200 as P
    return P


def test_library_exports_every_header_symbol(pkg):
    hdr = open(os.path.join(ROOT, "include", "qsim.h")).read()
    names = set(re.findall(r"\b(qsim_[a-z_0-9]+)\s*\(", hdr))
    assert len(names) >= 20
    lib = ctypes.CDLL(pkg.LIB_PATH)
    for nme in sorted(names):
        assert hasattr(lib, nme), nme
    assert names == set(pkg.EXPORTS)


def test_library_is_sm100a(pkg):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pkg.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings(pkg):
    lib = pkg._native.lib() if hasattr(pkg, "_native") else None
    from paper_quant_ph_0608239_b200 import _native as N
    lib = N.lib()
    for i, nme in enumerate(N.STATUS):
        assert lib.qsim_status_str(i).decode() == nme


def _plan(pkg, n, P, gates, fusion=True, policy=None):
    return pkg.plan_json(n, P, gates, fusion, policy)


def test_validation_codes(pkg):
    from paper_quant_ph_0608239_b200 import QsimError
    cases = [
        ([G.one_q(0, (1, 1, 0, 1))], 4),                          # not unitary
        ([G.ctrl([1], 1, G.PAULI_X)], 3),                          # control == target
        ([G.one_q(9, G.H)], 2),                                    # out of range
        ([G.perm_gate((), (0, 1), np.array([0, 1, 1, 2]))], 5),   # not a bijection
        ([G.perm_gate((0,), (0, 1), np.arange(4))], 3),            # control among targets
        ([G.swap(2, 2)], 3),
    ]
    for gates, code in cases:
        with pytest.raises(QsimError) as e:
            _plan(pkg, 4, 1, gates)
        assert e.value.status == code


def _check_plan(pkg, oracle_mod, n, P, init, gates, fusion=True, policy=None, block_fusion=True):
    js = pkg.plan_json(n, P, gates, fusion, policy, block_fusion)
    got = run_plan(js, n, init, gates)
    o = oracle_mod.Oracle(n)
    o.init_basis(init)
    o.run(gates)
    ref = o.amplitudes()
    assert np.max(np.abs(got - ref)) <= 1e-12
    return json.loads(js)


@pytest.mark.parametrize("P", [1, 2, 4])
def test_plan_random_brickwork(pkg, oracle_mod, P):
    n = 14
    gates = C.random_brickwork(n, 6, seed=11)
    d = _check_plan(pkg, oracle_mod, n, P, 0, gates)
    steps = d["plan"]["steps"]
    npass = sum(s["type"] == "pass" for s in steps)
    assert npass < len(gates) / 4  # fusion actually fuses
    if P > 1:
        assert any(s["type"] == "exchange" for s in steps)


def _pass_ops(d):
    return [op for s in d["plan"]["steps"] if s["type"] == "pass" for op in s["ops"]]


@pytest.mark.parametrize("P", [1, 2, 4])
def test_block_fusion_brickwork(pkg, oracle_mod, P):
    """Two-qubit block fusion (plan.cpp fuse_blocks): the brickwork's
    U2 (x) U2, CNOT, U2 (x) U2 clusters become 4x4 unitaries; executing the
    fused plan gives the oracle's state, and the fused pass program costs
    about half the FP64 work of the unfused one."""
    n = 14
    gates = C.random_brickwork(n, 8, seed=13)
    d = _check_plan(pkg, oracle_mod, n, P, 5, gates)
    d0 = _check_plan(pkg, oracle_mod, n, P, 5, gates, block_fusion=False)
    ops, ops0 = _pass_ops(d), _pass_ops(d0)
    assert not any(op["code"] == 7 for op in ops0)
    n_u4 = sum(op["code"] == 7 for op in ops)
    assert n_u4 >= len(gates) // 8

    def cost(ops):
        c = 0.0
        for op in ops:
            k = op["code"]
            bits = bin(op["cm"]).count("1")
            c += {0: 8.0, 1: 4.0, 3: 4.0, 7: 16.0 * 2 ** bits}.get(k, 0.0) / 2 ** bits
        return c
    assert cost(ops) < 0.6 * cost(ops0)


def test_block_fusion_mixed_predicates(pkg, oracle_mod):
    """Blocks next to controlled gates with out-of-cluster controls, phases on
    the pair, one-qubit runs, Toffolis and relabels: still the oracle's state."""
    n = 13
    rng = G.SplitMix64(77)
    gates = []
    for layer in range(4):
        for q in range(n):
            gates.append(G.one_q(q, G.haar_u2(rng)))
        for q in range(layer % 2, n - 1, 2):
            gates.append(G.cnot(q, q + 1))
        gates += [G.cphase(1, 2, 0.3 + layer), G.ctrl([5], 3, G.haar_u2(rng)), G.one_q(4, G.H),
                  G.one_q(4, G.haar_u2(rng)), G.toffoli(0, 6, 7), G.ctrl([8], 9, G.haar_u2(rng)),
                  G.one_q(8, G.haar_u2(rng)), G.one_q(9, G.haar_u2(rng)), G.swap(10, 11),
                  G.ctrl([2], 1, G.PAULI_X), G.one_q(2, G.R(0.7))]
    for P in (1, 2):
        d = _check_plan(pkg, oracle_mod, n, P, 11, gates)
        assert any(op["code"] == 7 for op in _pass_ops(d))


@pytest.mark.parametrize("P", [1, 2, 4])
def test_plan_perm_run(pkg, oracle_mod, P):
    """Consecutive permutations of one register (Shor's modular
    multiplications, and a mix of 0/1/2 controls) become one permrun step."""
    w = C.shor_order_finding(35, 3, 8, 6)
    d = _check_plan(pkg, oracle_mod, w.n, P, w.init, w.gates)
    runs = [s for s in d["plan"]["steps"] if s["type"] == "permrun"]
    assert len(runs) == 1 and len(runs[0]["gates"]) == 8
    assert not any(s["type"] == "perm" for s in d["plan"]["steps"])
    r = np.random.default_rng(5)
    tg = (2, 7, 4)
    gates = [G.one_q(q, G.H) for q in range(13)]
    for ctl in [(), (0,), (9, 12), (1,), (12,), (3, 5), ()]:
        gates.append(G.perm_gate(ctl, tg, r.permutation(8).astype(np.uint32)))
    gates.append(G.one_q(4, G.H))
    d = _check_plan(pkg, oracle_mod, 13, P, 0, gates)
    assert [len(s["gates"]) for s in d["plan"]["steps"] if s["type"] == "permrun"] == [7]


def test_plan_perm_run_fits_shared_memory(pkg, oracle_mod):
    """A run's R tables of 2^t uint16 and its two staged tiles must fit one
    CTA's shared memory (engine.h perm_run_smem_bytes): 20 perms on a 12-qubit
    register split into runs of 12 and 8 (226 KB >= 128 KB + 4 B + R * 8 KB)."""
    r = np.random.default_rng(9)
    n, tg = 16, tuple(range(12))
    gates = [G.one_q(q, G.H) for q in range(12, 16)]
    for j in range(20):
        gates.append(G.perm_gate((12 + j % 4,), tg, r.permutation(1 << 12).astype(np.uint32)))
    d = _check_plan(pkg, oracle_mod, n, 1, 5, gates)
    assert [len(s["gates"]) for s in d["plan"]["steps"] if s["type"] == "permrun"] == [12, 8]


def test_plan_break_even_blocks(pkg, oracle_mod):
    """Chain circuits: the strict block rule leaves most U2s unfused, so the
    planner also plans with break-even blocks and keeps the cheaper plan
    (fewer passes); the executed plan matches the oracle."""
    gates = C.random_chain(18, 6, seed=11, sweep=False)
    d = _check_plan(pkg, oracle_mod, 18, 1, 0, gates)
    n_pass = sum(s["type"] == "pass" for s in d["plan"]["steps"])
    strict = json.loads(_plan(pkg, 18, 1, gates, fusion=1 | 0x100))  # no gate-level blocks at all
    assert n_pass <= sum(s["type"] == "pass" for s in strict["plan"]["steps"])
    assert sum(op["code"] == 7 for op in _pass_ops(d)) > 0


def test_plan_qft_sharded(pkg, oracle_mod):
    w = C.qft_basis(14, 12345)
    d = _check_plan(pkg, oracle_mod, 14, 4, w.init, w.gates)
    assert sum(s["type"] == "relabel" for s in d["plan"]["steps"]) == 7


def test_plan_shor_sharded(pkg, oracle_mod):
    w = C.shor_order_finding(35, 3, 8, 6)
    _check_plan(pkg, oracle_mod, w.n, 2, w.init, w.gates)
    _check_plan(pkg, oracle_mod, w.n, 1, w.init, w.gates)


def test_plan_chain_three_global(pkg, oracle_mod):
    gates = C.random_chain(15, 2, seed=5, sweep=True)
    _check_plan(pkg, oracle_mod, 15, 8, 0, gates)


@pytest.mark.parametrize("P", [1, 4, 8])
def test_plan_generic_small(pkg, oracle_mod, P):
    n = 8
    rng = G.SplitMix64(4)
    gates = C.random_brickwork(n, 3, seed=2) + [G.toffoli(0, 5, 7), G.ctrl([7, 1], 3, G.haar_u2(rng)),
                                                G.perm_gate((6,), (0, 3, 7), np.array([3, 1, 4, 0, 7, 6, 5, 2])),
                                                G.swap(1, 6), G.cphase(7, 2, 0.4)]
    _check_plan(pkg, oracle_mod, n, P, 37, gates, fusion=True)
    _check_plan(pkg, oracle_mod, n, P, 37, gates, fusion=False)


def test_plan_controls_and_diagonals_on_global(pkg, oracle_mod):
    """Diagonal gates and controls on nonlocal qubits need no exchange
    (the optimisation P:623-628 and P:753-756 describe)."""
    n, P = 14, 4
    gates = [G.one_q(q, G.H) for q in range(12)]  # qubits 12,13 are never targeted -> global
    gates += [G.cphase(13, 2, 0.3), G.ctrl([12], 5, G.haar_u2(G.SplitMix64(1))), G.one_q(13, G.R(0.9)),
              G.toffoli(12, 13, 0)]
    d = _check_plan(pkg, oracle_mod, n, P, 0, gates)
    assert not any(s["type"] == "exchange" for s in d["plan"]["steps"])


def test_jit_kernels_compile_for_sm100a(pkg):
    """The pass-specialised kernels generated for a circuit with every gate
    kind (predicates on register/lane/warp/out-of-tile bits, swaps, phases,
    re-layouts) compile with NVRTC for sm_100a (no GPU needed)."""
    from tests.test_gpu_parity import kitchen_sink
    gates = kitchen_sink(14, seed=3)
    d = json.loads(_plan(pkg, 14, 2, gates, fusion=2))
    assert d["jit"]["ok"], d["jit"]["error"]
    assert d["jit"]["kernels"] >= 1
    # QFT passes: lazy phase flushes, the CTA-uniform phase prologue, Hadamard form
    w = C.qft_basis(20, 777)
    d = json.loads(_plan(pkg, 20, 1, w.gates, fusion=2))
    assert d["jit"]["ok"], d["jit"]["error"]
    # readout variants (<Q_i> fused into the last pass), with deferred flips
    d = json.loads(pkg.plan_json(14, 2, gates, fusion=2, readout=True))
    assert d["jit"]["ok"], d["jit"]["error"]


def test_relayout_barrier_forms(pkg, tmp_path, monkeypatch):
    """Re-layout barriers of the config-2 kernels (jit.cpp QSIM_JIT_BAR = 3):
    CTA barriers, warp barriers, and named barriers over one CTA half whose id
    is a function of the top warp bit only (an id always names the same four
    warps, so barriers of different forms cannot mix); the generated code
    holds at most two barriers per re-layout and all three forms occur."""
    monkeypatch.setenv("QSIM_JIT_DUMP", str(tmp_path))
    w = C.config2_random()
    d = json.loads(_plan(pkg, w.n, 1, w.gates, fusion=2))
    assert d["jit"]["ok"], d["jit"]["error"]
    srcs = [open(tmp_path / f).read() for f in sorted(os.listdir(tmp_path)) if f.endswith(".cu")]
    assert len(srcs) == d["jit"]["kernels"]
    n_cta = n_warp = n_half = n_trans = 0
    for src in srcs:
        named = re.findall(r'bar\.sync %0, (\d+);" :: "r"\(([^)]*\)[^)]*)\)', src)
        for cnt, idx in named:
            assert cnt == "128" and idx.replace(" ", "") == "1+((warp>>2)&1", idx
        n_half += len(named)
        n_warp += src.count("__syncwarp();")
        n_cta += src.count("__syncthreads();")
        n_trans += src.count("const int zzb")
    assert n_half > 0 and n_warp > 0 and n_cta > 0
    assert n_half + n_warp + n_cta <= 2 * n_trans


@pytest.mark.parametrize("policy", ["remap", "pairwise", "auto"])
def test_plan_global_policies(pkg, oracle_mod, policy):
    """Gates on nonlocal qubits by K-pair remap or by pairwise
    combine of partner shards; both give the oracle's state."""
    for P, n in ((2, 13), (4, 14), (8, 15)):
        gates = C.random_chain(n, 2, seed=P, sweep=True)
        d = _check_plan(pkg, oracle_mod, n, P, 3, gates, policy=policy)
        types = {s["type"] for s in d["plan"]["steps"]}
        if policy == "pairwise":
            assert "pairwise" in types
        if policy == "remap":
            assert "pairwise" not in types and "exchange" in types


def test_auto_policy_picks_pairwise_when_remap_would_thrash(pkg, oracle_mod):
    """One gate on the nonlocal qubit while every local qubit keeps being
    used: the auto policy combines partner shards instead of remapping."""
    n, P = 13, 2
    rng = G.SplitMix64(9)
    layer = lambda: [G.one_q(q, G.haar_u2(rng)) for q in range(12)]  # noqa: E731
    gates = layer() + [G.one_q(12, G.haar_u2(rng))] + [G.cnot(12, q) for q in range(12)] + layer() + layer()
    d = _check_plan(pkg, oracle_mod, n, P, 0, gates, policy="auto")
    types = [s["type"] for s in d["plan"]["steps"]]
    assert "pairwise" in types and "exchange" not in types


def _build_c_client(pkg, tmp_path):
    import subprocess
    exe = str(tmp_path / "abi_client")
    libdir = os.path.dirname(pkg.LIB_PATH)
    subprocess.check_call(["gcc", "-std=c11", "-O1", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "c", "abi_client.c"), "-o", exe,
                           "-L", libdir, "-l:libqsim_b200.so", "-Wl,-rpath," + libdir, "-lm"])
    return exe


def test_create_rank_argument_errors(pkg):
    """qsim_create_rank rejects bad rank counts, a missing NCCL id and a
    wrong shard size before touching the device."""
    import ctypes
    from paper_quant_ph_0608239_b200 import _native as N
    lib = N.lib()
    ctx = ctypes.c_void_p()
    assert lib.qsim_create_rank(20, 3, 0, None, None, 0, None, 0, None, ctypes.byref(ctx)) == 1
    assert lib.qsim_create_rank(20, 2, 0, None, None, 0, None, 0, None, ctypes.byref(ctx)) == 1
    assert lib.qsim_create_rank(20, 1, 0, None, ctypes.c_void_p(256), 123, None, 0, None, ctypes.byref(ctx)) == 1
    assert lib.qsim_create_rank(1, 4, 0, b"x" * 128, None, 0, None, 0, None, ctypes.byref(ctx)) == 1


def test_c_client_compiles_and_links(pkg, tmp_path):
    """A plain C program builds against include/qsim.h + libqsim_b200.so."""
    assert os.path.exists(_build_c_client(pkg, tmp_path))


@pytest.mark.gpu
def test_c_client_runs(pkg, tmp_path):
    """The same C program runs the engine with no Python/torch involvement."""
    import subprocess
    r = subprocess.run([_build_c_client(pkg, tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "abi_client ok" in r.stdout and "abi_client two-level ok" in r.stdout


def test_jit_key_implies_same_source(pkg):
    """The pass-kernel cache is keyed by jit_key: two passes that
    differ only in whether two ops share an out-of-tile control (one deduplicated
    (mout, vout) predicate vs two) generate different sources, so they must not
    share a key.  The planner's key check compares the generated source of every
    pass against every earlier pass with the same key, across all plans below."""
    rng = G.SplitMix64(11)
    n = 16
    base = [G.one_q(q, G.haar_u2(rng)) for q in range(4)]
    shared = base + [G.ctrl([15], 0, G.haar_u2(rng)), G.ctrl([15], 1, G.haar_u2(rng))]
    distinct = base + [G.ctrl([15], 0, G.haar_u2(rng)), G.ctrl([14], 1, G.haar_u2(rng))]
    for gates in (shared, distinct, shared[::-1], distinct[::-1]):
        js = json.loads(pkg.plan_json(n, 1, gates, key_check=True))
        assert js["jit"]["ok"], js["jit"]["error"]
    # the wider fuzz: circuits of every gate kind with out-of-tile controls
    for seed in range(6):
        gates = C.random_chain(n, 3, seed=seed, sweep=False)
        r = G.SplitMix64(100 + seed)
        for k in range(12):
            c = [12 + (k + seed) % 4] + ([13 + (k * 3 + seed) % 3] if k % 3 == 0 else [])
            c = sorted(set(c))
            gates.append(G.ctrl(c, k % 12, G.haar_u2(r)))
            gates.append(G.cphase(12 + (k + 2 * seed) % 4, k % 12, 0.1 * k + 0.05))
        js = json.loads(pkg.plan_json(n, 1, gates, key_check=True))
        assert js["jit"]["ok"], js["jit"]["error"]
