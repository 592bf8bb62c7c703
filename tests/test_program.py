"""The Appendix-A input format: parser, serialiser,
N_O, and execution on the GPU against the oracle."""
import os

import numpy as np
import pytest

from paper_quant_ph_0608239_b200.program import ProgramError, parse_program, run_program, serialize_program

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "appendix_a.qc")


def test_appendix_a_listing():
    p = parse_program(open(GOLDEN).read())
    assert (p.n, p.init, p.ranks) == (32, 0, 32)
    assert p.gate_count() == 32                     # N_O = L for H on all (Table IV)
    gates = p.gates()
    assert [g.target for g in gates] == list(range(32))
    sw = p.swaps()
    assert len(sw) == 6
    assert sw[0] == [(0, 27)] and sw[4] == [(30, 31)]
    assert sw[5] == [(31, 0), (1, 27), (2, 28), (3, 29), (4, 30)]
    meas = [i.args for i in p.body if i.op == "DO MEASUREMENT"]
    assert meas == [tuple(range(1, 27)) + (31,), (0, 27, 28, 29, 30)]


def test_round_trip():
    p = parse_program(open(GOLDEN).read())
    q = parse_program(serialize_program(p))
    assert (q.n, q.init, q.ranks) == (p.n, p.init, p.ranks)
    assert [(i.op, i.args) for i in q.body] == [(i.op, i.args) for i in p.body]
    assert serialize_program(parse_program("QUBITS 4\n")) == "QUBITS 4\nINITIAL STATE 0\n"


def test_gate_mnemonics():
    p = parse_program("qubits 3\nX 0\nYDAG 1\nR 2 2\nCNOT 0 1\nCPHASE -3 1 2\nCV 1 2 0\nTOFFOLI 0 1 2\nQSWAP 0 2\n")
    g = p.gates()
    assert [x.kind for x in g] == [0, 0, 0, 1, 1, 1, 1, 3]
    assert np.allclose(g[2].u, (1, 0, 0, 1j))                         # phi = 2 pi / 2^2
    assert np.allclose(g[4].u[3], np.exp(-2j * np.pi / 8))           # signed k: inverse phase
    assert g[6].controls == (0, 1) and g[6].target == 2
    assert np.allclose(g[5].u, (0, 1, 1, 0))                          # V(pi) = NOT


@pytest.mark.parametrize("text,frag", [
    ("H 0\n", "begin with QUBITS"),
    ("QUBITS 2\nH 2\n", "out of range"),
    ("QUBITS 2\nCNOT 1 1\n", "repeated"),
    ("QUBITS 2\nFOO 1\n", "unknown keyword"),
    ("QUBITS 4\nSWAP 2 0 1 2\n", "2K qubits"),
    ("QUBITS 2\nH x\n", "malformed integer"),
    ("QUBITS 2\nDO MEASUREMENT 0\n", "inside a measurement block"),
    ("QUBITS 2\nBEGIN MEASUREMENT\n", "unterminated"),
    ("QUBITS 2\nINITIAL STATE 4\n", "< 2^L"),
])
def test_errors_name_the_line(text, frag):
    with pytest.raises(ProgramError) as e:
        parse_program(text)
    assert frag in str(e.value)


@pytest.mark.gpu
@pytest.mark.parametrize("ranks", [1, 8])
def test_run_appendix_a_family_gpu(oracle_mod, ranks):
    """The Appendix-A program shrunk to 16 qubits (same structure: H on all with
    SWAP commands, measurement block with a 5-pair SWAP) on 1 shard and on 8
    virtual shards (SWAP commands become remaps): <Q_i> = 1/2, and a mixed
    program matches the oracle."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_quant_ph_0608239_b200 import QSim
    n = 16
    text = "QUBITS 16\nINITIAL STATE 0\nMPIPROCESSES 8\n" + "".join(f"H {q}\n" for q in range(13))
    for q in range(13, 16):
        text += f"SWAP 1 {q - 1 if q > 13 else 0} {q}\nH {q}\n"
    text += "BEGIN MEASUREMENT\nDO MEASUREMENT " + " ".join(map(str, range(1, 13))) + " 15\n"
    text += "SWAP 3 15 1 2 0 13 14\nDO MEASUREMENT 0 13 14\nEND MEASUREMENT\n"
    p = parse_program(text)
    sim = QSim(n, n_ranks=ranks, transport="local" if ranks == 1 else "virtual")
    res = run_program(p, sim)
    assert res.n_o == 16
    vals = [v for _, vs in res.measurements for v in vs]
    assert len(vals) == 16 and np.max(np.abs(np.array(vals) - 0.5)) < 1e-12
    if ranks > 1:
        assert res.remaps >= 1
    mixed = parse_program("QUBITS 16\nINITIAL STATE 37\n" + "".join(
        f"H {q}\nX {(q + 3) % 16}\nCNOT {q} {(q + 1) % 16}\nCPHASE {q % 5 + 1} {(q + 7) % 16} {q}\n"
        f"CV 2 {(q + 2) % 16} {(q + 9) % 16}\nTOFFOLI {q} {(q + 4) % 16} {(q + 11) % 16}\nYDAG {q}\nR -3 {q}\n"
        + (f"SWAP 1 {q} {15 - q}\n" if q < 8 else "") for q in range(16)) + "QSWAP 1 14\n")
    sim = QSim(n, n_ranks=ranks, transport="local" if ranks == 1 else "virtual")
    run_program(mixed, sim)
    o = oracle_mod.Oracle(n)
    o.init_basis(37)
    o.run(mixed.gates())
    assert np.max(np.abs(sim.get_amplitudes() - o.amplitudes())) <= 1e-11
