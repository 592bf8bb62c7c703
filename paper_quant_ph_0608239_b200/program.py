"""The simulator's text input format (Appendix A; §IV).

A program is a list of commands, one per line; a command is a keyword followed
by values.  Lines starting with "!" or "#" are comments, and so is anything
after a "!" (the listing's trailing comments).  Keywords are case-insensitive.

    QUBITS L                      size of the quantum computer
    INITIAL STATE x               basis state |x> (0 in the paper's listing)
    MPIPROCESSES P                number of processes (advisory; "not used by the OpenMP code")
    H q                           Hadamard (Eq. Hadamard)
    SWAP K a1..aK b1..bK          the qubit INTERCHANGE of Section III.B (not a quantum swap,
                                  P:1264-1265): pairs (a_i, b_i)
    BEGIN MEASUREMENT / DO MEASUREMENT q... / END MEASUREMENT

Appendix A shows only H, SWAP and measurement.  The other mnemonics (the gate
set of §II, Fig. 1; SPEC circuit-module reading) are

    X q, Y q, XDAG q, YDAG q      the pi/2 rotations of Eqs. Xoperation/Yoperation and inverses
    R k q                         phase shift diag(1, e^{i phi}), phi = 2 pi / 2^k (k signed)
    CNOT c t                      Eq. CNOT2
    CPHASE k c t                  controlled phase shift R(phi) on t, control c (Eq. COMM5)
    CV k c t                      controlled-V(phi) (Eq. COMM4)
    TOFFOLI c1 c2 t               Eq. Toffoli

plus `QSWAP a b`, the quantum swap gate (a relabel in this engine).  The
paper's "conditional operation" of Shor's algorithm has no text form; use the
C-ABI (`qsim_apply_perm`) for it.

Execution (`run_program`): gates are queued on a QSim; a SWAP command is an
explicit remap (`qsim_remap`) when it pairs a local with a nonlocal qubit of
the engine's current layout, else a no-op (the engine places qubits itself:
the command only moves data, the state it represents is unchanged); DO
MEASUREMENT returns the non-collapsing <Q_i> of the listed qubits (Eq. Shor7,
P:1061-1069).  N_O counts gate commands only (Table IV caption: "not
including swap commands"; all-H at L=27 gives N_O = 27).

Parsing and serialising are host-side marshalling; every gate runs in the
engine's kernels.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

# gate kinds of the C-ABI (include/qsim.h qsim_gate_kind)
_G_1Q, _G_CTRL, _G_SWAP = 0, 1, 3

_S2 = 1.0 / math.sqrt(2.0)
# 2x2 matrices, row-major (a0', a1') = U (a0, a1); P:231-259 as printed (reading R6)
_NAMED = {
    "H": (_S2, _S2, _S2, -_S2),
    "X": (_S2, 1j * _S2, 1j * _S2, _S2),
    "Y": (_S2, _S2, -_S2, _S2),
    "XDAG": (_S2, -1j * _S2, -1j * _S2, _S2),
    "YDAG": (_S2, -_S2, _S2, _S2),
}
_NOT = (0, 1, 1, 0)


def _phase(k: int) -> complex:
    phi = 2.0 * math.pi / (2.0 ** k) if k >= 0 else -2.0 * math.pi / (2.0 ** (-k))
    return complex(math.cos(phi), math.sin(phi))


def _v(k: int):
    e = _phase(k)
    return ((1 + e) / 2, (1 - e) / 2, (1 - e) / 2, (1 + e) / 2)


@dataclass
class GateRecord:
    """Duck-type of the gate records `pack_gates` accepts."""
    kind: int
    target: int = -1
    controls: Tuple[int, ...] = ()
    targets: Tuple[int, ...] = ()
    u: Tuple[complex, ...] = (1, 0, 0, 1)
    perm: object = None


@dataclass
class Instruction:
    op: str                       # keyword (upper case)
    args: Tuple[int, ...] = ()    # integers as written
    line: int = 0


@dataclass
class Program:
    n: int
    init: int = 0
    ranks: Optional[int] = None
    body: List[Instruction] = field(default_factory=list)

    def gate_count(self) -> int:
        return sum(1 for i in self.body if i.op in _GATE_ARITY)

    def swaps(self) -> List[List[Tuple[int, int]]]:
        return [_pairs(i) for i in self.body if i.op == "SWAP"]

    def gates(self) -> List[GateRecord]:
        """The gate commands in order (SWAP commands and measurements left out)."""
        return [g for i in self.body if i.op in _GATE_ARITY for g in [_gate(i)]]


# keyword -> number of integer arguments
_GATE_ARITY = {"H": 1, "X": 1, "Y": 1, "XDAG": 1, "YDAG": 1, "R": 2, "CNOT": 2, "CPHASE": 3, "CV": 3,
               "TOFFOLI": 3, "QSWAP": 2}


class ProgramError(ValueError):
    pass


def _pairs(ins: Instruction) -> List[Tuple[int, int]]:
    k = ins.args[0]
    return list(zip(ins.args[1:1 + k], ins.args[1 + k:1 + 2 * k]))


def _gate(ins: Instruction) -> GateRecord:
    a = ins.args
    op = ins.op
    if op in _NAMED:
        return GateRecord(_G_1Q, target=a[0], u=_NAMED[op])
    if op == "R":
        return GateRecord(_G_1Q, target=a[1], u=(1, 0, 0, _phase(a[0])))
    if op == "CNOT":
        return GateRecord(_G_CTRL, target=a[1], controls=(a[0],), u=_NOT)
    if op == "CPHASE":
        return GateRecord(_G_CTRL, target=a[2], controls=(a[1],), u=(1, 0, 0, _phase(a[0])))
    if op == "CV":
        return GateRecord(_G_CTRL, target=a[2], controls=(a[1],), u=_v(a[0]))
    if op == "TOFFOLI":
        return GateRecord(_G_CTRL, target=a[2], controls=(a[0], a[1]), u=_NOT)
    if op == "QSWAP":
        return GateRecord(_G_SWAP, targets=(a[0], a[1]))
    raise ProgramError(f"line {ins.line}: not a gate: {op}")


def parse_program(text: str) -> Program:
    """Appendix-A text -> Program.  Errors name the line."""
    prog: Optional[Program] = None
    in_meas = False
    for ln, raw in enumerate(text.splitlines(), 1):
        line = raw.split("!", 1)[0].strip()
        if not line or line.startswith("#"):
            continue
        w = line.split()
        key = w[0].upper()
        rest = w[1:]
        if key == "INITIAL" and rest and rest[0].upper() == "STATE":
            key, rest = "INITIAL STATE", rest[1:]
        elif key in ("BEGIN", "DO", "END") and rest and rest[0].upper() == "MEASUREMENT":
            key, rest = key + " MEASUREMENT", rest[1:]
        try:
            vals = tuple(int(x) for x in rest)
        except ValueError:
            raise ProgramError(f"line {ln}: malformed integer in {raw.strip()!r}") from None
        if key == "QUBITS":
            if prog is not None or len(vals) != 1 or not 1 <= vals[0] <= 62:
                raise ProgramError(f"line {ln}: QUBITS must come first, once, with 1 <= L <= 62")
            prog = Program(n=vals[0])
            continue
        if prog is None:
            raise ProgramError(f"line {ln}: program must begin with QUBITS")
        n = prog.n

        def check_qubits(qs):
            if any(q < 0 or q >= n for q in qs):
                raise ProgramError(f"line {ln}: qubit out of range 0..{n - 1}")
            if len(set(qs)) != len(qs):
                raise ProgramError(f"line {ln}: repeated qubit")

        if key == "INITIAL STATE":
            if len(vals) != 1 or not 0 <= vals[0] < (1 << n):
                raise ProgramError(f"line {ln}: INITIAL STATE needs one index < 2^L")
            prog.init = vals[0]
        elif key == "MPIPROCESSES":
            if len(vals) != 1 or vals[0] < 1:
                raise ProgramError(f"line {ln}: MPIPROCESSES needs one positive integer")
            prog.ranks = vals[0]
        elif key == "SWAP":
            if not vals or vals[0] < 1 or len(vals) != 1 + 2 * vals[0]:
                raise ProgramError(f"line {ln}: SWAP K needs 2K qubits")
            check_qubits(list(vals[1:]))
            prog.body.append(Instruction("SWAP", vals, ln))
        elif key == "BEGIN MEASUREMENT":
            if in_meas or vals:
                raise ProgramError(f"line {ln}: nested or malformed BEGIN MEASUREMENT")
            in_meas = True
            prog.body.append(Instruction(key, (), ln))
        elif key == "END MEASUREMENT":
            if not in_meas or vals:
                raise ProgramError(f"line {ln}: END MEASUREMENT without BEGIN")
            in_meas = False
            prog.body.append(Instruction(key, (), ln))
        elif key == "DO MEASUREMENT":
            if not in_meas or not vals:
                raise ProgramError(f"line {ln}: DO MEASUREMENT needs qubits inside a measurement block")
            check_qubits(list(vals))
            prog.body.append(Instruction(key, vals, ln))
        elif key in _GATE_ARITY:
            if len(vals) != _GATE_ARITY[key]:
                raise ProgramError(f"line {ln}: {key} takes {_GATE_ARITY[key]} integers")
            qs = list(vals[1:]) if key in ("R", "CPHASE", "CV") else list(vals)
            check_qubits(qs)
            prog.body.append(Instruction(key, vals, ln))
        else:
            raise ProgramError(f"line {ln}: unknown keyword {w[0]!r}")
    if prog is None:
        raise ProgramError("empty program (no QUBITS)")
    if in_meas:
        raise ProgramError("unterminated measurement block")
    return prog


def serialize_program(prog: Program) -> str:
    out = [f"QUBITS {prog.n}", f"INITIAL STATE {prog.init}"]
    if prog.ranks is not None:
        out.append(f"MPIPROCESSES {prog.ranks}")
    for i in prog.body:
        out.append(" ".join([i.op] + [str(x) for x in i.args]))
    return "\n".join(out) + "\n"


@dataclass
class RunResult:
    measurements: List[Tuple[Tuple[int, ...], List[float]]]  # (qubits, <Q_i>) per DO MEASUREMENT
    n_o: int                                                  # gate commands executed
    remaps: int                                               # SWAP commands executed as exchanges


def run_program(prog: Program, sim) -> RunResult:
    """Execute on a QSim of prog.n qubits (any number of shards)."""
    from .qsim import pack_gates
    if sim.n != prog.n:
        raise ProgramError(f"simulator has {sim.n} qubits, program {prog.n}")
    sim.init_basis(prog.init)
    meas, pending, remaps = [], [], 0
    M = sim.n - (sim.n_ranks - 1).bit_length()

    def flush():
        if pending:
            sim.run_circuit(pending, packed=pack_gates(pending))
            pending.clear()

    for ins in prog.body:
        if ins.op in _GATE_ARITY:
            pending.append(_gate(ins))
        elif ins.op == "SWAP":
            flush()
            if sim.n_ranks > 1:
                lay = sim.layout()
                loc, glo = [], []
                for a, b in _pairs(ins):
                    if lay[a] < M <= lay[b]:
                        loc.append(a), glo.append(b)
                    elif lay[b] < M <= lay[a]:
                        loc.append(b), glo.append(a)
                if loc:
                    sim.remap(loc, glo)
                    remaps += 1
        elif ins.op == "DO MEASUREMENT":
            flush()
            ex = sim.expectations()
            meas.append((ins.args, [float(ex[q]) for q in ins.args]))
    flush()
    return RunResult(meas, prog.gate_count(), remaps)


def main(argv=None) -> int:
    """python -m paper_quant_ph_0608239_b200.program FILE [--shards P]: run an
    Appendix-A program on this GPU and print one JSON line per DO MEASUREMENT."""
    import argparse
    import json
    import time

    ap = argparse.ArgumentParser(description=main.__doc__)
    ap.add_argument("file")
    ap.add_argument("--shards", type=int, default=1, help="virtual shards on this GPU (power of 2)")
    a = ap.parse_args(argv)
    from .qsim import QSim
    prog = parse_program(open(a.file).read())
    sim = QSim(prog.n, n_ranks=a.shards, transport="local" if a.shards == 1 else "virtual")
    t0 = time.perf_counter()
    res = run_program(prog, sim)
    sim.sync()
    dt = time.perf_counter() - t0
    for qs, vals in res.measurements:
        print(json.dumps({"qubits": list(qs), "Q": vals}))
    print(json.dumps({"L": prog.n, "N_O": res.n_o, "swap_commands_executed": res.remaps, "t_E_s": dt}))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
