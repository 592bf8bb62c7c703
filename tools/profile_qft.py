"""One QFT (config-4 structure) at n qubits through the engine: the command
profiled by ncu for the QFT passes (phase runs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_quant_ph_0608239_b200 import QSim  # noqa: E402
from workloads import circuits as C  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
w = C.qft_basis(n, 0x5A5A5A5 % (1 << n))
sim = QSim(n)
sim.set_option("timing", 1)
for _ in range(2):
    sim.init_basis(w.init)
    sim.run_circuit(w.gates)
    sim.sync()
st = sim.stats()
print("passes", st["passes"], "pass_ms", st["pass_ms"] / 2, "fp64 slots/amp/pass", st["pass_fp64_slots"] / st["passes"] / 2 ** n)
