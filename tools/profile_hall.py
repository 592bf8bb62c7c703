"""Run H on all L qubits (the paper's scaling test, default L = 30) twice
through the engine: the command profiled by ncu (one GPU)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_quant_ph_0608239_b200 import QSim  # noqa: E402
from workloads import circuits as C  # noqa: E402

w = C.h_on_all(int(sys.argv[1]) if len(sys.argv) > 1 else 30)
sim = QSim(w.n)
for _ in range(2):
    sim.init_basis(0)
    sim.run_circuit(w.gates)
    sim.sync()
print("norm", sim.norm(), "stats", sim.stats())
