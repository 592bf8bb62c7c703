"""Run one config-2 circuit (24 q, 1420 gates) through the engine: the
command profiled by ncu (one GPU)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_quant_ph_0608239_b200 import QSim  # noqa: E402
from workloads import circuits as C  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
w = C.config2_random()
sim = QSim(w.n)
for _ in range(reps):
    sim.init_basis(0)
    sim.run_circuit(w.gates)
    sim.sync()
print("norm", sim.norm(), "stats", sim.stats())
