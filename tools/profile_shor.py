"""Config 3 (Shor N=899, 28 q) through the engine: the command profiled by
ncu for the permutation run (k_perm_run) and the H / inverse-QFT passes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_quant_ph_0608239_b200 import QSim  # noqa: E402
from workloads import circuits as C  # noqa: E402

w = C.config3_shor()
sim = QSim(w.n)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    sim.init_basis(w.init)
    sim.run_circuit(w.gates)
    sim.sync()
print("norm", sim.norm(), "stats", sim.stats())
