import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_quant_ph_0608239_b200 import QSim
from workloads import circuits as C
sim = QSim(14)
sim.set_option("jit", 1)
sim.init_basis(0)
sim.run_circuit(C.random_brickwork(14, 3, 1))
sim.sync()
print("last_error:", sim.lib.qsim_last_error(sim.ctx).decode()[:3000])
print(sim.stats())
