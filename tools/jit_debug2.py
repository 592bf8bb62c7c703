import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_quant_ph_0608239_b200 import QSim
from workloads import circuits as C
for n, r in [(13, 1), (15, 4)]:
    for jit in (0, 1):
        sim = QSim(n, n_ranks=r, transport="local" if r == 1 else "virtual")
        sim.set_option("fusion", 1)
        sim.set_option("jit", jit)
        sim.init_basis(1)
        sim.run_circuit(C.random_brickwork(n, 4, seed=n))
        a = sim.get_amplitudes()
        print(n, r, jit, sim.stats()["jit_launches"], "err:", sim.lib.qsim_last_error(sim.ctx).decode()[:800])
