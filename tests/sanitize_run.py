"""Small workloads that exercise every kernel family, for compute-sanitizer
(racecheck / synccheck / memcheck) runs on one GPU:
  compute-sanitizer --tool racecheck python tests/sanitize_run.py
Fused tile passes with shared-memory re-layouts (JIT and interpreter tiers),
phase runs + the qsim_pass_tab companion kernel (QFT), the permutation run
(k_perm_run: cp.async double buffer, composed tables) and k_perm, exchanges
on 4 virtual shards, and the readouts (marginals, <Q_i>, two-level sampling).
Checked against the CPU oracle so a race that corrupts data also fails here."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_quant_ph_0608239_b200 import QSim  # noqa: E402
from workloads import circuits as C  # noqa: E402

n = int(os.environ.get("SAN_N", "14"))
cases = [("brick", n, 0, C.random_brickwork(n, 6, seed=2), 1, 1),
         ("brick-interp", n, 0, C.random_brickwork(n, 3, seed=3), 1, 0),
         ("qft", n, 5, C.qft_ladder(list(range(n)), swaps=True), 1, 1),
         ("chain-virt4", n, 0, C.random_chain(n, 2, seed=5, sweep=False), 4, 1)]
w = C.shor_order_finding(35, 3, 8, 6)
cases.append(("shor", w.n, w.init, w.gates, 1, 1))
bad = 0
for name, nq, init, gates, ranks, jit in cases:
    sim = QSim(nq, n_ranks=ranks, transport="local" if ranks == 1 else "virtual")
    sim.set_option("jit", jit)
    sim.init_basis(init)
    sim.run_circuit(gates)
    got = sim.get_amplitudes()
    o = oracle.Oracle(nq)
    o.init_basis(init)
    o.run(gates)
    err = float(np.max(np.abs(got - o.amplitudes())))
    p = sim.probabilities([0, nq - 1])
    ex = sim.expectations()
    shots = sim.measure(list(range(nq)), seed=3, shots=64)
    st = sim.stats()
    sim.close()
    ok = err <= 1e-11 and np.max(np.abs(p - o.probabilities([0, nq - 1]))) <= 1e-12
    bad += not ok
    print(f"{name}: n={nq} ranks={ranks} jit={jit} passes={st['passes']} perms={st['perm_launches']} "
          f"exchanges={st['exchanges']} max|d|={err:.2e} ok={ok}", flush=True)
sys.exit(1 if bad else 0)
