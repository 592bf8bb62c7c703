"""Pipelined pass kernel vs oracle with the persistent grid capped (many tiles per CTA)."""
import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    import numpy as np
    import oracle
    from paper_quant_ph_0608239_b200 import QSim
    from workloads import circuits as C
    n, depth = int(sys.argv[1]), int(sys.argv[2])
    seed = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    g = C.random_brickwork(n, depth, seed=seed)
    sim = QSim(n); sim.init_basis(0); sim.run_circuit(g); a = sim.get_amplitudes()
    o = oracle.Oracle(n); o.init_basis(0); o.run(g)
    err = float(np.max(np.abs(a - o.amplitudes())))
    print(json.dumps({"n": n, "depth": depth, "grid": os.environ.get("QSIM_PASS_GRID"), "pipe": os.environ.get("QSIM_JIT_PIPE"), "err": err, "passes": sim.stats()["passes"]}))
else:
    for env in [{"QSIM_JIT_PIPE": "0"}, {"QSIM_PASS_GRID": "3"}, {}]:
        for n, d, sd in [(22, 10, 3), (24, 40, 2), (24, 40, 3), (24, 8, 2), (23, 40, 2)]:
            subprocess.run([sys.executable, __file__, str(n), str(d), str(sd)], env={**os.environ, **env})
