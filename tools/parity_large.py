"""Full-state parity at paper scale (the "36 q" row's proxy):
the config-5 circuit family (H on all, 10 x (Haar U2 layer + CNOT chain),
per-position sweep) at n qubits on 8 virtual shards of one B200 (3 nonlocal
qubits, K-pair exchanges) against the CPU oracle at the same n, compared
amplitude by amplitude in chunks.  n = 33 needs 128 GiB on the GPU and
128 GiB of host RAM for the oracle.

usage: python tools/parity_large.py [n] [shards]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: parity check only)
from paper_quant_ph_0608239_b200 import QSim  # noqa: E402
from workloads import circuits as C  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 33
shards = int(sys.argv[2]) if len(sys.argv) > 2 else 8
gates = C.random_chain(n, 10, seed=5, sweep=True)

t0 = time.perf_counter()
sim = QSim(n, n_ranks=shards, transport="virtual" if shards > 1 else "local")
sim.init_basis(0)
sim.run_circuit(gates)
ex_gpu = sim.expectations()
nrm = sim.norm()
t_gpu = time.perf_counter() - t0
st = sim.stats()

t0 = time.perf_counter()
o = oracle.Oracle(n)
o.init_basis(0)
o.run(gates)
t_cpu = time.perf_counter() - t0
ex_cpu = o.expectations()

view = o.psi.view(np.complex128)
chunk = 1 << 26
err = 0.0
for first in range(0, 1 << n, chunk):
    g = sim.get_amplitudes(first, chunk)
    err = max(err, float(np.max(np.abs(g - view[first:first + chunk]))))
out = {"n": n, "shards": shards, "gates": len(gates), "max_abs_diff": err, "norm_dev": abs(1 - nrm),
       "max_expect_diff": float(np.max(np.abs(ex_gpu - ex_cpu))), "gpu_s": t_gpu, "oracle_s": t_cpu,
       "oracle_threads": oracle.Oracle.threads(), "exchanges": st["exchanges"], "passes": st["passes"],
       "ok": bool(err <= 1e-11 and abs(1 - nrm) <= 1e-12)}
print(json.dumps(out), flush=True)
