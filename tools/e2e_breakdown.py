"""Host-side timeline of one e2e step of bench.py's config 2 (plan cache off):
validation (qsim_run_circuit), then qsim_expectations (flush: plan + streamed
launches, expectation kernel, D2H)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_quant_ph_0608239_b200 import QSim, pack_gates  # noqa: E402
from workloads import circuits as C  # noqa: E402

w = C.config2_random()
packed = pack_gates(w.gates)
sim = QSim(w.n)
for _ in range(3):
    sim.init_basis(0); sim.run_circuit(w.gates, packed=packed); sim.expectations()
sim.set_option("plan_cache", 0)
ts = []
for _ in range(20):
    t0 = time.perf_counter()
    sim.init_basis(0)
    sim.run_circuit(w.gates, packed=packed)
    t1 = time.perf_counter()
    sim.expectations()
    t2 = time.perf_counter()
    ts.append((t1 - t0, t2 - t1))
ts.sort(key=lambda x: x[0] + x[1])
med = ts[len(ts) // 2]
st = sim.stats()
print({"enqueue_ms": med[0] * 1e3, "flush_to_result_ms": med[1] * 1e3, "total_ms": (med[0] + med[1]) * 1e3,
       "plan_ms_per_step": st["plan_ms"] / 23, "streamed_steps_per_step": st["streamed_steps"] / 20})
