"""A/B of the pass + exchange overlap on the virtual transport (8 shards on
one GPU): the config-5 family at n qubits, overlap on vs off; device time per
step (CUDA events) and the exchange / overlapped-step shares."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_quant_ph_0608239_b200 import QSim, pack_gates  # noqa: E402
from workloads import circuits as C  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
ranks = int(sys.argv[2]) if len(sys.argv) > 2 else 8
gates = C.random_chain(n, 10, seed=5, sweep=True)
packed = pack_gates(gates)
sim = QSim(n, n_ranks=ranks, transport="virtual")
for ov in (0, 2, 0, 2):
    sim.set_option("overlap", ov)
    sim.set_option("timing", 0)
    sim.init_basis(0); sim.run_circuit(gates, packed=packed); sim.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(sim.stream)
    sim.init_basis(0); sim.run_circuit(gates, packed=packed); sim.sync()
    e1.record(sim.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    sim.set_option("timing", 1)
    sim.reset_stats()
    sim.init_basis(0); sim.run_circuit(gates, packed=packed); sim.sync()
    st = sim.stats()
    print(json.dumps({"n": n, "shards": ranks, "overlap": ov, "ms_per_step": round(ms, 3),
                      "pass_ms": round(st["pass_ms"], 3), "exchange_ms": round(st["exchange_ms"], 3),
                      "overlap_ms": round(st["overlap_ms"], 3), "overlapped": st["overlapped"],
                      "exchanges": st["exchanges"], "passes": st["passes"]}), flush=True)
