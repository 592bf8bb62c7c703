"""A/B of the fused <Q_i> readout (option fuse_readout) on a workload:
init + circuit + qsim_expectations per step, device-timed, with the per-kind
event times.  usage: python tools/readout_ab.py [config4|config2|hallN|config3]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_quant_ph_0608239_b200 import QSim, pack_gates  # noqa: E402
from workloads import circuits as C  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "config4"
w = {"config4": C.config4_qft, "config2": C.config2_random, "config3": C.config3_shor}.get(wl)
w = w() if w else C.h_on_all(int(wl[4:]))
packed = pack_gates(w.gates)
sim = QSim(w.n)
for fuse in (1, 0, 1, 0):
    sim.set_option("fuse_readout", fuse)
    sim.set_option("timing", 0)
    sim.init_basis(w.init); sim.run_circuit(w.gates, packed=packed); sim.expectations()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 3
    e0.record(sim.stream)
    for _ in range(K):
        sim.init_basis(w.init); sim.run_circuit(w.gates, packed=packed); ex = sim.expectations()
    e1.record(sim.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    sim.set_option("timing", 1)
    sim.reset_stats()
    sim.init_basis(w.init); sim.run_circuit(w.gates, packed=packed); sim.expectations()
    st = sim.stats()
    print(json.dumps({"workload": wl, "fuse_readout": fuse, "ms_per_step": round(ms, 3),
                      "pass_ms": round(st["pass_ms"], 3), "reduce_ms": round(st["reduce_ms"], 3),
                      "fused_readouts": st["fused_readouts"]}), flush=True)
