"""A/B timing of engine options on config 2 (24 q, 1420 gates).
usage: python tools/pass_ab.py key=v1,v2 [key2=...]"""
import itertools
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_quant_ph_0608239_b200 import QSim, pack_gates  # noqa: E402
from workloads import circuits as C  # noqa: E402

wl = os.environ.get("PASS_AB_WORKLOAD", "config2")
if wl == "config2":
    w = C.config2_random()
elif wl.startswith("chain"):  # config-5 family at n qubits, e.g. chain28
    n = int(wl[5:])
    w = C.Workload("chain", n, 0, C.random_chain(n, 10, seed=5, sweep=True), {})
elif wl.startswith("qft"):
    w = C.qft_basis(int(wl[3:]), 12345)
elif wl.startswith("hall"):  # H on all n qubits (the paper's scaling test)
    w = C.h_on_all(int(wl[4:]))
elif wl == "shor":  # config 3 (28 q)
    w = C.config3_shor()
else:
    raise SystemExit("unknown PASS_AB_WORKLOAD " + wl)
packed = pack_gates(w.gates)
opts = {}
for a in sys.argv[1:]:
    k, v = a.split("=")
    opts[k] = [int(x) for x in v.split(",")]
keys = list(opts)
sim = QSim(w.n)
for combo in itertools.product(*[opts[k] for k in keys]) if keys else [()]:
    for k, v in zip(keys, combo):
        sim.set_option(k, v)
    sim.set_option("timing", 1)
    for _ in range(3):
        sim.init_basis(w.init); sim.run_circuit(w.gates, packed=packed); sim.sync()
    sim.reset_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 5
    e0.record(sim.stream)
    for _ in range(K):
        sim.init_basis(w.init); sim.run_circuit(w.gates, packed=packed)
        sim.sync()
    e1.record(sim.stream)
    torch.cuda.synchronize()
    st = sim.stats()
    ms = e0.elapsed_time(e1) / K
    print(json.dumps({"opts": dict(zip(keys, combo)), "ms_per_step": round(ms, 3),
                      "agu_per_s": len(w.gates) * 2 ** w.n / (ms / 1e3),
                      "pass_ms_per_launch": st["pass_ms"] / max(1, st["passes"]),
                      "passes_per_step": st["passes"] / K, "pass_GBps": st["pass_amp_bytes"] / (st["pass_ms"] / 1e3) / 1e9,
                      "perm_ms": st["perm_ms"] / K, "plan_ms": st["plan_ms"] / K}))
