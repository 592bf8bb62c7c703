"""Time every BASELINE.json config that fits one B200 (events, after a warm-up
run that also JIT-compiles): config 1 (adder 12 q), 2 (random 24 q),
3 (Shor 28 q), 4 (QFT 32 q, 64 GiB), 5-family at 30 q (1 GPU, and 8 virtual
shards = 3 nonlocal qubits exchanged by device copies)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_quant_ph_0608239_b200 import QSim, pack_gates  # noqa: E402
from workloads import circuits as C  # noqa: E402


def run(name, n, init, gates, ranks=1, reps=3, readout=None):
    sim = QSim(n, n_ranks=ranks, transport="local" if ranks == 1 else "virtual")
    sim.set_option("timing", 1)
    packed = pack_gates(gates)
    sim.init_basis(init); sim.run_circuit(gates, packed=packed); sim.sync()
    sim.reset_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(sim.stream)
    for _ in range(reps):
        sim.init_basis(init); sim.run_circuit(gates, packed=packed); sim.sync()
    e1.record(sim.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    st = sim.stats()
    out = {"config": name, "n": n, "ranks": ranks, "gates": len(gates), "ms": round(ms, 3),
           "agu_per_s": len(gates) * 2.0 ** n / (ms / 1e3),
           "passes": st["passes"] / reps, "pass_ms": st["pass_ms"] / reps, "perm_ms": st["perm_ms"] / reps,
           "generic_ms": st["generic_ms"] / reps, "exchange_ms": st["exchange_ms"] / reps,
           "exchanges": st["exchanges"] / reps,
           "pass_tflops": 2 * st["pass_fp64_slots"] / (st["pass_ms"] / 1e3) / 1e12 if st["pass_ms"] else None,
           "pass_GBps": st["pass_amp_bytes"] / (st["pass_ms"] / 1e3) / 1e9 if st["pass_ms"] else None}
    if readout:
        out.update(readout(sim))
    print(json.dumps(out), flush=True)
    sim.close()
    torch.cuda.empty_cache()


w1 = C.config1_adder()
run("1 adder", w1.n, w1.init, w1.gates, reps=20)
w2 = C.config2_random()
run("2 random", w2.n, w2.init, w2.gates)
w3 = C.config3_shor()
run("3 shor", w3.n, w3.init, w3.gates, reps=2)
w4 = C.config4_qft()
run("4 qft", 32, w4.init, w4.gates, reps=1)
g5 = C.random_chain(30, 10, seed=5, sweep=True)
run("5-family 30q", 30, 0, g5, reps=1)
run("5-family 30q virt8", 30, 0, g5, ranks=8, reps=1)
