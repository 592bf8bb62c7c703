"""Per-qubit-position single-gate bandwidth sweep (config 5's sweep, Fig. 6
analog P:1102-1114): one Haar U2 (and one H) on qubit p of an n-qubit state,
each its own pass; GB/s = 32 B x 2^n / kernel time, vs the measured HBM peak."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_quant_ph_0608239_b200 import QSim  # noqa: E402
from workloads import gates as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
reps = 5
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")) else 6545.0
sim = QSim(n)
sim.set_option("timing", 1)
sim.init_basis(0)
sim.run_circuit([G.one_q(q, G.H) for q in range(n)])
sim.sync()
rng = G.SplitMix64(5)
rows = []
for p in range(n):
    for name, u in (("H", G.H), ("U2", G.haar_u2(rng))):
        g = [G.one_q(p, u)]
        sim.run_circuit(g)
        sim.sync()
        sim.reset_stats()
        for _ in range(reps):
            sim.run_circuit(g)
            sim.sync()
        st = sim.stats()
        ms = (st["pass_ms"] + st["generic_ms"]) / reps
        gbs = 32.0 * 2 ** n / (ms / 1e3) / 1e9
        rows.append({"p": p, "gate": name, "ms": round(ms, 4), "GBps": round(gbs, 1), "frac_hbm": round(gbs / peak, 3)})
        print(json.dumps(rows[-1]), flush=True)
fr = [r["frac_hbm"] for r in rows]
print(json.dumps({"summary": True, "n": n, "min_frac": min(fr), "median_frac": sorted(fr)[len(fr) // 2],
                  "max_frac": max(fr)}))
