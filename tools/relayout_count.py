"""Static count of passes, re-layouts and fused blocks in the planner's plan of a workload (CPU only).
usage: python tools/relayout_count.py c2 chain30 c5-33"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_quant_ph_0608239_b200 as P
from workloads import circuits as C
cases = {"c2": (24, C.config2_random().gates), "chain30": (30, C.random_chain(30, 10, seed=5, sweep=True)),
         "c5-33": (33, C.random_chain(33, 10, seed=5, sweep=True))}
for name in sys.argv[1:] or ["c2"]:
    n, g = cases[name]
    d = json.loads(P.plan_json(n, 1, g))
    passes = [s for s in d["plan"]["steps"] if s["type"] == "pass"]
    tr = sum(1 for s in passes for o in s["ops"] if o["code"] == 4)
    u4 = sum(1 for s in passes for o in s["ops"] if o["code"] == 7)
    u2 = sum(1 for s in passes for o in s["ops"] if o["code"] in (0, 1))
    print(name, "passes", len(passes), "relayouts", tr, "u4", u4, "u2", u2, "configs", tr + len(passes),
          "fp64/amp", sum(d["jit"]["fp64_per_amp"]) if "jit" in d else None)
