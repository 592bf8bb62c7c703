"""Static plan statistics for a workload: passes, re-layouts, ops whose
predicate depends on lane/warp bits (select-based in the JIT kernel)."""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_quant_ph_0608239_b200 as P  # noqa: E402
from workloads import circuits as C  # noqa: E402

cases = {"c2": (24, C.config2_random().gates), "c4-24": (24, C.qft_basis(24, 123).gates),
         "c3": (28, C.config3_shor().gates), "c5-30": (30, C.random_chain(30, 10, 5, True))}
for name, (n, gates) in cases.items():
    d = json.loads(P.plan_json(n, 1, gates))
    passes = [s for s in d["plan"]["steps"] if s["type"] == "pass"]
    c = collections.Counter()
    for s in passes:
        for o in s["ops"]:
            if o["code"] == 4:
                c["trans"] += 1
            elif o["mlane"] or o["mwarp"]:
                c["sel_" + ("xs" if o["code"] == 2 else "phase" if o["code"] == 3 else "u2")] += 1
            else:
                c["plain_" + ("xs" if o["code"] == 2 else "phase" if o["code"] == 3 else "u2")] += 1
    print(name, "passes", len(passes), dict(sorted(c.items())))
