"""Register use / spills of the pass-specialised kernels of a workload,
compiled offline with nvcc -Xptxas -v (no GPU needed).
usage: [QSIM_JIT_3M=..] [QSIM_JIT_U4IL=..] python tools/jit_spills.py config2|chainN|qftN"""
import concurrent.futures as cf
import json
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_quant_ph_0608239_b200 import plan_json  # noqa: E402
from workloads import circuits as C  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "config2"
if wl == "config2":
    n, gates = 24, C.random_brickwork(24, 40, seed=2)
elif wl.startswith("chain"):
    n = int(wl[5:]); gates = C.random_chain(n, 10, seed=5, sweep=True)
elif wl.startswith("qft"):
    n = int(wl[3:]); w = C.qft_basis(n, 12345); gates = w.gates
d = tempfile.mkdtemp()
os.environ["QSIM_JIT_DUMP"] = d
js = json.loads(plan_json(n, 1, gates, key_check=True))
files = sorted(f for f in os.listdir(d) if f.endswith(".cu"))


def comp(f):
    r = subprocess.run(["/usr/local/cuda/bin/nvcc", "-std=c++17", "-arch=sm_100a", "-cubin", "-Xptxas", "-v",
                        "-diag-suppress=177", os.path.join(d, f), "-o", os.path.join(d, f + ".cubin")],
                       capture_output=True, text=True)
    m = re.search(r"(\d+) bytes spill stores", r.stderr)
    g = re.search(r"Used (\d+) registers", r.stderr)
    return f, int(m.group(1)) if m else -1, int(g.group(1)) if g else -1


with cf.ThreadPoolExecutor(16) as ex:
    res = list(ex.map(comp, files))
sp = [x[1] for x in res]
if os.environ.get("JIT_SPILLS_VERBOSE"):
    for r in res: print(r)
print(json.dumps({"workload": wl, "3m": os.environ.get("QSIM_JIT_3M"), "il": os.environ.get("QSIM_JIT_U4IL"),
                  "kernels": len(res), "spill_total": sum(sp), "spill_max": max(sp),
                  "fp64_per_amp": sum(js["jit"]["fp64_per_amp"])}))
