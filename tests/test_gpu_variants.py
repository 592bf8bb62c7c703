"""GPU checks that need their own process (-m gpu): the on-disk JIT cache
(environment read at library load) and the opt-in paper-scale parity run."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

_RUN = r'''
import json, sys
import numpy as np
sys.path.insert(0, {root!r})
import oracle
from paper_quant_ph_0608239_b200 import QSim
from workloads import circuits as C
n, shards, kind = {n}, {shards}, {kind!r}
init = 0
if kind == "brick":
    gates = C.random_brickwork(n, 40, seed=3)
elif kind == "qft":
    w = C.qft_basis(n, 0x5A5A5A5A5 % (1 << n))
    gates, init = w.gates, w.init
else:
    gates = C.random_chain(n, 10, seed=5, sweep=True)
sim = QSim(n, n_ranks=shards, transport="virtual" if shards > 1 else "local")
sim.set_option("overlap", {overlap})
sim.init_basis(init)
sim.run_circuit(gates)
nrm = sim.norm()
o = oracle.Oracle(n)
o.init_basis(init)
o.run(gates)
view = o.psi.view(np.complex128)
err, chunk = 0.0, 1 << 26
for first in range(0, 1 << n, chunk):
    g = sim.get_amplitudes(first, min(chunk, (1 << n) - first))
    err = max(err, float(np.max(np.abs(g - view[first:first + g.size]))))
st = sim.stats()
print(json.dumps({{"n": n, "shards": shards, "gates": len(gates), "max_abs_diff": err, "norm_dev": abs(1 - nrm),
                  "exchanges": st["exchanges"], "overlapped": st["overlapped"], "passes": st["passes"],
                  "jit_compile_ms": st["jit_compile_ms"], "jit_kernels": st["jit_kernels"]}}))
'''


def _run(n, shards, kind, env=None, timeout=600, overlap=1):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    code = _RUN.format(root=ROOT, n=n, shards=shards, kind=kind, overlap=overlap)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=timeout,
                       env={**os.environ, **(env or {})})
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.skipif(not os.environ.get("QSIM_LARGE_PARITY"), reason="opt-in: set QSIM_LARGE_PARITY=<n> (33 takes ~25 min)")
def test_large_full_state_parity():
    """SURVEY §8(c)'s proxy for the 36-qubit row: the config-5 family at n
    qubits on 8 virtual shards vs the oracle at n, amplitude by amplitude
    (n = 33: 128 GiB on the GPU and in host RAM).  Result recorded in
    profiles/r1_parity_33q_8shards.json."""
    n = int(os.environ["QSIM_LARGE_PARITY"])
    # overlap = 2: the pass + exchange overlap runs on the virtual shards too
    d = _run(n, 8, os.environ.get("QSIM_LARGE_KIND", "chain"), timeout=3600,
             overlap=int(os.environ.get("QSIM_LARGE_OVERLAP", "2")))
    print(json.dumps(d))
    assert d["max_abs_diff"] <= 1e-11 and d["norm_dev"] <= 1e-12
    assert d["exchanges"] >= 1 and d["passes"] >= 1  # 3 nonlocal qubits: the sharded path ran


def test_jit_disk_cache(tmp_path):
    """The pass kernels a process compiled are loaded from the on-disk cache
    by the next process (no NVRTC), with the same results; QSIM_JIT_CACHE_DIR=off
    bypasses it."""
    env = {"QSIM_JIT_CACHE_DIR": str(tmp_path)}
    a = _run(18, 1, "chain", env)
    files = [f for f in os.listdir(tmp_path) if f.endswith(".bin")]
    assert len(files) == a["jit_kernels"] > 0
    b = _run(18, 1, "chain", env)
    assert b["max_abs_diff"] == a["max_abs_diff"] <= 1e-11
    assert b["jit_compile_ms"] < 0.25 * a["jit_compile_ms"], (a["jit_compile_ms"], b["jit_compile_ms"])
    c = _run(18, 1, "chain", {"QSIM_JIT_CACHE_DIR": "off"})
    assert c["max_abs_diff"] == a["max_abs_diff"] and c["jit_compile_ms"] > 2 * b["jit_compile_ms"]
