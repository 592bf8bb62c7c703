"""Modelled weak scaling of the config-5 family: n = 33 + log2 N
qubits on N B200 (N = 8: config 5 itself, 36 q, 128 GiB per GPU).

The plan is the engine's own (host planner, plan_json with generated-kernel
FP64 counts).  Per step:
  - a pass costs max(FP64-pipe instructions per amp x 2^M / F, 32 B x 2^M / H),
    F = the FP64 rate the fused passes reach on one B200 (measured: the bench's
    config5_family_33q line, default 23.2 TFLOP/s executed), H = 0.85 x the
    measured HBM copy peak;
  - a K-pair exchange sends (2^K - 1)/2^K of the shard per direction over
    NVLink at B GB/s (default 0.75 x 900 GB/s per direction; NCCL peer
    send/recv on NVSwitch is not measurable on this one-GPU pool) plus, for
    non-contiguous blocks, the pack/unpack copies at H;
  - an overlapped pass + exchange (runtime `overlap`) costs max(pass, exchange)
    + one block of the pass (the first block computes before any transfer).
usage: python tools/model_scaling.py [F_tflops] [B_gbs]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_quant_ph_0608239_b200 import plan_json  # noqa: E402
from workloads import circuits as C  # noqa: E402

F = float(sys.argv[1]) * 1e12 if len(sys.argv) > 1 else 23.2e12
B = float(sys.argv[2]) * 1e9 if len(sys.argv) > 2 else 0.75 * 900e9
peaks = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
H = 0.85 * (json.load(open(peaks))["hbm_gbs"] * 1e9 if os.path.exists(peaks) else 6.55e12)


def model(n, P):
    gates = C.random_chain(n, 10, seed=5, sweep=True)
    d = json.loads(plan_json(n, P, gates, key_check=True, overlap=P > 1))  # the plan the NCCL runtime makes
    fp = iter(d["jit"]["fp64_per_amp"])
    M = d["plan"]["M"]
    amps = float(1 << M)
    steps = d["plan"]["steps"]
    t = t_pass = t_x = 0.0
    n_pass = n_x = n_ov = 0
    i = 0
    while i < len(steps):
        s = steps[i]
        if s["type"] == "pass":
            tp = max(next(fp) * amps * 2 / F, 32 * amps / H)
            n_pass += 1
            nx = steps[i + 1] if i + 1 < len(steps) else None
            if P > 1 and nx and nx["type"] == "exchange" and not (set(nx["lpos"]) & (set(s["tp"]) | set(s["tp_out"]))):
                K = len(nx["lpos"])
                tx = (2 ** K - 1) / 2 ** K * 16 * amps / B
                t += max(tp, tx) + tp / 2 ** K
                t_pass += tp
                t_x += tx
                n_x += 1
                n_ov += 1
                i += 2
                continue
            t += tp
            t_pass += tp
        elif s["type"] == "exchange":
            K = len(s["lpos"])
            contiguous = sorted(s["lpos"]) == list(range(M - K, M))
            tx = (2 ** K - 1) / 2 ** K * 16 * amps / B + (0 if contiguous else 2 * 16 * amps * (2 ** K - 1) / 2 ** K / H)
            t += tx
            t_x += tx
            n_x += 1
        elif s["type"] in ("perm", "permrun", "generic", "phase", "pairwise"):
            tp = 32 * amps / H if s["type"] != "pairwise" else 32 * amps / B
            t += tp
        i += 1
    return {"N": P, "n": n, "M": M, "gates": len(gates), "passes": n_pass, "exchanges": n_x, "overlapped": n_ov,
            "t_pass_s": round(t_pass, 4), "t_exchange_s": round(t_x, 4), "t_step_s": round(t, 4),
            "agu_per_s": len(gates) * 2.0 ** n / t}


rows = [model(33 + g, 1 << g) for g in range(4)]
base = rows[0]["agu_per_s"]
for r in rows:
    r["weak_eff"] = round(r["agu_per_s"] / (r["N"] * base), 3)
    print(json.dumps(r))
print(json.dumps({"assumptions": {"fp64_tflops": F / 1e12, "hbm_gbs_eff": H / 1e9, "nvlink_gbs_per_dir": B / 1e9}}))
