"""Per-pass table of one config-2 step from an ncu report of its 14 pass
launches (tools/profile_round.sh: the last step of tools/profile_pass.py 3),
with the generator's executed FP64 per amplitude, the plan's re-layouts and
blocks, and each pass's FP64 + re-layout serial bound.
usage: python tools/ncu_perpass.py REPORT.ncu-rep"""
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402  (peaks and the re-layout bandwidth)
from paper_quant_ph_0608239_b200 import plan_json  # noqa: E402
from workloads import circuits as C  # noqa: E402

STALLS = ("no_instruction", "barrier", "long_scoreboard", "short_scoreboard", "mio_throttle", "math_pipe_throttle")

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
to_ns = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9, "s": 1e9}[
    units[col["gpu__time_duration.sum"]]]

w = C.config2_random()
d = json.loads(plan_json(w.n, 1, w.gates, key_check=True))
passes = [s for s in d["plan"]["steps"] if s["type"] == "pass"]
fps = d["jit"]["fp64_per_amp"]
amps = float(1 << w.n)
fp64_peak, hbm = 34.2e12, 6548.2e9
print("# config 2: every pass of one step (ncu --clock-control none, the last step of tools/profile_pass.py 3)")
print("# fp64/amp = executed FP64-pipe instructions per amplitude (generator count); eff = achieved / 34.2 TFLOP/s")
print("# bound = max(FP64 at 34.2 TFLOP/s + re-layouts at %.1f TB/s, 32 B/amp at 6548 GB/s); meas/bound >= 1"
      % (bench.SMEM_RELAYOUT_GBS / 1e3))
tot_ns = tot_b = 0.0
for i, (r, st, fp) in enumerate(zip(data, passes, fps)):
    ns = float(r[col["gpu__time_duration.sum"]]) * to_ns
    rel = sum(1 for o in st["ops"] if o["code"] == 4)
    u4 = sum(1 for o in st["ops"] if o["code"] == 7)
    t_fp = 2 * fp * amps / fp64_peak
    t_sm = rel * 32 * amps / (bench.SMEM_RELAYOUT_GBS * 1e9)
    bound = max(t_fp + t_sm, 32 * amps / hbm) * 1e9
    tot_ns += ns
    tot_b += bound
    st_txt = " ".join("stall_%s=%.2f" % (k, float(r[col["smsp__average_warps_issue_stalled_%s_per_issue_active.ratio"
                                                          % k]])) for k in STALLS)
    print("pass %2d ns=%9.0f fp64_pipe_pct=%5.1f issue_pct=%5.1f %s fp64/amp=%3.0f eff=%.2f relayouts=%2d u4=%2d "
          "bound_ns=%8.0f meas/bound=%.2f" % (
              i, ns, float(r[col["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]]),
              float(r[col["smsp__issue_active.avg.pct_of_peak_sustained_active"]]), st_txt, fp,
              2 * fp * amps / (ns * 1e-9) / fp64_peak, rel, u4, bound, ns / bound))
print("step: %.3f ms measured, %.3f ms serial bound (meas/bound %.2f)" % (tot_ns / 1e6, tot_b / 1e6, tot_ns / tot_b))
