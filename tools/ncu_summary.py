"""Summarise an ncu --set full report: key metrics, stall reasons, opcode mix."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, units, v = r[0], r[1], r[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "launch__grid_size", "launch__occupancy_limit_registers"]
for k in keys:
    if k in h:
        i = h.index(k)
        print(f"{k:70s} {v[i]} {units[i]}")
st = [(h[i][len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(v[i] or 0))
      for i in range(len(h)) if h[i].startswith("smsp__average_warps_issue_stalled") and h[i].endswith("per_issue_active.ratio")]
print("stalls/issue:", ", ".join(f"{k}={x:.2f}" for k, x in sorted(st, key=lambda t: -t[1])[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
iS, iE, iSrc = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed"), hh.index("Source")
samp, ex = collections.Counter(), collections.Counter()
for row in rows[2:]:
    if len(row) <= iE or row[0] in ("Kernel Name", "Address"):
        continue
    t = row[iSrc].strip().split()
    if not t:
        continue
    o = t[1] if t[0].startswith("@") else t[0]
    o = o.split(".")[0]
    samp[o] += float(row[iS] or 0)
    ex[o] += float(row[iE] or 0)
ts, te = sum(samp.values()), sum(ex.values())
print("opcode mix (stall-sample %, instruction %):")
for o, s in samp.most_common(14):
    print(f"   {o:10s} {100 * s / ts:5.1f}% {100 * ex[o] / te:5.1f}%")
