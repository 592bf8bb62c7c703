"""Hottest SASS instructions of the first profiled kernel with their top stall reasons,
and stall-reason totals by instruction class."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr, out, k = None, [], 0
for r in rows:
    if r and r[0] == "Kernel Name":
        k += 1
        if k > 1:
            break
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        out.append(r)
ist = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
iS = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[iS] or 0) for r in out) or 1
by = {}
for n, r in enumerate(out):
    reasons = sorted(((hdr[i][6:], float(r[i] or 0)) for i in ist), key=lambda x: -x[1])
    by[n] = reasons
for n, r in sorted(enumerate(out), key=lambda x: -float(x[1][iS] or 0))[:top]:
    rs = ", ".join(f"{a}={100 * b / tot:.1f}" for a, b in by[n][:3] if b)
    print(f"{n:5d} {100 * float(r[iS] or 0) / tot:5.1f}%  {r[1].strip()[:48]:48s} {rs}")
agg = {}
for n, r in enumerate(out):
    for a, b in by[n]:
        agg[a] = agg.get(a, 0) + b
print("totals:", ", ".join(f"{a}={100 * b / tot:.1f}%" for a, b in sorted(agg.items(), key=lambda x: -x[1])[:10]))
