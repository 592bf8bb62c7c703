"""Stall samples of the first profiled kernel by program segment (SASS order)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
nseg = int(sys.argv[2]) if len(sys.argv) > 2 else 20
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
out, k = [], 0
for r in rows:
    if r and r[0] == "Kernel Name":
        k += 1
        if k > 1:
            break
        continue
    if not r or r[0] == "Address" or len(r) < 4:
        continue
    out.append((r[1].strip(), float(r[2] or 0)))
tot = sum(x[1] for x in out) or 1
seg = max(1, len(out) // nseg)
for i in range(0, len(out), seg):
    ch = out[i:i + seg]
    ops = {}
    for t, _ in ch:
        w = t.split()
        o = (w[1] if w[0].startswith("@") and len(w) > 1 else w[0]).split(".")[0]
        ops[o] = ops.get(o, 0) + 1
    hot = max(ch, key=lambda x: x[1])
    print(f"{i:5d} {100 * sum(x[1] for x in ch) / tot:5.1f}%  {sorted(ops.items(), key=lambda x: -x[1])[:4]}  hot: {hot[0][:40]} {100 * hot[1] / tot:.1f}%")
