"""Copy the outputs of tools/profile_round.sh (gpurun_out/) into profiles/
as round-`r` artifacts, with the ncu summaries.  usage: python tools/collect_artifacts.py [round]"""
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
r = sys.argv[1] if len(sys.argv) > 1 else "r1"


def summary(rep):
    out = []
    for tool, head in (("ncu_summary.py", None), ("ncu_hot.py", "# hot instructions (tools/ncu_hot.py)"),
                       ("ncu_segments.py", "# stall samples by program segment (tools/ncu_segments.py)")):
        txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", tool), rep], capture_output=True,
                             text=True).stdout
        if head:
            out += ["", head]
            txt = "\n".join(txt.splitlines()[:14] if tool == "ncu_hot.py" else txt.splitlines())
        out.append(txt.rstrip())
    return "\n".join(out) + "\n"


for src, dst in (("bench.json", "bench.json"), ("launches.csv", "bench_launches.csv"),
                 ("configs.jsonl", "configs.jsonl"), ("paper.jsonl", "paper_benchmarks.jsonl"),
                 ("sweep30.jsonl", "position_sweep_30q.jsonl"), ("bench_reference.json", "bench_reference.json"),
                 ("relayout_bench.jsonl", "relayout_bench.jsonl"), ("gran_bench.jsonl", "tile_granularity_30q.jsonl")):
    if os.path.exists(os.path.join(G, src)) and os.path.getsize(os.path.join(G, src)):
        shutil.copy(os.path.join(G, src), os.path.join(P, f"{r}_{dst}"))
for rep, dst in (("prof_pass.ncu-rep", "pass_c2.txt"), ("prof_qft.ncu-rep", "pass_qft.txt"),
                 ("prof_perm.ncu-rep", "perm_run_bulk.txt")):
    if os.path.exists(os.path.join(G, rep)):
        open(os.path.join(P, f"{r}_{dst}"), "w").write(summary(os.path.join(G, rep)))
t = open(os.path.join(P, f"{r}_pass_c2.txt")).read()
rd = float(re.search(r"dram__bytes_read.sum\s+([\d.]+) Mbyte", t).group(1)) * 1e6
wr = float(re.search(r"dram__bytes_write.sum\s+([\d.]+) Mbyte", t).group(1)) * 1e6
json.dump({"kernel": "qsim_pass", "workload": "config 2 (24 q, block-fused, low-qubit remap, 3M blocks), launch 11 of "
           "tools/profile_pass.py", "dram_bytes_read_per_launch": int(round(rd)),
           "dram_bytes_write_per_launch": int(round(wr)), "dram_bytes_per_launch": int(round(rd + wr)),
           "algorithmic_bytes_per_launch": 536870912,
           "source": f"profiles/{r}_pass_c2.txt (ncu --set full --clock-control none)"},
          open(os.path.join(P, "pass_traffic.json"), "w"))
print("collected into profiles/ as", r)
