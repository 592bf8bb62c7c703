#!/bin/bash
# Round evidence on one B200: bench line, ncu launch list of the same bench
# command, one ncu --set full capture of a config-2 pass (tools/profile_pass.py).
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench=$?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "launches=$?"
python tools/profile_pass.py > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:qsim_pass -s 10 -c 1 -o gpurun_out/prof_pass \
    python tools/profile_pass.py > gpurun_out/ncu_full.log 2>&1; echo "full=$?"
# per-config timings, the paper's benchmarks, a QFT pass capture, the reference arm
python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs=$?"
python tools/bench_paper.py > gpurun_out/paper.jsonl 2> gpurun_out/paper.err; echo "paper=$?"
python tools/profile_qft.py 28 > gpurun_out/qft_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:qsim_pass -s 4 -c 1 -o gpurun_out/prof_qft \
    python tools/profile_qft.py 28 > gpurun_out/ncu_qft.log 2>&1; echo "qft=$?"
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
echo "reference=$?"
