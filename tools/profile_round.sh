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
