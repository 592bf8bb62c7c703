#!/bin/bash
# Round evidence on one B200 (run under gpurun; outputs in gpurun_out/, copy
# the summaries into profiles/ with the round prefix):
#   bench line, ncu launch list of the same bench command, ncu --set full
#   captures of a config-2 pass, a QFT pass (the pass itself: ^qsim_pass$, not
#   the qsim_pass_tab companion), the permutation run, per-pass metrics of a
#   config-2 step; per-config timings, the paper's benchmarks, the position
#   sweep and the reference arm.
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench=$?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/ncu_launches.log 2>&1; echo "launches=$?"
python tools/profile_pass.py > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:^qsim_pass$ -s 10 -c 1 -o gpurun_out/prof_pass -f \
    python tools/profile_pass.py > gpurun_out/ncu_full.log 2>&1; echo "full=$?"
python tools/profile_qft.py 28 > gpurun_out/qft_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:^qsim_pass$ -s 4 -c 1 -o gpurun_out/prof_qft -f \
    python tools/profile_qft.py 28 > gpurun_out/ncu_qft.log 2>&1; echo "qft=$?"
python tools/profile_shor.py > gpurun_out/shor_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_perm_run -s 1 -c 1 -o gpurun_out/prof_perm -f \
    python tools/profile_shor.py > gpurun_out/ncu_perm.log 2>&1; echo "perm=$?"
python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs=$?"
python tools/bench_paper.py > gpurun_out/paper.jsonl 2> gpurun_out/paper.err; echo "paper=$?"
python tools/sweep.py 30 > gpurun_out/sweep30.jsonl 2>&1; echo "sweep=$?"
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
echo "reference=$?"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/relayout_bench tools/relayout_bench.cu && \
/tmp/relayout_bench > gpurun_out/relayout_bench.jsonl 2>&1; echo "relayout_bench=$?"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gran_bench tools/gran_bench.cu && \
/tmp/gran_bench 30 > gpurun_out/gran_bench.jsonl 2>&1; echo "gran_bench=$?"
ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio --clock-control none -k regex:^qsim_pass$ -s 28 -c 14 -o gpurun_out/prof_perpass -f \
    python tools/profile_pass.py 3 > gpurun_out/ncu_perpass.log 2>&1; echo "perpass=$?"
