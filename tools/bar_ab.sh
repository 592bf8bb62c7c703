# A/B of the re-layout barrier forms (QSIM_JIT_BAR) and warp-slot keeping
# (QSIM_PLAN_KEEPWARP): pass timings (BAR_AB_PARITY=1: GPU parity first).
export QSIM_JIT_CACHE_DIR=off
if [ "${BAR_AB_PARITY:-0}" = 1 ]; then
  QSIM_FUZZ_SEEDS=80 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -x -q -m gpu 2>&1 | tail -3
fi
for wl in ${BAR_AB_WL:-config2 chain30 qft28 shor hall30}; do
  for rep in 1 2; do
  for m in ${BAR_AB_MODES:-"0 0" "2 0" "2 1" "3 0" "3 1"}; do set -- $(echo $m | tr , ' ')
    echo "wl=$wl bar=$1 keepwarp=$2"; PASS_AB_WORKLOAD=$wl QSIM_JIT_BAR=$1 QSIM_PLAN_KEEPWARP=$2 timeout 300 python tools/pass_ab.py 2>&1 | tail -1
  done; done
done
