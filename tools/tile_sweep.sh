#!/bin/bash
# tile width x kernel variant sweep on config 2 (rebuilds the library per tile width)
for tb in 12 11; do
  QSB_TILE_BITS=$tb python -m paper_quant_ph_0608239_b200.build --force > /dev/null 2>&1
  for v in "QSIM_JIT_PIPE=0" "QSIM_JIT_PIPE=1" "QSIM_JIT_PIPE=0 QSIM_JIT_MINB=3"; do
    echo "== tile=$tb $v"; env $v python tools/pass_ab.py
  done
done
python -m paper_quant_ph_0608239_b200.build --force > /dev/null 2>&1
