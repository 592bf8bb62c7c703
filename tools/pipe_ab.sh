#!/bin/bash
# interleaved A/B of the JIT pass variants on config 2
for rep in 1 2; do
  for v in 0 1; do
    echo "== QSIM_JIT_PIPE=$v"; QSIM_JIT_PIPE=$v python tools/pass_ab.py
  done
done
