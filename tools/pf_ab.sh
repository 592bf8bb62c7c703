#!/bin/bash
# A/B of JIT generator env variants on config 2 (one process per variant)
for v in "$@"; do
  echo "== $v"
  env $v python tools/pass_ab.py
done
