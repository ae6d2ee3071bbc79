#!/bin/bash
# Time n=15 dense under environment variations (developer tool). Usage: tools/sweep_env.sh "VAR=a VAR2=b" "VAR=c" ...
for cfg in "$@"; do
  echo -n "$cfg : "
  env $cfg timeout 120 python tools/diag_n15.py ${N:-15} 2>&1 | tail -1
done
