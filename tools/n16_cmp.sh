#!/bin/bash
# developer: compare libraries at n=15/16 (usage: tools/n16_cmp.sh lib1 lib2 ...)
for L in "$@"; do
  for N in 15 16; do
    echo -n "$L n=$N: "; PTDR_LIB_NAME=$L timeout 200 python tools/diag_n15.py $N 2>&1 | tail -1
  done
done
