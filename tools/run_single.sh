#!/bin/bash
# runs on the GPU box: single-system latency of each variant library
cd $GRAFT_REPO_ROOT
for v in "$@"; do
  for cfg in "2 256 256" "4 256 256" "4 512 256"; do
    set -- $cfg
    XQR_B200_LIB=tools/_var/$v/lib.so timeout 300 python tools/variant_bench.py --single --limbs $1 --m $2 --n $3 --reps 7 2>&1 | tail -1
  done
done
