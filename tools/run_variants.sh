#!/bin/bash
# runs on the GPU box
cd $GRAFT_REPO_ROOT
for v in "$@"; do
  XQR_B200_LIB=tools/_var/$v/lib.so timeout 300 python tools/variant_bench.py --batch 296 --reps 3 2>&1 | tail -1
done
