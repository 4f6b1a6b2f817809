#!/bin/bash
# runs on the GPU box: single-system factorisation/back-substitution spans per library / env setting
#   tools/single_cmp.sh "label|ENV=.. ENV2=..|lib" ...   (lib "" = in-tree)
cd $GRAFT_REPO_ROOT
for spec in "$@"; do
  IFS='|' read -r label envs lib <<< "$spec"
  for m in 256 512; do
    out=$(env $envs XQR_B200_LIB=$lib timeout 300 python tools/trace_single.py --reps 2 --m $m 2>&1 | tail -n 1)
    echo "$label m=$m: $out"
  done
done
