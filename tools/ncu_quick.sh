#!/bin/bash
# runs on the GPU box: quick ncu (warp states, instruction stats) of one batched wave per library variant
#   tools/ncu_quick.sh name [name...]   (name "default" = the in-tree library)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "$@"; do
  lib=""; [ "$v" != default ] && lib=tools/_var/$v/lib.so
  XQR_B200_LIB=$lib timeout 600 ncu --section WarpStateStats --section InstructionStats --section SchedulerStats --section ComputeWorkloadAnalysis \
     --clock-control none -k regex:mgs_cta_kernel -c 1 -o gpurun_out/q_$v python tools/profile_batched.py 4 128 128 296 1 > gpurun_out/q_$v.log 2>&1
done
