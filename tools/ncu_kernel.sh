#!/bin/bash
# One full ncu capture of a kernel (regex) in a few Kochi-1.0 steps.
#   tools/ncu_kernel.sh TAG REGEX [SKIP] [COUNT]   -> gpurun_out/TAG.ncu-rep
set -u
TAG=$1; RX=$2; SKIP=${3:-4}; CNT=${4:-1}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" --launch-skip $SKIP \
    --launch-count $CNT -o gpurun_out/$TAG python tools/profile_step.py --steps 4 > gpurun_out/$TAG.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/$TAG.log
