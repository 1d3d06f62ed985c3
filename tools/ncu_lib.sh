#!/bin/bash
# ncu full capture of the march kernels of a given library build
#   tools/ncu_lib.sh TAG LIB [REGEX] [SKIP] [COUNT]
set -u
TAG=$1; LIB=$2; RX=${3:-k_march}; SKIP=${4:-4}; CNT=${5:-4}
mkdir -p gpurun_out
TSUNAMI_B200_LIB=$LIB timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" --launch-skip $SKIP \
    --launch-count $CNT -o gpurun_out/$TAG python tools/profile_step.py --steps 4 > gpurun_out/$TAG.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/$TAG.log
