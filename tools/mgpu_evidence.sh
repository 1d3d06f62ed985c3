#!/bin/bash
# Multi-GPU parity evidence on one box: every tests/test_gpu_multi.py case
# at the box's GPU count through tools/mgpu_check.py, JSON lines kept.
#   tools/mgpu_evidence.sh TAG        (results in gpurun_out/TAG_mgpu_*)
set -u
TAG=${1:-mg}
O=gpurun_out
mkdir -p $O
N=$(python -c 'import torch; print(torch.cuda.device_count())')
echo "gpus=$N"
timeout 1500 python -m pytest tests/test_gpu_multi.py -m gpu -v > $O/${TAG}_mgpu_pytest_n$N.log 2>&1
echo "pytest rc=$?"; tail -3 $O/${TAG}_mgpu_pytest_n$N.log
port=29611
for spec in "kochi 0.001 40 minmax" "quad_wetdry 0 30 minmax" "kochi 0.01 20 packed" "kochi 0.001 40 packed" \
            "fuzz 0 60 packed" "fuzz 0 60 minmax"; do
  set -- $spec
  extra=""
  [ "$1" = kochi ] && extra="--scale $2"
  [ "$1" = fuzz ] && extra="--seeds 48"
  port=$((port+1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 \
     --master-port $port tools/mgpu_check.py --system $1 --steps $3 --plan $4 $extra \
     >> $O/${TAG}_mgpu_check_n$N.jsonl 2>> $O/${TAG}_mgpu_check_n$N.err
  echo "$spec rc=$?"
done
