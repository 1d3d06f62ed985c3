#!/bin/bash
# Multi-GPU evidence on one 4-GPU box: tools/mgpu_evidence.sh at 4 and 2
# GPUs (bitwise against one GPU), then bench.py at 1 / 2 / 4 GPUs on Kochi-1.0
# (K = 20 and 200), config 5 (strong) and config 5 weak.
#   tools/scale_evidence.sh TAG        (results in gpurun_out/TAG_*)
set -u
O=gpurun_out; mkdir -p $O
TAG=${1:-e}
bash tools/mgpu_evidence.sh ${TAG}
CUDA_VISIBLE_DEVICES=0,1 bash tools/mgpu_evidence.sh ${TAG}
for n in 1 2 4; do
  devs=$(python -c "print(','.join(str(i) for i in range($n)))")
  for spec in "kochi20 --steps 20 --warmup 5" "kochi200 --steps 200 --warmup 5" "cfg5 --config cfg5 --steps 10 --warmup 3" "cfg5weak --config cfg5weak --steps 10 --warmup 3"; do
    set -- $spec; name=$1; shift
    if [ $n = 1 ]; then CUDA_VISIBLE_DEVICES=$devs timeout 900 python bench.py --gpus 1 "$@" --no-cpu > $O/${TAG}_${name}_n$n.json 2> $O/${TAG}_${name}_n$n.err
    else CUDA_VISIBLE_DEVICES=$devs timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $n "$@" --no-cpu > $O/${TAG}_${name}_n$n.json 2> $O/${TAG}_${name}_n$n.err; fi
    echo "$name n=$n rc=$?"; python -c "
import json; d=json.load(open('$O/${TAG}_${name}_n$n.json')); print(round(d['value'],2), round(d['ms_per_step'],4), d['e2e']['value'])" 2>/dev/null
  done
done
