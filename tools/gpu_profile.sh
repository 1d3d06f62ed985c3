#!/bin/bash
# One GPU box pass: parity tests, the 1-GPU bench line, the reference arm,
# the ncu launch list and one full capture of the step's two big kernels.
#   tools/gpu_profile.sh TAG    (results in gpurun_out/TAG_*)
set -u
TAG=${1:-run}
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/${TAG}_pytest.log
timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?"; cat $O/${TAG}_bench.json
timeout 300 python bench.py --impl reference --steps 2 > $O/${TAG}_ref.json 2> $O/${TAG}_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu > $O/${TAG}_ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_march|k_mass" \
    --launch-skip 10 --launch-count 5 -o $O/${TAG}_full python bench.py --steps 2 --warmup 3 --no-cpu \
    > $O/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:"k_xops" --launch-skip 4 --launch-count 2 \
    -o $O/${TAG}_xops python bench.py --steps 2 --warmup 3 --no-cpu > $O/${TAG}_ncu_xops.log 2>&1; echo "ncu xops rc=$?"
