#!/bin/bash
# Round profile capture (run on the GPU box from the repo root):
#   bash tools/profile_round.sh TAG
# 1. the default bench (must exit 0 before anything runs under ncu)
# 2. ncu launch lists (gpu__time_duration per launch) of the C2 / C3 benches
# 3. one ncu --set full capture of each dominant kernel
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err || { echo "bench failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_c2_train_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-secondary --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_c3_infer_launches.csv \
    python bench.py --workload c3-infer --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_train_fast -s 3 -c 1 \
    -o $OUT/${TAG}_prof_train python bench.py --steps 1 --warmup 3 --no-secondary --no-cpu-baseline > $OUT/${TAG}_ncu_train.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_infer_ws -s 3 -c 1 \
    -o $OUT/${TAG}_prof_infer python bench.py --workload c3-infer --steps 1 --warmup 3 --no-cpu-baseline > $OUT/${TAG}_ncu_infer.log 2>&1
echo done
