#!/bin/bash
# Round profile capture (run on the GPU box from the repo root):
#   bash tools/profile_round.sh TAG
# 1. every bench workload (each must exit 0 before anything runs under ncu)
# 2. ncu launch lists (gpu__time_duration per launch) of the C2 / C3 benches
# 3. one ncu --set full capture of each dominant kernel
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
python tools/int_peaks.py --out $OUT/${TAG}_int_peaks.json > /dev/null 2>&1
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err || { echo "bench failed"; exit 1; }
for w in c1-train c3-infer c4-train c4-sweep c5-sparse; do
  timeout 1500 python bench.py --workload $w > $OUT/${TAG}_bench_$w.json 2> $OUT/${TAG}_bench_$w.err || echo "bench $w failed"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_c2_train_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-secondary --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_c3_infer_launches.csv \
    python bench.py --workload c3-infer --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_train_spec -s 3 -c 1 \
    -o $OUT/${TAG}_prof_train python bench.py --steps 1 --warmup 3 --no-secondary --no-cpu-baseline > $OUT/${TAG}_ncu_train.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_infer_solo -s 3 -c 1 \
    -o $OUT/${TAG}_prof_infer python bench.py --workload c3-infer --steps 1 --warmup 3 --no-cpu-baseline > $OUT/${TAG}_ncu_infer.log 2>&1
[ -n "${SKIP_C4_NCU:-}" ] || timeout 1500 ncu --set full --import-source on --clock-control none -k k_train -s 3 -c 1 \
    -o $OUT/${TAG}_prof_c4train python bench.py --workload c4-train --steps 1 --warmup 3 --no-cpu-baseline > $OUT/${TAG}_ncu_c4.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_sparse_train -s 3 -c 1 \
    -o $OUT/${TAG}_prof_c5train python bench.py --workload c5-sparse --steps 1 --warmup 3 --no-cpu-baseline > $OUT/${TAG}_ncu_c5train.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_sparse_infer -s 2 -c 1 \
    -o $OUT/${TAG}_prof_c5infer python bench.py --workload c5-sparse --steps 1 --warmup 3 --no-cpu-baseline > $OUT/${TAG}_ncu_c5infer.log 2>&1
echo done
