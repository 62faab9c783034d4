#!/bin/bash
# Profile evidence for one round (run under gpurun from the repo root):
#   1) the bench command plain, 2) its per-launch list (gpu__time_duration),
#   3) one full capture of each dominant kernel (lag moments L2, fused conv-hist, conv).
set -u
OUT=gpurun_out/prof_round
mkdir -p $OUT
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > $OUT/plain.json 2> $OUT/plain.err && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"ddcca|lag_zone|conv|solve|zone_reduce|assemble|rect_sums|batch_epilogue|tree_level|hist" \
    --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"conv_hist_kernel" -c 1 \
    -o $OUT/conv_hist $CMD > $OUT/ncu_full1.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"lag_zone_kernel" -s 1 -c 1 \
    -o $OUT/lag_zone $CMD > $OUT/ncu_full2.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"conv_c_kernel" -c 1 \
    -o $OUT/conv_c $CMD > $OUT/ncu_full3.log 2>&1
echo "profile rc=$?"
