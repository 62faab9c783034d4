#!/bin/bash
# Profile evidence for one round (run under gpurun from the repo root, ONE GPU):
#   1) the bench command plain (must exit 0 before any ncu pass),
#   2) its per-launch list (gpu__time_duration + DRAM bytes, --clock-control none),
#   3) one full capture of each dominant kernel (tcgen05 conv-hist, lag moments, tcgen05 hidden-layer
#      conv) and of the
#      HBM-bound window sums (rect_sums).
# Usage: tools/profile_round.sh [workload]   -> gpurun_out/prof_round/
set -u
WL=${1:-caltech256}
OUT=gpurun_out/prof_round
mkdir -p $OUT
CMD="python bench.py --workload $WL --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > $OUT/plain.json 2> $OUT/plain.err || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"ddcca|lag_|conv|solve|whiten|finalize|gram_kernel|eig2|finish|taps_prep|zone_reduce|assemble|rect_sums|batch_epilogue|tree_level|hist|sym_eig|iq_" \
    --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
# tensor-core conv launches of one step: 6 in the fit (responses mode, layer 1), then 6 in the
# transform (histogram mode)
ncu --set full --import-source on --clock-control none -k regex:"conv_hist_tc_kernel" -s 8 -c 1 \
    -o $OUT/conv_hist $CMD > $OUT/ncu_full1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"lag_tma_kernel" -s 4 -c 1 \
    -o $OUT/lag_tma $CMD > $OUT/ncu_full2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"conv_hist_tc_kernel" -s 2 -c 1 \
    -o $OUT/conv_resp $CMD > $OUT/ncu_full3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"rect_sums_kernel" -s 1 -c 1 \
    -o $OUT/rect_sums $CMD > $OUT/ncu_full4.log 2>&1
echo "profile rc=$?"
