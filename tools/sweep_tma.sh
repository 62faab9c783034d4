for cfg in ${SWEEP_CFGS:-"3 96" "4 96" "6 96" "4 48" "6 48" "8 48" "2 192" "3 144"}; do
set -- $cfg
DDCCA_TMA_STAGES=$1 DDCCA_TMA_ROWS=$2 python bench.py --workload caltech256 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sw.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/sw.json')); k=d['kernels']
print('ns=$1 rows=$2', round(k['moments_l1']['ms_per_step'],2), round(k['moments_l2']['ms_per_step'],2))"
done
