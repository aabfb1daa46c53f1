#!/bin/bash
set -u
OUT=gpurun_out/r3j; mkdir -p $OUT
python bench.py --no-cpu-baseline --no-c5 --no-chained > $OUT/bench.json 2>$OUT/bench.log
python -c "
import json; d=json.load(open('$OUT/bench.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'])
print({k: v for k, v in d['kernels_ms_per_step'].items() if 'colsum' in k or 'rowdot' in k or 'ct_' in k})"
ZKDL_COLSUM_TC=0 python bench.py --no-cpu-baseline --no-c5 --no-chained --steps 3 > $OUT/bench_off.json 2>/dev/null
python -c "
import json; d=json.load(open('$OUT/bench_off.json')); print('TC off', d['value'], d['ms_per_step'], {k: v for k, v in d['kernels_ms_per_step'].items() if 'colsum' in k})"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_colsum_tma --csv python bench.py --steps 1 --warmup 1 --profile-mode --no-cpu-baseline --no-c5 --no-chained --streams 1 > $OUT/ncu_colsum.csv 2>/dev/null; echo ncu=$?
grep -E "k_colsum_tma" $OUT/ncu_colsum.csv | head -30 | awk -F'","' '{print \$5, \$(NF-2), \$NF}' | head -30
