#!/bin/bash
# A/B of the hot product bodies: FP64-pipe product (ZKDL_FR64=1) against the integer CIOS (=0).
set -u
OUT=gpurun_out/r2c; mkdir -p $OUT
for V in 1 0; do
  ZKDL_FR64=$V python -c "from paper_2307_16273_b200 import build; build.build(force=True)" > $OUT/build_$V.txt 2>&1
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sumcheck_vs_oracle or relu_vs_oracle or c5_vs_oracle or c2_full or fcn_tiny" > $OUT/parity_$V.txt 2>&1; echo "fr64=$V parity exit=$?"; tail -1 $OUT/parity_$V.txt
  timeout 600 python bench.py --no-cpu-baseline --no-chained > $OUT/c4_$V.json 2> $OUT/c4_$V.log; echo "c4 exit=$?"
  timeout 300 python bench.py --config C5 --c5-log 26 --no-cpu-baseline > $OUT/c5_$V.json 2> $OUT/c5_$V.log; echo "c5 exit=$?"
  python -c "
import json
d = json.load(open('$OUT/c4_$V.json')); c = json.load(open('$OUT/c5_$V.json'))
print('FR64=$V C4 ms', round(d['ms_per_step'],3), 'dom', d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'])
print('   kernels', {k: v for k, v in list(d['kernels_ms_per_step'].items())[:6]})
print('FR64=$V C5 ms', round(c['ms_per_step'],3), c['roofline']['achieved'], c['roofline']['frac'])"
done
ZKDL_FR64=1 python -c "from paper_2307_16273_b200 import build; build.build(force=True)" > /dev/null 2>&1
