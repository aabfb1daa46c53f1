#!/bin/bash
# i-round fold rounds: L1 prefetch of the next pair (ZKDL_IR_PF) A/B
for v in "ZKDL_IR_PF=1" "ZKDL_IR_PF=0"; do
  rm -rf build/obj; ZKDL_DEFS="$v" python -c "from paper_2307_16273_b200 import build; build.build(force=True, verbose=False)"
  timeout 600 python bench.py --no-cpu-baseline --no-c5 --no-chained > gpurun_out/v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/v.json')); k=d['kernels_ms_per_step']; print('$v', round(d['ms_per_step'],3), 'i5', k.get('k_relu_iround_f<5>'), 'i7', k.get('k_relu_iround_f<7>'), 'frac', d['roofline']['frac'])"
done
