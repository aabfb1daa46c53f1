#!/bin/bash
# the Gram kernel's grid (ZKDL_GRAM_WAVES) in the window and alone
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for W in 1 2 3 1 2; do
  ZKDL_GRAM_WAVES=$W timeout 600 python bench.py --no-cpu-baseline --no-c5 --no-chained > gpurun_out/p.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/p.json')); k=d['kernels_ms_per_step']; print('waves=$W', round(d['ms_per_step'],3), 'gram(serial pass)', k.get('k_relu_gram'))"
done
