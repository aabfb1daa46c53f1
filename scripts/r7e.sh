#!/bin/bash
# window vs the restriction kernels' tensor-core (TMEM, large smem) paths beside the zkReLU's one-wave Gram
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for E in "X=1" "ZKDL_ROWDOT_TC=0 ZKDL_COLSUM_TC=0" "ZKDL_COLSUM_TC=0" "ZKDL_ROWDOT_TC=0" "X=1"; do
  env $E timeout 600 python bench.py --no-cpu-baseline --no-c5 --no-chained > gpurun_out/p.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/p.json')); k=d['kernels_ms_per_step']; print('$E:', round(d['ms_per_step'],3))"
done
