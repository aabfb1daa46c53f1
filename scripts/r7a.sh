#!/bin/bash
# D3d window: the matmul families' persistent sumcheck footprint beside the zkReLU
python -c "import __graft_entry__ as g; g.build()" > /dev/null
run() {
  env $1 timeout 600 python bench.py --no-cpu-baseline --no-c5 --no-chained $2 > gpurun_out/v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/v.json')); k=d['kernels_ms_per_step']; print('$1 $2:', round(d['ms_per_step'],3), 'sc_all', k.get('k_sc_all'), 'i5', k.get('k_relu_iround_f<5>'), 'gram', k.get('k_relu_gram'))"
}
run "X=1" ""
run "ZKDL_SCALL_T=128" ""
run "ZKDL_SCALL_T=128" "--mm-budget 18"
run "X=1" "--mm-budget 12"
run "ZKDL_SCALL_T=128" "--mm-streams 4 --mm-budget 37"
run "X=1" "--relu-priority 0"
