#!/bin/bash
# where the zkReLU hands its rounds to the persistent kernel (ZKDL_IPERSIST_LOG: rounds with <= 2^L pairs)
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for L in 16 15 14 17 16; do
  ZKDL_IPERSIST_LOG=$L timeout 600 python bench.py --no-cpu-baseline --no-c5 --no-chained > gpurun_out/p.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/p.json')); k=d['kernels_ms_per_step']; print('L=$L', round(d['ms_per_step'],3), 'ipersist', k.get('k_relu_ipersist'), 'i5', k.get('k_relu_iround_f<5>'))"
done
