#!/bin/bash
# Gram kernel variants (timing + the relu parity tests for the default)
for v in "GR_SELFGATE=1" "GR_SELFGATE=0"; do
  rm -rf build/obj; ZKDL_DEFS="$v" python -c "from paper_2307_16273_b200 import build; build.build(force=True, verbose=False)"
  timeout 600 python bench.py --no-cpu-baseline --no-c5 --no-chained > gpurun_out/h.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/h.json')); k=d['kernels_ms_per_step']; print('$v C4', d['ms_per_step'], 'gram', k.get('k_relu_gram'))"
done
rm -rf build/obj; python -c "from paper_2307_16273_b200 import build; build.build(force=True, verbose=False)"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "relu or c2 or fcn" 2>&1 | tail -2
