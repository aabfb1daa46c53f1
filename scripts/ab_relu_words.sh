#!/bin/bash
# A/B of the zkReLU word-sourced rounds 0/1 (ZKDL_RELU_WORDS) in the C4 bench (under gpurun)
for w in 1 0 1 0; do
  ZKDL_RELU_WORDS=$w timeout 300 python bench.py --no-c5 --no-cpu-baseline --steps 10 2>/dev/null | tail -1 | W=$w python -c "
import json, os, sys
d = json.loads(sys.stdin.read()); k = d['kernels_ms_per_step']
print('words', os.environ['W'], round(d['ms_per_step'], 3), round(d['e2e']['value'] * 16e3, 3), {x: k[x] for x in k if 'relu' in x})"
done
