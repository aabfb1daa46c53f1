#!/bin/bash
# serial kernel tables with the fused zkReLU claim MLEs on / off (under gpurun)
for f in 1 0; do
  ZKDL_MLE4_FUSED=$f timeout 120 python bench.py --no-c5 --no-cpu-baseline --steps 5 --streams 1 --mm-streams 1 > gpurun_out/m$f.json 2> gpurun_out/m$f.log
  F=$f python -c "
import json, os
d = json.load(open('gpurun_out/m' + os.environ['F'] + '.json')); k = d['kernels_ms_per_step']
print('fused', os.environ['F'], round(d['ms_per_step'], 3), {x: k[x] for x in k if 'mle4' in x or 'rowdot_i32' in x or 'dot_fr' in x})"
done
