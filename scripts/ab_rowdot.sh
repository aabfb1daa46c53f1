#!/bin/bash
# serial kernel tables (no stream overlap) for the tensor-core row dots (under gpurun)
for i in 1 2; do
  timeout 120 python bench.py --no-c5 --no-cpu-baseline --steps 5 --streams 1 --mm-streams 1 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read()); k = d['kernels_ms_per_step']
print(round(d['ms_per_step'], 3), {x: k[x] for x in k if 'rowdot' in x or 'colsum' in x})"
done
