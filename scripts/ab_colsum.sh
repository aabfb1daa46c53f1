#!/bin/bash
# serial kernel tables (no stream overlap) for the column sums: rows path on / off (under gpurun)
for r in 1 0 1; do
  ZKDL_COLSUM_ROWS=$r timeout 120 python bench.py --no-c5 --no-cpu-baseline --steps 5 --streams 1 --mm-streams 1 2>/dev/null | R=$r python -c "
import json, os, sys
d = json.loads(sys.stdin.read()); k = d['kernels_ms_per_step']
print('rows', os.environ['R'], round(d['ms_per_step'], 3), {x: k[x] for x in k if 'colsum' in x})"
done
