#!/bin/bash
# window time vs the matmul streams' SM budget
for B in 12 20 28 37; do for S in 2 3; do
  python bench.py --no-cpu-baseline --no-c5 --no-chained --steps 5 --mm-budget $B --mm-streams $S > /tmp/b.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/b.json')); print('budget $B streams $S', round(d['ms_per_step'],3), 'frac', d['roofline']['frac'])"
done; done
