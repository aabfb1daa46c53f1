#!/bin/bash
set -u
python -c "from paper_2307_16273_b200 import build; build.build(verbose=False)"
for MS in 8 4 2; do for MB in 148 64; do
  python bench.py --no-cpu-baseline --no-c5 --steps 5 --merge-streams $MS --merge-budget $MB > /tmp/b.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/b.json')); print('[merge streams $MS budget $MB]', round(d['ms_per_step'],3), 'chained', d['n3_chained_window']['ms_per_step'])"
done; done
