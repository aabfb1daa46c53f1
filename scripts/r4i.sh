#!/bin/bash
set -u
python -c "from paper_2307_16273_b200 import build; build.build(verbose=False)"
for S in 1 0; do for i in 1 2 3; do
  python bench.py --no-cpu-baseline --chain-serial $S > /tmp/b.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/b.json')); print('[serial $S run $i]', round(d['ms_per_step'],3), 'chained', d['n3_chained_window']['ms_per_step'])"
done; done
