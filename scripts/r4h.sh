#!/bin/bash
set -u
python -c "from paper_2307_16273_b200 import build; build.build(verbose=False)"
timeout 900 python -m pytest tests/test_gpu_chain.py -x -q 2>&1 | tail -1
for i in 1 2 3 4; do
  python bench.py --no-cpu-baseline --no-c5 --steps 5 > /tmp/b.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/b.json')); print('[run $i]', round(d['ms_per_step'],3), 'chained', d['n3_chained_window']['ms_per_step'])"
done
