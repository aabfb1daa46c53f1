#!/bin/bash
set -u
OUT=gpurun_out/r2i; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
for P in 1 0; do
  timeout 600 python bench.py --no-cpu-baseline --no-c5 --no-chained --pipeline $P > $OUT/c4_p$P.json 2> $OUT/c4_p$P.log; echo "pipe $P exit=$?"
  python -c "
import json
d = json.load(open('$OUT/c4_p$P.json'))
print('pipeline $P: C4 ms', round(d['ms_per_step'],3), 'value', d['value'], 'frac', d['roofline']['frac'], d['roofline'].get('frac_of_measured_product_rate'), 'e2e', d['e2e']['value'], 'launches', d['gpu_launches'])"
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fcn or async" > $OUT/fcn.txt 2>&1; echo "fcn tests exit=$?"; tail -2 $OUT/fcn.txt
