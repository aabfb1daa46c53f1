#!/bin/bash
set -u
OUT=gpurun_out/r2j; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "e2e_int16 or fcn_tiny or async" > $OUT/t.txt 2>&1; echo "tests exit=$?"; tail -3 $OUT/t.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.log; echo "bench exit=$?"; tail -2 $OUT/bench.log
python -c "
import json
d = json.load(open('$OUT/bench.json'))
print('C4', d['value'], d['ms_per_step'], 'e2e', d['e2e'], 'frac', d['roofline']['frac'], d['roofline'].get('frac_of_measured_product_rate'))
print('chained', d['n3_chained_window']['ms_per_step'], 'c5', d.get('c5_sharded',{}).get('ms_per_proof'))
print('cpu', json.dumps(d.get('cpu_baseline'))[:1200])"
