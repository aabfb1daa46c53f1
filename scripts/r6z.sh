#!/bin/bash
# full GPU suite, smoke, two bench lines
set -u
OUT=gpurun_out/${TAG:-r6z}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=5 > $OUT/gpu_tests.txt 2>&1; echo "tests exit=$?"; tail -3 $OUT/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke exit=$?"; tail -1 $OUT/smoke.txt
for i in 1 2; do timeout 900 python bench.py > $OUT/bench$i.json 2> $OUT/bench$i.log; echo "bench exit=$?"
python -c "
import json
d = json.load(open('$OUT/bench$i.json'))
print('C4', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], d['roofline'].get('frac_of_measured_product_rate'), d['clocks']['sm_mhz'], d['clocks']['reasons'])
print('chained', d['n3_chained_window']['ms_per_step'], 'c5', d.get('c5_sharded',{}).get('ms_per_proof'))"
done
