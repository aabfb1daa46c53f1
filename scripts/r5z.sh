#!/bin/bash
# closing run (round 2, session 3): full GPU suite, smoke, bench lines, C5 sweep, launch list and ncu capture
set -u
OUT=gpurun_out/${TAG:-r5z}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > $OUT/gpu_tests.txt 2>&1; echo "tests exit=$?"; tail -3 $OUT/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke exit=$?"; tail -1 $OUT/smoke.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.log; echo "bench exit=$?"
for M in 22 24 26 28 30; do timeout 400 python bench.py --config C5 --c5-log $M > $OUT/c5_m$M.json 2> $OUT/c5_m$M.log; echo "c5 $M exit=$?"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 1 --profile-mode --no-cpu-baseline --no-c5 --no-chained --streams 1 > /dev/null 2>&1; echo "launch list exit=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_relu_iround_f --launch-skip 2 --launch-count 1 -o $OUT/iround1 -f python bench.py --steps 1 --warmup 1 --profile-mode --no-cpu-baseline --no-c5 --no-chained --streams 1 > $OUT/ncu_iround.log 2>&1; echo "ncu iround exit=$?"
python -c "
import json
d = json.load(open('$OUT/bench.json'))
print('C4', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], d['roofline'].get('frac_of_measured_product_rate'), d['clocks'])
print('chained', d['n3_chained_window']['ms_per_step'], 'c5', d.get('c5_sharded',{}).get('ms_per_proof'))
for M in (22, 24, 26, 28, 30):
    c = json.load(open('$OUT/c5_m%d.json' % M)); print('C5', M, c['ms_per_step'], c['roofline']['frac'])"
