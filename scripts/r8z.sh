#!/bin/bash
# closing run (round 2, session 3): full GPU suite, smoke, bench lines, C5 sweep, launch list, ncu of the dominant kernel
set -u
OUT=gpurun_out/${TAG:-r8z}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=5 > $OUT/gpu_tests.txt 2>&1; echo "tests exit=$?"; tail -2 $OUT/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke exit=$?"; tail -1 $OUT/smoke.txt
for i in 1 2; do timeout 900 python bench.py > $OUT/bench$i.json 2> $OUT/bench$i.log; echo "bench exit=$?"
python -c "
import json
d = json.load(open('$OUT/bench$i.json'))
print('C4', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], d['roofline'].get('frac_of_measured_product_rate'), d['clocks']['sm_mhz'], d['clocks']['reasons'])
print('chained', d['n3_chained_window']['ms_per_step'], 'c5', d.get('c5_sharded',{}).get('ms_per_proof'))"
done
for M in 22 26 30; do timeout 400 python bench.py --config C5 --c5-log $M > $OUT/c5_m$M.json 2> $OUT/c5_m$M.log; echo "c5 $M exit=$?"; done
P="python bench.py --steps 1 --warmup 1 --profile-mode --no-cpu-baseline --no-c5 --no-chained --streams 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $P > /dev/null 2>&1; echo "launch list exit=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_relu_iround_f --launch-skip 2 --launch-count 1 -o $OUT/iround2 -f $P > $OUT/ncu_i2.log 2>&1; echo "ncu exit=$?"
timeout 900 ncu --set full --clock-control none -k regex:k_relu_ipersist --launch-count 1 -o $OUT/ipersist -f $P > $OUT/ncu_ip.log 2>&1; echo "ncu ipersist exit=$?"
