#!/bin/bash
# Round-1 closing run (under gpurun, ONE GPU): full GPU suite, smoke, bench lines, C4 launch list.
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/final_gpu_tests.txt 2>&1; echo "tests exit=$?"; tail -1 $OUT/final_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/final_smoke.txt 2>&1; echo "smoke exit=$?"; tail -1 $OUT/final_smoke.txt
timeout 600 python bench.py > $OUT/r1m_bench.json 2> $OUT/r1m_bench.log; echo "bench exit=$?"
timeout 300 python bench.py --config C5 --c5-log 26 > $OUT/r1m_c5.json 2>/dev/null; echo "c5 exit=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_r1m.csv python bench.py --steps 1 --warmup 1 --profile-mode --no-cpu-baseline --no-c5 --streams 1 > /dev/null 2>&1; echo "launch list exit=$?"
python -c "
import json
d = json.load(open('$OUT/r1m_bench.json')); c = json.load(open('$OUT/r1m_c5.json'))
print('C4', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'])
print('C5', c['ms_per_step'], c['roofline']['achieved'], c['roofline']['frac'])"
