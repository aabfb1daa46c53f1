#!/bin/bash
# e2e uploads on two streams; product-rate variants; source-level ncu of the dominant kernel
set -u
OUT=gpurun_out/r3a; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/fr64_bench scripts/fr64_bench.cu && /tmp/fr64_bench > $OUT/fr64_rates.txt 2>&1; cat $OUT/fr64_rates.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "e2e or fcn_tiny" > $OUT/t.txt 2>&1; echo "tests exit=$?"; tail -3 $OUT/t.txt
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.log; echo "bench exit=$?"; tail -2 $OUT/bench.log
python -c "
import json
d = json.load(open('$OUT/bench.json'))
print('C4', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'])"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_relu_iround_f --launch-skip 2 --launch-count 1 -o $OUT/iround1 -f python bench.py --steps 1 --warmup 1 --profile-mode --no-cpu-baseline --no-c5 --no-chained --streams 1 > $OUT/ncu.log 2>&1; echo "ncu exit=$?"
