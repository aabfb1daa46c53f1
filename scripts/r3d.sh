#!/bin/bash
# parity suite + bench after the k_sc_all / transcript latency changes
set -u
OUT=gpurun_out/r3d; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.txt 2>&1; echo "tests exit=$?"; tail -3 $OUT/gpu_tests.txt
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.log; echo "bench exit=$?"; tail -2 $OUT/bench.log
python -c "
import json
d = json.load(open('$OUT/bench.json'))
print('C4', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'])
print('chained', d['n3_chained_window']['ms_per_step'], 'c5', d.get('c5_sharded',{}).get('ms_per_proof'))
print({k: v for k, v in d['kernels_ms_per_step'].items()})
print('chain kernels', d['n3_chained_window'].get('kernels_ms_one_window_serialised'))"
