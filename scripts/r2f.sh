#!/bin/bash
set -u
OUT=gpurun_out/r2f; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_chain.py -x -q -k "rescale" > $OUT/rescale.txt 2>&1; echo "rescale exit=$?"; tail -25 $OUT/rescale.txt
timeout 1500 python -m pytest tests/test_gpu_chain.py -q -k "full" > $OUT/chain_full.txt 2>&1; echo "chain full exit=$?"; tail -25 $OUT/chain_full.txt
timeout 900 python bench.py --no-cpu-baseline --no-c5 > $OUT/bench.json 2> $OUT/bench.log; echo "bench exit=$?"; tail -3 $OUT/bench.log
python -c "
import json
d = json.load(open('$OUT/bench.json'))
print('C4', d['value'], d['ms_per_step'], d['roofline']['frac'])
print('chained', json.dumps(d.get('n3_chained_window'))[:1500])"
