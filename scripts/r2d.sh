#!/bin/bash
# Round 2: chained window with the top layer (loss + rescale) on the GPU, then the bench line.
set -u
OUT=gpurun_out/r2d; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_chain.py -x -q -k "tiny or mid or rescale" > $OUT/chain_small.txt 2>&1; echo "chain small exit=$?"; tail -30 $OUT/chain_small.txt
timeout 1500 python -m pytest tests/test_gpu_chain.py -x -q -k "full" > $OUT/chain_full.txt 2>&1; echo "chain full exit=$?"; tail -30 $OUT/chain_full.txt
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "shard" > $OUT/shard.txt 2>&1; echo "shard exit=$?"; tail -3 $OUT/shard.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.log; echo "bench exit=$?"; tail -3 $OUT/bench.log
python -c "
import json
d = json.load(open('$OUT/bench.json'))
print('C4', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'])
print('chained', d.get('n3_chained_window'))
print('cpu', json.dumps(d.get('cpu_baseline'))[:800])"
