#!/bin/bash
set -u
OUT=gpurun_out/r2g; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests/test_gpu_chain.py -q -k "full" > $OUT/chain_full.txt 2>&1; echo "chain full exit=$?"; tail -5 $OUT/chain_full.txt
timeout 900 python bench.py --no-cpu-baseline --no-c5 > $OUT/bench.json 2> $OUT/bench.log; echo "bench exit=$?"; tail -2 $OUT/bench.log
python -c "
import json
d = json.load(open('$OUT/bench.json'))
print('C4', d['value'], d['ms_per_step'], d['roofline']['frac'])
print('chained', json.dumps(d.get('n3_chained_window'))[:900])"
timeout 600 ncu --set full --import-source on --clock-control none -k 'regex:iround_f<1>' --launch-skip 6 --launch-count 1 -o $OUT/iround1 python bench.py --steps 1 --warmup 1 --profile-mode --no-cpu-baseline --no-c5 --no-chained --streams 1 > $OUT/ncu_iround.log 2>&1; echo "ncu iround exit=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k 'regex:k_sc_all' --launch-skip 20 --launch-count 1 -o $OUT/scall python bench.py --steps 1 --warmup 1 --profile-mode --no-cpu-baseline --no-c5 --no-chained --streams 1 > $OUT/ncu_scall.log 2>&1; echo "ncu scall exit=$?"
