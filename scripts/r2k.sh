#!/bin/bash
set -u
OUT=gpurun_out/r2k; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "rowdot" > $OUT/rowdot.txt 2>&1; echo "rowdot exit=$?"; tail -15 $OUT/rowdot.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_toggles.py -x -q -k "matmul_vs_oracle or restriction or window_full or c1_golden or readme" > $OUT/mm.txt 2>&1; echo "mm exit=$?"; tail -3 $OUT/mm.txt
for T in 1 0; do
  ZKDL_ROWDOT_TMA=$T timeout 600 python bench.py --no-cpu-baseline --no-c5 --no-chained > $OUT/c4_tma$T.json 2> $OUT/c4_tma$T.log
  python -c "
import json
d = json.load(open('$OUT/c4_tma$T.json'))
k = d['kernels_ms_per_step']
print('TMA=$T C4 ms', round(d['ms_per_step'],3), {x: k[x] for x in k if 'rowdot' in x or 'colsum' in x})"
done
timeout 600 ncu --set full --clock-control none -k k_rowdot_tma --launch-skip 8 --launch-count 1 -o $OUT/tma python bench.py --steps 1 --warmup 1 --profile-mode --no-cpu-baseline --no-c5 --no-chained --streams 1 > $OUT/ncu_tma.log 2>&1; echo "ncu exit=$?"
