#!/bin/bash
# Round-1 final measurement (under gpurun, ONE GPU): the default bench line, the C5 line, the sweep,
# then the ncu launch lists and full sets of the top kernels (C4 and C5).
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python bench.py > $OUT/r1j_bench.json 2> $OUT/r1j_bench.log; echo "bench exit=$?"
timeout 300 python bench.py --config C5 --c5-log 26 > $OUT/r1j_c5.json 2> $OUT/r1j_c5.log; echo "c5 exit=$?"
bash scripts/profile_r1j.sh > $OUT/profile_r1j_all.log 2>&1; echo "profiles exit=$?"
ls -la $OUT | tail -30
