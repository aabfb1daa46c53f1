#!/bin/bash
# Round-1 closing ncu evidence (under gpurun, ONE GPU): the C4 launch list and full sets of the top kernels
# after the column-sum change, including the 512 MB column sum (5th k_colsum_i32 launch of the window).
set -u
OUT=gpurun_out; mkdir -p $OUT
CMD="python bench.py --steps 1 --warmup 1 --profile-mode --no-cpu-baseline --no-c5 --streams 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_r1k.csv $CMD > /dev/null 2>&1
echo "launch list exit=$?"
ncu --set full --clock-control none --import-source on -k regex:"^k_colsum" -s 4 -c 1 -o $OUT/prof_r1k_colsum -f $CMD > /dev/null 2>&1
python scripts/ncu_summary.py $OUT/prof_r1k_colsum.ncu-rep > $OUT/ncu_prof_r1k_k_colsum_i32_big.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"^k_rowdot_tc" -s 1 -c 1 -o $OUT/prof_r1k_rowdot -f $CMD > /dev/null 2>&1
python scripts/ncu_summary.py $OUT/prof_r1k_rowdot.ncu-rep > $OUT/ncu_prof_r1k_k_rowdot_tc_big.txt 2>&1
rm -f $OUT/*.ncu-rep
