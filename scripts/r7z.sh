#!/bin/bash
# evidence for the round-2 (session 3) state: launch list, ncu of the Gram kernel, the cell-sourced round 0 and
# the dominant fold round, the C5 sweep
set -u
OUT=gpurun_out/${TAG:-r7z}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.txt 2>&1
for M in 22 24 26 28 30; do timeout 400 python bench.py --config C5 --c5-log $M > $OUT/c5_m$M.json 2> $OUT/c5_m$M.log; echo "c5 $M exit=$?"; done
P="python bench.py --steps 1 --warmup 1 --profile-mode --no-cpu-baseline --no-c5 --no-chained --streams 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $P > /dev/null 2>&1; echo "launch list exit=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_relu_gram$ --launch-count 1 -o $OUT/gram -f $P > $OUT/ncu_gram.log 2>&1; echo "ncu gram exit=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_relu_iround_f --launch-count 1 -o $OUT/iround0 -f $P > $OUT/ncu_i0.log 2>&1; echo "ncu round0 exit=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_relu_iround_f --launch-skip 2 --launch-count 1 -o $OUT/iround2 -f $P > $OUT/ncu_i2.log 2>&1; echo "ncu round2 exit=$?"
