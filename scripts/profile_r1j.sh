#!/bin/bash
# Round-1 final ncu evidence (under gpurun, ONE GPU): C4 launch list + full sets of the top zkReLU kernels,
# C5 (m = 26) launch list + full sets of the integer round 0 and the factored round kernel.
set -u
OUT=gpurun_out; mkdir -p $OUT
bash scripts/profile.sh r1j "k_relu_iround_f k_relu_gram" > $OUT/profile_r1j.log 2>&1
C5="python bench.py --config C5 --c5-log 26 --steps 1 --warmup 1 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_r1j_c5.csv $C5 > $OUT/ncu_launches_r1j_c5.log 2>&1
echo "c5 launch list exit=$?"
for K in k_sc_round0_int k_sc_round2f; do
  ncu --set full --clock-control none --import-source on -k regex:"^$K" -s 0 -c 1 -o $OUT/prof_r1j_c5_$K -f $C5 > $OUT/ncu_full_r1j_c5_$K.log 2>&1
  echo "full c5 $K exit=$?"
  python scripts/ncu_summary.py $OUT/prof_r1j_c5_$K.ncu-rep > $OUT/ncu_prof_r1j_c5_$K.txt 2>&1
done
ncu --set full --clock-control none -k regex:"^k_sc_round2f" -s 1 -c 1 -o $OUT/prof_r1j_c5_round1 -f $C5 > /dev/null 2>&1
python scripts/ncu_summary.py $OUT/prof_r1j_c5_round1.ncu-rep > $OUT/ncu_prof_r1j_c5_k_sc_round2f_mode3.txt 2>&1
rm -f $OUT/*.ncu-rep
ls -la $OUT | tail -30
