#!/bin/bash
# ncu evidence for one C4 window (run under gpurun, ONE GPU).  Outputs land in gpurun_out/.
#   bash scripts/profile.sh [tag] [kernels...]
# The bench runs with --streams 1 under ncu (ncu serialises kernels anyway).
set -u
TAG=${1:-r1}
shift || true
KS=${*:-"k_relu_iround k_relu_gram k_sc_all k_colsum_i32 k_rowdot_i32"}
OUT=gpurun_out
mkdir -p $OUT
CMD="python bench.py --steps 1 --warmup 1 --profile-mode --no-cpu-baseline --streams 1"
# 1) every launch with its device time (cold-cache, serialised: compare shares, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launches_$TAG.log 2>&1
echo "launch list exit=$?"
# 2) full sets of the top kernels (first launch of each)
for K in $KS; do
  ncu --set full --clock-control none --import-source on -k regex:"^$K" -s 0 -c 1 -o $OUT/prof_${TAG}_$K -f $CMD > $OUT/ncu_full_${TAG}_$K.log 2>&1
  echo "full $K exit=$?"
  python scripts/ncu_summary.py $OUT/prof_${TAG}_$K.ncu-rep > $OUT/ncu_prof_${TAG}_$K.txt 2>&1
done
ls -la $OUT
