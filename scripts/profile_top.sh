#!/bin/bash
# ncu --set full of selected kernels from one C4 window (under gpurun, ONE GPU).  bash scripts/profile_top.sh TAG 'k1 k2 ...'
TAG=${1:-r1}; KS=${2:-"k_relu_iround k_relu_bitsums2 k_sc_round"}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --profile-mode --no-cpu-baseline"
for K in $KS; do
  ncu --set full --clock-control none --import-source on -k regex:"^${K}" -s 0 -c 1 -o gpurun_out/prof_${TAG}_$K -f $CMD > gpurun_out/ncu_full_${TAG}_$K.log 2>&1
  echo "full $K exit=$?"
done
