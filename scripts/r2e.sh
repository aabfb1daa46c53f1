#!/bin/bash
# Claim merge at n = 0 / bits (the C3 rescale aux), the shard tests, then the zkReLU i-round CTA shape A/B.
set -u
OUT=gpurun_out/r2e; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_chain.py -x -q -k "claim_merge" > $OUT/cm.txt 2>&1; echo "cm exit=$?"; tail -20 $OUT/cm.txt
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "shard" > $OUT/shard.txt 2>&1; echo "shard exit=$?"; tail -3 $OUT/shard.txt
for CFG in "256 2" "128 3" "128 2"; do
  set -- $CFG
  ZKDL_DEFS="ZKDL_IR_LB_T=$1 ZKDL_IR_LB_B=$2" python -c "from paper_2307_16273_b200 import build; build.build(force=True)" > /dev/null 2>&1
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "relu_vs_oracle or c2_full or relu_round_paths" > $OUT/relu_$1_$2.txt 2>&1; echo "lb $1 $2 parity exit=$?"; tail -1 $OUT/relu_$1_$2.txt
  timeout 600 python bench.py --no-cpu-baseline --no-chained --no-c5 > $OUT/c4_$1_$2.json 2> $OUT/c4_$1_$2.log
  python -c "
import json
d = json.load(open('$OUT/c4_$1_$2.json'))
k = d['kernels_ms_per_step']
print('LB $1 $2: C4 ms', round(d['ms_per_step'],3), 'frac', d['roofline']['frac'], {x: k[x] for x in k if 'iround' in x})"
done
python -c "from paper_2307_16273_b200 import build; build.build(force=True)" > /dev/null 2>&1
