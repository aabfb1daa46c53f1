#!/bin/bash
# A/B of compile-time i-round settings on the C4-sized zkReLU proof (kbench: per-kernel times + proof digest)
# bash scripts/ab_iround.sh TAG "DEFS1" "DEFS2" ...   (each DEFS a space-separated NAME=VALUE list; "" = default)
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
i=0
for DEFS in "$@"; do
  rm -f build/obj/relu.o paper_2307_16273_b200/libzkdl.so
  ZKDL_DEFS="$DEFS" python -c "from paper_2307_16273_b200 import build; build.build(verbose=False)" || { echo "build failed: $DEFS"; continue; }
  timeout 300 python scripts/kbench.py --logD 23 --m --reps 5 > $OUT/v$i.json 2> $OUT/v$i.log
  python - "$DEFS" $OUT/v$i.json <<'PY'
import json, sys
d = json.load(open(sys.argv[2]))["relu_logD23"]
k = {n: v for n, v in d["kernels_ms"].items() if "iround" in n or "gram" in n or "persist" in n}
print(f"[{sys.argv[1]}] relu {d['ms']} ms digest {d['digest']} {k}")
PY
  i=$((i+1))
done
rm -f build/obj/relu.o paper_2307_16273_b200/libzkdl.so
