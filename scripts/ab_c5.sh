#!/bin/bash
# A/B of compile-time settings of the product-sumcheck kernels on C5 statements (kbench: ms + digests)
# bash scripts/ab_c5.sh "DEFS1" "DEFS2" ...
set -u
for DEFS in "$@"; do
  rm -f build/obj/sumcheck.o paper_2307_16273_b200/libzkdl.so
  ZKDL_DEFS="$DEFS" python -c "from paper_2307_16273_b200 import build; build.build(verbose=False)" || { echo "build failed: $DEFS"; continue; }
  timeout 300 python scripts/kbench.py --logD 0 --m 24 26 --reps 3 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin)
print('[$DEFS]', {k: (v['ms'], v['digest']) for k, v in d.items()})"
done
rm -f build/obj/sumcheck.o paper_2307_16273_b200/libzkdl.so
