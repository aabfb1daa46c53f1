#!/bin/bash
# chained window vs the product-sumcheck body switch and the derived-X=1 i-rounds
set -u
for DEFS in "ZKDL_SC_MULW=1" "ZKDL_SC_MULW=3"; do
  rm -f build/obj/sumcheck.o paper_2307_16273_b200/libzkdl.so
  ZKDL_DEFS="$DEFS" python -c "from paper_2307_16273_b200 import build; build.build(verbose=False)"
  for V in 1 0; do
    ZKDL_IR_DERIVE=$V python bench.py --no-cpu-baseline --no-c5 --steps 5 > /tmp/b.json 2>/dev/null
    python -c "
import json; d=json.load(open('/tmp/b.json')); print('[$DEFS] derive $V', round(d['ms_per_step'],3), 'chained', d['n3_chained_window']['ms_per_step'])"
  done
done
rm -f build/obj/sumcheck.o paper_2307_16273_b200/libzkdl.so
