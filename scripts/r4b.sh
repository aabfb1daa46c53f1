#!/bin/bash
# chained window: the batched claim-merge eq tables (current) against the per-claim version (abtmp/)
set -u
run() { python bench.py --no-cpu-baseline --no-c5 --steps 5 > /tmp/b.json 2>/dev/null; python -c "
import json; d=json.load(open('/tmp/b.json')); c=d['n3_chained_window']; print('$1', 'C4', round(d['ms_per_step'],3), 'chained', c['ms_per_step'], c['launches_one_window'])"; }
python -c "from paper_2307_16273_b200 import build; build.build(verbose=False)"
run new; run new
cp paper_2307_16273_b200/csrc/chain.cu /tmp/chain_new.cu; cp paper_2307_16273_b200/csrc/tables.cu /tmp/tables_new.cu
cp abtmp/chain.cu abtmp/tables.cu paper_2307_16273_b200/csrc/
python -c "from paper_2307_16273_b200 import build; build.build(verbose=False)"
run old; run old
cp /tmp/chain_new.cu paper_2307_16273_b200/csrc/chain.cu; cp /tmp/tables_new.cu paper_2307_16273_b200/csrc/tables.cu
