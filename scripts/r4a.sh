#!/bin/bash
set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests/test_gpu_chain.py -x -q 2>&1 | tail -2
python bench.py --no-cpu-baseline --no-c5 --steps 3 > /tmp/b.json 2>/dev/null
python -c "
import json; d=json.load(open('/tmp/b.json')); c=d['n3_chained_window']; print('C4', round(d['ms_per_step'],3), 'chained', c['ms_per_step'], c['launches_one_window']); print(c['kernel_launches_one_window']); print(c['kernels_ms_one_window_serialised'])"
bash scripts/ab_c5.sh "" "ZKDL_SC_MULW=1"
