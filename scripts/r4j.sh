#!/bin/bash
set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_toggles.py -x -q -k "c5 or sumcheck or matmul or fcn_window or rescale or merge" 2>&1 | tail -2
for V in 1 0; do ZKDL_SC_DERIVE=$V timeout 300 python scripts/kbench.py --logD 0 --m 24 26 --reps 3 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print('derive $V', {k: (v['ms'], v['digest'], {n: t for n, t in v['kernels_ms'].items() if 'round2f' in n or 'inv' in n}) for k, v in d.items()})"; done
