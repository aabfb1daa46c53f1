#!/bin/bash
set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_toggles.py -x -q -k "relu" 2>&1 | tail -3
for V in 0 1; do ZKDL_IR_DERIVE=$V timeout 300 python scripts/kbench.py --logD 23 --m --reps 3 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin)['relu_logD23']; print('derive $V', d['ms'], d['digest'], {k:v for k,v in d['kernels_ms'].items() if 'iround' in k or 'jround' in k or 'uinv' in k})"; done
