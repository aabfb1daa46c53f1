#!/bin/bash
# Round 2: the claim-chained window on the GPU (tiny / mid / full size), the changed verifier call sites.
set -u
OUT=gpurun_out/r2b; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_chain.py -x -q -k "tiny or mid" > $OUT/chain_small.txt 2>&1; echo "chain small exit=$?"; tail -30 $OUT/chain_small.txt
timeout 1500 python -m pytest tests/test_gpu_chain.py -x -q -k "full" --durations=5 > $OUT/chain_full.txt 2>&1; echo "chain full exit=$?"; tail -30 $OUT/chain_full.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "readme or window_full" > $OUT/parity_changed.txt 2>&1; echo "parity exit=$?"; tail -5 $OUT/parity_changed.txt
