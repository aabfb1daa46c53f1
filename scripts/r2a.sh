#!/bin/bash
# Round 2, first GPU call: host facts, the new/changed GPU tests, the C5 sweep on one GPU, sanitizer.
set -u
OUT=gpurun_out/r2a; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
(nproc; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; lscpu | head -20) > $OUT/host.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_toggles.py tests/test_gpu_parity.py -m gpu -x -q -k "restriction_paths or rowdot or c5_large" > $OUT/tests_new.txt 2>&1; echo "new tests exit=$?"; tail -3 $OUT/tests_new.txt
for M in 22 24 26 28 30; do
  timeout 400 python bench.py --config C5 --c5-log $M > $OUT/c5_m$M.json 2> $OUT/c5_m$M.log; echo "c5 m=$M exit=$?"
done
for T in racecheck synccheck memcheck; do
  timeout 600 compute-sanitizer --tool $T --print-limit 20 python scripts/sanitize_small.py > $OUT/sanitizer_$T.txt 2>&1; echo "sanitizer $T exit=$?"; tail -3 $OUT/sanitizer_$T.txt
done
