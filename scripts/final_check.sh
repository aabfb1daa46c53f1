#!/bin/bash
# Full GPU suite, smoke, and the bench lines (under gpurun, ONE GPU)
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/final_gpu_tests.txt 2>&1; echo "tests exit=$?"; tail -3 $OUT/final_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/final_smoke.txt 2>&1; echo "smoke exit=$?"; tail -2 $OUT/final_smoke.txt
timeout 600 python bench.py > $OUT/r1k_bench.json 2> $OUT/r1k_bench.log; echo "bench exit=$?"
python scripts/kt.py relu colsum rowdot sc_all < $OUT/r1k_bench.json
timeout 300 python bench.py --config C5 --c5-log 26 > $OUT/r1k_c5.json 2>/dev/null; echo "c5 exit=$?"
python scripts/kt.py sc_ < $OUT/r1k_c5.json
