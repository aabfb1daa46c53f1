#!/bin/bash
# chained-window stage layouts (scripts/chain_stages.py)
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for cfg in "1 4 0" "1 4 1" "0 4 1" "1 0 0" "0 0 0"; do
  set -- $cfg
  echo "=== rescale stream $1, late streams $2, after relu $3"
  CHAIN_RESCALE_STREAM=$1 CHAIN_LATE_STREAMS=$2 CHAIN_LATE_AFTER=$3 timeout 300 python scripts/chain_stages.py 2>&1 | grep -v "^\[bench\]" | tail -28
done
