#!/bin/bash
# chained window: stage-1 stream counts (rescale stream, 4 late streams beside stage 3)
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for nmm in 2 4 8 2 4; do
  echo "=== mm streams $nmm"
  CHAIN_MM_STREAMS=$nmm timeout 300 python scripts/chain_stages.py 2>&1 | grep -v "^\[bench\]" | grep "end\|joined\|relu proved\|W\[2"
done
