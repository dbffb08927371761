#!/bin/bash
# K2/K3 grid-sizing sweep on the bench's own tail roofline (tools/tail_sweep.sh <workload>)
W=${1:-domain}
for b in 2 4 8 16; do
  MPB_LAYOUT_BLOCKS_PER_SM=$b python bench.py --workload $W --steps 5 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('blocks_per_sm=$b', round(d['ms_per_step'],4), 'ms/step', {k[:22]: round(v['us_per_launch'],1) for k,v in r['tail'].items()})"
done
