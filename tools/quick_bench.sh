#!/bin/bash
# quick bench summary lines: tools/quick_bench.sh "<bench args>" ...
for a in "$@"; do
  python bench.py $a --no-e2e --no-cpu-baseline 2>/tmp/qb.err | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$a', '|', d['config']['workload'], '%.1fM tok/s'%(d['value']/1e6), '%.4f ms/step'%d['ms_per_step'], 'graph', d['cuda_graph'], 'launches', d['gpu_launches'], 'router %.4f ms'%r['ms_per_launch'], 'frac %.3f'%r['frac'], 'share %.3f'%r['share_of_step'], d['clocks'], {k[:12]: round(v['us_per_launch'],1) for k,v in r.get('tail',{}).items()})" || tail -5 /tmp/qb.err
done
