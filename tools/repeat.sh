#!/bin/bash
nvidia-smi --query-gpu=name,clocks.sm,clocks.mem,clocks.max.mem,power.draw,power.limit,temperature.gpu --format=csv
for i in 1 2 3; do
  for w in c2 full c3; do
    steps=200; [ $w = c3 ] && steps=20
    timeout 300 python bench.py --workload $w --steps $steps --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$i $w', '%.2f Gq/s'%(d['value']/1e9), 'ms/step %.4f'%d['ms_per_step'])"
  done
done
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu --format=csv
