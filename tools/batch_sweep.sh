#!/bin/bash
for m in 1 2 4 8; do
  NMQ_BATCH_MULT=$m timeout 300 python bench.py --steps 40 --sets 2 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('mult $m', '%.2f Gq/s'%(d['value']/1e9), 'ms %.4f'%d['ms_per_step'])"
done
