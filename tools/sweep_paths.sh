#!/bin/bash
# Bench every kernel family of the in-tree library on the three workloads.
# usage: tools/sweep_paths.sh TAG [paths...]   (3 = warp-tile, 2 = tcgen05, 1 = generic)
TAG=${1:-paths}; shift
PATHS=${@:-3 2}
mkdir -p gpurun_out
for p in $PATHS; do
  for w in c2 c3 full; do
    steps=200; [ $w = c3 ] && steps=20
    NMQ_KERNEL_PATH=$p timeout 300 python bench.py --workload $w --steps $steps --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "
import json,sys
t=sys.stdin.read().strip().splitlines()
try:
    d=json.loads(t[-1]); print('path$p $w', '%.3f Gq/s'%(d['value']/1e9), 'ms %.4f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], d['clocks']['sm_mhz'])
except Exception: print('path$p $w FAILED', t[-3:])" | tee -a gpurun_out/${TAG}_results.txt
  done
done
