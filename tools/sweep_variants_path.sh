#!/bin/bash
# Bench library variants (tools/variants/) with one kernel family forced.
# usage: tools/sweep_variants_path.sh TAG PATH [workloads]
TAG=$1; P=$2; shift 2; WLS=${@:-c2 c3 full}
mkdir -p gpurun_out
for lib in tools/variants/libnmq_*.so; do
  n=$(basename $lib .so)
  for w in $WLS; do
    steps=200; [ $w = c3 ] && steps=20
    NMQ_KERNEL_PATH=$P NMQ_LIB=$PWD/$lib timeout 300 python bench.py --workload $w --steps $steps --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "
import json,sys
t=sys.stdin.read().strip().splitlines()
try:
    d=json.loads(t[-1]); print('$n p$P $w', '%.3f Gq/s'%(d['value']/1e9), 'ms %.4f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], d['clocks']['sm_mhz'])
except Exception: print('$n p$P $w FAILED', t[-3:])" | tee -a gpurun_out/${TAG}_results.txt
  done
done
