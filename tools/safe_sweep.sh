#!/bin/bash
# Hang-check every variant (tools/hang_probe.py, 5 s watchdog per launch),
# then bench the ones that pass.  usage: tools/safe_sweep.sh TAG PATH
TAG=$1; P=$2
mkdir -p gpurun_out
for lib in tools/variants/libnmq_*.so; do
  n=$(basename $lib .so)
  if NMQ_LIB=$PWD/$lib NMQ_KERNEL_PATH=$P timeout 120 python tools/hang_probe.py 132736 300000 2100000 > gpurun_out/${TAG}_${n}_probe.txt 2>&1; then
    for w in c2 c3 full; do
      steps=200; [ $w = c3 ] && steps=20
      NMQ_KERNEL_PATH=$P NMQ_LIB=$PWD/$lib timeout 120 python bench.py --workload $w --steps $steps --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "
import json,sys
t=sys.stdin.read().strip().splitlines()
try:
    d=json.loads(t[-1]); print('$n p$P $w', '%.3f Gq/s'%(d['value']/1e9), 'ms %.4f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], d['clocks']['sm_mhz'])
except Exception: print('$n p$P $w FAILED', t[-3:])" | tee -a gpurun_out/${TAG}_results.txt
    done
  else
    echo "$n p$P HANG/FAIL: $(tail -1 gpurun_out/${TAG}_${n}_probe.txt)" | tee -a gpurun_out/${TAG}_results.txt
  fi
done
