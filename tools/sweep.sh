#!/bin/bash
# Sweep library variants (tools/variants/libnmq_*.so) over the bench workloads.
TAG=${1:-sweep}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --tb=line > gpurun_out/${TAG}_pytest.log 2>&1
tail -4 gpurun_out/${TAG}_pytest.log
for lib in tools/variants/libnmq_*.so; do
  n=$(basename $lib .so)
  for w in c2 c3 full; do
    steps=200; [ $w = c3 ] && steps=20
    NMQ_LIB=$PWD/$lib timeout 300 python bench.py --workload $w --steps $steps --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$n $w', '%.3f Gq/s'%(d['value']/1e9), 'ms %.4f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], d['clocks']['sm_mhz'])" | tee -a gpurun_out/${TAG}_results.txt
  done
done
