#!/bin/bash
TAG=${1:-r01e}
for w in c2 c3 full; do
  steps=200; [ $w = c3 ] && steps=20
  timeout 300 python bench.py --workload $w --steps $steps --no-cpu-baseline --e2e-steps 0 > gpurun_out/${TAG}_bench_$w.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/${TAG}_bench_$w.json').read().strip().splitlines()[-1]); print('$w', '%.2f Gq/s'%(d['value']/1e9), 'frac %.3f'%d['roofline']['frac'])"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fast_kernel" -s 3 -c 1 -o gpurun_out/${TAG}_prof_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fast_kernel" -s 3 -c 1 -o gpurun_out/${TAG}_prof_full python bench.py --workload full --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ls gpurun_out | grep $TAG
