#!/bin/bash
# One gpurun iteration: GPU parity tests, variant sweep (sweep.sh), optional
# ncu --set full capture of one workload with the in-tree library.
# usage: tools/gpu_iter.sh TAG [ncu_workload]
TAG=${1:-iter}; WL=${2:-}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv,noheader > gpurun_out/${TAG}_smi.txt
bash tools/sweep.sh $TAG
if [ -n "$WL" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fast_kernel" -s 3 -c 1 \
    -o gpurun_out/${TAG}_prof_$WL python bench.py --workload $WL --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${TAG}_ncu.log 2>&1
  tail -2 gpurun_out/${TAG}_ncu.log
fi
