#!/bin/bash
# ncu --set full of one kernel family (NMQ_KERNEL_PATH) on one workload.
# usage: tools/prof_path.sh TAG PATH WORKLOAD [kernel-regex]
TAG=$1; P=$2; WL=$3; K=${4:-"fast_kernel|warp_kernel"}
mkdir -p gpurun_out
NMQ_KERNEL_PATH=$P timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"$K" -s 3 -c 1 -o gpurun_out/${TAG}_p${P}_$WL \
  python bench.py --workload $WL --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${TAG}_p${P}_$WL.log 2>&1
tail -1 gpurun_out/${TAG}_p${P}_$WL.log
