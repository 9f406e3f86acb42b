#!/bin/bash
# ncu --set full of the fast kernel for one library variant and workload.
# usage: tools/prof_variant.sh TAG VARIANT WORKLOAD
TAG=$1; V=$2; WL=$3
mkdir -p gpurun_out
NMQ_LIB=$PWD/tools/variants/libnmq_$V.so timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"fast_kernel" -s 3 -c 1 -o gpurun_out/${TAG}_${V}_$WL \
  python bench.py --workload $WL --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${TAG}_${V}_$WL.log 2>&1
tail -1 gpurun_out/${TAG}_${V}_$WL.log
