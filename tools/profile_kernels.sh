#!/bin/bash
# ncu --set full captures (one launch each) of the shipped kernels behind the
# bench lines + the launch list of the default bench command.  GPU box only.
#   tools/profile_kernels.sh TAG   -> gpurun_out/TAG_{c2,c3,full,fp32_path,c4_scatter}.ncu-rep,
#                                     gpurun_out/TAG_launches_c2.csv
TAG=${1:-r02}
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
NCU="timeout 600 ncu --set full --clock-control none --import-source on -c 1"
for w in c2 c3 full; do
  $NCU -k regex:fast_kernel -s 3 -o gpurun_out/${TAG}_$w $B --workload $w --no-subresults > /dev/null 2>&1
done
$NCU -k regex:fused_kernel -s 3 -o gpurun_out/${TAG}_fp32_path $B > /dev/null 2>&1
$NCU -k regex:bin_scatter -s 2 -o gpurun_out/${TAG}_c4_scatter $B --workload c4 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ls -la gpurun_out | grep $TAG
