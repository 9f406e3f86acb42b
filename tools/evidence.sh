#!/bin/bash
# Round evidence: launch list + ncu --set full of the default kernel for the
# three workloads, PCIe probe.  usage: tools/evidence.sh TAG
TAG=${1:-ev}
mkdir -p gpurun_out
python tools/pcie_probe.py > gpurun_out/${TAG}_pcie.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fast_kernel|warp_kernel|fused_kernel|fetch_kernel" --csv --log-file gpurun_out/${TAG}_launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
for w in c2 c3 full; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fast_kernel" -s 3 -c 1 -o gpurun_out/${TAG}_$w python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${TAG}_ncu_$w.log 2>&1
done
ls gpurun_out | grep $TAG
