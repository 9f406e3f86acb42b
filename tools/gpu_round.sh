#!/bin/bash
# One gpurun call: parity tests, bench, ncu launch list, ncu --set full of the fused kernel.
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
nproc > gpurun_out/${TAG}_nproc.txt
timeout 600 python -m pytest tests -q -m gpu --tb=line > gpurun_out/${TAG}_pytest_gpu.log 2>&1
tail -5 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
cat gpurun_out/${TAG}_bench.json
timeout 600 python bench.py --workload c3 --steps 20 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${TAG}_bench_c3.json 2>&1
timeout 600 python bench.py --workload full --steps 50 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${TAG}_bench_full.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fused_kernel|fast_kernel|fetch_kernel|sample_kernel|pdf_kernel" --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fused_kernel|fast_kernel" -s 3 -c 1 -o gpurun_out/${TAG}_prof_eval python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${TAG}_ncu_full.log 2>&1
tail -3 gpurun_out/${TAG}_ncu_full.log
ls -la gpurun_out
