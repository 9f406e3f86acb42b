#!/bin/bash
# Round-end evidence in one gpurun call: GPU tests, smoke, every bench
# workload, the reference arm, compute-sanitizer, and the ncu captures of the
# shipped kernels (tools/profile_kernels.sh).  usage: tools/final_evidence.sh TAG
TAG=${1:-final}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/${TAG}_smi.txt
NMQ_PARITY_REPORT=1 timeout 1200 python -m pytest tests -q -s -m gpu --tb=short > gpurun_out/${TAG}_pytest_gpu_full.log 2>&1
grep -E "PARITY" gpurun_out/${TAG}_pytest_gpu_full.log > gpurun_out/${TAG}_parity_report.txt
tail -3 gpurun_out/${TAG}_pytest_gpu_full.log | tee gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err
for w in c3 full c4 c5 train kl; do
  timeout 600 python bench.py --workload $w > gpurun_out/${TAG}_bench_$w.json 2> gpurun_out/${TAG}_bench_$w.err
done
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_bench_reference.json 2>&1
./tools/sanitize.sh ${TAG}san > gpurun_out/${TAG}_sanitize_summary.txt 2>&1
./tools/profile_kernels.sh ${TAG} > /dev/null 2>&1
for f in gpurun_out/${TAG}_bench_*.json; do echo "$f: $(head -c 300 $f)"; done
