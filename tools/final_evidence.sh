#!/bin/bash
# Round-end evidence in one gpurun call: GPU tests, smoke, every bench
# workload, the reference arm, launch list + ncu --set full of the headline
# kernel.  usage: tools/final_evidence.sh TAG
TAG=${1:-final}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/${TAG}_smi.txt
timeout 900 python -m pytest tests -q -m gpu --tb=short > gpurun_out/${TAG}_pytest_gpu.log 2>&1; tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err
for w in c3 full c4 c5 train kl; do
  timeout 600 python bench.py --workload $w > gpurun_out/${TAG}_bench_$w.json 2> gpurun_out/${TAG}_bench_$w.err
done
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_bench_reference.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fast_kernel" --csv --log-file gpurun_out/${TAG}_launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fast_kernel" -s 3 -c 1 -o gpurun_out/${TAG}_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
for f in gpurun_out/${TAG}_bench_*.json; do echo "$f: $(tail -c 400 $f | head -c 400)"; done
