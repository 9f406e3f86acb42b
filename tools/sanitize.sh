#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over small launches of
# every kernel family (race detection).  usage: tools/sanitize.sh TAG
TAG=${1:-san}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for p in 2 1; do
    NMQ_KERNEL_PATH=$p timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 \
      python tools/sanitize_run.py > gpurun_out/${TAG}_${tool}_p$p.log 2>&1
    echo "$tool path$p rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/${TAG}_${tool}_p$p.log | tail -1)"
  done
done
