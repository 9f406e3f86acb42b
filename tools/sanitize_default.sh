mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  NMQ_KERNEL_PATH=0 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/san2_${tool}.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san2_${tool}.log | tail -1) $(grep -c 'sanitize_run ok' gpurun_out/san2_${tool}.log)"
done
