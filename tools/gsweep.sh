#!/bin/bash
for G in 3 4 5 6 7; do
  echo "G=$G"; NMQ_G=$G NMQ_LIB=$PWD/tools/libnmq_trace.so python tools/trace_run.py c2 2>&1 | tail -4 | head -2
  NMQ_G=$G NMQ_LIB=$PWD/tools/libnmq_gs.so timeout 300 python bench.py --steps 100 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('  c2 %.2f Gq/s'%(d['value']/1e9))"
done
