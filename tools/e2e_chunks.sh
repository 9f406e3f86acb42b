#!/bin/bash
# e2e (host buffers through nm_eval_host) vs the streaming chunk size.
mkdir -p gpurun_out
for c in ${CHUNKS:-131072 262144 524288}; do
  NMQ_STREAM_CHUNK=$c timeout 300 python bench.py --workload c2 --steps 50 --no-cpu-baseline --e2e-steps 30 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('chunk $c', 'e2e %.3f Gq/s'%(d['e2e']['value']/1e9), 'kernel %.2f Gq/s'%(d['value']/1e9))" | tee -a gpurun_out/e2e_chunks.txt
done
