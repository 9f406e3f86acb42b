#!/bin/bash
# bench.py's e2e (the drop-in call, pageable inputs alternating over 2 sets) vs host threads
for rep in 1 2; do for th in 6 8 12 16; do
  NMQ_HOST_THREADS=$th timeout 300 python bench.py --no-subresults --no-cpu-baseline --steps 50 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('threads $th e2e', round(d['e2e']['value']/1e6,1))"
done; done
