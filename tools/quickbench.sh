#!/bin/bash
# quick C2/C3/full throughput of the default build and variants (GPU box):
#   tools/quickbench.sh [variant ...]   (variant = paper_2305_02678_b200/variants/libnmq_<v>.so)
run() {  # lib label workload
  NMQ_LIB=$1 timeout 300 python bench.py --steps 300 --workload $3 --no-cpu-baseline --e2e-steps 0 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', '$3', round(d['value']/1e9,2), 'Gq/s frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
}
W=${WORKLOADS:-c2}
for w in $W; do run paper_2305_02678_b200/libnmq.so default $w; done
for v in "$@"; do for w in $W; do run paper_2305_02678_b200/variants/libnmq_$v.so $v $w; done; done
