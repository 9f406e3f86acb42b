for lib in tools/variants/libnmq_*.so; do
  n=$(basename $lib .so)
  NMQ_LIB=$PWD/$lib NMQ_KERNEL_PATH=2 timeout 120 python tools/hang_probe.py 132736 300000 2100000 > /dev/null 2>&1 || { echo "$n HANG"; continue; }
  NMQ_KERNEL_PATH=2 NMQ_LIB=$PWD/$lib timeout 120 python bench.py --workload c3 --steps 20 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$n c3', '%.3f Gq/s'%(d['value']/1e9), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
