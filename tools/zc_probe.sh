for zc in 0 1; do
  NMQ_HOST_ZEROCOPY=$zc timeout 120 python bench.py --workload c2 --steps 50 --no-cpu-baseline --e2e-steps 30 2>&1 | tail -1 | python -c "
import json,sys
t=sys.stdin.read()
try:
  d=json.loads(t); print('zc $zc e2e %.3f Gq/s kernel %.2f'%(d['e2e']['value']/1e9, d['value']/1e9))
except Exception: print('zc $zc FAILED', t[-400:])"
done
NMQ_HOST_ZEROCOPY=1 timeout 120 python -m pytest tests -m gpu -q -k "host or stream" 2>&1 | tail -2
