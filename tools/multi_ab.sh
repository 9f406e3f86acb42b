# A/B of the multi-material launch policies on C4 (i.i.d. ids): device-side
# proportional shares (default) vs even 1/n_mats shares + host-count checked mode
for split in 0 1 0 1; do
  NMQ_MULTI_SPLIT=$split timeout 600 python bench.py --workload c4 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('split=$split', 'binned %.2f async %.2f'%(d['value']/1e9, d['binned_async']['value']/1e9))"
done
