import numpy as np, time
print(open('/sys/kernel/mm/transparent_hugepage/enabled').read().strip(), open('/sys/kernel/mm/transparent_hugepage/defrag').read().strip())
try:
    from numpy._core import multiarray as ma
except ImportError:
    from numpy.core import multiarray as ma
print("numpy madvise hugepage:", ma._get_madvise_hugepage())
n=1920*1080
for k in range(3):
    t=time.perf_counter(); a=np.empty((n,3)); a.fill(1.0); b=np.empty(n,np.int64); b.fill(1); print("alloc+touch %.2f ms" % (1e3*(time.perf_counter()-t)))
