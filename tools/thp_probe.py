"""First-touch cost of fresh result-sized arrays (C2: 2.07M x 3 float64 +
2.07M int64) with numpy's MADV_HUGEPAGE hint on and off, single-threaded
fill vs the library's threaded copy-out."""
import time
import numpy as np
try:
    from numpy._core import multiarray as ma
except ImportError:
    from numpy.core import multiarray as ma
print(open('/sys/kernel/mm/transparent_hugepage/enabled').read().strip(),
      open('/sys/kernel/mm/transparent_hugepage/defrag').read().strip())
n = 1920 * 1080
for hint in (True, False, True, False):
    prev = ma._set_madvise_hugepage(hint)
    ts = []
    for k in range(5):
        t = time.perf_counter()
        a = np.empty((n, 3)); a.fill(1.0); b = np.empty(n, np.int64); b.fill(1)
        ts.append(1e3 * (time.perf_counter() - t))
        del a, b
    ma._set_madvise_hugepage(prev)
    print("madvise hugepage", hint, "alloc+touch ms", [round(x, 2) for x in ts])
