"""Zero-copy host eval: where the time goes — inputs from pinned host
memory and/or rgb to pinned host memory, the fused kernel reading/writing
over PCIe directly (nm_eval with UVA host pointers)."""
import ctypes, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2305_02678_b200 import _lib

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
class A: workload = "c2"; sets = 1
mat, n, sets = bench.build_workload(A, 0, dev)
q = sets[0]
hq = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in q.items()}
for k in hq: hq[k].copy_(q[k])
rgb_d = torch.empty((n, 3), device=dev)
rgb_h = torch.empty((n, 3), pin_memory=True)
lib = _lib.load(); h = mat.device_material(dev)
st = torch.cuda.current_stream(dev)

def run(src, rgb):
    return lambda: lib.nm_eval(h.ptr, n, src["uv"].data_ptr(), src["lod"].data_ptr(), 1, src["u_rr"].data_ptr(),
                               src["wi"].data_ptr(), src["wo"].data_ptr(), rgb.data_ptr(), None, None,
                               ctypes.c_void_p(st.cuda_stream))

def ev_time(fn, k=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(k): fn()
    e1.record(st); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k

for name, src, rgb in (("dev in / dev out", q, rgb_d), ("host in / dev out", hq, rgb_d),
                       ("dev in / host out", q, rgb_h), ("host in / host out", hq, rgb_h)):
    ms = ev_time(run(src, rgb))
    print("%-20s %.3f ms  %.3f Gq/s" % (name, ms, n / ms / 1e6))
ref = rgb_d.clone(); run(hq, rgb_h)(); torch.cuda.synchronize()
print("host-out == dev-out:", torch.equal(ref.cpu(), rgb_h))
