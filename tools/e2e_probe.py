"""Where the e2e (host-buffer) time goes: the public call vs the raw
nm_eval_host call vs plain copies of the same bytes."""
import ctypes, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2305_02678_b200 import neural, _lib, _io

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
class A: workload = "c2"; sets = 2
mat, n, sets = bench.build_workload(A, 0, dev)
q = sets[0]
hq = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in q.items()}
for k in hq: hq[k].copy_(q[k])
hn = {k: v.numpy() for k, v in hq.items()}
print({k: (v.dtype, v.shape) for k, v in hn.items()})
out = torch.empty((n, 3), dtype=torch.float32, pin_memory=True).numpy()
lib = _lib.load(); h = mat.device_material(dev)
st = torch.cuda.current_stream(dev)

def ev_time(fn, k=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(st)
    for _ in range(k): fn()
    e1.record(st); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k, (time.perf_counter() - t0) * 1e3 / k

api = lambda: neural.eval_material(mat, hn["uv"], hn["lod"], hn["wi"], hn["wo"], hn["u_rr"], fp16=True,
                                   return_level=False, out=out)
for chunk in (1 << 18, 1 << 19, 1 << 20, n):
    raw = lambda: lib.nm_eval_host(h.ptr, n, hn["uv"].ctypes.data, hn["lod"].ctypes.data, 1,
                                   hn["u_rr"].ctypes.data, hn["wi"].ctypes.data, hn["wo"].ctypes.data,
                                   out.ctypes.data, chunk, ctypes.c_void_p(st.cuda_stream))
    print("raw nm_eval_host chunk %d: %.3f ms (wall %.3f)" % ((chunk,) + ev_time(raw)))
print("public api: %.3f ms (wall %.3f)" % ev_time(api))
d = {k: torch.empty_like(v, device=dev) for k, v in hq.items()}
drgb = torch.empty((n, 3), device=dev); hrgb = torch.from_numpy(out)
def h2d():
    for k in ("uv", "lod", "u_rr", "wi", "wo"): d[k].copy_(hq[k], non_blocking=True)
def d2h(): hrgb.copy_(drgb, non_blocking=True)
print("h2d only: %.3f ms" % ev_time(h2d)[0])
print("d2h only: %.3f ms" % ev_time(d2h)[0])
s2 = torch.cuda.Stream()
def both():
    ev = torch.cuda.Event(); ev.record(st); s2.wait_event(ev)
    with torch.cuda.stream(s2): d2h()
    h2d()
    ev2 = torch.cuda.Event(); ev2.record(s2); st.wait_event(ev2)
print("h2d || d2h: %.3f ms" % ev_time(both)[0])
