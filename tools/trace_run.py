"""Per-phase cycle breakdown of the fast kernel (needs a -DNMQ_TRACE build in $NMQ_LIB)."""
import ctypes, os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2305_02678_b200 import _lib, synth
lib = _lib.load()
lib.nm_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
dev = torch.device("cuda", 0)
wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
mat = synth.material("2x32", 4096, 4096, seed=0, device=dev)
n = 1920 * 1080
q = synth.queries(n, mat.latent.n_levels, seed=1, device=dev)
h = mat.device_material(dev)
rgb = torch.empty((n, 3), device=dev); ws = torch.empty((n, 3), device=dev); pdf = torch.empty(n, device=dev)
sp = torch.cuda.current_stream().cuda_stream
def go():
    if wl == "c2":
        _lib.check(lib.nm_eval(h.ptr, n, q["uv"].data_ptr(), q["lod"].data_ptr(), 1, q["u_rr"].data_ptr(), q["wi"].data_ptr(), q["wo"].data_ptr(), rgb.data_ptr(), None, None, sp))
    elif wl == "full":
        _lib.check(lib.nm_query(h.ptr, n, q["uv"].data_ptr(), q["lod"].data_ptr(), 1, q["u_rr"].data_ptr(), q["wi"].data_ptr(), q["wo"].data_ptr(), q["u3"].data_ptr(), rgb.data_ptr(), ws.data_ptr(), pdf.data_ptr(), None, sp))
    else:
        _lib.check(lib.nm_sample_pdf(h.ptr, n, q["uv"].data_ptr(), q["lod"].data_ptr(), 1, q["u_rr"].data_ptr(), q["wi"].data_ptr(), q["u3"].data_ptr(), ws.data_ptr(), pdf.data_ptr(), None, None, sp))
for _ in range(3): go()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 64)()
lib.nm_trace_read(buf, 64, 1)
for _ in range(10): go()
torch.cuda.synchronize()
lib.nm_trace_read(buf, 64, 1)
a = np.array(buf[:32], dtype=np.float64).reshape(4, 8)[:, :5]
tiles = n / 128 * 10
names = ["work", "barrier", "issue", "overlap", "mma_wait"]
for w in range(4):
    tot = a[w].sum()
    print(f"warp{w}: per-tile cycles total {tot/tiles:8.0f}  " + "  ".join(f"{nm} {a[w,k]/tiles:7.0f} ({100*a[w,k]/tot:4.1f}%)" for k, nm in enumerate(names)))
