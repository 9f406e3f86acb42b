"""Does the box let kernels read pageable host memory (HMM / ATS)?  If so,
time the eval kernel reading the drop-in's pageable numpy inputs in place."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2305_02678_b200 import _io, _lib, synth
from cuda.bindings import runtime as rt
for name in ("cudaDevAttrPageableMemoryAccess", "cudaDevAttrPageableMemoryAccessUsesHostPageTables",
             "cudaDevAttrConcurrentManagedAccess", "cudaDevAttrHostNativeAtomicSupported"):
    err, v = rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, name), 0)
    print(name, v)
err, v = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrPageableMemoryAccess, 0)
if v:
    dev = torch.device("cuda", 0)
    lib = _lib.load()
    mat = synth.material("2x32", 4096, 4096, seed=0, device=dev)
    h = mat.device_material(dev)
    n = 1920 * 1080
    q = synth.queries(n, mat.latent.n_levels, seed=1, device=dev)
    hq = {k: np.ascontiguousarray(v.cpu().numpy()) for k, v in q.items()}
    rgb = np.empty((n, 3), np.float32)
    sp = _io.stream_ptr(dev)
    for k in range(5):
        t = time.perf_counter()
        _lib.check(lib.nm_eval(h.ptr, n, hq["uv"].ctypes.data, hq["lod"].ctypes.data, 1, hq["u_rr"].ctypes.data,
                               hq["wi"].ctypes.data, hq["wo"].ctypes.data, rgb.ctypes.data, None, None, sp))
        torch.cuda.synchronize()
        print("eval reading pageable memory in place: %.2f ms" % (1e3 * (time.perf_counter() - t)))
