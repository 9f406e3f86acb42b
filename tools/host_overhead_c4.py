"""Host submission cost of one nm_eval_multi call (C4, BINNED_ASYNC and
BINNED) vs its wall time: does the host keep the GPU fed?"""
import ctypes, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2305_02678_b200 import _lib, synth
from paper_2305_02678_b200.synth import C4_RESOLUTIONS
lib = _lib.load()
dev = torch.device("cuda", 0)
mats = [synth.material("2x32", w, h, seed=10 + k, device=dev) for k, (w, h) in enumerate(C4_RESOLUTIONS)]
hs = [m.device_material(dev) for m in mats]
n = 1920 * 1080
q = synth.queries(n, min(m.latent.n_levels for m in mats), seed=1, device=dev)
ids = torch.randint(0, len(mats), (n,), device=dev, dtype=torch.int32)
rgb = torch.empty((n, 3), device=dev)
wsb = int(lib.nm_multi_workspace_bytes(n, len(mats)))
ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
ptrs = (ctypes.c_void_p * len(mats))(*[h.ptr for h in hs])
sp = torch.cuda.current_stream().cuda_stream
for mode, name in ((_lib.NM_MULTI_BINNED_ASYNC, "binned_async"), (_lib.NM_MULTI_BINNED, "binned")):
    call = lambda: lib.nm_eval_multi(ptrs, len(mats), n, ids.data_ptr(), q["uv"].data_ptr(), q["lod"].data_ptr(), 1,
                                     q["u_rr"].data_ptr(), q["wi"].data_ptr(), q["wo"].data_ptr(), rgb.data_ptr(),
                                     mode, ws.data_ptr(), wsb, sp)
    for _ in range(5): call()
    torch.cuda.synchronize()
    K = 50
    t0 = time.perf_counter()
    for _ in range(K): call()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name}: host submit {1e6 * (t1 - t0) / K:.1f} us/call, wall {1e6 * (t2 - t0) / K:.1f} us/call")
