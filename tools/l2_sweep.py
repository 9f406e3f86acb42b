"""GPU time per C2 launch vs number of rotating input sets and batch size."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2305_02678_b200 import _lib, synth
lib = _lib.load()
dev = torch.device("cuda", 0)
mat = synth.material("2x32", 4096, 4096, seed=0, device=dev)
h = mat.device_material(dev)
sp = torch.cuda.current_stream().cuda_stream
for mult in (1, 4):
    n = 1920 * 1080 * mult
    sets = [synth.queries(n, mat.latent.n_levels, seed=1 + s, device=dev) for s in range(3)]
    rgb = torch.empty((n, 3), device=dev)
    for nsets in (1, 2, 3):
        args = [(h.ptr, n, q["uv"].data_ptr(), q["lod"].data_ptr(), 1, q["u_rr"].data_ptr(),
                 q["wi"].data_ptr(), q["wo"].data_ptr(), rgb.data_ptr(), None, None, sp)
                for q in sets[:nsets]]
        for i in range(6):
            lib.nm_eval(*args[i % nsets])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 60 if mult == 1 else 20
        e0.record()
        for i in range(K):
            lib.nm_eval(*args[i % nsets])
        e1.record()
        torch.cuda.synchronize()
        us = 1e3 * e0.elapsed_time(e1) / K
        print(f"mult {mult} sets {nsets}: {us:8.1f} us/launch  {n / us / 1e3:6.2f} Gq/s")
