"""Host submission cost of one fused launch vs its GPU time (C2 eval)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2305_02678_b200 import _lib, synth
lib = _lib.load()
dev = torch.device("cuda", 0)
mat = synth.material("2x32", 4096, 4096, seed=0, device=dev)
n = 1920 * 1080
q = synth.queries(n, mat.latent.n_levels, seed=1, device=dev)
h = mat.device_material(dev)
rgb = torch.empty((n, 3), device=dev)
sp = torch.cuda.current_stream().cuda_stream
args = (h.ptr, n, q["uv"].data_ptr(), q["lod"].data_ptr(), 1, q["u_rr"].data_ptr(),
        q["wi"].data_ptr(), q["wo"].data_ptr(), rgb.data_ptr(), None, None, sp)
for _ in range(10):
    lib.nm_eval(*args)
torch.cuda.synchronize()
K = 200
t0 = time.perf_counter()
for _ in range(K):
    lib.nm_eval(*args)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host submit {1e6 * (t1 - t0) / K:.1f} us/launch, wall {1e6 * (t2 - t0) / K:.1f} us/launch")
# graph replay
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        a2 = list(args)
        a2[-1] = torch.cuda.current_stream().cuda_stream
        for _ in range(20):
            lib.nm_eval(*a2)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(f"graph replay {1e3 * e0.elapsed_time(e1) / 200:.1f} us/launch-equivalent "
      f"-> {n / (e0.elapsed_time(e1) / 200 / 1e3) / 1e9:.2f} Gq/s")
