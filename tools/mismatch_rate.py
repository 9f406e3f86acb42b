"""How many C2 rows the resolve must re-evaluate: rows whose fast-path fp16
decoder direction inputs differ from the reference rounding (nm_decoder_inputs),
and how many the fast check queues (nm_eval_debug_tw dumps the fast values)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2305_02678_b200 import _io, _lib, synth

dev = torch.device("cuda", 0)
lib = _lib.load()
mat = synth.material("2x32", 4096, 4096, seed=0, device=dev)
h = mat.device_material(dev)
n = 1920 * 1080
q = synth.queries(n, mat.latent.n_levels, seed=1, device=dev)
sp = _io.stream_ptr(dev)
rgb = torch.empty((n, 3), device=dev)
dbg = torch.empty((n, 14), device=dev)
_lib.check(lib.nm_eval_debug_tw(h.ptr, n, q["uv"].data_ptr(), q["lod"].data_ptr(), 1, q["u_rr"].data_ptr(),
                                q["wi"].data_ptr(), q["wo"].data_ptr(), rgb.data_ptr(), dbg.data_ptr(), sp))
z = torch.empty((n, 8), device=dev)
_lib.check(lib.nm_fetch(h.ptr, n, q["uv"].data_ptr(), q["lod"].data_ptr(), 1, q["u_rr"].data_ptr(),
                        z.data_ptr(), None, None, None, sp))
x16 = torch.empty((n, 12), dtype=torch.int16, device=dev)
_lib.check(lib.nm_decoder_inputs(h.ptr, n, z.data_ptr(), q["wi"].data_ptr(), q["wo"].data_ptr(), None, None,
                                 x16.data_ptr(), sp))
torch.cuda.synchronize()
fast = dbg[:, :12].half().view(torch.int16)
diff = (fast != x16).any(dim=1)
print(f"rows {n}: fast fp16 inputs differ from the reference rounding on {int(diff.sum())} rows "
      f"({100 * diff.float().mean().item():.3f} %), values {int((fast != x16).sum())}")
