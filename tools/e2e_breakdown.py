"""Where the drop-in e2e call's time goes (C2 batch, pageable fp32 numpy in):
eval_material total, nm_eval_host alone, the output dtype widening, and a
plain pageable H2D/D2H of the same bytes.  GPU box: python tools/e2e_breakdown.py"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2305_02678_b200 import _io, _lib, neural, synth

dev = torch.device("cuda", 0)
mat = synth.material("2x32", 4096, 4096, seed=0, device=dev)
n = 1920 * 1080
q = synth.queries(n, mat.latent.n_levels, seed=1, device=dev)
hq = {k: v.cpu().numpy() for k, v in q.items()}
lib = _lib.load()
h = mat.device_material(dev)


def t(fn, k=10):
    fn()
    torch.cuda.synchronize()
    s = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - s) / k


rgb = np.empty((n, 3), np.float32)
lv = np.empty(n, np.int32)
print("eval_material (f64 f, int64 level)  %.2f ms" % t(lambda: neural.eval_material(
    mat, hq["uv"], hq["lod"], hq["wi"], hq["wo"], hq["u_rr"], fp16=True)))
f64o = np.empty((n, 3)); lv64 = np.empty(n, np.int64)
print("nm_eval_host_ref -> f64/int64       %.2f ms" % t(lambda: _lib.check(lib.nm_eval_host_ref(h.ptr, n, hq["uv"].ctypes.data, hq["lod"].ctypes.data, 1, hq["u_rr"].ctypes.data, hq["wi"].ctypes.data, hq["wo"].ctypes.data, f64o.ctypes.data, None, lv64.ctypes.data, 0, _io.stream_ptr(dev)))))
print("nm_eval_host pageable -> f32/int32  %.2f ms" % t(lambda: _lib.check(lib.nm_eval_host(
    h.ptr, n, hq["uv"].ctypes.data, hq["lod"].ctypes.data, 1, hq["u_rr"].ctypes.data, hq["wi"].ctypes.data,
    hq["wo"].ctypes.data, rgb.ctypes.data, None, lv.ctypes.data, _io.STREAM_CHUNK, _io.stream_ptr(dev)))))
print("widen rgb f64 + level i64           %.2f ms" % t(lambda: (rgb.astype(np.float64), lv.astype(np.int64))))
allin = np.concatenate([hq[k].reshape(-1) for k in ("uv", "lod", "u_rr", "wi", "wo")])
d = torch.empty(allin.size, device=dev)
print("pageable H2D %d MB                  %.2f ms" % (allin.nbytes >> 20, t(lambda: d.copy_(torch.from_numpy(allin)))))
out = np.empty(n * 4, np.float32)
print("pageable D2H %d MB                  %.2f ms" % (out.nbytes >> 20, t(lambda: torch.from_numpy(out).copy_(d[: n * 4]))))
# fresh result arrays every call (what the drop-in returns) vs reused ones
def fresh():
    f = np.empty((n, 3)); l = np.empty(n, np.int64)
    _lib.check(lib.nm_eval_host_ref(h.ptr, n, hq["uv"].ctypes.data, hq["lod"].ctypes.data, 1, hq["u_rr"].ctypes.data,
                                    hq["wi"].ctypes.data, hq["wo"].ctypes.data, f.ctypes.data, None, l.ctypes.data, 0,
                                    _io.stream_ptr(dev)))
print("nm_eval_host_ref, fresh outputs      %.2f ms" % t(fresh))
def touch():
    f = np.empty((n, 3)); l = np.empty(n, np.int64); f.fill(0); l.fill(0)
print("np.empty + fill (first touch)        %.2f ms" % t(touch))
