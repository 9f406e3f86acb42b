"""Small launches of every query entry point, the multi-material modes, LoD
and training kernels (for compute-sanitizer; partial tiles included)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from oracle import nm_oracle as O
from paper_2305_02678_b200 import neural, render, train, mlp
from paper_2305_02678_b200.latent import LatentPyramid

rng = np.random.default_rng(0)
mat = neural.NeuralMaterial.create(neural.NeuralMaterialConfig(), rng)
mat.latent = LatentPyramid(O.random_pyramid(rng, 64, 32).levels)
n = 1000 + 37
uv = rng.random((n, 2)).astype(np.float32)
lod = (rng.random(n) * 5).astype(np.float32)
urr = rng.random(n).astype(np.float32)
wi, wo = O.draw_direction_pairs(rng, n)
wi, wo = wi.astype(np.float32), wo.astype(np.float32)
u3 = rng.random((n, 3)).astype(np.float32)
neural.eval_material(mat, uv, lod, wi, wo, urr, fp16=True)
neural.sample_pdf(mat, uv, lod, urr, wi, u3)
neural.query(mat, uv, lod, urr, wi, wo, u3)
neural.eval_material(mat, uv, lod, wi, wo, urr, fp16=False)
# float64 coordinates (nm_fetch_f64 / nm_query_f64), trilinear, in-kernel spp mean
uv64 = rng.random((n, 2)); lod64 = rng.random(n) * 5; urr64 = rng.random(n)
neural.eval_material(mat, uv64, lod64, wi, wo, urr64, fp16=True)
neural.sample_pdf(mat, uv64, lod64, urr64, wi, u3)
neural.query(mat, uv64, lod64, urr64, wi, wo, u3)
mat.latent.fetch(uv64, lod64, urr64)
mat.latent.fetch_trilinear(uv, lod)
neural.eval_material_spp(mat, uv[:1024], lod[:1024], wi[:1024], wo[:1024], urr[:1024], 16)
z, _ = mat.latent.fetch(uv, lod, urr)
neural.eval_brdf(mat, z, wi, wo, fp16=True)
neural.infer_proxy(mat, z, wi, fp16=True)
mats = [mat, neural.NeuralMaterial.create(neural.NeuralMaterialConfig(brdf_hidden="2x16"), rng)]
mats[1].latent = LatentPyramid(O.random_pyramid(rng, 32, 32).levels)
ids = rng.integers(0, 2, n).astype(np.int32)
for mode in ("binned", "binned_async", "divergent"):
    neural.eval_material_multi(mats, ids, uv, lod, wi, wo, urr, mode=mode)
for mode in ("binned", "binned_async"):
    neural.sample_pdf_multi(mats, ids, uv, lod, urr, wi, u3, mode=mode)
    neural.query_multi(mats, ids, uv, lod, urr, wi, wo, u3, mode=mode)
render.cone_level(rng.random(n).astype(np.float32), rng.random(n).astype(np.float32),
                  rng.random(n).astype(np.float32), rng.random(n).astype(np.float32), 100.0, 6)
net = mlp.Mlp.create((20, 32, 32, 3), rng)
out, cache = train.forward_cached(net, rng.normal(size=(n, 20)).astype(np.float32))
train.backward(net, cache, rng.normal(size=(n, 3)).astype(np.float32))
mat.latent.accumulate_texel_grads(mat.latent.zero_grads(), uv, np.zeros(n, np.int64), rng.normal(size=(n, 8)).astype(np.float32))
# KL sampler loss (std + isotropic)
for cfg in (neural.NeuralMaterialConfig(), neural.NeuralMaterialConfig(sampler_isotropic=True)):
    km = neural.NeuralMaterial.create(cfg, rng)
    train.sampler_loss_and_grads(km, rng.normal(size=(n, 8)).astype(np.float32), wi.astype(np.float64), rng)
# per-vertex shading context (two materials)
from types import SimpleNamespace
scene = SimpleNamespace(objects=[SimpleNamespace(material="a"), SimpleNamespace(material="b")],
                        materials={"a": render.NeuralBinding(mats[0], fp16=True),
                                   "b": render.NeuralBinding(mats[1], fp16=False)})
ctx = render.VertexShading(scene, SimpleNamespace(lod=True, force_level=None, fp16=False),
                           SimpleNamespace(obj=ids, uv=uv), wo, lod, rng)
ctx.eval(wi); ctx.sample(rng); ctx.pdf(wi)
# host-buffer eval: zero-copy (pinned) and staged (pageable) paths
import ctypes
from paper_2305_02678_b200 import _lib, _io
lib = _lib.load()
h = mat.device_material(None)
pin = {k: torch.from_numpy(v).pin_memory() for k, v in (("uv", uv), ("lod", lod), ("urr", urr), ("wi", wi), ("wo", wo))}
rgb_pin = torch.empty((n, 3)).pin_memory()
rgb_pg = np.empty((n, 3), np.float32)
for src, dst in ((pin, rgb_pin.data_ptr()), ({"uv": uv, "lod": lod, "urr": urr, "wi": wi, "wo": wo}, rgb_pg.ctypes.data)):
    ptr = {k: (v.data_ptr() if isinstance(v, torch.Tensor) else v.ctypes.data) for k, v in src.items()}
    _lib.check(lib.nm_eval_host(h.ptr, n, ptr["uv"], ptr["lod"], 1, ptr["urr"], ptr["wi"], ptr["wo"], dst,
                                None, None, 256, _io.stream_ptr(h.device)))
assert np.array_equal(rgb_pin.numpy(), rgb_pg)
# the drop-in's reference dtypes through the pinned bounce pipeline (several chunks)
f64o, lv64 = np.empty((n, 3)), np.empty(n, np.int64)
_lib.check(lib.nm_eval_host_ref(h.ptr, n, uv.ctypes.data, lod.ctypes.data, 1, urr.ctypes.data, wi.ctypes.data,
                                wo.ctypes.data, f64o.ctypes.data, None, lv64.ctypes.data, 256, _io.stream_ptr(h.device)))
assert np.array_equal(f64o, rgb_pg.astype(np.float64))
# float64 directions (nm_query_f64 / nm_eval_z_f64) and the decoder-input hook
wi64, wo64 = O.draw_direction_pairs(rng, n)
neural.eval_material(mat, uv64, lod64, wi64, wo64, urr64, fp16=True)
neural.eval_brdf(mat, z, wi64, wo64, fp16=True)
x16 = torch.empty((n, 12), dtype=torch.int16, device="cuda")
zt = torch.from_numpy(np.ascontiguousarray(z, np.float32)).cuda()
w64 = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (wi64, wo64)]
_lib.check(lib.nm_decoder_inputs(h.ptr, n, zt.data_ptr(), None, None, w64[0].data_ptr(), w64[1].data_ptr(),
                                 x16.data_ptr(), _io.stream_ptr(h.device)))
torch.cuda.synchronize()
print("sanitize_run ok")
