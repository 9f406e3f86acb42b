"""The renderer-side callers of the query path (reference ``render.py``):
level of detail from ray cones (``footprint_to_level`` :334-337 and the
footprint inside ``_surface_frames_and_level`` :423-445) and the per-vertex
shading context (``_VertexShading`` :340-420, with the material bindings
``NeuralBinding`` :170-183).  Only these pieces of the reference renderer
touch the query path; the path tracer itself is out of scope.

The LoD functions run on the GPU (csrc/nmq_lod.cu) in float64 like the
reference.
numpy in -> numpy out (float64, the reference's dtype); torch CUDA in ->
torch out on the same device (``cone_level`` returns the fp32 lod the query
entry points take, so it can feed ``neural.eval_material`` directly).
"""

import numpy as np
import torch

from . import _io, _lib, neural, proxy


def footprint_to_level(area_texels, n_levels):
    """Fractional mip level from footprint area in level-0 texels^2:
    clip(0.5 * log2(max(area, 1)), 0, n_levels - 1) (render.py:334-337)."""
    if int(n_levels) < 1:
        raise ValueError("n_levels must be >= 1")
    np_mode = _io.is_numpy_like(area_texels)
    dev = _io.cuda_device(None if np_mode else area_texels.device)
    if np_mode:
        a = np.asarray(area_texels, dtype=np.float64)
        shape = a.shape
        t = torch.from_numpy(np.ascontiguousarray(a.reshape(-1))).to(dev)
    else:
        shape = tuple(area_texels.shape)
        t = area_texels.to(device=dev, dtype=torch.float64).reshape(-1).contiguous()
    out = torch.empty_like(t)
    lib = _lib.load()
    _lib.check(lib.nm_footprint_level(t.numel(), t.data_ptr(), int(n_levels), out.data_ptr(),
                                      _io.stream_ptr(dev)), "nm_footprint_level")
    out = out.reshape(shape)
    return out.cpu().numpy() if np_mode else out


def cone_level(cone_w, cone_s, t, cos_hit, density, n_levels):
    """Level of a ray-cone footprint at a surface hit (render.py:436-443):
    width = cone_w + cone_s * t, diameter = width / max(|cos_hit|, 0.05),
    area = (diameter * density)^2 texels^2, level = footprint_to_level(area).
    `density` (texels per unit length, Quad/Sphere.texel_density) may be a
    scalar or per hit.  Returns the fp32 lod of the query API."""
    if int(n_levels) < 1:
        raise ValueError("n_levels must be >= 1")
    np_mode = _io.is_numpy_like(cone_w)
    dev = _io.cuda_device(None if np_mode else cone_w.device)
    w = _io.as_rows(cone_w, 1, dev, "cone_w")
    n = w.numel()
    s = _io.as_rows(cone_s, 1, dev, "cone_s")
    tt = _io.as_rows(t, 1, dev, "t")
    c = _io.as_rows(cos_hit, 1, dev, "cos_hit")
    for name, v in (("cone_s", s), ("t", tt), ("cos_hit", c)):
        if v.numel() != n:
            raise ValueError(f"{name}: expected {n} values, got {v.numel()}")
    d, stride = _io.as_vec(density, n, dev, "density")
    lod = torch.empty((n,), device=dev, dtype=torch.float32)
    lib = _lib.load()
    _lib.check(lib.nm_cone_level(n, w.data_ptr(), s.data_ptr(), tt.data_ptr(), c.data_ptr(),
                                 d.data_ptr(), stride, int(n_levels), lod.data_ptr(),
                                 _io.stream_ptr(dev)), "nm_cone_level")
    return lod.cpu().numpy() if np_mode else lod


class NeuralBinding:
    """A scene material backed by a neural material (render.py:170-183)."""
    kind = "neural"

    def __init__(self, mat, fp16=False):
        self.mat = mat
        self.fp16 = fp16

    @property
    def resolution(self):
        return self.mat.latent.width, self.mat.latent.height

    @property
    def n_levels(self):
        return self.mat.latent.n_levels


class VertexShading:
    """Per-vertex material context (render.py:340-420), GPU-resident.

    Groups the vertices by material name (sorted, so the random stream is the
    reference's), then per neural group fetches the latent codes (``nm_fetch``,
    Russian-roulette level from ``rng.random(ns)``) and infers the analytic
    proxy once (``nm_infer_proxy``); ``eval`` decodes the BRDF from the cached
    codes (``nm_eval_z``), ``sample``/``pdf`` reuse the cached 9-float proxy
    blocks (``nm_sample`` / ``nm_pdf``).  Codes, proxies and the per-group row
    indices stay on the device between calls.

    ``scene`` needs ``objects[i].material`` (name) and ``materials`` (name ->
    binding), ``cfg`` ``lod``, ``force_level``, ``fp16`` (and optionally
    ``assert_pdf_consistency``), ``hits`` ``obj`` and ``uv`` — the reference
    renderer's own objects work unchanged.  Analytic (``kind ==
    "reference"``) bindings are not on the neural query path and raise
    NotImplementedError.  numpy in -> float64 numpy out (the reference's
    dtypes); torch CUDA in -> fp32 tensors on that device."""

    def __init__(self, scene, cfg, hits, wo_local, level, rng):
        self.scene = scene
        self.cfg = cfg
        self.hits = hits
        self.np_mode = _io.is_numpy_like(wo_local)
        self.dev = _io.cuda_device(None if self.np_mode else wo_local.device)
        self.wo = _io.as_rows(wo_local, 3, self.dev, "wo_local")
        # numpy callers pass float64 (the reference renderer does): levels, taps
        # and T.wo are formed from the float64 values (nm_fetch_f64, eval_brdf's
        # float64 route); the fp32 copy feeds the sampler and proxy as the
        # reference narrows them (neural.py:358)
        self.wo64 = _io.as_rows64(wo_local, 3, self.dev, "wo_local") if self.np_mode else None
        self.n = self.wo.shape[0]
        obj = np.asarray(hits.obj if _io.is_numpy_like(hits.obj) else hits.obj.cpu().numpy())
        names = [scene.objects[int(i)].material for i in obj]
        if len(names) != self.n:
            raise ValueError("hits and wo_local must share the batch size")
        uv = (_io.as_rows64 if self.np_mode else _io.as_rows)(hits.uv, 2, self.dev, "uv")
        ftype = torch.float64 if self.np_mode else torch.float32
        lv_all = None
        if cfg.lod and cfg.force_level is None:
            lv_all = level if isinstance(level, torch.Tensor) else np.asarray(level, np.float64)
        self.groups = []  # (binding, device row indices, fp16, z, proxy)
        name_arr = np.array(names, dtype=object)
        lib = _lib.load()
        stream = _io.stream_ptr(self.dev)
        for name in sorted(set(names)):
            sel = np.flatnonzero(name_arr == name)
            binding = scene.materials[name]
            if binding.kind != "neural":
                raise NotImplementedError(
                    f"material {name!r}: analytic '{binding.kind}' bindings are not on the neural query path")
            ns = sel.size
            idx = torch.from_numpy(sel).to(self.dev)
            if cfg.force_level is not None:
                lod = torch.full((ns,), float(cfg.force_level), device=self.dev, dtype=ftype)
            elif lv_all is None:
                lod = torch.zeros((ns,), device=self.dev, dtype=ftype)
            elif isinstance(lv_all, torch.Tensor):
                lod = lv_all.to(self.dev, ftype).reshape(-1)[idx].contiguous()
            else:
                lod = torch.from_numpy(lv_all.reshape(-1)[sel].astype(np.float64)).to(self.dev, ftype)
            fp16 = bool(cfg.fp16 or binding.fp16)
            mat = binding.mat
            h = mat.device_material(self.dev, precise=not fp16)
            u_rr = torch.from_numpy(np.asarray(rng.random(ns), np.float64)).to(self.dev, ftype)
            uv_g = uv[idx].contiguous()
            z = torch.empty((ns, neural.LATENT_CHANNELS), device=self.dev)
            chosen = torch.empty((ns,), device=self.dev, dtype=torch.int32)
            if ns:
                fetch = lib.nm_fetch_f64 if self.np_mode else lib.nm_fetch
                _lib.check(fetch(h.ptr, ns, uv_g.data_ptr(), lod.data_ptr(), 1, u_rr.data_ptr(),
                                 z.data_ptr(), chosen.data_ptr(), None, None, stream), "nm_fetch")
            wo_g = self.wo[idx].contiguous()
            pp = neural.infer_proxy(mat, z, wo_g, fp16=fp16) if ns else None
            wo_e = self.wo64[idx].contiguous() if self.wo64 is not None else wo_g  # for eval
            self.groups.append((binding, idx, fp16, z, pp, wo_g, wo_e))

    def _result(self, t):
        return _io.out(t, self.np_mode)

    def eval(self, wi_local):
        """BRDF values at (wi_local, wo_local) per vertex (render.py:377-389)."""
        rows = _io.as_rows64 if self.np_mode else _io.as_rows
        wi = rows(wi_local, 3, self.dev, "wi_local")
        if wi.shape[0] != self.n:
            raise ValueError("wi_local must have one row per vertex")
        out = torch.zeros((self.n, 3), device=self.dev)
        for binding, idx, fp16, z, _, _, wo_e in self.groups:
            if idx.numel():
                f, _ = neural.eval_brdf(binding.mat, z, wi[idx].contiguous(), wo_e, fp16=fp16)
                out[idx] = f
        return self._result(out)

    def sample(self, rng):
        """(wi, pdf): proxy samples from u = rng.random((ns, 3)) per group in
        the reference's order, and their mixture pdf (render.py:391-409)."""
        wi = torch.zeros((self.n, 3), device=self.dev)
        pdf = torch.zeros((self.n,), device=self.dev)
        for _, idx, _, _, pp, wo_g, _ in self.groups:
            ns = idx.numel()
            u = torch.from_numpy(np.asarray(rng.random((ns, 3)), np.float32)).to(self.dev)
            if not ns:
                continue
            w = proxy.sample(pp, wo_g, u)
            p = proxy.pdf(pp, wo_g, w)
            if getattr(self.cfg, "assert_pdf_consistency", False):
                again = proxy.pdf(pp, wo_g, w)
                assert torch.allclose(p, again, atol=1e-6)
            wi[idx] = w
            pdf[idx] = p.reshape(-1)
        return self._result(wi), self._result(pdf)

    def pdf(self, wi_local):
        """Mixture pdf of wi_local under each vertex's cached proxy (render.py:411-420)."""
        wi = _io.as_rows(wi_local, 3, self.dev, "wi_local")
        if wi.shape[0] != self.n:
            raise ValueError("wi_local must have one row per vertex")
        out = torch.zeros((self.n,), device=self.dev)
        for _, idx, _, _, pp, wo_g, _ in self.groups:
            if idx.numel():
                out[idx] = proxy.pdf(pp, wo_g, wi[idx].contiguous()).reshape(-1)
        return self._result(out)
