"""Neural material query API — drop-in for ``neuralmat.neural``.

Same names and argument meaning as the reference (neural.py:82-419):
``NeuralMaterialConfig``, ``NeuralMaterial`` (``create``, ``half``,
``invalidate_half``, ``clamp_warnings``), ``eval_brdf``, ``eval_material``,
``infer_proxy``, ``save_archive`` / ``load_archive``.  Every query runs in
the fused sm_100a kernels of ``libnmq.so``; there is no CPU path.

Two fused entry points go beyond the reference's per-stage calls:
``sample_pdf`` (fetch + sampler + sample + pdf, the renderer's BSDF-sampling
step, render.py:368-372 + 401-402) and ``query`` (one fetch feeding eval,
the sampler, sample and pdf).

Precision: ``fp16=True`` is the reference's fp16 inference path
(``NeuralMaterial.half()``: fp16 weights and texels, fp16-rounded layer-0
inputs, fp32 accumulation and fp32 hidden activations), reproduced on the
tensor cores with a hi/lo split of the hidden activations.
"""

import ctypes
import io
import json
import os
import struct

import numpy as np
import torch

from . import _io, _lib, mlp
from ._handle import DeviceMaterial
from .latent import LATENT_CHANNELS, LatentPyramid, read_pyramid, write_pyramid
from .proxy import ProxyParams

N_FRAMES = 2
PARAM_DIM = 9  # encoder input width (texture.py:25)
ARCHIVE_MAGIC = b"NMATARC1"


def parse_arch(s):
    n, w = s.lower().split("x")
    return (int(w),) * int(n)


class NeuralMaterialConfig:
    def __init__(self, brdf_hidden="2x32", sampler_hidden="3x32", encoder_hidden="3x32",
                 n_frames=N_FRAMES, albedo_head=False, use_frames=True, vanilla_extra_width=12,
                 sampler_isotropic=False, param_dim=PARAM_DIM, channels=LATENT_CHANNELS):
        self.brdf_hidden = brdf_hidden
        self.sampler_hidden = sampler_hidden
        self.encoder_hidden = encoder_hidden
        self.n_frames = n_frames
        self.albedo_head = albedo_head
        self.use_frames = use_frames
        self.vanilla_extra_width = vanilla_extra_width
        self.sampler_isotropic = sampler_isotropic
        self.param_dim = param_dim
        self.channels = channels

    def to_json(self):
        return dict(self.__dict__)

    @classmethod
    def from_json(cls, d):
        return cls(**d)


class NeuralMaterial:
    def __init__(self, cfg, encoder, frame_layer, brdf_decoder, sampler_decoder, latent=None):
        self.cfg = cfg
        self.encoder = encoder
        self.frame_layer = frame_layer
        self.brdf_decoder = brdf_decoder
        self.sampler_decoder = sampler_decoder
        self.latent = latent
        self._half = None
        self._dev = {}

    @classmethod
    def create(cls, cfg, rng):
        """Random init consuming `rng` in the reference's order (neural.py:117-141):
        frame layer, BRDF decoder, sampler decoder, encoder."""
        c = cfg.channels
        frame = None
        if cfg.use_frames:
            frame = mlp.Mlp.create((c, 6 * cfg.n_frames), rng, out_act=mlp.ACT_LINEAR,
                                   weight_scale=0.1)
            frame.layers[0].b[:] = np.tile([0.0, 0.0, 1.0, 1.0, 0.0, 0.0], cfg.n_frames)
            brdf_sizes = (c + 6 * cfg.n_frames, *parse_arch(cfg.brdf_hidden),
                          6 if cfg.albedo_head else 3)
        else:
            brdf_sizes = (c + 6, cfg.vanilla_extra_width, *parse_arch(cfg.brdf_hidden),
                          6 if cfg.albedo_head else 3)
        brdf = mlp.Mlp.create(brdf_sizes, rng)
        sampler = mlp.Mlp.create((c + 3, *parse_arch(cfg.sampler_hidden),
                                  2 if cfg.sampler_isotropic else 9), rng)
        encoder = mlp.Mlp.create((cfg.param_dim, *parse_arch(cfg.encoder_hidden), c), rng)
        return cls(cfg, encoder, frame, brdf, sampler)

    # --- fp16 inference copies and their device residency ------------------------
    def invalidate_half(self):
        self._half = None
        for h in self._dev.values():
            if hasattr(h, "close"):
                h.close()
        self._dev = {}

    def _master_fingerprint(self):
        """Checksum of the fp32 master weights and pyramid (in-place edits)."""
        parts = []
        for net in (self.frame_layer, self.brdf_decoder, self.sampler_decoder):
            if net is not None:
                for l in net.layers:
                    parts.append((np.asarray(l.w, np.float32).tobytes(), np.asarray(l.b, np.float32).tobytes()))
        lat = self.latent.fingerprint() if isinstance(self.latent, LatentPyramid) else None
        return hash(tuple(parts)), lat

    def half(self):
        if self._half is None:
            latent = None
            if isinstance(self.latent, LatentPyramid):
                latent = LatentPyramid([l.astype(np.float32) for l in self.latent.half_copy()])
                latent._frozen = True  # the reference caches its render copy too (neural.py:147-161)
            self._half = {
                "frame": mlp.quantize(self.frame_layer) if self.frame_layer is not None else None,
                "brdf": mlp.quantize(self.brdf_decoder),
                "sampler": mlp.quantize(self.sampler_decoder),
                "latent": latent,
            }
        return self._half

    def clamp_warnings(self):
        h = self.half()
        total = h["brdf"].clamped + h["sampler"].clamped
        if h["frame"] is not None:
            total += h["frame"].clamped
        return total

    def device_material(self, device=None, precise=False):
        """The immutable device copy on `device`, built once and cached like
        half(): fp16 weights re-tiled for tcgen05 + fp16 texels (the fp16
        inference path), or with `precise` the fp32 master weights (as fp16
        hi/lo pairs) + the fp32 master pyramid (the reference's fp16=False path)."""
        dev = _io.cuda_device(device)
        if precise:
            # the reference's fp16=False path reads the fp32 master weights and
            # pyramid live (neural.py:288-293): rebuild when either changed
            key = (dev.index, "fp32")
            h = self._dev.get(key)
            fp = self._master_fingerprint()
            if h is not None and self._dev.get((dev.index, "fp32-fp")) != fp:
                h.close()
                h = None
            if h is None:
                if isinstance(self.latent, DeviceLatent):
                    raise NotImplementedError(
                        "a device-only fp16 latent pyramid has no fp32 master copy (use fp16=True)")
                q = self.half()
                if self.latent is not None:
                    blob, fp32 = self.latent.texel_blob()
                    w, hh, nl = self.latent.width, self.latent.height, self.latent.n_levels
                else:
                    blob, fp32, w, hh, nl = np.zeros((1, 8), np.float32), True, 1, 1, 1
                h = DeviceMaterial(dev, w, hh, nl, blob, fp32, q["frame"], q["brdf"], q["sampler"],
                                   use_frames=self.cfg.use_frames, n_frames=self.cfg.n_frames,
                                   albedo_head=self.cfg.albedo_head,
                                   sampler_isotropic=self.cfg.sampler_isotropic,
                                   masters=(self.frame_layer, self.brdf_decoder, self.sampler_decoder))
                self._dev[key] = h
                self._dev[(dev.index, "fp32-fp")] = fp
            return h
        h = self._dev.get(dev.index)
        if h is None:
            q = self.half()
            lat = self.latent
            if isinstance(lat, DeviceLatent):
                blob, w, hh, nl = lat.texels, lat.width, lat.height, lat.n_levels
            elif lat is not None:
                blob = np.concatenate([l.reshape(-1, LATENT_CHANNELS) for l in lat.half_copy()])
                w, hh, nl = lat.width, lat.height, lat.n_levels
            else:  # latent-less material: eval_brdf / infer_proxy from given codes
                blob, w, hh, nl = np.zeros((1, 8), np.float16), 1, 1, 1
            h = DeviceMaterial(dev, w, hh, nl, blob, False, q["frame"], q["brdf"], q["sampler"],
                               use_frames=self.cfg.use_frames, n_frames=self.cfg.n_frames,
                               albedo_head=self.cfg.albedo_head,
                               sampler_isotropic=self.cfg.sampler_isotropic)
            self._dev[dev.index] = h
        return h


class DeviceLatent:
    """A latent pyramid that lives only on the device as fp16 texels
    (texels, 8) — for synthetic 4K..15K pyramids too large to build on the
    host.  Used as ``NeuralMaterial.latent`` by the benchmarks."""

    def __init__(self, texels, width, height):
        from .latent import level_shapes
        shapes = level_shapes(width, height)
        need = sum(h * w for h, w in shapes)
        if texels.dtype != torch.float16 or tuple(texels.shape) != (need, LATENT_CHANNELS):
            raise ValueError(f"expected ({need}, 8) fp16 texels")
        self.texels = texels.contiguous()
        self.width, self.height, self.n_levels = int(width), int(height), len(shapes)
        self.shapes = shapes

    @property
    def channels(self):
        return LATENT_CHANNELS

    def half_copy(self):
        out, ofs = [], 0
        host = self.texels.cpu().numpy()
        for h, w in self.shapes:
            out.append(host[ofs:ofs + h * w].reshape(h, w, 8))
            ofs += h * w
        return out


def _require_fp16(fp16):
    if not fp16:
        raise NotImplementedError("this entry point implements the fp16 inference path (fp16=True)")


def _launch(fn, *args):
    _lib.check(fn(*args), fn.__name__)


def eval_brdf(mat, z, wi, wo, fp16=False):
    """BRDF values (and albedo when enabled) from latent codes (neural.py:273-300).
    Directions below the horizon yield zero."""
    np_mode = _io.is_numpy_like(z)
    h = mat.device_material(None if np_mode else z.device, precise=not fp16)
    dev = h.device
    z_t = _io.as_rows(z, LATENT_CHANNELS, dev, "z")
    n = z_t.shape[0]
    # float64 directions fp32 cannot hold exactly stay float64: the reference
    # forms T.wi / T.wo from its float64 arrays (neural.py:280-287)
    d64 = _io.inexact_f64(wi) or _io.inexact_f64(wo)
    rows = _io.as_rows64 if d64 else _io.as_rows
    wi_t = rows(wi, 3, dev, "wi")
    wo_t = rows(wo, 3, dev, "wo")
    if wi_t.shape[0] != n or wo_t.shape[0] != n:
        raise ValueError("z, wi and wo must share the batch size")
    f = _io.empty(n, 3, dev)
    alb = _io.empty(n, 3, dev) if mat.cfg.albedo_head else None
    lib = _lib.load()
    _launch(lib.nm_eval_z_f64 if d64 else lib.nm_eval_z, h.ptr, n, z_t.data_ptr(), wi_t.data_ptr(),
            wo_t.data_ptr(), f.data_ptr(), _io.ptr(alb), _io.stream_ptr(dev))
    return _io.out(f, np_mode), (None if alb is None else _io.out(alb, np_mode))


class _QueryInputs:
    def __init__(self, mat, uv, level, u_rr, need, fp16=True, **dirs):
        self.np_mode = _io.is_numpy_like(uv)
        self.h = mat.device_material(None if self.np_mode else uv.device, precise=not fp16)
        dev = self.dev = self.h.device
        # float64 coordinates or directions fp32 cannot hold exactly keep
        # float64 (nm_query_f64: levels / taps / T.w as the reference forms them)
        self.f64 = any(_io.inexact_f64(x) for x in (uv, level, u_rr)) or \
            any(_io.inexact_f64(dirs[k]) for k in need if k in ("wi", "wo"))
        if self.f64:
            self.uv = _io.as_rows64(uv, 2, dev, "uv")
            n = self.n = self.uv.shape[0]
            self.lod, self.lod_stride = _io.as_vec64(level, n, dev, "level")
            self.urr, _ = _io.as_vec64(u_rr, n, dev, "u_rr")
        else:
            self.uv = _io.as_rows(uv, 2, dev, "uv")
            n = self.n = self.uv.shape[0]
            self.lod, self.lod_stride = _io.as_vec(level, n, dev, "level")
            self.urr, _ = _io.as_vec(u_rr, n, dev, "u_rr")
        for k in need:
            t = (_io.as_rows64 if self.f64 and k in ("wi", "wo") else _io.as_rows)(dirs[k], 3, dev, k)
            if t.shape[0] != n:
                raise ValueError(f"{k}: batch {t.shape[0]} != {n}")
            setattr(self, k, t)


def _host_eval(mat, uv, level, wi, wo, u_rr, out, return_level):
    """eval_material on host (numpy) arrays through nm_eval_host, all in
    native code: pinned buffers go zero-copy (one fused launch over PCIe),
    pageable ones stream in chunks (H2D / fused kernel / D2H overlapped on
    three internal streams).  Returns (f, albedo, level) with the reference's
    dtypes (f/albedo float64, level int64; f is `out` when given), or None if
    the arrays are not plain host rows."""
    n = np.shape(uv)[0] if np.ndim(uv) == 2 else 0
    if n == 0:
        return None
    if any(_io.inexact_f64(x) for x in (uv, level, u_rr, wi, wo)):
        return None  # float64 coordinates / directions: the device path's nm_query_f64
    h_uv, h_wi, h_wo = _io.host_rows(uv, 2, "uv"), _io.host_rows(wi, 3, "wi"), _io.host_rows(wo, 3, "wo")
    h_lod = np.ascontiguousarray(np.asarray(level, dtype=np.float32)).reshape(-1)
    h_urr = np.ascontiguousarray(np.asarray(u_rr, dtype=np.float32)).reshape(-1)
    if h_uv is None or h_wi is None or h_wo is None or h_urr.shape[0] != n \
            or h_lod.shape[0] not in (1, n) or h_wi.shape[0] != n or h_wo.shape[0] != n:
        return None
    if out is not None and (out.dtype != np.float32 or out.shape != (n, 3) or not out.flags.c_contiguous):
        return None
    h = mat.device_material(None)
    lib = _lib.load()
    lod_stride = int(h_lod.shape[0] == n)
    if out is None:
        # the reference's dtypes straight from the library (widened on the
        # device; pageable buffers through its pinned bounce pipeline)
        f = _io.result_array((n, 3), np.float64)
        alb = _io.result_array((n, 3), np.float64) if mat.cfg.albedo_head else None
        lv = _io.result_array((n,), np.int64) if return_level else None
        _launch(lib.nm_eval_host_ref, h.ptr, n, h_uv.ctypes.data, h_lod.ctypes.data, lod_stride,
                h_urr.ctypes.data, h_wi.ctypes.data, h_wo.ctypes.data, f.ctypes.data,
                None if alb is None else alb.ctypes.data, None if lv is None else lv.ctypes.data,
                _io.REF_CHUNK, _io.stream_ptr(h.device))
        return f, alb, lv
    alb = np.empty((n, 3), np.float32) if mat.cfg.albedo_head else None
    lv = np.empty(n, np.int32) if return_level else None
    _launch(lib.nm_eval_host, h.ptr, n, h_uv.ctypes.data, h_lod.ctypes.data, lod_stride,
            h_urr.ctypes.data, h_wi.ctypes.data, h_wo.ctypes.data, out.ctypes.data,
            None if alb is None else alb.ctypes.data, None if lv is None else lv.ctypes.data,
            _io.STREAM_CHUNK, _io.stream_ptr(h.device))
    return (out, None if alb is None else alb.astype(np.float64),
            None if lv is None else lv.astype(np.int64))


def eval_material(mat, uv, level, wi, wo, u_rr, fp16=False, return_level=True, out=None):
    """Fetch (Russian-roulette level + bilinear) and decode in ONE fused
    kernel, returning (f, albedo, chosen_level) (neural.py:303-309).
    `out` may pass a preallocated (B,3) fp32 device tensor, or a host (ideally
    pinned) fp32 buffer, for f.  Large host batches without albedo or level
    outputs stream through the GPU in overlapped chunks."""
    if fp16 and _io.is_numpy_like(uv) and (out is None or isinstance(out, np.ndarray)):
        r = _host_eval(mat, uv, level, wi, wo, u_rr, out, return_level)
        if r is not None:
            return r
    q = _QueryInputs(mat, uv, level, u_rr, ("wi", "wo"), fp16=fp16, wi=wi, wo=wo)
    on_dev = isinstance(out, torch.Tensor) and out.is_cuda
    f = out if on_dev else _io.empty(q.n, 3, q.dev)
    alb = _io.empty(q.n, 3, q.dev) if mat.cfg.albedo_head else None
    lv = _io.empty(q.n, 1, q.dev, torch.int32) if return_level else None
    lib = _lib.load()
    if q.f64:
        _launch(lib.nm_query_f64, q.h.ptr, _lib.NM_QUERY_EVAL, q.n, q.uv.data_ptr(), q.lod.data_ptr(),
                q.lod_stride, q.urr.data_ptr(), q.wi.data_ptr(), q.wo.data_ptr(), None, f.data_ptr(),
                _io.ptr(alb), None, None, None, _io.ptr(lv), _io.stream_ptr(q.dev))
    else:
        _launch(lib.nm_eval, q.h.ptr, q.n, q.uv.data_ptr(), q.lod.data_ptr(), q.lod_stride,
                q.urr.data_ptr(), q.wi.data_ptr(), q.wo.data_ptr(), f.data_ptr(), _io.ptr(alb),
                _io.ptr(lv), _io.stream_ptr(q.dev))
    if out is not None and not on_dev:  # host buffer (numpy or pinned CPU tensor)
        (torch.from_numpy(out) if isinstance(out, np.ndarray) else out).copy_(f)
        f_res = out
    else:
        f_res = _io.out(f, q.np_mode)
    return (f_res, None if alb is None else _io.out(alb, q.np_mode),
            None if lv is None else _io.out(lv, q.np_mode, np.int64))


def eval_material_spp(mat, uv, level, wi, wo, u_rr, spp, fp16=True, out=None):
    """eval_material reduced to the per-pixel mean over `spp` consecutive
    samples inside the kernel (the renderer's accumulation, render.py:565):
    rows are pixel * spp + s; returns the (B / spp, 3) image (fp32 tensor for
    torch callers, float64 numpy otherwise)."""
    _require_fp16(fp16)
    for x, name in ((uv, "uv"), (level, "level"), (u_rr, "u_rr"), (wi, "wi"), (wo, "wo")):
        _io.check_exact_f32(x, name)  # no float64 spp entry point
    q = _QueryInputs(mat, uv, level, u_rr, ("wi", "wo"), fp16=fp16, wi=wi, wo=wo)
    if spp <= 0 or spp & (spp - 1) or q.n % spp:
        raise ValueError("spp must be a power of two dividing the batch")
    img = out if isinstance(out, torch.Tensor) and out.is_cuda else _io.empty(q.n // spp, 3, q.dev)
    lib = _lib.load()
    _launch(lib.nm_eval_spp, q.h.ptr, q.n, q.uv.data_ptr(), q.lod.data_ptr(), q.lod_stride, q.urr.data_ptr(),
            q.wi.data_ptr(), q.wo.data_ptr(), int(spp), img.data_ptr(), _io.stream_ptr(q.dev))
    return _io.out(img, q.np_mode)


def infer_proxy(mat, z, wi, fp16=False):
    """Sampler parameters for latent codes and conditioning directions
    (neural.py:353-362 + proxy_from_raw :317-331)."""
    np_mode = _io.is_numpy_like(z)
    h = mat.device_material(None if np_mode else z.device, precise=not fp16)
    dev = h.device
    z_t = _io.as_rows(z, LATENT_CHANNELS, dev, "z")
    n = z_t.shape[0]
    wi_t = _io.as_rows(wi, 3, dev, "wi")
    if wi_t.shape[0] != n:
        raise ValueError("z and wi must share the batch size")
    p9 = _io.empty(n, 9, dev)
    lib = _lib.load()
    _launch(lib.nm_infer_proxy, h.ptr, n, z_t.data_ptr(), wi_t.data_ptr(), p9.data_ptr(),
            _io.stream_ptr(dev))
    return ProxyParams.from_block(p9, np_mode)


def sample_pdf(mat, uv, level, u_rr, wi, u, fp16=True, return_params=False, return_level=False):
    """Fused fetch + sampler decoder + proxy + sample + pdf: returns
    (ws, pdf[, params][, level]) with ws = sample(params, wi, u), pdf = pdf(params, wi, ws)."""
    q = _QueryInputs(mat, uv, level, u_rr, ("wi", "u"), fp16=fp16, wi=wi, u=u)
    ws = _io.empty(q.n, 3, q.dev)
    p = _io.empty(q.n, 1, q.dev)
    p9 = _io.empty(q.n, 9, q.dev) if return_params else None
    lv = _io.empty(q.n, 1, q.dev, torch.int32) if return_level else None
    lib = _lib.load()
    if q.f64:
        _launch(lib.nm_query_f64, q.h.ptr, _lib.NM_QUERY_SAMPLE_PDF, q.n, q.uv.data_ptr(), q.lod.data_ptr(),
                q.lod_stride, q.urr.data_ptr(), q.wi.data_ptr(), None, q.u.data_ptr(), None, None,
                ws.data_ptr(), p.data_ptr(), _io.ptr(p9), _io.ptr(lv), _io.stream_ptr(q.dev))
    else:
        _launch(lib.nm_sample_pdf, q.h.ptr, q.n, q.uv.data_ptr(), q.lod.data_ptr(), q.lod_stride,
                q.urr.data_ptr(), q.wi.data_ptr(), q.u.data_ptr(), ws.data_ptr(), p.data_ptr(),
                _io.ptr(p9), _io.ptr(lv), _io.stream_ptr(q.dev))
    res = (_io.out(ws, q.np_mode), _io.out(p, q.np_mode))
    if return_params:
        res = res + (ProxyParams.from_block(p9, q.np_mode),)
    if return_level:
        res = res + (_io.out(lv, q.np_mode, np.int64),)
    return res


def query(mat, uv, level, u_rr, wi, wo, u, fp16=True, return_level=False):
    """One full query (fetch -> eval(wi, wo) -> proxy(wi) -> sample(u) -> pdf):
    returns (f, ws, pdf[, level])."""
    q = _QueryInputs(mat, uv, level, u_rr, ("wi", "wo", "u"), fp16=fp16, wi=wi, wo=wo, u=u)
    f = _io.empty(q.n, 3, q.dev)
    ws = _io.empty(q.n, 3, q.dev)
    p = _io.empty(q.n, 1, q.dev)
    lv = _io.empty(q.n, 1, q.dev, torch.int32) if return_level else None
    lib = _lib.load()
    if q.f64:
        _launch(lib.nm_query_f64, q.h.ptr, _lib.NM_QUERY_FULL, q.n, q.uv.data_ptr(), q.lod.data_ptr(),
                q.lod_stride, q.urr.data_ptr(), q.wi.data_ptr(), q.wo.data_ptr(), q.u.data_ptr(), f.data_ptr(),
                None, ws.data_ptr(), p.data_ptr(), None, _io.ptr(lv), _io.stream_ptr(q.dev))
    else:
        _launch(lib.nm_query, q.h.ptr, q.n, q.uv.data_ptr(), q.lod.data_ptr(), q.lod_stride,
                q.urr.data_ptr(), q.wi.data_ptr(), q.wo.data_ptr(), q.u.data_ptr(), f.data_ptr(),
                ws.data_ptr(), p.data_ptr(), _io.ptr(lv), _io.stream_ptr(q.dev))
    res = (_io.out(f, q.np_mode), _io.out(ws, q.np_mode), _io.out(p, q.np_mode))
    if return_level:
        res = res + (_io.out(lv, q.np_mode, np.int64),)
    return res


MULTI_MODES = {"divergent": _lib.NM_MULTI_DIVERGENT, "binned": _lib.NM_MULTI_BINNED,
               "binned_async": _lib.NM_MULTI_BINNED_ASYNC}


def eval_material_multi(mats, mat_id, uv, level, wi, wo, u_rr, mode="binned", fp16=True, out=None):
    """Per-query material selection (the renderer's per-vertex material groups,
    render.py:352-356): f[i] = eval_material(mats[mat_id[i]], ...)[0][i].
    mode "binned" sorts queries into per-material segments with warp-level
    counting and runs the coherent fused kernel per segment (ids validated:
    one host round trip); "binned_async" skips the round trip (segment sizes
    stay on the device; out-of-range ids leave their rows untouched);
    "divergent" decodes mixed tiles directly.  Returns f (B, 3)."""
    _require_fp16(fp16)
    if mode not in MULTI_MODES:
        raise ValueError(f"mode must be one of {sorted(MULTI_MODES)}")
    mats = list(mats)
    if not mats:
        raise ValueError("no materials")
    np_mode = _io.is_numpy_like(uv)
    handles = [m.device_material(None if np_mode else uv.device) for m in mats]
    dev = handles[0].device
    if any(h.device != dev for h in handles):
        raise ValueError("materials must live on the same device")
    uv_t = _io.as_rows(uv, 2, dev, "uv", exact=True)
    n = uv_t.shape[0]
    lod_t, lod_stride = _io.as_vec(level, n, dev, "level", exact=True)
    urr_t, _ = _io.as_vec(u_rr, n, dev, "u_rr", exact=True)
    wi_t = _io.as_rows(wi, 3, dev, "wi")
    wo_t = _io.as_rows(wo, 3, dev, "wo")
    if isinstance(mat_id, torch.Tensor):
        ids = mat_id.to(device=dev, dtype=torch.int32).reshape(-1).contiguous()
    else:
        ids = torch.from_numpy(np.ascontiguousarray(np.asarray(mat_id).reshape(-1), np.int32)).to(dev)
    if ids.numel() != n or wi_t.shape[0] != n or wo_t.shape[0] != n:
        raise ValueError("mat_id, uv, wi and wo must share the batch size")
    f = out if isinstance(out, torch.Tensor) and out.is_cuda else _io.empty(n, 3, dev)
    lib = _lib.load()
    ws_bytes = int(lib.nm_multi_workspace_bytes(n, len(handles)))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    ptrs = (ctypes.c_void_p * len(handles))(*[h.ptr for h in handles])
    _launch(lib.nm_eval_multi, ptrs, len(handles), n, ids.data_ptr(), uv_t.data_ptr(),
            lod_t.data_ptr(), lod_stride, urr_t.data_ptr(), wi_t.data_ptr(), wo_t.data_ptr(),
            f.data_ptr(), MULTI_MODES[mode], ws.data_ptr(), ws_bytes, _io.stream_ptr(dev))
    return _io.out(f, np_mode)


def _multi_inputs(mats, mat_id, uv, level, u_rr, dirs):
    mats = list(mats)
    if not mats:
        raise ValueError("no materials")
    np_mode = _io.is_numpy_like(uv)
    handles = [m.device_material(None if np_mode else uv.device) for m in mats]
    dev = handles[0].device
    if any(h.device != dev for h in handles):
        raise ValueError("materials must live on the same device")
    uv_t = _io.as_rows(uv, 2, dev, "uv", exact=True)
    n = uv_t.shape[0]
    lod_t, lod_stride = _io.as_vec(level, n, dev, "level", exact=True)
    urr_t, _ = _io.as_vec(u_rr, n, dev, "u_rr", exact=True)
    d = {k: _io.as_rows(v, 3, dev, k, exact=k in ("wi", "wo")) for k, v in dirs.items()}
    if isinstance(mat_id, torch.Tensor):
        ids = mat_id.to(device=dev, dtype=torch.int32).reshape(-1).contiguous()
    else:
        ids = torch.from_numpy(np.ascontiguousarray(np.asarray(mat_id).reshape(-1), np.int32)).to(dev)
    if ids.numel() != n or any(t.shape[0] != n for t in d.values()):
        raise ValueError("mat_id, uv and the directions must share the batch size")
    lib = _lib.load()
    ws_bytes = int(lib.nm_multi_workspace_bytes(n, len(handles)))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    ptrs = (ctypes.c_void_p * len(handles))(*[h.ptr for h in handles])
    return np_mode, dev, n, ptrs, len(handles), ids, uv_t, lod_t, lod_stride, urr_t, d, ws, ws_bytes


def sample_pdf_multi(mats, mat_id, uv, level, u_rr, wi, u, mode="binned", fp16=True, return_params=False):
    """sample_pdf with a material per row (the renderer's per-vertex material
    groups for the sampler side, render.py:361-372, 391-409): binned by
    material id on the device; returns (ws, pdf[, params])."""
    _require_fp16(fp16)
    if mode not in MULTI_MODES:
        raise ValueError(f"mode must be one of {sorted(MULTI_MODES)}")
    np_mode, dev, n, ptrs, k, ids, uv_t, lod_t, stride, urr_t, d, wsp, ws_bytes = _multi_inputs(
        mats, mat_id, uv, level, u_rr, {"wi": wi, "u": u})
    ws = _io.empty(n, 3, dev)
    p = _io.empty(n, 1, dev)
    p9 = _io.empty(n, 9, dev) if return_params else None
    lib = _lib.load()
    _launch(lib.nm_sample_pdf_multi, ptrs, k, n, ids.data_ptr(), uv_t.data_ptr(), lod_t.data_ptr(), stride,
            urr_t.data_ptr(), d["wi"].data_ptr(), d["u"].data_ptr(), ws.data_ptr(), p.data_ptr(), _io.ptr(p9),
            MULTI_MODES[mode], wsp.data_ptr(), ws_bytes, _io.stream_ptr(dev))
    res = (_io.out(ws, np_mode), _io.out(p, np_mode))
    if return_params:
        res = res + (ProxyParams.from_block(p9, np_mode),)
    return res


def query_multi(mats, mat_id, uv, level, u_rr, wi, wo, u, mode="binned", fp16=True):
    """query() with a material per row: (f, ws, pdf), binned on the device."""
    _require_fp16(fp16)
    if mode not in MULTI_MODES:
        raise ValueError(f"mode must be one of {sorted(MULTI_MODES)}")
    np_mode, dev, n, ptrs, k, ids, uv_t, lod_t, stride, urr_t, d, wsp, ws_bytes = _multi_inputs(
        mats, mat_id, uv, level, u_rr, {"wi": wi, "wo": wo, "u": u})
    f = _io.empty(n, 3, dev)
    ws = _io.empty(n, 3, dev)
    p = _io.empty(n, 1, dev)
    lib = _lib.load()
    _launch(lib.nm_query_multi, ptrs, k, n, ids.data_ptr(), uv_t.data_ptr(), lod_t.data_ptr(), stride,
            urr_t.data_ptr(), d["wi"].data_ptr(), d["wo"].data_ptr(), d["u"].data_ptr(), f.data_ptr(),
            ws.data_ptr(), p.data_ptr(), MULTI_MODES[mode], wsp.data_ptr(), ws_bytes, _io.stream_ptr(dev))
    return _io.out(f, np_mode), _io.out(ws, np_mode), _io.out(p, np_mode)


# --- archive (NMATARC1, neural.py:368-419) -------------------------------------

def save_archive(path, mat, include_encoder=False):
    latent_name = None
    if mat.latent is not None:
        latent_name = os.path.basename(os.path.splitext(path)[0]) + ".latents"
        with open(os.path.join(os.path.dirname(path), latent_name), "wb") as f:
            write_pyramid(f, mat.latent)
    header = {
        "config": mat.cfg.to_json(),
        "latent_file": latent_name,
        "has_encoder": bool(include_encoder and mat.encoder is not None),
        "clamped_warnings": mat.clamp_warnings(),
    }
    hbytes = json.dumps(header, sort_keys=True).encode("utf-8")
    with open(path, "wb") as f:
        f.write(ARCHIVE_MAGIC)
        f.write(struct.pack("<I", len(hbytes)))
        f.write(hbytes)
        if mat.cfg.use_frames:
            mlp.write_blob(f, mat.frame_layer)
        mlp.write_blob(f, mat.brdf_decoder)
        mlp.write_blob(f, mat.sampler_decoder)
        if header["has_encoder"]:
            mlp.write_blob(f, mat.encoder)


def load_archive(path):
    with open(path, "rb") as f:
        if f.read(8) != ARCHIVE_MAGIC:
            raise ValueError("not a neural material archive")
        (hlen,) = struct.unpack("<I", f.read(4))
        header = json.loads(f.read(hlen).decode("utf-8"))
        cfg = NeuralMaterialConfig.from_json(header["config"])
        frame = mlp.read_blob(f)[0] if cfg.use_frames else None
        brdf = mlp.read_blob(f)[0]
        sampler = mlp.read_blob(f)[0]
        encoder = mlp.read_blob(f)[0] if header.get("has_encoder") else None
    latent = None
    if header.get("latent_file"):
        with open(os.path.join(os.path.dirname(path), header["latent_file"]), "rb") as f:
            latent = read_pyramid(f)
    return NeuralMaterial(cfg, encoder, frame, brdf, sampler, latent)
