"""Training-side kernels — drop-ins for the reference's
network engine and latent-gradient scatter used by its offline baking loop
(``training.py``):

* ``forward_cached(net, x)`` / ``backward(net, cache, out_grad)`` —
  ``Mlp.forward_cached`` / ``Mlp.backward`` (reference mlp.py:90-116):
  float32 forward, float64 reverse chain (the reference promotes to float64
  at its first leaky layer), dW = g^T x and db = sum g reduced over the
  batch on the GPU (csrc/nmq_train.cu).
* ``sampler_loss_and_grads(mat, z, wi, rng, target_and_grad=None, us=None)``
  — the KL sampler loss (training.py:219-273): network passes on the fp32
  engine, float64 per-row heads in csrc/nmq_kl.cu.
* ``accumulate_texel_grads(pyramid, grad_levels, uv, chosen, z_grad)`` —
  ``LatentPyramid.accumulate_texel_grads`` (latent.py:109-119): the exact
  adjoint of the fetch, scattered with atomics; adds into ``grad_levels``
  in place like the reference.

numpy in -> numpy out with the reference's dtypes; the device work is on
the current CUDA stream.  Also attached as ``Mlp.forward_cached`` /
``Mlp.backward`` and ``LatentPyramid.accumulate_texel_grads``.
"""

import ctypes

import numpy as np
import torch

from . import _io, _lib
from .latent import LATENT_CHANNELS, LatentPyramid
from .mlp import ACT_CODES, ACT_LINEAR, Mlp


def _weights(net):
    return np.ascontiguousarray(np.concatenate(
        [np.concatenate([l.w, l.b[:, None]], axis=1).ravel() for l in net.layers]), np.float32)


class _DeviceMlp:
    """nm_mlp handle for one network on one device (weights re-uploaded per
    forward_cached call so an optimizer step between calls is always seen)."""

    def __init__(self, net, dev):
        lib = _lib.load()
        self.keep = []
        d = _lib.NetDesc()
        fi = np.ascontiguousarray([l.w.shape[1] for l in net.layers], np.int32)
        fo = np.ascontiguousarray([l.w.shape[0] for l in net.layers], np.int32)
        act = np.ascontiguousarray([ACT_CODES[l.act] for l in net.layers], np.int32)
        w32 = _weights(net)
        self.keep += [fi, fo, act, w32]
        d.n_layers = len(net.layers)
        d.fan_in = fi.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        d.fan_out = fo.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        d.act = act.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        d.weights = w32.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        h = ctypes.c_void_p()
        with torch.cuda.device(dev):
            _lib.check(lib.nm_mlp_create(ctypes.byref(d), dev.index, ctypes.byref(h)), "nm_mlp_create")
        self.ptr, self.dev, self.lib = h.value, dev, lib
        self.shapes = [l.w.shape for l in net.layers]

    def set_weights(self, net):
        """Re-upload only when the weights changed since the last upload
        (an optimizer step in between); a synchronous copy otherwise costs a
        host round trip per call."""
        w32 = _weights(net)
        if np.array_equal(w32, self.keep[3]):
            return
        with torch.cuda.device(self.dev):
            _lib.check(self.lib.nm_mlp_set_weights(self.ptr, w32.ctypes.data), "nm_mlp_set_weights")
        self.keep[3] = w32

    def __del__(self):
        try:
            self.lib.nm_mlp_destroy(self.ptr)
        except Exception:
            pass


class GpuCache:
    """What backward needs from forward_cached (device buffers)."""

    def __init__(self, handle, batch, buf, np_mode):
        self.handle, self.batch, self.buf, self.np_mode = handle, batch, buf, np_mode


def _handle(net, dev):
    shapes = [l.w.shape for l in net.layers]
    h = getattr(net, "_gpu", None)
    if h is None or h.dev != dev or h.shapes != shapes:
        h = _DeviceMlp(net, dev)
        net._gpu = h
    else:
        h.set_weights(net)
    return h


def forward_cached(net, x):
    """(out (B, out) float32, cache) — reference Mlp.forward_cached (mlp.py:90-101)."""
    np_mode = _io.is_numpy_like(x)
    dev = _io.cuda_device(None if np_mode else x.device)
    xt = _io.as_rows(x, net.layers[0].w.shape[1], dev, "x")
    if xt.dim() == 1:
        xt = xt[None, :]
    B = xt.shape[0]
    h = _handle(net, dev)
    lib = _lib.load()
    out = torch.empty((B, net.layers[-1].w.shape[0]), device=dev, dtype=torch.float32)
    buf = torch.empty(max(1, int(lib.nm_mlp_cache_bytes(h.ptr, B))), device=dev, dtype=torch.uint8)
    _lib.check(lib.nm_mlp_forward_cached(h.ptr, B, xt.data_ptr(), out.data_ptr(), buf.data_ptr(),
                                         _io.stream_ptr(dev)), "nm_mlp_forward_cached")
    cache = GpuCache(h, B, buf, np_mode)
    return (out.cpu().numpy() if np_mode else out), cache


def backward(net, cache, out_grad):
    """([(dW, db), ...], dx) of sum(out * out_grad) — reference Mlp.backward
    (mlp.py:103-116); float64 except the last layer's (dW, db) when it is
    linear, float32 like the reference."""
    h, B, dev = cache.handle, cache.batch, cache.handle.dev
    g = _io.as_rows(out_grad, net.layers[-1].w.shape[0], dev, "out_grad")
    if g.dim() == 1:
        g = g[None, :]
    if g.shape[0] != B:
        raise ValueError("output gradient shape mismatch")
    lib = _lib.load()
    n_params = int(lib.nm_mlp_params(h.ptr))
    dp = torch.empty(n_params, device=dev, dtype=torch.float64)
    dx = torch.empty((B, net.layers[0].w.shape[1]), device=dev, dtype=torch.float64)
    _lib.check(lib.nm_mlp_backward(h.ptr, B, cache.buf.data_ptr(), g.data_ptr(), dp.data_ptr(),
                                   dx.data_ptr(), _io.stream_ptr(dev)), "nm_mlp_backward")
    grads, o = [], 0
    for i, l in enumerate(net.layers):
        fo, fi = l.w.shape
        blk = dp[o:o + fo * (fi + 1)].reshape(fo, fi + 1)
        o += fo * (fi + 1)
        dw, db = blk[:, :fi], blk[:, fi]
        if i == len(net.layers) - 1 and l.act == ACT_LINEAR:  # reference keeps float32 here
            dw, db = dw.float(), db.float()
        grads.append((dw, db))
    if cache.np_mode:
        return [(a.cpu().numpy(), b.cpu().numpy()) for a, b in grads], dx.cpu().numpy()
    return grads, dx


def accumulate_texel_grads(pyramid, grad_levels, uv, chosen, z_grad):
    """Scatter z_grad onto the four bilinear taps of each query at its chosen
    level, ADDING into grad_levels in place (latent.py:109-119).  grad_levels:
    the reference's list of per-level (H, W, C) float32 arrays, or one device
    tensor (texels, 8) float32 in the pyramid's level layout."""
    if pyramid.channels != LATENT_CHANNELS:
        raise NotImplementedError("the GPU scatter handles 8-channel latents")
    list_mode = isinstance(grad_levels, (list, tuple))
    np_mode = _io.is_numpy_like(uv)
    h = pyramid.device_material(None if np_mode else uv.device)
    dev = h.device
    uv_t = _io.as_rows(uv, 2, dev, "uv")
    n = uv_t.shape[0]
    if isinstance(chosen, torch.Tensor):
        lv = chosen.to(device=dev, dtype=torch.int32).reshape(-1)
    else:
        lv = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(np.asarray(chosen), (n,)), np.int32)).to(dev)
    if lv.numel() == 1 and n != 1:
        lv = lv.expand(n).contiguous()
    zg = _io.as_rows(z_grad, LATENT_CHANNELS, dev, "z_grad")
    if zg.shape[0] != n or lv.numel() != n:
        raise ValueError("uv, chosen and z_grad must share the batch size")
    if list_mode:
        flat = torch.from_numpy(np.concatenate(
            [np.asarray(g, np.float32).reshape(-1, LATENT_CHANNELS) for g in grad_levels])).to(dev)
    else:
        flat = grad_levels
    lib = _lib.load()
    _lib.check(lib.nm_texel_grads(h.ptr, n, uv_t.data_ptr(), lv.data_ptr(), zg.data_ptr(),
                                  flat.data_ptr(), _io.stream_ptr(dev)), "nm_texel_grads")
    if list_mode:
        host = flat.cpu().numpy()
        o = 0
        for g in grad_levels:
            k = g.shape[0] * g.shape[1]
            g[...] = host[o:o + k].reshape(g.shape)
            o += k
    return grad_levels


def sampler_loss_and_grads(mat, z, wi, rng, target_and_grad=None, us=None):
    """KL-style sampler loss and its gradients for the sampler decoder —
    reference training.sampler_loss_and_grads (training.py:219-273) with the
    default target _brdf_target_and_grad (training.py:187-216).

    Returns (loss, grads), grads in Mlp.backward's layout.  The three network
    passes (sampler forward, BRDF decoder forward + input backward at the 2B
    samples, sampler backward) run on the fp32 network engine; the per-row
    heads (proxy, the two lobe samples, the luminance target and its
    direction derivative through the frames, grad log pdf, the sample and raw
    Jacobians) are float64 CUDA kernels (csrc/nmq_kl.cu).  `us` fixes the
    two (b, 2) uniform draws, else they come from `rng` in the reference's
    order; `target_and_grad(wo) -> (f (b,), df (b, 3))` replaces the default
    target (called on host arrays, like the reference's gradient oracles).
    numpy in -> numpy out (float64 loss, the reference's gradient dtypes)."""
    cfg = mat.cfg
    if cfg.channels != LATENT_CHANNELS:
        raise NotImplementedError("the GPU sampler loss handles 8-channel latents")
    np_mode = _io.is_numpy_like(z)
    dev = _io.cuda_device(None if np_mode else z.device)
    if np_mode:
        z64 = np.atleast_2d(np.asarray(z, np.float64))
        wi64 = np.atleast_2d(np.asarray(wi, np.float64))
        zt = torch.from_numpy(np.ascontiguousarray(z64, np.float32)).to(dev)
        wit = torch.from_numpy(np.ascontiguousarray(wi64)).to(dev)
    else:
        zt = z.to(dev, torch.float32).reshape(-1, LATENT_CHANNELS).contiguous()
        wit = (wi if isinstance(wi, torch.Tensor) else torch.as_tensor(np.asarray(wi, np.float64))) \
            .to(dev, torch.float64).reshape(-1, 3).contiguous()
    b = zt.shape[0]
    if wit.shape[0] != b or zt.shape[1] != LATENT_CHANNELS:
        raise ValueError("z must be (b, 8) and wi (b, 3)")
    iso = bool(cfg.sampler_isotropic)
    lib = _lib.load()
    st = _io.stream_ptr(dev)
    inp = torch.cat([zt.double(), wit], 1).float().contiguous()
    raw, cache = forward_cached(mat.sampler_decoder, inp)
    u_d, u_s = us if us is not None else (rng.random((b, 2)), rng.random((b, 2)))
    ud, us_t = ((u.to(dev, torch.float64).contiguous() if isinstance(u, torch.Tensor)
                 else torch.from_numpy(np.ascontiguousarray(u, np.float64)).to(dev)) for u in (u_d, u_s))
    frames = bool(cfg.use_frames)
    nf = int(cfg.n_frames) if frames else 0
    raw_f = forward_cached(mat.frame_layer, zt)[0] if frames else None
    in_w = LATENT_CHANNELS + (6 * nf if frames else 6)
    x2 = torch.empty((2 * b, in_w), device=dev, dtype=torch.float32)
    scr = torch.empty((b, _lib.NM_KL_SCRATCH), device=dev, dtype=torch.float64)
    _lib.check(lib.nm_kl_sample(b, int(frames), nf, int(iso), raw.data_ptr(), _io.ptr(raw_f), zt.data_ptr(),
                                wit.data_ptr(), ud.data_ptr(), us_t.data_ptr(), x2.data_ptr(), scr.data_ptr(),
                                st), "nm_kl_sample")
    if target_and_grad is None:
        y, cache_b = forward_cached(mat.brdf_decoder, x2)
        out_w = y.shape[1]
        tgt = torch.empty(2 * b, device=dev, dtype=torch.float64)
        lum = torch.empty(2 * b, device=dev, dtype=torch.float64)
        og = torch.empty((2 * b, out_w), device=dev, dtype=torch.float32)
        _lib.check(lib.nm_kl_target(b, out_w, y.data_ptr(), scr.data_ptr(), tgt.data_ptr(), lum.data_ptr(),
                                    og.data_ptr(), st), "nm_kl_target")
        _, dx = backward(mat.brdf_decoder, cache_b, og)
        dtgt = torch.empty((2 * b, 3), device=dev, dtype=torch.float64)
        _lib.check(lib.nm_kl_target_dir(b, int(frames), nf, _io.ptr(raw_f), dx.data_ptr(), scr.data_ptr(),
                                        lum.data_ptr(), dtgt.data_ptr(), st), "nm_kl_target_dir")
    else:
        host = scr.cpu().numpy()
        f_d, df_d = target_and_grad(host[:, 0:3])
        f_s, df_s = target_and_grad(host[:, 3:6])
        tgt = torch.from_numpy(np.concatenate([np.asarray(f_d, np.float64).reshape(-1),
                                               np.asarray(f_s, np.float64).reshape(-1)])).to(dev)
        dtgt = torch.from_numpy(np.ascontiguousarray(np.concatenate(
            [np.asarray(df_d, np.float64).reshape(-1, 3), np.asarray(df_s, np.float64).reshape(-1, 3)]))).to(dev)
    draw = torch.empty((b, 2 if iso else 9), device=dev, dtype=torch.float32)
    rows = torch.empty(b, device=dev, dtype=torch.float64)
    _lib.check(lib.nm_kl_grad(b, int(iso), raw.data_ptr(), wit.data_ptr(), scr.data_ptr(), tgt.data_ptr(),
                              dtgt.data_ptr(), draw.data_ptr(), rows.data_ptr(), st), "nm_kl_grad")
    loss = float(np.mean(rows.cpu().numpy()))
    grads, _ = backward(mat.sampler_decoder, cache, draw)
    if np_mode:
        grads = [(dw.cpu().numpy(), db.cpu().numpy()) for dw, db in grads]
    return loss, grads


# drop-in methods, as on the reference's classes
Mlp.forward_cached = forward_cached
Mlp.backward = backward
LatentPyramid.accumulate_texel_grads = accumulate_texel_grads
LatentPyramid.zero_grads = lambda self: [np.zeros_like(l) for l in self.levels]
