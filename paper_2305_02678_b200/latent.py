"""Hierarchical 8-channel latent texture — drop-in for ``neuralmat.latent``.

``LatentPyramid.fetch`` (reference latent.py:84-98) runs on the GPU through
``nm_fetch``: Russian-roulette level choice (latent.py:76-82) and
wrap-addressed bilinear taps (latent.py:56-74) computed exactly like the
reference (float64 texel coordinates), so chosen levels and tap indices are
bit-identical, and the blend is float64 like the reference's, so z is
bit-identical too.

Like the reference, a pyramid's ``levels`` may be edited in place between
fetches (the baking loop's Adam step, training.py:305-356): the device copy
is refreshed whenever the levels' content changed (a full-array checksum per
fetch).  The fp16 render copy built by ``NeuralMaterial.half()`` is cached
until ``invalidate_half()``, exactly like the reference's (neural.py:144-161).

Texels are uploaded as fp16 when every value is fp16-representable (the
render copy ``half_copy()``, which is what the fp16 query path reads) and as
fp32 otherwise, so a fetch always sees exactly the pyramid's values.
"""

import struct

import numpy as np
import torch

from . import _io, _lib
from ._handle import DeviceMaterial

LATENT_CHANNELS = 8
PYRAMID_MAGIC = b"NLATPYR1"


def level_shapes(width, height):
    """(h, w) per level: halve with max(1, .//2) until 1x1 (latent.py:28-38)."""
    out, w, h = [], int(width), int(height)
    while True:
        out.append((h, w))
        if w == 1 and h == 1:
            return out
        w, h = max(1, w // 2), max(1, h // 2)


class LatentPyramid:
    def __init__(self, levels):
        c = levels[0].shape[2] if levels and levels[0].ndim == 3 else None
        for lvl in levels:
            if lvl.ndim != 3 or lvl.shape[2] != c:
                raise ValueError("levels must be (H, W, C) with a shared C")
        self.levels = [np.ascontiguousarray(l, dtype=np.float32) for l in levels]
        self._dev = {}
        self._fp = {}
        self._frozen = False  # True for the cached render copy (NeuralMaterial.half())

    @classmethod
    def zeros(cls, width, height, channels=LATENT_CHANNELS):
        return cls([np.zeros((h, w, channels), np.float32) for h, w in level_shapes(width, height)])

    @property
    def n_levels(self):
        return len(self.levels)

    @property
    def channels(self):
        return self.levels[0].shape[2]

    @property
    def width(self):
        return self.levels[0].shape[1]

    @property
    def height(self):
        return self.levels[0].shape[0]

    def invalidate(self):
        """Drop device copies (they are also refreshed automatically when the
        levels' content changes)."""
        for h in self._dev.values():
            h.close()
        self._dev = {}
        self._fp = {}

    def fingerprint(self):
        """Content checksum of every level (float32 bits: wrapping sum and xor
        of 64-bit words, plus the shapes) — detects in-place edits."""
        out = []
        for l in self.levels:
            a = np.ascontiguousarray(l, dtype=np.float32)
            flat = a.reshape(-1)
            if flat.size % 2:
                flat = np.concatenate([flat, np.zeros(1, np.float32)])
            u = flat.view(np.uint64)
            out.append((a.shape, int(np.add.reduce(u, dtype=np.uint64)), int(np.bitwise_xor.reduce(u))))
        return tuple(out)

    def half_copy(self):
        """fp16 render copy: clip to +-65504, round to nearest even (latent.py:124-126)."""
        return [np.clip(l, -65504, 65504).astype(np.float16) for l in self.levels]

    def texel_blob(self):
        """(texels, C) array of all levels back to back, fp16 when exact."""
        flat = np.concatenate([l.reshape(-1, self.channels) for l in self.levels])
        h = flat.astype(np.float16)
        if np.array_equal(h.astype(np.float32), flat, equal_nan=True):
            return h, False
        return flat, True

    def device_material(self, device=None):
        dev = _io.cuda_device(device)
        h = self._dev.get(dev.index)
        if h is not None and not self._frozen:
            if self._fp.get(dev.index) != self.fingerprint():  # levels edited in place
                h.close()
                h = None
        if h is None:
            if [l.shape[:2] for l in self.levels] != level_shapes(self.width, self.height):
                raise ValueError("levels do not follow the max(1, n//2) halving chain")
            blob, fp32 = self.texel_blob()
            h = DeviceMaterial(dev, self.width, self.height, self.n_levels, blob, latent_fp32=fp32)
            self._dev[dev.index] = h
            if not self._frozen:
                self._fp[dev.index] = self.fingerprint()
        return h

    def fetch(self, uv, level, u_rr, return_taps=False):
        """(z (B,C) float32, chosen (B,) int64); torch in -> torch out."""
        if self.channels != LATENT_CHANNELS:
            raise NotImplementedError("the GPU fetch handles 8-channel latents")
        np_mode = _io.is_numpy_like(uv)
        h = self.device_material(None if np_mode else uv.device)
        dev = h.device
        # float64 coordinates fp32 cannot hold exactly stay float64 (nm_fetch_f64)
        f64 = any(_io.inexact_f64(x) for x in (uv, level, u_rr))
        rows, vec = (_io.as_rows64, _io.as_vec64) if f64 else (_io.as_rows, _io.as_vec)
        uv_t = rows(uv, 2, dev, "uv")
        n = uv_t.shape[0]
        lod_t, lod_stride = vec(level, n, dev, "level")
        urr_t, _ = vec(u_rr, n, dev, "u_rr")
        z = _io.empty(n, 8, dev)
        lv = _io.empty(n, 1, dev, torch.int32)
        taps = _io.empty(n, 8, dev, torch.int32) if return_taps else None
        wts = _io.empty(n, 4, dev) if return_taps else None
        lib = _lib.load()
        fn = lib.nm_fetch_f64 if f64 else lib.nm_fetch
        _lib.check(fn(h.ptr, n, uv_t.data_ptr(), lod_t.data_ptr(), lod_stride, urr_t.data_ptr(), z.data_ptr(),
                      lv.data_ptr(), _io.ptr(taps), _io.ptr(wts), _io.stream_ptr(dev)), fn.__name__)
        res = (_io.out(z, np_mode, np.float32), _io.out(lv, np_mode, np.int64))
        if return_taps:
            t = taps.reshape(n, 4, 2)
            xs, ys = t[..., 0], t[..., 1]
            res = res + (_io.out(xs, np_mode, np.int64), _io.out(ys, np_mode, np.int64),
                         _io.out(wts, np_mode, np.float64))
        return res

    def fetch_trilinear(self, uv, level):
        """Deterministic trilinear fetch (optional filtering mode): the roulette
        fetch's expectation (1 - f) bilinear(floor l) + f bilinear(ceil l)
        (latent.py:84-92), float64 from the two fp32 bilinear fetches."""
        if self.channels != LATENT_CHANNELS:
            raise NotImplementedError("the GPU fetch handles 8-channel latents")
        np_mode = _io.is_numpy_like(uv)
        h = self.device_material(None if np_mode else uv.device)
        dev = h.device
        uv_t = _io.as_rows(uv, 2, dev, "uv", exact=True)
        n = uv_t.shape[0]
        lod_t, lod_stride = _io.as_vec(level, n, dev, "level", exact=True)
        z = _io.empty(n, 8, dev)
        lib = _lib.load()
        _lib.check(lib.nm_fetch_trilinear(h.ptr, n, uv_t.data_ptr(), lod_t.data_ptr(), lod_stride, z.data_ptr(),
                                          None, _io.stream_ptr(dev)), "nm_fetch_trilinear")
        return _io.out(z, np_mode, np.float32)

    def fetch_level(self, uv, level):
        """Deterministic fetch at integer `level` (latent.py:100-107)."""
        n = np.atleast_2d(np.asarray(uv) if _io.is_numpy_like(uv) else uv.cpu().numpy()).shape[0]
        zeros = np.zeros(n, np.float32) if _io.is_numpy_like(uv) else torch.zeros(n, device=uv.device)
        return self.fetch(uv, float(int(level)), zeros)[0]


def write_pyramid(stream, pyr):
    """NLATPYR1 file: magic, <IIII w,h,levels,channels, fp16 levels (latent.py:157-163)."""
    stream.write(PYRAMID_MAGIC)
    stream.write(struct.pack("<IIII", pyr.width, pyr.height, pyr.n_levels, pyr.channels))
    for lvl in pyr.half_copy():
        stream.write(lvl.astype("<f2").tobytes())


def read_pyramid(stream):
    """latent.py:166-179"""
    if stream.read(8) != PYRAMID_MAGIC:
        raise ValueError("not a latent pyramid file")
    w, h, n_levels, c = struct.unpack("<IIII", stream.read(16))
    shapes = level_shapes(w, h)
    if len(shapes) != n_levels:
        raise ValueError("corrupt pyramid header")
    levels = []
    for hh, ww in shapes:
        data = np.frombuffer(stream.read(2 * hh * ww * c), dtype="<f2")
        if data.size != hh * ww * c:
            raise ValueError("truncated pyramid file")
        levels.append(data.reshape(hh, ww, c).astype(np.float32))
    return LatentPyramid(levels)
