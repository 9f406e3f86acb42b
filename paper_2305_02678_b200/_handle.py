"""Owner of one ``nm_material*`` (an immutable device copy of a material:
re-tiled fp16 weights + latent texels) — the replacement for the
reference's lazily built ``NeuralMaterial.half()`` cache (neural.py:147-161)."""

import ctypes

import numpy as np
import torch

from . import _lib
from .mlp import ACT_CODES


def _net_desc(qnet, keep, master=None):
    """Fill an NetDesc from a QuantizedMlp (or an empty one for None); with
    `master` (the fp32 Mlp) also its fp32 weights in the same access order."""
    d = _lib.NetDesc()
    if qnet is None:
        d.n_layers = 0
        return d
    if master is not None:
        w32 = np.ascontiguousarray(np.concatenate(
            [np.concatenate([l.w, l.b[:, None]], axis=1).ravel() for l in master.layers]), np.float32)
        keep.append(w32)
        d.weights = w32.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
    fi = np.ascontiguousarray([s[1] for s in qnet.shapes], dtype=np.int32)
    fo = np.ascontiguousarray([s[0] for s in qnet.shapes], dtype=np.int32)
    act = np.ascontiguousarray([ACT_CODES[a] for a in qnet.acts], dtype=np.int32)
    packed = np.ascontiguousarray(qnet.packed.view(np.uint16))
    keep.extend([fi, fo, act, packed])
    d.n_layers = len(qnet.shapes)
    d.fan_in = fi.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    d.fan_out = fo.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    d.act = act.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    d.packed = packed.ctypes.data_as(ctypes.POINTER(ctypes.c_uint16))
    return d


class DeviceMaterial:
    """One material resident on one CUDA device."""

    def __init__(self, device, width, height, n_levels, latent, latent_fp32=False,
                 frame=None, brdf=None, sampler=None, use_frames=True, n_frames=2,
                 albedo_head=False, sampler_isotropic=False, masters=None):
        lib = _lib.load()
        keep = []
        desc = _lib.MaterialDesc()
        desc.channels = 8
        desc.use_frames = int(bool(use_frames))
        desc.n_frames = int(n_frames)
        desc.albedo_head = int(bool(albedo_head))
        desc.sampler_isotropic = int(bool(sampler_isotropic))
        m = masters or (None, None, None)  # fp32 Mlps: the precise (fp16=False) path
        desc.precise = int(masters is not None)
        desc.frame = _net_desc(frame if use_frames else None, keep, m[0])
        desc.brdf = _net_desc(brdf, keep, m[1])
        desc.sampler = _net_desc(sampler, keep, m[2])
        desc.width, desc.height, desc.n_levels = int(width), int(height), int(n_levels)
        desc.latent_fp32 = int(bool(latent_fp32))
        if isinstance(latent, torch.Tensor):
            if latent.device.type != "cuda" or latent.device.index != device.index:
                latent = latent.to(device)
            latent = latent.contiguous()
            keep.append(latent)
            desc.latent = latent.data_ptr()
            desc.latent_on_device = 1
        else:
            arr = np.ascontiguousarray(latent)
            keep.append(arr)
            desc.latent = arr.ctypes.data
            desc.latent_on_device = 0
        handle = ctypes.c_void_p()
        with torch.cuda.device(device):
            rc = lib.nm_material_create(ctypes.byref(desc), device.index, ctypes.byref(handle))
        _lib.check(rc, "nm_material_create")
        self.ptr = handle.value
        self.device = device
        self._lib = lib
        info = _lib.MaterialInfo()
        _lib.check(lib.nm_material_info_get(self.ptr, ctypes.byref(info)))
        self.info = info

    def level_table(self):
        n = self.info.n_levels
        w = np.zeros(n, np.int32)
        h = np.zeros(n, np.int32)
        off = np.zeros(n, np.int64)
        _lib.check(self._lib.nm_material_levels(self.ptr, w.ctypes.data, h.ctypes.data, off.ctypes.data))
        return w, h, off

    def close(self):
        if getattr(self, "ptr", None):
            self._lib.nm_material_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
