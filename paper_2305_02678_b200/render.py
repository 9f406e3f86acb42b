"""Level of detail from ray cones — the renderer step that produces the
fractional lod consumed by the query path (reference ``render.py``:
``footprint_to_level`` :334-337 and the footprint inside
``_surface_frames_and_level`` :423-445).  Only these functions of the
reference renderer are on the query path; the path tracer itself is out of
scope.

Both run on the GPU (csrc/nmq_lod.cu) in float64 like the reference.
numpy in -> numpy out (float64, the reference's dtype); torch CUDA in ->
torch out on the same device (``cone_level`` returns the fp32 lod the query
entry points take, so it can feed ``neural.eval_material`` directly).
"""

import numpy as np
import torch

from . import _io, _lib


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
