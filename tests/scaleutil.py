"""Test infrastructure for parity at the BASELINE configs' real sizes:
the oracle (oracle/nm_oracle.py) evaluated on a seeded subset of a batch
whose material lives on the GPU (4096^2 .. 15360^2 pyramids generated on the
device).  Only tests import this module."""

import numpy as np
import torch

from oracle import nm_oracle as O


def oracle_material(mat, handle):
    """The oracle's copy of a device material: the same fp16 networks, and a
    pyramid whose taps are gathered from the device latent buffer."""
    def net(m):
        return None if m is None else O.Net([(l.w, l.b, l.act) for l in m.layers])

    om = O.Material(O.Config(**mat.cfg.to_json()), net(mat.frame_layer), net(mat.brdf_decoder),
                    net(mat.sampler_decoder))
    w, h, off = handle.level_table()
    lat = mat.latent.texels  # (texels, 8) fp16 on the device
    off_t = torch.as_tensor(off, device=lat.device)
    w_t = torch.as_tensor(w.astype(np.int64), device=lat.device)

    def gather(level, ys, xs):
        gid = off_t[level] + torch.as_tensor(ys, device=lat.device) * w_t[level] + torch.as_tensor(
            xs, device=lat.device)
        return lat[gid].float().cpu().numpy()

    shapes = [(int(hh), int(ww)) for ww, hh in zip(w, h)]
    pyr = O.GatherPyramid(shapes, gather)
    om._half = {"frame": O.quantize(om.frame) if om.frame is not None else None,
                "brdf": O.quantize(om.brdf), "sampler": O.quantize(om.sampler), "latent": pyr}
    return om


def subset_rows(n, k, seed=0):
    """~k rows: a stride sample over the whole batch plus the partial last tile."""
    stride = max(1, n // k)
    rows = np.arange(0, n, stride)
    last = np.arange((n // 128) * 128, n)
    rng = np.random.default_rng(seed)
    extra = rng.integers(0, n, size=min(4096, n))
    return np.unique(np.concatenate([rows, last, extra]))


def host(q, rows):
    return {k: v[torch.as_tensor(rows, device=v.device)].cpu().numpy() for k, v in q.items()}
