"""Seeded synthetic workloads (BASELINE.json configs C1..C5), generated on
the device with torch's Philox generator so 2M..530M-query batches and
4K..15K latent pyramids never touch the host.

Directions follow the reference's benchmark recipe:
(wi, wo) from half/difference vectors with both above the horizon
(reference geom.py:138-173, re-drawn by rejection), uv ~ U[0,1)^2,
lod ~ U[0, L-1), u_rr ~ U[0,1), u3 ~ U[0,1)^3, all fp32.
"""

import math

import numpy as np
import torch

from .latent import level_shapes
from .neural import DeviceLatent, NeuralMaterial, NeuralMaterialConfig

# C4: five texture sets sized from the paper's Table 1
C4_RESOLUTIONS = [(15360, 15360), (3712, 3712), (8192, 8192), (4480, 4480), (7104, 7104)]


def device_latent(width, height, seed, device):
    """Standard-normal latents, one draw for the whole pyramid, stored as
    the fp16 render copy (texels, 8)."""
    n = sum(h * w for h, w in level_shapes(width, height))
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    t = torch.empty((n, 8), device=device, dtype=torch.float32)
    chunk = 1 << 24
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        t[s:e].normal_(generator=g)
    return DeviceLatent(t.to(torch.float16), width, height)


def material(brdf_hidden="2x32", width=4096, height=4096, seed=0, device="cuda", **cfg):
    """Random-init material (reference init order) + device latent pyramid."""
    mat = NeuralMaterial.create(NeuralMaterialConfig(brdf_hidden=brdf_hidden, **cfg),
                                np.random.default_rng(seed))
    mat.latent = device_latent(width, height, seed + 1000, torch.device(device))
    return mat


def _hemisphere(u1, u2):
    z = 1.0 - u1
    r = torch.sqrt(torch.clamp(1.0 - z * z, min=0.0))
    phi = 2.0 * math.pi * u2
    return torch.stack([r * torch.cos(phi), r * torch.sin(phi), z], -1)


def _frame_from_normal(n):
    # fallback tangent: n x e_k, k = argmin |n_k|  (geom.py:82-93)
    k = torch.argmin(n.abs(), dim=-1)
    e = torch.nn.functional.one_hot(k, 3).to(n.dtype)
    t0 = torch.linalg.cross(n, e)
    t0 = t0 / t0.norm(dim=-1, keepdim=True)
    c = torch.linalg.cross(n, t0)
    b = c / c.norm(dim=-1, keepdim=True)
    t = torch.linalg.cross(b, n)
    return t, b, n


def direction_pairs(n, gen, device):
    """(wi, wo), both with z > 0, via half/difference vectors."""
    wi = torch.empty((n, 3), device=device)
    wo = torch.empty((n, 3), device=device)
    got = 0
    while got < n:
        m = max(64, int(2.3 * (n - got)))
        u = torch.rand((m, 4), device=device, generator=gen, dtype=torch.float64)
        h = _hemisphere(u[:, 0], u[:, 1])
        d = _hemisphere(u[:, 2], u[:, 3])
        t, b, nn = _frame_from_normal(h)
        a = d[:, 0:1] * t + d[:, 1:2] * b + d[:, 2:3] * nn
        r = 2.0 * (a * h).sum(-1, keepdim=True) * h - a
        ok = torch.nonzero((a[:, 2] > 0) & (r[:, 2] > 0)).squeeze(1)[: n - got]
        k = ok.numel()
        wi[got:got + k] = a[ok].float()
        wo[got:got + k] = r[ok].float()
        got += k
    return wi, wo


def queries(n, n_levels, seed, device, need=("uv", "lod", "u_rr", "wi", "wo", "u3")):
    device = torch.device(device)
    gen = torch.Generator(device=device)
    gen.manual_seed(int(seed))
    out = {}
    out["uv"] = torch.rand((n, 2), device=device, generator=gen)
    out["lod"] = torch.rand((n,), device=device, generator=gen) * (n_levels - 1)
    out["u_rr"] = torch.rand((n,), device=device, generator=gen)
    out["wi"], out["wo"] = direction_pairs(n, gen, device)
    out["u3"] = torch.rand((n, 3), device=device, generator=gen)
    return {k: v.contiguous() for k, v in out.items() if k in need}

