"""Analytic two-lobe sampling proxy — drop-in for ``neuralmat.proxy``.

``ProxyParams`` holds the renderer's 9-float per-query block (wd, ws, mu_d,
alpha, rho, mu_s; reference proxy.py:37-84) as one (B, 9) fp32 device tensor.
``sample`` (proxy.py:168-180) and ``pdf`` (proxy.py:129-135) run on the GPU
(``nm_sample`` / ``nm_pdf``).  Numpy callers get float64 numpy results like
the reference; torch callers get fp32 device tensors.
"""

import numpy as np
import torch

from . import _io, _lib

ALPHA_FLOOR = 1e-4
RHO_CLAMP = float(np.sqrt(1.0 - 1e-4))


class ProxyParams:
    __slots__ = ("data", "_np")

    def __init__(self, wd, ws, mu_d, alpha, rho, mu_s, device=None):
        """Reference constructor signature; floors alpha, clamps rho
        (proxy.py:42-50)."""
        np_mode = all(_io.is_numpy_like(v) for v in (wd, ws, mu_d, alpha, rho, mu_s))
        if np_mode:
            wd = np.atleast_1d(np.asarray(wd, np.float64))
            ws = np.atleast_1d(np.asarray(ws, np.float64))
            mu_d = np.atleast_2d(np.asarray(mu_d, np.float64))
            alpha = np.maximum(np.atleast_2d(np.asarray(alpha, np.float64)), ALPHA_FLOOR)
            rho = np.clip(np.atleast_1d(np.asarray(rho, np.float64)), -RHO_CLAMP, RHO_CLAMP)
            mu_s = np.atleast_2d(np.asarray(mu_s, np.float64))
            block = np.concatenate([wd[:, None], ws[:, None], mu_d, alpha, rho[:, None], mu_s], axis=1)
            dev = _io.cuda_device(device)
            self.data = torch.from_numpy(np.ascontiguousarray(block, np.float32)).to(dev)
        else:
            dev = _io.cuda_device(device if device is not None else next(
                v.device for v in (wd, ws, mu_d, alpha, rho, mu_s) if isinstance(v, torch.Tensor)))

            def col(v, k):
                t = v if isinstance(v, torch.Tensor) else torch.as_tensor(np.asarray(v, np.float32))
                t = t.to(dev, torch.float32)
                return t.reshape(-1, k)

            a = col(alpha, 2).clamp_min(ALPHA_FLOOR)
            r = col(rho, 1).clamp(-RHO_CLAMP, RHO_CLAMP)
            self.data = torch.cat([col(wd, 1), col(ws, 1), col(mu_d, 2), a, r, col(mu_s, 2)], 1).contiguous()
        self._np = np_mode

    @classmethod
    def from_block(cls, block, numpy_mode=False):
        """Wrap a (B, 9) fp32 device tensor produced by the kernels."""
        p = cls.__new__(cls)
        p.data = block
        p._np = numpy_mode
        return p

    def __len__(self):
        return self.data.shape[0]

    def _col(self, sl):
        t = self.data[:, sl]
        return t.cpu().numpy().astype(np.float64) if self._np else t

    @property
    def wd(self):
        return self._col(0)

    @property
    def ws(self):
        return self._col(1)

    @property
    def mu_d(self):
        return self._col(slice(2, 4))

    @property
    def alpha(self):
        return self._col(slice(4, 6))

    @property
    def rho(self):
        return self._col(6)

    @property
    def mu_s(self):
        return self._col(slice(7, 9))

    @property
    def s(self):
        r = self.rho
        return np.sqrt(1.0 - r ** 2) if self._np else torch.sqrt(1.0 - r * r)

    def det(self):
        """alpha_x * alpha_y * sqrt(1 - rho^2) (proxy.py:76-78)."""
        a = self.alpha
        return a[:, 0] * a[:, 1] * self.s

    def matrix(self):
        """The 3x3 slope warp M per batch entry (proxy.py:64-74)."""
        a, r, s, ms = self.alpha, self.rho, self.s, self.mu_s
        z = np.zeros if self._np else (lambda n: torch.zeros(n, device=self.data.device))
        o = np.ones if self._np else (lambda n: torch.ones(n, device=self.data.device))
        n = len(self)
        rows = [[a[:, 0], z(n), -ms[:, 0]], [a[:, 1] * r, a[:, 1] * s, -ms[:, 1]], [z(n), z(n), o(n)]]
        if self._np:
            return np.stack([np.stack(rw, -1) for rw in rows], 1)
        return torch.stack([torch.stack(rw, -1) for rw in rows], 1)

    def diffuse_normal(self):
        """Axis of the tilted cosine lobe, normalize(-mu_d.x, -mu_d.y, 1) (proxy.py:80-84)."""
        md = self.mu_d
        if self._np:
            v = np.stack([-md[:, 0], -md[:, 1], np.ones(len(self))], -1)
            return v / np.linalg.norm(v, axis=-1, keepdims=True)
        v = torch.stack([-md[:, 0], -md[:, 1], torch.ones(len(self), device=md.device)], -1)
        return v / v.norm(dim=-1, keepdim=True)

    def take(self, idx):
        if isinstance(idx, np.ndarray):
            idx = torch.from_numpy(idx).to(self.data.device)
        return ProxyParams.from_block(self.data[idx].reshape(-1, 9).contiguous(), self._np)

    def as_array(self):
        return self.data.cpu().numpy().astype(np.float64)


def _dirs(x, n, dev, name):
    t = _io.as_rows(x, 3, dev, name)
    if t.shape[0] != n:
        if t.shape[0] == 1:
            t = t.expand(n, 3).contiguous()
        else:
            raise ValueError(f"{name}: batch {t.shape[0]} does not match params batch {n}")
    return t


def sample(params, wi, u):
    """Map u in [0,1)^3 to an outgoing direction (may be below the horizon)."""
    dev = params.data.device
    n = len(params)
    np_mode = params._np or _io.is_numpy_like(wi)
    wi_t = _dirs(wi, n, dev, "wi")
    u_t = _dirs(u, n, dev, "u")
    wo = _io.empty(n, 3, dev)
    lib = _lib.load()
    _lib.check(lib.nm_sample(n, params.data.data_ptr(), wi_t.data_ptr(), u_t.data_ptr(),
                             wo.data_ptr(), _io.stream_ptr(dev)), "nm_sample")
    return _io.out(wo, np_mode)


def pdf(params, wi, wo):
    """Mixture density w_d p_d(wo) + w_s p_s(wi, wo)."""
    dev = params.data.device
    n = len(params)
    np_mode = params._np or _io.is_numpy_like(wi)
    wi_t = _dirs(wi, n, dev, "wi")
    wo_t = _dirs(wo, n, dev, "wo")
    p = _io.empty(n, 1, dev)
    lib = _lib.load()
    _lib.check(lib.nm_pdf(n, params.data.data_ptr(), wi_t.data_ptr(), wo_t.data_ptr(),
                          p.data_ptr(), _io.stream_ptr(dev)), "nm_pdf")
    return _io.out(p, np_mode)


def normalize_check(params, wi, n_samples, rng, chunk=2_000_000):
    """MC estimate of the full-sphere integral of pdf by uniform-sphere
    sampling (proxy.py:183-196); the pdf runs on the GPU (nm_pdf)."""
    if len(params) != 1:
        raise ValueError("normalize_check expects a single parameter set")
    total, done = 0.0, 0
    while done < n_samples:
        m = min(chunk, n_samples - done)
        u = rng.random((m, 2))
        z = 1.0 - 2.0 * u[:, 0]
        r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
        phi = 2.0 * np.pi * u[:, 1]
        d = np.stack([r * np.cos(phi), r * np.sin(phi), z], -1)  # geom.sample_uniform_sphere
        rep = params.take(np.zeros(m, dtype=np.int64))
        total += float(np.sum(pdf(rep, np.broadcast_to(np.asarray(wi, np.float64), (m, 3)), d)))
        done += m
    return total * 4.0 * np.pi / n_samples
