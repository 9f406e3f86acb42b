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
