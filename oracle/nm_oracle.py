"""CPU oracle for the neural-material query path — TEST INFRASTRUCTURE ONLY.

This module is a from-scratch numpy restatement of the reference
implementation's query hot path (``/root/reference/pkg/src/neuralmat``,
"neuralmat", arXiv 2305.02678).  It exists so that

* ``tests/`` can check the CUDA kernels against a CPU implementation on the
  GPU box (where ``/root/reference`` does not exist), and
* ``bench.py`` can time a CPU baseline (``cpu_baseline`` / ``--impl
  reference``).

It is NEVER imported by the product package ``paper_2305_02678_b200`` (the
product path has no CPU fallback).  Parity of this restatement with the real
reference is pinned by ``tests/test_oracle_golden.py`` against golden vectors
that ``oracle/make_golden.py`` produced by importing the reference itself.

Arithmetic follows the reference exactly: float64 for texel coordinates,
bilinear weights, frames and proxy math; float32 GEMMs over fp16-rounded
inputs for the "fused" fp16 path.  Each function cites the reference
``file:line`` it restates (paths relative to ``pkg/src/neuralmat``).
"""

import numpy as np

LATENT_CHANNELS = 8          # latent.py:17
LEAKY_SLOPE = 0.01           # mlp.py:16
FP16_MAX = 65504.0           # mlp.py:17
ALPHA_FLOOR = 1e-4           # proxy.py:32
RHO_CLAMP = np.sqrt(1.0 - 1e-4)  # proxy.py:33
PARAM_DIM = 9                # texture.py:25 (encoder input width)
N_FRAMES = 2                 # neural.py:30

ACT_LINEAR = "linear"
ACT_LEAKY = "leaky_relu"


# ---------------------------------------------------------------------------
# geometry helpers (geom.py)

def _unit(v):
    """geom.py:23-24"""
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def _mirror(w, m):
    """geom.py:31-33: 2 (w.m) m - w"""
    return 2.0 * np.sum(w * m, axis=-1)[..., None] * m - w


def fallback_tangent(n):
    """geom.py:82-89: n x e_k, k = argmin |n_k| (first index on ties)."""
    n = np.asarray(n, dtype=np.float64)
    k = np.argmin(np.abs(n), axis=-1)
    e = np.zeros_like(n)
    e[np.arange(n.shape[0]), k] = 1.0
    return _unit(np.cross(n, e))


def uniform_sphere(u):
    """geom.py:121-126"""
    u = np.asarray(u, dtype=np.float64)
    z = 1.0 - 2.0 * u[..., 0]
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    phi = 2.0 * np.pi * u[..., 1]
    return np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=-1)


def uniform_hemisphere(u):
    """geom.py:112-118"""
    u = np.asarray(u, dtype=np.float64)
    z = 1.0 - u[..., 0]
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    phi = 2.0 * np.pi * u[..., 1]
    return np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=-1)


def _basis_from_normal(n):
    """geom.py:60-93 (frame_from_normal = orthonormal_frame(n, fallback))."""
    t0 = fallback_tangent(n)
    c = np.cross(n, t0)
    b = c / np.linalg.norm(c, axis=-1, keepdims=True)
    nn = _unit(n)
    t = np.cross(b, nn)
    return t, b, nn


def half_diff_directions(u):
    """geom.py:138-151: (wi, wo) from half/difference vectors."""
    u = np.asarray(u, dtype=np.float64)
    h = uniform_hemisphere(u[..., 0:2])
    d = uniform_hemisphere(u[..., 2:4])
    t, b, n = _basis_from_normal(h)
    wi = d[..., 0:1] * t + d[..., 1:2] * b + d[..., 2:3] * n
    return wi, _mirror(wi, h)


def draw_direction_pairs(rng, n):
    """geom.py:154-173: rejection loop keeping pairs with both z > 0."""
    wi = np.empty((n, 3))
    wo = np.empty((n, 3))
    got = 0
    while got < n:
        need = n - got
        m = max(64, int(2.3 * need))
        a, b = half_diff_directions(rng.random((m, 4)))
        keep = np.flatnonzero((a[:, 2] > 0.0) & (b[:, 2] > 0.0))[:need]
        wi[got:got + keep.size] = a[keep]
        wo[got:got + keep.size] = b[keep]
        got += keep.size
    return wi, wo


# ---------------------------------------------------------------------------
# latent pyramid (latent.py)

def pyramid_shapes(width, height):
    """latent.py:28-38: halve with max(1, .//2) until 1x1."""
    shapes = []
    w, h = width, height
    while True:
        shapes.append((h, w))
        if w == 1 and h == 1:
            return shapes
        w, h = max(1, w // 2), max(1, h // 2)


class Pyramid:
    """Latent pyramid: list of (H, W, C) float32 levels (latent.py:21-26)."""

    def __init__(self, levels):
        self.levels = [np.ascontiguousarray(l, dtype=np.float32) for l in levels]

    @property
    def n_levels(self):
        return len(self.levels)

    def half_levels(self):
        """latent.py:124-126: clip to +-65504, RNE to fp16."""
        return [np.clip(l, -FP16_MAX, FP16_MAX).astype(np.float16) for l in self.levels]

    def render_copy(self):
        """neural.py:150-154: fp16 texels widened back to fp32."""
        return Pyramid([l.astype(np.float32) for l in self.half_levels()])

    def taps(self, level, uv):
        """latent.py:56-74: wrap-addressed bilinear taps in float64."""
        h, w = self.levels[level].shape[:2]
        uv = np.asarray(uv, dtype=np.float64)
        x = uv[..., 0] * w - 0.5
        y = uv[..., 1] * h - 0.5
        xf, yf = np.floor(x), np.floor(y)
        fx, fy = x - xf, y - yf
        x0 = xf.astype(np.int64) % w
        y0 = yf.astype(np.int64) % h
        x1 = (x0 + 1) % w
        y1 = (y0 + 1) % h
        gx, gy = 1.0 - fx, 1.0 - fy
        wts = np.stack([gx * gy, fx * gy, gx * fy, fx * fy], axis=-1)
        return (np.stack([x0, x1, x0, x1], axis=-1),
                np.stack([y0, y0, y1, y1], axis=-1), wts)

    def choose_level(self, level, u_rr):
        """latent.py:76-82: Russian-roulette level pick."""
        top = self.n_levels - 1
        lv = np.clip(np.asarray(level, dtype=np.float64), 0, top)
        lo = np.floor(lv)
        pick = lo + (np.asarray(u_rr) < (lv - lo))
        return np.clip(pick, 0, top).astype(np.int64)

    def fetch(self, uv, level, u_rr):
        """latent.py:84-98 -> (z (B,C) float32, chosen (B,) int64)."""
        uv = np.atleast_2d(np.asarray(uv, dtype=np.float64))
        chosen = self.choose_level(np.broadcast_to(level, uv.shape[:-1]), u_rr)
        z = np.empty(uv.shape[:-1] + (self.levels[0].shape[2],), dtype=np.float32)
        for lv in np.unique(chosen):
            m = chosen == lv
            xs, ys, wts = self.taps(int(lv), uv[m])
            tex = self.levels[int(lv)][ys, xs]
            z[m] = np.sum(tex * wts[..., None], axis=-2, dtype=np.float64)
        return z, chosen

    def accumulate_texel_grads(self, grad_levels, uv, chosen, z_grad):
        """latent.py:109-119: exact adjoint of fetch — scatter z_grad onto the
        four bilinear taps of each query (float64 contributions added into the
        caller's float32 gradient images)."""
        uv = np.atleast_2d(np.asarray(uv, dtype=np.float64))
        chosen = np.broadcast_to(chosen, uv.shape[:-1])
        z_grad = np.asarray(z_grad)
        for l in np.unique(chosen):
            sel = chosen == l
            xs, ys, wts = self.taps(int(l), uv[sel])
            contrib = wts[..., None] * z_grad[sel][..., None, :]
            np.add.at(grad_levels[int(l)], (ys, xs), contrib)

    def fetch_level(self, uv, level):
        """latent.py:100-107: deterministic fetch at one integer level."""
        uv = np.atleast_2d(np.asarray(uv, dtype=np.float64))
        xs, ys, wts = self.taps(int(level), uv)
        tex = self.levels[int(level)][ys, xs]
        return np.sum(tex * wts[..., None], axis=-2, dtype=np.float64).astype(np.float32)


class GatherPyramid(Pyramid):
    """A pyramid whose texels live elsewhere (the 4K..15K pyramids of the
    BASELINE configs, resident on the GPU): the same fetch as Pyramid.fetch
    (latent.py:84-98) — float64 taps, weights and weighted sum, narrowed to
    float32 — with the four taps of each query read through
    ``gather(level, ys, xs) -> (..., 4, C) float32``."""

    def __init__(self, shapes, gather, channels=LATENT_CHANNELS):
        # zero-size stand-ins: taps() only reads each level's (H, W)
        self.levels = [np.empty((h, w, 0), np.float32) for h, w in shapes]
        self.gather = gather
        self.channels = channels

    def fetch(self, uv, level, u_rr):
        uv = np.atleast_2d(np.asarray(uv, dtype=np.float64))
        chosen = self.choose_level(np.broadcast_to(level, uv.shape[:-1]), u_rr)
        z = np.empty(uv.shape[:-1] + (self.channels,), dtype=np.float32)
        for lv in np.unique(chosen):
            m = chosen == lv
            xs, ys, wts = self.taps(int(lv), uv[m])
            tex = np.asarray(self.gather(int(lv), ys, xs), np.float32)
            z[m] = np.sum(tex * wts[..., None], axis=-2, dtype=np.float64)
        return z, chosen


def fetch_trilinear(pyr, uv, level):
    """Deterministic trilinear fetch: the expectation of the roulette fetch
    over u_rr, stated in latent.py:84-92 and checked by
    tests/test_acceptance.py:242-255 — (1 - f) * fetch_level(floor l) +
    f * fetch_level(ceil l), l clipped to [0, L-1] as in choose_level
    (latent.py:76-82), evaluated in float64 from the two float32 bilinear
    fetches (latent.py:100-107) and narrowed to float32."""
    uv = np.atleast_2d(np.asarray(uv, dtype=np.float64))
    lv = np.clip(np.broadcast_to(np.asarray(level, dtype=np.float64), uv.shape[:-1]), 0, pyr.n_levels - 1)
    lo = np.floor(lv)
    f = lv - lo
    hi = np.minimum(lo + 1, pyr.n_levels - 1)
    z = np.empty(uv.shape[:-1] + (pyr.levels[0].shape[2],), dtype=np.float32)
    for l in np.unique(lo):
        m = lo == l
        a = pyr.fetch_level(uv[m], int(l)).astype(np.float64)
        h = int(min(l + 1, pyr.n_levels - 1))
        b = pyr.fetch_level(uv[m], h).astype(np.float64)
        fm = f[m][:, None]
        z[m] = ((1.0 - fm) * a + fm * b).astype(np.float32)
    return z


def random_pyramid(rng, width, height, channels=LATENT_CHANNELS):
    """Synthetic latents, one standard_normal draw per level in order
    (the reference tests' generator, tests/test_latent.py:10-14)."""
    return Pyramid([rng.standard_normal((h, w, channels)).astype(np.float32)
                    for h, w in pyramid_shapes(width, height)])


# ---------------------------------------------------------------------------
# MLP engine (mlp.py)

def _act(x, act):
    """mlp.py:27-30"""
    return x if act == ACT_LINEAR else np.where(x >= 0.0, x, LEAKY_SLOPE * x)


class Net:
    """fp32 master network: list of (w (out,in) f32, b (out,) f32, act)."""

    def __init__(self, layers):
        self.layers = [(np.ascontiguousarray(w, np.float32), np.ascontiguousarray(b, np.float32), a)
                       for w, b, a in layers]

    @classmethod
    def random(cls, sizes, rng, out_act=ACT_LINEAR, weight_scale=1.0):
        """mlp.py:57-69: He-style fan-in uniform init, zero biases; the RNG
        is consumed layer by layer exactly like the reference."""
        layers = []
        last = len(sizes) - 2
        for i in range(len(sizes) - 1):
            fan_in, fan_out = sizes[i], sizes[i + 1]
            bound = weight_scale * np.sqrt(6.0 / fan_in)
            w = rng.uniform(-bound, bound, size=(fan_out, fan_in))
            layers.append((w, np.zeros(fan_out), out_act if i == last else ACT_LEAKY))
        return cls(layers)

    @property
    def in_dim(self):
        return self.layers[0][0].shape[1]

    @property
    def out_dim(self):
        return self.layers[-1][0].shape[0]

    def forward(self, x):
        """mlp.py:79-88: fp32 forward."""
        x = np.asarray(x, dtype=np.float32)
        for w, b, a in self.layers:
            x = _act(x @ w.T + b, a)
        return x


def _act_grad(pre, act):
    """mlp.py:33-36 (a float64 array for leaky layers: the reference's
    backward promotes to float64 from the first leaky layer on)."""
    return 1.0 if act == ACT_LINEAR else np.where(pre >= 0.0, 1.0, LEAKY_SLOPE)


def forward_cached(net, x):
    """mlp.py:90-101: fp32 forward keeping every layer input and pre-activation."""
    x = np.asarray(x, dtype=np.float32)
    inputs, pres = [x], []
    for w, b, a in net.layers:
        pre = inputs[-1] @ w.T + b
        pres.append(pre)
        inputs.append(_act(pre, a))
    return inputs[-1], (inputs, pres)


def backward(net, cache, out_grad):
    """mlp.py:103-116: gradients of sum(out * out_grad) -> ([(dW, db)], dx)."""
    inputs, pres = cache
    g = np.asarray(out_grad, dtype=np.float32)
    grads = [None] * len(net.layers)
    for i in range(len(net.layers) - 1, -1, -1):
        w, b, a = net.layers[i]
        g = g * _act_grad(pres[i], a)
        grads[i] = (g.T @ inputs[i], g.sum(axis=0))
        g = g @ w
    return grads, g


class HalfNet:
    """Quantized network (mlp.py:165-233): fp16 weights packed per layer as
    [w_row(fan_in), bias] per output neuron."""

    def __init__(self, shapes, acts, packed, clamped=0):
        self.shapes = list(shapes)
        self.acts = list(acts)
        self.packed = np.asarray(packed, dtype=np.float16)
        self.clamped = clamped
        self.views = []
        ofs = 0
        for out, fan_in in self.shapes:
            blk = self.packed[ofs:ofs + out * (fan_in + 1)].reshape(out, fan_in + 1)
            self.views.append((blk[:, :fan_in].astype(np.float32),
                               blk[:, fan_in].astype(np.float32)))
            ofs += out * (fan_in + 1)

    def forward(self, x):
        """mlp.py:196-208: round input to fp16 once, fp32 layers after."""
        x = np.asarray(x).astype(np.float16).astype(np.float32)
        for (w, b), a in zip(self.views, self.acts):
            x = _act(x @ w.T + b, a)
        return x


def quantize(net):
    """mlp.py:214-233: clamp to +-65504 (counted), RNE fp16, access order."""
    parts, shapes, acts, clamped = [], [], [], 0
    for w, b, a in net.layers:
        blk = np.concatenate([w, b[:, None]], axis=1)
        clamped += int(np.count_nonzero(np.abs(blk) > FP16_MAX))
        parts.append(np.clip(blk, -FP16_MAX, FP16_MAX).astype(np.float16).ravel())
        shapes.append(w.shape)
        acts.append(a)
    return HalfNet(shapes, acts, np.concatenate(parts), clamped)


# ---------------------------------------------------------------------------
# neural material (neural.py)

def brdf_output(y):
    """neural.py:37-39"""
    return np.maximum(np.expm1(np.minimum(y, 60.0)), 0.0)


def quad_tanh(x):
    """neural.py:46-49"""
    ax = np.abs(x)
    return np.clip(x * (1.0 + 0.5 * ax) / (1.0 + ax + 0.5 * x * x), -1.0, 1.0)


def quad_sinh(x):
    """neural.py:58-60"""
    return x * (1.0 + x * x / 6.0)


def softmax_pair(a, b):
    """neural.py:67-71"""
    m = np.maximum(a, b)
    ea, eb = np.exp(a - m), np.exp(b - m)
    return ea / (ea + eb), eb / (ea + eb)


def parse_arch(s):
    """neural.py:77-79: "NxW" -> (W,)*N"""
    n, w = s.lower().split("x")
    return (int(w),) * int(n)


class Config:
    """neural.py:82-96 (same field names and defaults)."""

    def __init__(self, brdf_hidden="2x32", sampler_hidden="3x32", encoder_hidden="3x32",
                 n_frames=N_FRAMES, albedo_head=False, use_frames=True,
                 vanilla_extra_width=12, sampler_isotropic=False, param_dim=PARAM_DIM,
                 channels=LATENT_CHANNELS):
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


class Material:
    """Networks + latents of one neural material (neural.py:106-161)."""

    def __init__(self, cfg, frame, brdf, sampler, encoder=None, latent=None):
        self.cfg = cfg
        self.frame = frame
        self.brdf = brdf
        self.sampler = sampler
        self.encoder = encoder
        self.latent = latent
        self._half = None

    @classmethod
    def random(cls, cfg, rng):
        """neural.py:117-141 (RNG consumed in the same order: frame layer,
        BRDF decoder, sampler decoder, encoder)."""
        c = cfg.channels
        brdf_out = 6 if cfg.albedo_head else 3
        frame = None
        if cfg.use_frames:
            frame = Net.random((c, 6 * cfg.n_frames), rng, weight_scale=0.1)
            w, _, a = frame.layers[0]
            frame.layers[0] = (w, np.tile(np.float32([0, 0, 1, 1, 0, 0]), cfg.n_frames), a)
            sizes = (c + 6 * cfg.n_frames, *parse_arch(cfg.brdf_hidden), brdf_out)
        else:
            sizes = (c + 6, cfg.vanilla_extra_width, *parse_arch(cfg.brdf_hidden), brdf_out)
        brdf = Net.random(sizes, rng)
        sampler = Net.random((c + 3, *parse_arch(cfg.sampler_hidden),
                              2 if cfg.sampler_isotropic else 9), rng)
        encoder = Net.random((cfg.param_dim, *parse_arch(cfg.encoder_hidden), c), rng)
        return cls(cfg, frame, brdf, sampler, encoder)

    def half(self):
        """neural.py:147-161: cached fp16 inference copies."""
        if self._half is None:
            self._half = {
                "frame": quantize(self.frame) if self.frame is not None else None,
                "brdf": quantize(self.brdf),
                "sampler": quantize(self.sampler),
                "latent": self.latent.render_copy() if self.latent is not None else None,
            }
        return self._half


def frames_from_raw(raw):
    """neural.py:207-233 -> (t, b, n), each (B, N, 3) float64."""
    raw = np.atleast_2d(np.asarray(raw, dtype=np.float64))
    nb = raw.shape[0]
    r = raw.reshape(nb, raw.shape[1] // 6, 6)
    rn, rt = r[..., 0:3], r[..., 3:6].copy()
    n = rn / np.maximum(np.linalg.norm(rn, axis=-1, keepdims=True), 1e-12)
    c = np.cross(n, rt)
    cl = np.linalg.norm(c, axis=-1, keepdims=True)
    bad = cl[..., 0] < 1e-8
    if np.any(bad):
        rt[bad] = fallback_tangent(n[bad])
        c = np.cross(n, rt)
        cl = np.linalg.norm(c, axis=-1, keepdims=True)
    b = c / np.maximum(cl, 1e-12)
    return np.cross(b, n), b, n


def frame_transform(frames, w):
    """neural.py:185-196: (t_i.w, b_i.w, n_i.w) over frames -> (B, 3N)."""
    t, b, n = frames
    w = w[:, None, :]
    out = np.stack([np.sum(t * w, -1), np.sum(b * w, -1), np.sum(n * w, -1)], axis=-1)
    return out.reshape(w.shape[0], -1)


def eval_brdf(mat, z, wi, wo, fp16=False):
    """neural.py:273-300 -> (f (B,3) f64, albedo or None)."""
    wi = np.atleast_2d(np.asarray(wi, dtype=np.float64))
    wo = np.atleast_2d(np.asarray(wo, dtype=np.float64))
    z64 = np.atleast_2d(np.asarray(z, dtype=np.float64))
    if mat.cfg.use_frames:
        if fp16:
            raw = mat.half()["frame"].forward(np.atleast_2d(z).astype(np.float32))
        else:
            raw = mat.frame.forward(z64.astype(np.float32))
        fr = frames_from_raw(raw)
        zin = np.atleast_2d(z) if fp16 else z64
        inp = np.concatenate([zin, frame_transform(fr, wi), frame_transform(fr, wo)], axis=-1)
    else:
        inp = np.concatenate([z64, wi, wo], axis=-1)
    inp = inp.astype(np.float32)
    y = mat.half()["brdf"].forward(inp) if fp16 else mat.brdf.forward(inp)
    y = np.asarray(y, dtype=np.float64)
    up = ((wi[:, 2] > 0.0) & (wo[:, 2] > 0.0))[:, None]
    f = np.where(up, brdf_output(y[:, 0:3]), 0.0)
    if mat.cfg.albedo_head:
        return f, np.where(up, np.maximum(y[:, 3:6], 0.0), 0.0)
    return f, None


def eval_material(mat, uv, level, wi, wo, u_rr, fp16=False):
    """neural.py:303-309"""
    pyr = mat.half()["latent"] if fp16 else mat.latent
    z, chosen = pyr.fetch(uv, level, u_rr)
    f, albedo = eval_brdf(mat, z, wi, wo, fp16=fp16)
    return f, albedo, chosen


# ---------------------------------------------------------------------------
# analytic proxy (proxy.py)

class Proxy:
    """proxy.py:37-84: 9 parameters with alpha floor / rho clamp applied."""

    def __init__(self, wd, ws, mu_d, alpha, rho, mu_s):
        self.wd = np.atleast_1d(np.asarray(wd, dtype=np.float64))
        self.ws = np.atleast_1d(np.asarray(ws, dtype=np.float64))
        self.mu_d = np.atleast_2d(np.asarray(mu_d, dtype=np.float64))
        self.alpha = np.maximum(np.atleast_2d(np.asarray(alpha, dtype=np.float64)), ALPHA_FLOOR)
        self.rho = np.clip(np.atleast_1d(np.asarray(rho, dtype=np.float64)), -RHO_CLAMP, RHO_CLAMP)
        self.mu_s = np.atleast_2d(np.asarray(mu_s, dtype=np.float64))

    def __len__(self):
        return self.wd.shape[0]

    def subset(self, idx):
        return Proxy(self.wd[idx], self.ws[idx], self.mu_d[idx], self.alpha[idx],
                     self.rho[idx], self.mu_s[idx])

    def as_array(self):
        """(B, 9) in the order wd, ws, mu_d(2), alpha(2), rho, mu_s(2)."""
        return np.concatenate([self.wd[:, None], self.ws[:, None], self.mu_d, self.alpha,
                               self.rho[:, None], self.mu_s], axis=1)

    @property
    def s(self):
        return np.sqrt(1.0 - self.rho ** 2)

    def det(self):
        """proxy.py:76-78"""
        return self.alpha[:, 0] * self.alpha[:, 1] * self.s

    def warp(self):
        """proxy.py:64-74: slope-space matrix M."""
        m = np.zeros((len(self), 3, 3))
        m[:, 0, 0] = self.alpha[:, 0]
        m[:, 0, 2] = -self.mu_s[:, 0]
        m[:, 1, 0] = self.alpha[:, 1] * self.rho
        m[:, 1, 1] = self.alpha[:, 1] * self.s
        m[:, 1, 2] = -self.mu_s[:, 1]
        m[:, 2, 2] = 1.0
        return m

    def diffuse_axis(self):
        """proxy.py:80-84"""
        v = np.stack([-self.mu_d[:, 0], -self.mu_d[:, 1], np.ones_like(self.wd)], axis=-1)
        return _unit(v)


RAW_WD, RAW_MUDX, RAW_MUDY, RAW_WS, RAW_AX, RAW_AY, RAW_RHO, RAW_MUSX, RAW_MUSY = range(9)


def proxy_from_raw(raw, isotropic=False):
    """neural.py:314-331"""
    raw = np.atleast_2d(np.asarray(raw, dtype=np.float64))
    if isotropic:
        wd = 0.5 * (quad_tanh(raw[:, 0]) + 1.0)
        a = 0.5 * (quad_tanh(raw[:, 1]) + 1.0)
        z = np.zeros_like(wd)
        return Proxy(wd, 1.0 - wd, np.stack([z, z], -1), np.stack([a, a], -1), z,
                     np.stack([z, z], -1))
    wd, ws = softmax_pair(raw[:, RAW_WD], raw[:, RAW_WS])
    return Proxy(wd, ws, quad_sinh(raw[:, (RAW_MUDX, RAW_MUDY)]),
                 0.5 * (quad_tanh(raw[:, (RAW_AX, RAW_AY)]) + 1.0),
                 quad_tanh(raw[:, RAW_RHO]), quad_sinh(raw[:, (RAW_MUSX, RAW_MUSY)]))


def infer_proxy(mat, z, wi, fp16=False):
    """neural.py:353-362"""
    z = np.atleast_2d(np.asarray(z, dtype=np.float64))
    wi = np.atleast_2d(np.asarray(wi, dtype=np.float64))
    inp = np.concatenate([z, wi], axis=-1).astype(np.float32)
    raw = mat.half()["sampler"].forward(inp) if fp16 else mat.sampler.forward(inp)
    return proxy_from_raw(raw, isotropic=mat.cfg.sampler_isotropic)


def _half_vector(wi, wo):
    """proxy.py:87-101: normalized wi+wo flipped to h.z >= 0, validity."""
    h = wi + wo
    hl = np.sqrt(np.sum(h * h, axis=-1))
    ok = hl > 1e-9
    h = h / np.maximum(hl, 1e-12)[..., None]
    h = h * np.where(h[..., 2] < 0.0, -1.0, 1.0)[..., None]
    return h, ok


def _inverse_warp(p, h):
    """proxy.py:104-111: q = M^-1 h in closed form."""
    ax, ay, s = p.alpha[:, 0], p.alpha[:, 1], p.s
    q0 = (h[:, 0] + p.mu_s[:, 0] * h[:, 2]) / ax
    q1 = ((h[:, 1] + p.mu_s[:, 1] * h[:, 2]) / ay - p.rho * q0) / s
    return np.stack([q0, q1, h[:, 2]], axis=-1)


def pdf_diffuse(p, wo):
    """proxy.py:114-116"""
    return np.maximum(np.sum(wo * p.diffuse_axis(), axis=-1), 0.0) / np.pi


def pdf_specular(p, wi, wo):
    """proxy.py:119-126"""
    h, ok = _half_vector(wi, wo)
    q = _inverse_warp(p, h)
    q2 = np.sum(q * q, axis=-1)
    coh = np.abs(np.sum(wo * h, axis=-1))
    val = h[:, 2] * (1.0 / p.det()) / (4.0 * np.pi * q2 * q2 * np.maximum(coh, 1e-12))
    return np.where(ok & (h[:, 2] > 0.0), np.maximum(val, 0.0), 0.0)


def pdf(p, wi, wo):
    """proxy.py:129-135"""
    wi = np.atleast_2d(np.asarray(wi, dtype=np.float64))
    wo = np.atleast_2d(np.asarray(wo, dtype=np.float64))
    return p.wd * pdf_diffuse(p, wo) + p.ws * pdf_specular(p, wi, wo)


def ndf_sample(u):
    """proxy.py:138-146: unit-roughness NDF sample."""
    u = np.asarray(u, dtype=np.float64)
    tan2 = u[..., 0] / np.maximum(1.0 - u[..., 0], 1e-12)
    ct = 1.0 / np.sqrt(1.0 + tan2)
    st = np.sqrt(np.maximum(0.0, 1.0 - ct * ct))
    phi = 2.0 * np.pi * u[..., 1]
    return np.stack([st * np.cos(phi), st * np.sin(phi), ct], axis=-1)


def sample_diffuse(p, u2):
    """proxy.py:149-156"""
    g = p.diffuse_axis() + uniform_sphere(u2)
    return g / np.maximum(np.linalg.norm(g, axis=-1, keepdims=True), 1e-9)


def sample_specular(p, wi, u2):
    """proxy.py:159-165"""
    g = np.einsum("bij,bj->bi", p.warp(), ndf_sample(u2))
    h = g / np.maximum(np.linalg.norm(g, axis=-1, keepdims=True), 1e-12)
    return _mirror(wi, h)


def sample(p, wi, u):
    """proxy.py:168-180: u0 picks the lobe, (u1, u2) drive it."""
    wi = np.atleast_2d(np.asarray(wi, dtype=np.float64))
    u = np.atleast_2d(np.asarray(u, dtype=np.float64))
    diff = u[:, 0] < p.wd
    wo = np.empty_like(wi)
    if np.any(diff):
        wo[diff] = sample_diffuse(p.subset(diff), u[diff, 1:3])
    if np.any(~diff):
        spec = ~diff
        wo[spec] = sample_specular(p.subset(spec), wi[spec], u[spec, 1:3])
    return wo


def normalize_check(p, wi, n_samples, rng, chunk=2_000_000):
    """proxy.py:183-196: MC estimate of the sphere integral of pdf."""
    total, done = 0.0, 0
    while done < n_samples:
        m = min(chunk, n_samples - done)
        d = uniform_sphere(rng.random((m, 2)))
        rep = p.subset(np.zeros(m, dtype=np.int64))
        total += float(np.sum(pdf(rep, np.broadcast_to(wi, (m, 3)), d)))
        done += m
    return total * 4.0 * np.pi / n_samples


# ---------------------------------------------------------------------------
# one full query (the chain SURVEY §8d times): fetch -> eval -> proxy -> sample -> pdf

def full_query(mat, uv, lod, u_rr, wi, wo, u3, fp16=True):
    """render.py:368-372 + 385-386 + 401-402 chained for one batch."""
    pyr = mat.half()["latent"] if fp16 else mat.latent
    z, chosen = pyr.fetch(uv, lod, u_rr)
    f, _ = eval_brdf(mat, z, wi, wo, fp16=fp16)
    p = infer_proxy(mat, z, wi, fp16=fp16)
    ws = sample(p, wi, u3)
    return f, ws, pdf(p, wi, ws), p, chosen


# ---------------------------------------------------------------------------
# LoD from ray cones (render.py) — the step that produces the query's lod

def footprint_to_level(area_texels, n_levels):
    """render.py:334-337: fractional mip level of a footprint area given in
    level-0 texels^2."""
    lvl = 0.5 * np.log2(np.maximum(np.asarray(area_texels, dtype=np.float64), 1.0))
    return np.clip(lvl, 0.0, n_levels - 1)


def cone_level(cone_w, cone_s, t, cos_hit, density, n_levels):
    """render.py:436-443 (_surface_frames_and_level): ray-cone width at the hit,
    foreshortened by the hit cosine (floored at 0.05), squared in texels."""
    width = np.asarray(cone_w, np.float64) + np.asarray(cone_s, np.float64) * np.asarray(t, np.float64)
    diam = width / np.maximum(np.abs(np.asarray(cos_hit, np.float64)), 0.05)
    area = (diam * np.asarray(density, np.float64)) ** 2
    return footprint_to_level(area, n_levels)


# ---------------------------------------------------------------------------
# KL sampler loss (training.py:187-273) — SURVEY §8 f4

EPS_KL = 1e-4                                  # training.py:45
LUM_WEIGHTS = np.array([0.2126, 0.7152, 0.0722])  # training.py:46
_TINY = 1e-30                                  # training.py:47


def _quad_tanh_grad(x):
    """neural.py:53-56"""
    ax = np.abs(x)
    den = 1.0 + ax + 0.5 * x * x
    return (1.0 + ax) / (den * den)


def _kl_target(mat, z, wi, wo):
    """training.py:187-216: lum(f) cos(theta_o) + eps and its wo-derivative
    (frames and decoder supply values and direction derivatives only)."""
    up = wo[:, 2] > 0.0
    woz = np.maximum(wo[:, 2], 0.0)
    if mat.cfg.use_frames:
        fr = frames_from_raw(mat.frame.forward(z.astype(np.float32)))
        inp = np.concatenate([z, frame_transform(fr, wi), frame_transform(fr, wo)], -1)
    else:
        fr = None
        inp = np.concatenate([z, wi, wo], -1)
    y, cache = forward_cached(mat.brdf, inp.astype(np.float32))
    y = np.asarray(y, np.float64)
    lum = brdf_output(y[:, 0:3]) @ LUM_WEIGHTS
    target = np.where(up, lum * woz, 0.0) + EPS_KL
    og = np.zeros_like(y, dtype=np.float32)
    og[:, 0:3] = (LUM_WEIGHTS * np.where(y[:, 0:3] > 0.0, np.exp(np.minimum(y[:, 0:3], 60.0)), 0.0)
                  * woz[:, None]).astype(np.float32)
    _, din = backward(mat.brdf, cache, og)
    din = np.asarray(din, np.float64)
    c = z.shape[1]
    if fr is not None:  # neural.py:198-205 transform adjoint on the wo block
        nf = mat.cfg.n_frames
        g = din[:, c + 3 * nf:].reshape(-1, nf, 3)
        t, b, n = fr
        dt = np.sum(g[..., 0:1] * t + g[..., 1:2] * b + g[..., 2:3] * n, axis=1)
    else:
        dt = din[:, c + 3:]
    dt = dt + lum[:, None] * np.array([0.0, 0.0, 1.0])
    return target, np.where(up[:, None], dt, 0.0)


def _grad_log_pdf(p, wi, wo):
    """proxy.py:203-250: (p, d log p / d wo), subgradient 0 at the kinks."""
    nd = p.diffuse_axis()
    dn = np.sum(wo * nd, -1)
    pd = np.maximum(dn, 0.0) / np.pi
    dpd = np.where((dn > 0.0)[:, None], nd / np.pi, 0.0)
    hs = wi + wo
    hl = np.linalg.norm(hs, axis=-1)
    ok = hl > 1e-9
    h = hs / np.maximum(hl, 1e-12)[:, None]
    flip = np.where(h[:, 2] < 0.0, -1.0, 1.0)
    h = h * flip[:, None]
    hz = ok & (h[:, 2] > 0.0)
    q = _inverse_warp(p, h)
    qn2 = np.maximum(np.sum(q * q, -1), _TINY)
    coh = np.sum(wo * h, -1)
    with np.errstate(divide="ignore", invalid="ignore"):
        ps = np.where(hz, h[:, 2] / (p.det() * 4.0 * np.pi * qn2 * qn2 * np.maximum(np.abs(coh), 1e-12)), 0.0)
    ax, ay, s, rho = p.alpha[:, 0], p.alpha[:, 1], p.s, p.rho
    mtq = np.stack([q[:, 0] / ax - q[:, 1] * rho / (ax * s), q[:, 1] / (ay * s),
                    q[:, 0] * p.mu_s[:, 0] / ax
                    + q[:, 1] * (p.mu_s[:, 1] / (ay * s) - p.mu_s[:, 0] * rho / (ax * s)) + q[:, 2]], -1)
    inv_coh = np.where(np.abs(coh) < 1e-12, 0.0, 1.0 / np.where(coh == 0.0, 1.0, coh))
    dlog_dh = (np.stack([0 * ps, 0 * ps, 1.0 / np.maximum(h[:, 2], 1e-12)], -1)
               - 4.0 * mtq / qn2[:, None] - wo * inv_coh[:, None])
    proj = dlog_dh - h * np.sum(h * dlog_dh, -1)[:, None]
    dlog_ps = flip[:, None] * proj / np.maximum(hl, 1e-12)[:, None] - h * inv_coh[:, None]
    dps = np.where(hz[:, None], ps[:, None] * dlog_ps, 0.0)
    pm = p.wd * pd + p.ws * ps
    dp = p.wd[:, None] * dpd + p.ws[:, None] * dps
    return pm, dp / np.maximum(pm, _TINY)[:, None]


def sampler_loss_and_grads(mat, z, wi, us):
    """training.py:219-273 with the default target and fixed uniforms
    us = (u_d, u_s): the reparameterized KL estimate over both lobes and
    the sampler decoder's gradients -> (loss, [(dW, db), ...])."""
    z = np.atleast_2d(np.asarray(z, np.float64))
    wi = np.atleast_2d(np.asarray(wi, np.float64))
    b = z.shape[0]
    iso = mat.cfg.sampler_isotropic
    raw, cache = forward_cached(mat.sampler, np.concatenate([z, wi], -1).astype(np.float32))
    raw = np.asarray(raw, np.float64)
    p = proxy_from_raw(raw, isotropic=iso)
    u_d, u_s = (np.asarray(u, np.float64) for u in us)
    # samples + aux (proxy.py:149-165)
    v = uniform_sphere(u_d)
    nd = p.diffuse_axis()
    g = nd + v
    gl = np.maximum(np.linalg.norm(g, axis=-1), 1e-9)
    wo_d = g / gl[:, None]
    m = ndf_sample(u_s)
    gs = np.einsum("bij,bj->bi", p.warp(), m)
    gls = np.linalg.norm(gs, axis=-1)
    h = gs / np.maximum(gls, 1e-12)[:, None]
    wo_s = _mirror(wi, h)
    f_d, df_d = _kl_target(mat, z, wi, wo_d)
    f_s, df_s = _kl_target(mat, z, wi, wo_s)
    p_d, dl_d = _grad_log_pdf(p, wi, wo_d)
    p_s, dl_s = _grad_log_pdf(p, wi, wo_s)
    ell_d = np.log(np.maximum(p_d, _TINY)) - np.log(f_d)
    ell_s = np.log(np.maximum(p_s, _TINY)) - np.log(f_s)
    loss = float(np.mean(p.wd * ell_d + p.ws * ell_s))
    brk_d = dl_d - df_d / f_d[:, None]
    brk_s = dl_s - df_s / f_s[:, None]
    # d wo / d mu_d (proxy.py:253-266)
    vlen = np.sqrt(1.0 + np.sum(p.mu_d ** 2, -1))
    g_mu_d = np.empty((b, 2))
    for k in range(2):
        e = np.zeros_like(nd)
        e[:, k] = -1.0
        dnd = (e - nd * np.sum(nd * e, -1)[:, None]) / vlen[:, None]
        dwo = (dnd - wo_d * np.sum(wo_d * dnd, -1)[:, None]) / gl[:, None]
        g_mu_d[:, k] = p.wd * np.sum(brk_d * dwo, -1)
    # d wo / d (ax, ay, rho, msx, msy) (proxy.py:269-282)
    ay, s, rho = p.alpha[:, 1], p.s, p.rho
    dg = np.zeros((b, 3, 5))
    dg[:, 0, 0] = m[:, 0]
    dg[:, 1, 1] = rho * m[:, 0] + s * m[:, 1]
    dg[:, 1, 2] = ay * (m[:, 0] - rho * m[:, 1] / s)
    dg[:, 0, 3] = -m[:, 2]
    dg[:, 1, 4] = -m[:, 2]
    dh = (dg - h[..., None] * np.sum(h[..., None] * dg, 1)[:, None, :]) / gls[:, None, None]
    js = 2.0 * h[..., None] * np.sum(wi[..., None] * dh, 1)[:, None, :] \
        + 2.0 * np.sum(wi * h, -1)[:, None, None] * dh
    g_spec = p.ws[:, None] * np.einsum("bi,bik->bk", brk_s, js)
    # raw-output Jacobian (neural.py:334-350)
    draw = np.zeros_like(raw)
    if iso:
        draw[:, 0] = (ell_d - ell_s) * 0.5 * _quad_tanh_grad(raw[:, 0])
        draw[:, 1] = (g_spec[:, 0] + g_spec[:, 1]) * 0.5 * _quad_tanh_grad(raw[:, 1])
    else:
        wd, ws = softmax_pair(raw[:, RAW_WD], raw[:, RAW_WS])
        sj = wd * ws
        draw[:, 0] = (ell_d - ell_s) * sj
        draw[:, 3] = (ell_s - ell_d) * sj
        draw[:, 1:3] = g_mu_d * (1.0 + 0.5 * raw[:, 1:3] ** 2)
        draw[:, 4:6] = g_spec[:, 0:2] * 0.5 * _quad_tanh_grad(raw[:, 4:6])
        draw[:, 6] = g_spec[:, 2] * _quad_tanh_grad(raw[:, 6])
        draw[:, 7:9] = g_spec[:, 3:5] * (1.0 + 0.5 * raw[:, 7:9] ** 2)
    draw /= b
    grads, _ = backward(mat.sampler, cache, draw.astype(np.float32))
    return loss, grads


# ---------------------------------------------------------------------------
# chi-square goodness-of-fit harness for spherical samplers (chi2.py:13-72):
# the reference's validation recipe for sample() against pdf()

def _chi2_bin_masses(pdf_fn, res_theta, res_phi, z_lo, z_hi, quad):
    """chi2.py:13-27: integral of the density over each (cos theta, phi) bin."""
    dz = (z_hi - z_lo) / res_theta
    dphi = 2.0 * np.pi / res_phi
    zi = z_lo + dz * (np.arange(res_theta * quad) + 0.5) / quad
    pj = dphi * (np.arange(res_phi * quad) + 0.5) / quad
    zz, pp = np.meshgrid(zi, pj, indexing="ij")
    rr = np.sqrt(np.maximum(0.0, 1.0 - zz ** 2))
    dirs = np.stack([rr * np.cos(pp), rr * np.sin(pp), zz], axis=-1).reshape(-1, 3)
    vals = np.asarray(pdf_fn(dirs), np.float64).reshape(res_theta * quad, res_phi * quad)
    cell = (dz / quad) * (dphi / quad)
    return vals.reshape(res_theta, quad, res_phi, quad).sum(axis=(1, 3)) * cell


def _chi2_pearson(observed, expected, min_expected):
    """chi2.py:30-43: pool small cells, scale, Pearson statistic, p-value."""
    from scipy import stats
    exp_flat, obs_flat = expected.ravel(), observed.ravel()
    big = exp_flat >= min_expected
    exp_p = np.append(exp_flat[big], exp_flat[~big].sum())
    obs_p = np.append(obs_flat[big], obs_flat[~big].sum())
    keep = exp_p > 1e-9
    exp_p, obs_p = exp_p[keep], obs_p[keep]
    exp_p = exp_p * (obs_p.sum() / exp_p.sum())
    stat = float(np.sum((obs_p - exp_p) ** 2 / exp_p))
    dof = exp_p.size - 1
    return stat, dof, float(stats.chi2.sf(stat, dof))


def chi_square_test(sample_fn, pdf_fn, n_samples, res_theta=16, res_phi=32, significance=0.01,
                    sphere=True, quad=48, min_expected=5.0):
    """chi2.py:46-72 -> (passed, p_value, statistic, dof)."""
    z_lo, z_hi = (-1.0, 1.0) if sphere else (0.0, 1.0)
    dirs = np.asarray(sample_fn(n_samples), np.float64)
    z = np.clip(dirs[:, 2], z_lo, np.nextafter(z_hi, -np.inf))
    phi = np.arctan2(dirs[:, 1], dirs[:, 0]) % (2.0 * np.pi)
    iz = ((z - z_lo) / (z_hi - z_lo) * res_theta).astype(np.int64)
    ip = np.minimum((phi / (2.0 * np.pi) * res_phi).astype(np.int64), res_phi - 1)
    observed = np.zeros((res_theta, res_phi))
    np.add.at(observed, (iz, ip), 1.0)
    expected = _chi2_bin_masses(pdf_fn, res_theta, res_phi, z_lo, z_hi, quad) * n_samples
    stat, dof, p = _chi2_pearson(observed, expected, min_expected)
    return p > significance, p, stat, dof
