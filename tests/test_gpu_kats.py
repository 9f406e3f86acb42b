"""The reference's own known-answer and statistical tests for the query path,
run on the CUDA kernels.  Each test cites the reference test
it mirrors (paths under /root/reference/pkg).
"""

import numpy as np
import pytest

from conftest import rel_err
from test_gpu_parity import check_rel

pytestmark = pytest.mark.gpu


def _params(wd=0.5, mu_d=(0.0, 0.0), alpha=(0.5, 0.5), rho=0.0, mu_s=(0.0, 0.0)):
    """tests/test_proxy.py:8-10 (make_params)."""
    from paper_2305_02678_b200 import proxy
    return proxy.ProxyParams(wd, 1.0 - wd, mu_d, alpha, rho, mu_s)


def _random_params(rng, mu_d_scale=0.0):
    """tests/test_proxy.py:13-19."""
    wd = rng.uniform(0.2, 0.8)
    mu_d = rng.uniform(-1.0, 1.0, 2) * mu_d_scale
    alpha = rng.uniform(0.2, 1.0, 2)
    rho = rng.uniform(-0.8, 0.8)
    mu_s = rng.uniform(-0.5, 0.5, 2)
    return _params(wd, mu_d, alpha, rho, mu_s)


def _random_wi(rng, min_cos=0.3):
    """tests/test_proxy.py:22-25 (uniform hemisphere, z floored, normalized)."""
    u = rng.random((1, 2))
    z = u[:, 0]
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    phi = 2.0 * np.pi * u[:, 1]
    w = np.stack([r * np.cos(phi), r * np.sin(phi), z], -1)
    w[0, 2] = max(w[0, 2], min_cos)
    return w / np.linalg.norm(w, axis=-1, keepdims=True)


# --- proxy pdf goldens at the zenith (tests/test_proxy.py:39-55) -------------

def test_pdf_zenith_goldens_through_nm_pdf():
    from paper_2305_02678_b200 import proxy
    z = np.array([[0.0, 0.0, 1.0]])
    cases = [(_params(wd=1.0), 1.0 / np.pi),
             (_params(wd=0.0, alpha=(1.0, 1.0)), 1.0 / (4.0 * np.pi)),
             (_params(wd=0.5, alpha=(1.0, 1.0)), 0.5 / np.pi + 0.5 / (4.0 * np.pi))]
    for p, want in cases:
        got = proxy.pdf(p, z, z)[0]
        assert got == pytest.approx(want, rel=1e-6), (got, want)  # fp32 kernel vs the exact value


def test_proxy_matrix_det_and_diffuse_normal():
    """ProxyParams.matrix / det / diffuse_normal (proxy.py:64-84, tests/test_proxy.py:72-81)."""
    from oracle import nm_oracle as O
    rng = np.random.default_rng(3)
    p = _random_params(rng, mu_d_scale=0.5)
    m = p.matrix()
    assert m.shape == (1, 3, 3)
    assert np.allclose(np.linalg.det(m), p.det(), rtol=1e-6)
    b = p.as_array()
    ref = O.Proxy(b[:, 0], b[:, 1], b[:, 2:4], b[:, 4:6], b[:, 6], b[:, 7:9])
    assert np.allclose(m, ref.warp(), atol=1e-7)
    assert np.allclose(p.diffuse_normal(), ref.diffuse_axis(), atol=1e-7)


# --- MC normalization, +-1 % (tests/test_proxy.py:114-135) --------------------

@pytest.mark.parametrize("case", ["diffuse", "specular", "mixture"])
def test_normalization_on_gpu_pdf(case):
    from paper_2305_02678_b200 import proxy
    if case == "diffuse":
        rng, p, wi, n = np.random.default_rng(4), _params(wd=1.0), np.array([0.0, 0.0, 1.0]), 1_000_000
    elif case == "specular":
        rng = np.random.default_rng(5)
        p = _params(wd=0.0, alpha=(0.4, 0.7), rho=0.4, mu_s=(0.3, -0.2))
        wi, n = np.array([0.4, -0.2, 0.8]), 4_000_000
    else:
        rng = np.random.default_rng(6)
        p = _params(wd=0.35, mu_d=(0.0, 0.0), alpha=(0.6, 0.3), rho=-0.5, mu_s=(-0.4, 0.1))
        wi, n = np.array([-0.3, 0.1, 0.9]), 4_000_000
    wi = wi / np.linalg.norm(wi)
    est = proxy.normalize_check(p, wi, n, rng)
    assert abs(est - 1.0) < 0.01, est


# --- chi-square sample() vs pdf() on the GPU (tests/test_proxy.py:138-160) -----

def test_chi_square_gpu_sampler_vs_gpu_pdf():
    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import proxy
    rng = np.random.default_rng(7)
    passed = 0
    for i in range(5):
        params = _random_params(rng, mu_d_scale=0.5 if i % 2 else 0.0)
        wi = _random_wi(rng)[0]
        srng = np.random.default_rng(100 + i)

        def sample_fn(n):
            rep = params.take(np.zeros(n, dtype=np.int64))
            return proxy.sample(rep, np.broadcast_to(wi, (n, 3)), srng.random((n, 3)))

        def pdf_fn(dirs):
            rep = params.take(np.zeros(dirs.shape[0], dtype=np.int64))
            return proxy.pdf(rep, np.broadcast_to(wi, dirs.shape), dirs)

        ok, pval, stat, dof = O.chi_square_test(sample_fn, pdf_fn, 200_000)
        passed += int(ok)
    assert passed >= 4


def test_chi_square_fused_sampler_of_a_material():
    """The fused kernel's own sample()/pdf() (nm_sample_pdf) for one texel of
    a random material (the validate recipe, cli.py:91-114)."""
    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import neural, proxy
    from paper_2305_02678_b200.latent import LatentPyramid
    rng = np.random.default_rng(11)
    mat = neural.NeuralMaterial.create(neural.NeuralMaterialConfig(), rng)
    mat.latent = LatentPyramid(O.random_pyramid(rng, 32, 32).levels)
    wi = _random_wi(rng)[0].astype(np.float32)
    uv = np.array([[0.3, 0.6]], np.float32)
    _, _, p = neural.sample_pdf(mat, uv, 0.0, np.zeros(1, np.float32), wi[None], np.full((1, 3), 0.5, np.float32),
                                return_params=True)
    srng = np.random.default_rng(12)

    def sample_fn(n):
        ws, pdf_s = neural.sample_pdf(mat, np.broadcast_to(uv, (n, 2)), 0.0, np.zeros(n, np.float32),
                                      np.broadcast_to(wi, (n, 3)), srng.random((n, 3)).astype(np.float32))
        return ws

    def pdf_fn(dirs):
        rep = p.take(np.zeros(dirs.shape[0], dtype=np.int64))
        return proxy.pdf(rep, np.broadcast_to(wi, dirs.shape), dirs)

    ok, pval, stat, dof = O.chi_square_test(sample_fn, pdf_fn, 200_000)
    assert ok, (pval, stat, dof)


# --- Russian-roulette level pick: unbiased at l = 1.3 (tests/test_latent.py:41-53)

def test_roulette_expectation_level_1p3():
    from oracle import nm_oracle as O
    from paper_2305_02678_b200.latent import LatentPyramid
    rng = np.random.default_rng(2)
    pyr = LatentPyramid(O.random_pyramid(rng, 16, 16).levels)
    uv = np.array([0.37, 0.81])
    n = 100_000
    z, chosen = pyr.fetch(np.tile(uv, (n, 1)), 1.3, rng.random(n))
    z = z.astype(np.float64)
    target = 0.7 * pyr.fetch_level(uv[None, :], 1) + 0.3 * pyr.fetch_level(uv[None, :], 2)
    err = np.abs(z.mean(axis=0) - target[0])
    sigma = z.std(axis=0) / np.sqrt(n)
    assert np.all(err <= 3.0 * sigma + 1e-7)
    assert abs(np.mean(chosen == 2) - 0.3) < 0.01


def test_texel_center_identity_and_integer_level():
    """tests/test_latent.py:23-38: a texel-center fetch at an integer level
    returns that texel; integer levels never roulette."""
    from oracle import nm_oracle as O
    from paper_2305_02678_b200.latent import LatentPyramid
    rng = np.random.default_rng(1)
    pyr = LatentPyramid(O.random_pyramid(rng, 16, 16).levels)
    uv = np.array([[(3 + 0.5) / 16, (5 + 0.5) / 16]])
    z, _ = pyr.fetch(uv, 0.0, np.zeros(1))
    assert np.allclose(z[0], pyr.levels[0][5, 3], atol=1e-7)
    _, ch = pyr.fetch(np.tile(uv, (1000, 1)), 2.0, rng.random(1000))
    assert np.all(ch == 2)


# --- learned frames: canonical and degenerate (tests/test_neural.py:20-30, 61-67)

def _frames_material(bias, n_frames=2, seed=0):
    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import mlp, neural
    from paper_2305_02678_b200.latent import LatentPyramid
    rng = np.random.default_rng(seed)
    mat = neural.NeuralMaterial.create(neural.NeuralMaterialConfig(n_frames=n_frames), rng)
    mat.frame_layer = mlp.Mlp([mlp.Layer(np.zeros((6 * n_frames, 8), np.float32),
                                         np.asarray(bias, np.float32), mlp.ACT_LINEAR)])
    mat.latent = LatentPyramid(O.random_pyramid(rng, 32, 32).levels)
    return mat


def _eval_vs_oracle(mat, n=4099, seed=1, paths=(2, 1)):
    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import _lib, neural
    from test_gpu_parity import _oracle_from
    rng = np.random.default_rng(seed)
    uv = rng.random((n, 2)).astype(np.float32)
    lod = (rng.random(n) * (mat.latent.n_levels - 1)).astype(np.float32)
    urr = rng.random(n).astype(np.float32)
    wi, wo = O.draw_direction_pairs(rng, n)
    wi, wo = wi.astype(np.float32), wo.astype(np.float32)
    f_ref, _, ch_ref = O.eval_material(_oracle_from(mat), uv, lod, wi, wo, urr, fp16=True)
    lib = _lib.load()
    try:
        for path in paths:
            lib.nm_set_kernel_path(path)
            f, _, ch = neural.eval_material(mat, uv, lod, wi, wo, urr, fp16=True)
            assert np.array_equal(ch, ch_ref)
            check_rel(f, f_ref, what=f"path {path}")
    finally:
        lib.nm_set_kernel_path(0)


def test_canonical_frames_decode_like_the_reference():
    """Zero frame weights, bias (0,0,1, 1,0,0) per frame: T.w = (w, w)."""
    _eval_vs_oracle(_frames_material(np.tile([0.0, 0.0, 1.0, 1.0, 0.0, 0.0], 2)))


def test_degenerate_tangent_fallback_on_gpu():
    """Tangent parallel to the normal in both frames: the fallback tangent
    n x e_argmin|n| (geom.py:82-89) on every row — the fast kernel queues
    them (conditioning +inf) and resolves exactly; the generic kernel takes
    the exact path directly."""
    _eval_vs_oracle(_frames_material([0.0, 0.0, 1.0, 0.0, 0.0, 1.0] * 2))


def test_near_degenerate_and_mixed_frames():
    """Frame 1 canonical, frame 2 with a tangent at 1e-7 from its normal
    (just inside the reference's |c| < 1e-8 threshold after normalization
    for some rows, outside for others)."""
    _eval_vs_oracle(_frames_material([0.0, 0.0, 1.0, 1.0, 0.0, 0.0, 0.0, 0.0, 1.0, 1e-8, 0.0, 1.0]))


# --- device copies follow in-place edits (reference semantics: fetch reads
# the live levels, training.py:305-356; fp16=False reads live weights) --------

def test_fetch_sees_in_place_level_edits():
    from oracle import nm_oracle as O
    from paper_2305_02678_b200.latent import LatentPyramid
    rng = np.random.default_rng(21)
    pyr = LatentPyramid(O.random_pyramid(rng, 16, 16).levels)
    uv = rng.random((512, 2)).astype(np.float32)
    z0, _ = pyr.fetch(uv, 1.5, rng.random(512))
    for l in pyr.levels:  # an optimizer step in place
        l *= 0.5
        l += 0.25
    urr = rng.random(512)
    z1, _ = pyr.fetch(uv, 1.5, urr)
    z_ref, _ = O.Pyramid(pyr.levels).fetch(uv, 1.5, urr)
    assert np.array_equal(z1, z_ref)


def test_fp32_path_sees_in_place_weight_edits():
    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import neural
    from paper_2305_02678_b200.latent import LatentPyramid
    from test_gpu_parity import _oracle_from
    rng = np.random.default_rng(22)
    mat = neural.NeuralMaterial.create(neural.NeuralMaterialConfig(), rng)
    mat.latent = LatentPyramid(O.random_pyramid(rng, 16, 16).levels)
    n = 1000
    z = rng.standard_normal((n, 8)).astype(np.float32)
    wi, wo = O.draw_direction_pairs(rng, n)
    neural.eval_brdf(mat, z, wi, wo, fp16=False)
    mat.brdf_decoder.layers[-1].b[:] += 0.5  # in place
    f, _ = neural.eval_brdf(mat, z, wi, wo, fp16=False)
    f_ref, _ = O.eval_brdf(_oracle_from(mat), z, wi, wo, fp16=False)
    check_rel(f, f_ref, max_tol=1e-3, mean_tol=1e-5, what="fp32 path after edit")


# --- deterministic trilinear filtering (optional mode; exact oracle from
# latent.py:84-107, tests/test_acceptance.py:242-255) ------------------------

def test_trilinear_fetch_bit_exact():
    from oracle import nm_oracle as O
    from paper_2305_02678_b200.latent import LatentPyramid
    rng = np.random.default_rng(31)
    for w, h in ((64, 64), (24, 20)):  # power-of-two and non-power-of-two levels
        opyr = O.random_pyramid(rng, w, h)
        pyr = LatentPyramid(opyr.levels)
        n = 5000
        uv = (rng.random((n, 2)) * 3 - 1).astype(np.float32)  # wraps
        lod = (rng.random(n) * (pyr.n_levels + 1) - 0.5).astype(np.float32)  # clips at both ends
        z = pyr.fetch_trilinear(uv, lod)
        z_ref = O.fetch_trilinear(opyr, uv, lod)
        assert z.dtype == np.float32 and np.array_equal(z, z_ref), np.abs(z - z_ref).max()


def test_trilinear_is_the_roulette_expectation():
    """Mean of roulette fetches at l = 1.3 -> the trilinear fetch within 3 sigma."""
    from oracle import nm_oracle as O
    from paper_2305_02678_b200.latent import LatentPyramid
    rng = np.random.default_rng(2)
    pyr = LatentPyramid(O.random_pyramid(rng, 16, 16).levels)
    uv = np.array([0.37, 0.81], np.float32)
    n = 100_000
    z, _ = pyr.fetch(np.tile(uv, (n, 1)), np.float32(1.3), rng.random(n).astype(np.float32))
    zt = pyr.fetch_trilinear(uv[None, :], np.float32(1.3))[0].astype(np.float64)
    z = z.astype(np.float64)
    assert np.all(np.abs(z.mean(0) - zt) <= 3.0 * z.std(0) / np.sqrt(n) + 1e-7)



# --- float64 coordinates (the reference's dtype): levels, taps and z bit-exact
# for inputs fp32 cannot represent (latent.py:59-82) ---------------------------

def test_float64_coordinates_bit_exact_at_boundaries():
    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import neural
    from paper_2305_02678_b200.latent import LatentPyramid
    from test_gpu_parity import _oracle_from
    rng = np.random.default_rng(41)
    mat = neural.NeuralMaterial.create(neural.NeuralMaterialConfig(), rng)
    mat.latent = LatentPyramid(O.random_pyramid(rng, 24, 40).levels)  # npot levels
    n = 20000
    w0, h0 = 24, 40
    # texel-boundary coordinates: u*w - 0.5 within ~1e-13 of an integer, and
    # u_rr within 1e-13 of the level fraction (the float32 rounding of either
    # would flip the tap or the level)
    k = rng.integers(-40, 80, size=(n, 2)).astype(np.float64)
    uv = (k + 0.5) / np.array([w0, h0]) + rng.choice([-1e-13, 1e-13, 0.0], size=(n, 2))
    lod = rng.random(n) * (mat.latent.n_levels - 1)
    urr = (lod - np.floor(lod)) + rng.choice([-1e-13, 1e-13], size=n)
    pyr = O.Pyramid(mat.latent.levels)
    z_ref, ch_ref = pyr.fetch(uv, lod, urr)
    z, ch = mat.latent.fetch(uv, lod, urr)
    assert np.array_equal(ch, ch_ref) and np.array_equal(z, z_ref)
    zh, chh, xs, ys, _ = mat.half()["latent"].fetch(uv, lod, urr, return_taps=True)
    hz, hch = O.Pyramid(mat.half()["latent"].levels).fetch(uv, lod, urr)
    assert np.array_equal(chh, hch) and np.array_equal(zh, hz)
    wi, wo = O.draw_direction_pairs(rng, n)
    f_ref, _, ch2 = O.eval_material(_oracle_from(mat), uv, lod, wi.astype(np.float32), wo.astype(np.float32),
                                    urr, fp16=True)
    f, _, ch3 = neural.eval_material(mat, uv, lod, wi.astype(np.float32), wo.astype(np.float32), urr, fp16=True)
    assert np.array_equal(ch3, ch2)
    check_rel(f, f_ref, what="float64 coordinates")
    # float32-narrowed, the same inputs would pick other levels / taps on some rows
    _, ch32 = pyr.fetch(uv.astype(np.float32), lod.astype(np.float32), urr.astype(np.float32))
    assert not np.array_equal(ch32, ch_ref)
