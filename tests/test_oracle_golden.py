"""Pin the numpy oracle (oracle/nm_oracle.py) to the golden vectors that the
REAL reference produced (oracle/make_golden.py).  CPU only."""

import os

import numpy as np
import pytest

from conftest import golden_cases, golden_config, golden_levels, golden_nets, load_golden
from oracle import nm_oracle as O

CASES = golden_cases()


def oracle_material(g):
    cfg = O.Config(**golden_config(g))
    frame = O.Net(golden_nets(g, "frame")) if int(g["frame_n"]) else None
    mat = O.Material(cfg, frame, O.Net(golden_nets(g, "brdf")), O.Net(golden_nets(g, "sampler")))
    mat.latent = O.Pyramid(golden_levels(g))
    return mat


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference_fp16_path(name):
    g = load_golden(name)
    mat = oracle_material(g)
    f, ws, pdf_ws, p, chosen = O.full_query(mat, g["uv"].astype(np.float64),
                                            g["lod"].astype(np.float64),
                                            g["u_rr"].astype(np.float64),
                                            g["wi"].astype(np.float64),
                                            g["wo"].astype(np.float64),
                                            g["u3"].astype(np.float64))
    assert np.array_equal(chosen, g["chosen"])
    z, _ = mat.half()["latent"].fetch(g["uv"], g["lod"], g["u_rr"])
    assert np.array_equal(z, g["z"])
    np.testing.assert_allclose(f, g["f"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(p.as_array(), g["params"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(ws, g["ws"], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(pdf_ws, g["pdf_ws"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(O.pdf(p, g["wi"], g["wo"]), g["pdf_wo"], rtol=1e-9, atol=1e-12)
    if "albedo" in g:
        _, alb = O.eval_brdf(mat, z, g["wi"], g["wo"], fp16=True)
        np.testing.assert_allclose(alb, g["albedo"], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("name", [c for c in CASES if "xs" in load_golden(c)])
def test_oracle_taps_bit_exact(name):
    g = load_golden(name)
    pyr = oracle_material(g).half()["latent"]
    for lv in np.unique(g["chosen"]):
        m = g["chosen"] == lv
        xs, ys, wts = pyr.taps(int(lv), g["uv"][m].astype(np.float64))
        assert np.array_equal(xs, g["xs"][m]) and np.array_equal(ys, g["ys"][m])
        assert np.array_equal(wts, g["wts"][m])


def test_oracle_fp32_path_matches_reference():
    g = load_golden("c1_2x32")
    mat = oracle_material(g)
    f32, _ = O.eval_brdf(mat, g["z"], g["wi"], g["wo"], fp16=False)
    np.testing.assert_allclose(f32, g["f_fp32path"], rtol=1e-12, atol=1e-12)


def test_oracle_proxy_kat():
    g = load_golden("proxy_kat")
    b = g["params"].astype(np.float64)
    p = O.Proxy(b[:, 0], b[:, 1], b[:, 2:4], b[:, 4:6], b[:, 6], b[:, 7:9])
    wi = g["wi"].astype(np.float64)
    ws = O.sample(p, wi, g["u3"].astype(np.float64))
    np.testing.assert_allclose(ws, g["ws"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(O.pdf(p, wi, ws), g["pdf_ws"], rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(O.pdf(p, wi, g["wo"]), g["pdf_wo"], rtol=1e-10, atol=1e-14)


def test_oracle_random_material_matches_reference_init():
    """Oracle init consumes the RNG like the reference (neural.py:117-141)."""
    for name in ("c1_2x32", "vanilla", "isotropic"):
        g = load_golden(name)
        mat = O.Material.random(O.Config(**golden_config(g)), np.random.default_rng(int(g["seed"])))
        for prefix, net in (("brdf", mat.brdf), ("sampler", mat.sampler), ("frame", mat.frame)):
            if net is None:
                continue
            for (w, b, a), (gw, gb, ga) in zip(net.layers, golden_nets(g, prefix)):
                assert np.array_equal(w, gw) and np.array_equal(b, gb) and a == ga


def test_oracle_zenith_pdf_goldens():
    """tests/test_proxy.py:39-55 analytic goldens."""
    z = np.array([[0.0, 0.0, 1.0]])

    def mk(wd, alpha):
        return O.Proxy(wd, 1 - wd, [[0, 0]], [alpha], 0.0, [[0, 0]])

    assert O.pdf(mk(1.0, (0.5, 0.5)), z, z)[0] == pytest.approx(1 / np.pi, rel=1e-12)
    assert O.pdf(mk(0.0, (1.0, 1.0)), z, z)[0] == pytest.approx(1 / (4 * np.pi), rel=1e-9)
    assert O.pdf(mk(0.5, (1.0, 1.0)), z, z)[0] == pytest.approx(0.5 / np.pi + 0.5 / (4 * np.pi), rel=1e-9)


def test_lod_from_ray_cones_matches_reference():
    """render._surface_frames_and_level / footprint_to_level goldens
    (produced by the reference renderer itself, oracle/make_golden.py)."""
    from oracle import nm_oracle as O
    g = load_golden("lod")
    lv = O.cone_level(g["cone_w"], g["cone_s"], g["t"], g["cos_hit"], g["density"], int(g["n_levels"]))
    assert np.array_equal(lv, g["level"])
    assert np.array_equal(O.footprint_to_level(g["area"], int(g["n_levels"])), g["area_level"])


def test_training_side_oracle_matches_reference():
    """forward_cached / backward / accumulate_texel_grads restatements
    against the reference's own outputs (tests/golden/train.npz)."""
    g = load_golden("train")
    for tag in ("brdf", "samp", "wide", "deep"):
        n = int(g[f"{tag}_n"])
        net = O.Net([(g[f"{tag}_w{i}"], g[f"{tag}_b{i}"], "linear" if int(g[f"{tag}_a{i}"]) == 0 else "leaky_relu")
                     for i in range(n)])
        out, cache = O.forward_cached(net, g[f"{tag}_x"])
        assert np.array_equal(out, g[f"{tag}_out"])
        grads, dx = O.backward(net, cache, g[f"{tag}_g"])
        assert np.array_equal(dx, g[f"{tag}_dx"])
        for i in range(n):
            assert np.array_equal(grads[i][0], g[f"{tag}_dw{i}"])
            assert np.array_equal(grads[i][1], g[f"{tag}_db{i}"])
    levels = []
    i = 0
    while f"tg_grad{i}" in g:
        levels.append(np.zeros_like(g[f"tg_grad{i}"]))
        i += 1
    pyr = O.Pyramid([np.zeros_like(l) for l in levels])
    pyr.accumulate_texel_grads(levels, g["tg_uv"].astype(np.float64), g["tg_level"], g["tg_zgrad"])
    for i, l in enumerate(levels):
        assert np.array_equal(l, g[f"tg_grad{i}"])


@pytest.mark.parametrize("tag", ["std", "oneframe", "vanilla", "iso", "albedo", "wide"])
def test_kl_sampler_loss_oracle_matches_reference(tag):
    """oracle.sampler_loss_and_grads against the reference's own
    training.sampler_loss_and_grads (tests/golden/kl.npz)."""
    import json
    g = load_golden("kl")
    cfg = O.Config(**json.loads(str(g[f"{tag}_config"])))

    def net(prefix):
        n = int(g[f"{tag}_{prefix}_n"])
        return O.Net([(g[f"{tag}_{prefix}_w{i}"], g[f"{tag}_{prefix}_b{i}"],
                       O.ACT_LINEAR if int(g[f"{tag}_{prefix}_a{i}"]) == 0 else O.ACT_LEAKY)
                      for i in range(n)]) if n else None

    mat = O.Material(cfg, net("frame"), net("brdf"), net("sampler"))
    loss, grads = O.sampler_loss_and_grads(mat, g[f"{tag}_z"], g[f"{tag}_wi"], (g[f"{tag}_ud"], g[f"{tag}_us"]))
    assert abs(loss - float(g[f"{tag}_loss"])) <= 1e-12 * abs(float(g[f"{tag}_loss"]))
    for i, (dw, db) in enumerate(grads):
        for a, want in ((dw, g[f"{tag}_dw{i}"]), (db, g[f"{tag}_db{i}"])):
            assert np.abs(a - want).max() <= 1e-6 * np.abs(want).max() + 1e-12


def _reference():
    import importlib
    import sys
    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference not mounted")
    if src not in sys.path:
        sys.path.insert(0, src)
    return importlib.import_module("neuralmat")


def test_oracle_trilinear_is_the_reference_expectation():
    """O.fetch_trilinear == (1-f) fetch_level(lo) + f fetch_level(hi) of the
    reference pyramid (latent.py:84-107, test_acceptance.py:251)."""
    _reference()
    from neuralmat import latent as RL
    rng = np.random.default_rng(5)
    opyr = O.random_pyramid(rng, 32, 32)
    rpyr = RL.LatentPyramid([l.copy() for l in opyr.levels])
    uv = rng.random((300, 2)).astype(np.float32)
    for lvl in (0.0, 1.3, 2.75, 4.0, 9.0):
        lv = min(float(np.float32(lvl)), rpyr.n_levels - 1)  # the level as the fp32 the kernels take
        lo = int(np.floor(lv))
        hi = min(lo + 1, rpyr.n_levels - 1)
        f = lv - lo
        want = ((1.0 - f) * rpyr.fetch_level(uv, lo).astype(np.float64)
                + f * rpyr.fetch_level(uv, hi).astype(np.float64)).astype(np.float32)
        assert np.array_equal(O.fetch_trilinear(opyr, uv, np.full(300, lvl, np.float32)), want)


def test_oracle_chi2_harness_matches_reference():
    """O.chi_square_test restates chi2.py:46-72: same statistic on the same samples."""
    _reference()
    from neuralmat import chi2 as RC
    from neuralmat import proxy as RP
    p = RP.ProxyParams(0.4, 0.6, (0.1, -0.2), (0.5, 0.3), 0.2, (0.1, 0.05))
    wi = np.array([0.2, 0.1, 0.97]) / np.linalg.norm([0.2, 0.1, 0.97])

    def run(test):
        rng = np.random.default_rng(9)

        def sample_fn(n):
            rep = p.take(np.zeros(n, dtype=np.int64))
            return RP.sample(rep, np.broadcast_to(wi, (n, 3)), rng.random((n, 3)))

        def pdf_fn(d):
            rep = p.take(np.zeros(d.shape[0], dtype=np.int64))
            return RP.pdf(rep, np.broadcast_to(wi, d.shape), d)

        return test(sample_fn, pdf_fn, 50_000)

    ok_r, p_r, s_r, d_r = run(RC.chi_square_test)
    ok_o, p_o, s_o, d_o = run(O.chi_square_test)
    assert (ok_r, d_r) == (ok_o, d_o) and s_r == pytest.approx(s_o, rel=1e-12) and p_r == pytest.approx(p_o, rel=1e-9)


def oracle_decoder_inputs(mat, z, wi, wo):
    """The BRDF decoder's fp16 direction inputs as the reference forms them
    (neural.py:282-287), from the oracle's frames: fp16 bit patterns."""
    raw = mat.half()["frame"].forward(np.atleast_2d(z).astype(np.float32))
    fr = O.frames_from_raw(raw)
    x = np.concatenate([O.frame_transform(fr, wi), O.frame_transform(fr, wo)], axis=-1)
    return x.astype(np.float32).astype(np.float16).view(np.uint16)


def test_oracle_float64_inputs_bit_exact():
    """Genuinely float64 uv / level / u_rr / wi / wo (the reference renderer's
    dtype): levels and z bit-exact, the decoder's fp16 direction inputs
    bit-exact (own frames, the degenerate fallback, a near-degenerate
    tangent), colours to 1e-12."""
    g = load_golden("f64_inputs")
    mat = oracle_material(g)
    f, _, chosen = O.eval_material(mat, g["uv"], g["lod"], g["wi"], g["wo"], g["u_rr"], fp16=True)
    assert np.array_equal(chosen, g["chosen"])
    np.testing.assert_allclose(f, g["f"], rtol=1e-12, atol=1e-12)
    z, _ = mat.half()["latent"].fetch(g["uv"], g["lod"], g["u_rr"])
    assert np.array_equal(z, g["z"])
    assert np.array_equal(oracle_decoder_inputs(mat, z, g["wi"], g["wo"]), g["x16"])
    for tag in ("degen", "near"):
        m2 = oracle_material(g)
        m2.frame = O.Net([(np.zeros((12, 8), np.float32), g[f"bias_{tag}"], "linear")])
        m2._half = None
        assert np.array_equal(oracle_decoder_inputs(m2, z, g["wi"], g["wo"]), g[f"x16_{tag}"]), tag
