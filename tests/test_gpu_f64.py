"""The reference's own float64 inputs (its renderer passes float64 uv,
level, u_rr and directions, render.py:369) and the exact fp16 rounding of
the BRDF decoder's direction inputs (neural.py:282-287).

Goldens: tests/golden/f64_inputs.npz and vertex_f64.npz, written by the
reference itself (oracle/make_golden.py make_f64_case / make_vertex_f64_case).
The decoder inputs are compared as fp16 bit patterns: bit-exact.
"""

import numpy as np
import pytest
import torch

from conftest import load_golden
from test_gpu_parity import _oracle_from, check_rel, our_material
from test_oracle_golden import oracle_decoder_inputs

pytestmark = pytest.mark.gpu


def _decoder_inputs(mat, z, wi, wo):
    """nm_decoder_inputs: (n, 12) uint16 fp16 bit patterns; float64 numpy
    directions go in as float64, fp32 ones as fp32."""
    from paper_2305_02678_b200 import _io, _lib
    lib = _lib.load()
    h = mat.device_material(None)
    dev = h.device
    n = z.shape[0]
    z_t = torch.from_numpy(np.ascontiguousarray(z, np.float32)).to(dev)
    out = torch.empty((n, 12), dtype=torch.int16, device=dev)
    if np.asarray(wi).dtype == np.float64:
        wi_t = torch.from_numpy(np.ascontiguousarray(wi)).to(dev)
        wo_t = torch.from_numpy(np.ascontiguousarray(wo)).to(dev)
        args = (None, None, wi_t.data_ptr(), wo_t.data_ptr())
    else:
        wi_t = torch.from_numpy(np.ascontiguousarray(wi, np.float32)).to(dev)
        wo_t = torch.from_numpy(np.ascontiguousarray(wo, np.float32)).to(dev)
        args = (wi_t.data_ptr(), wo_t.data_ptr(), None, None)
    _lib.check(lib.nm_decoder_inputs(h.ptr, n, z_t.data_ptr(), *args, out.data_ptr(), _io.stream_ptr(dev)))
    return out.cpu().numpy().view(np.uint16)


def _with_frame_bias(g, bias):
    from paper_2305_02678_b200 import mlp
    mat = our_material(g)
    mat.frame_layer = mlp.Mlp([mlp.Layer(np.zeros((12, 8), np.float32), np.asarray(bias, np.float32),
                                         mlp.ACT_LINEAR)])
    return mat


def test_decoder_inputs_bit_exact_vs_reference_golden():
    """The reference's own fp16 decoder inputs on float64 directions: the
    material's frames, the degenerate fallback tangent on every row, a
    tangent 1e-8 from the normal."""
    g = load_golden("f64_inputs")
    assert np.array_equal(_decoder_inputs(our_material(g), g["z"], g["wi"], g["wo"]), g["x16"])
    for tag in ("degen", "near"):
        mat = _with_frame_bias(g, g[f"bias_{tag}"])
        assert np.array_equal(_decoder_inputs(mat, g["z"], g["wi"], g["wo"]), g[f"x16_{tag}"]), tag


@pytest.mark.parametrize("f64", [False, True])
def test_decoder_inputs_bit_exact_at_scale(f64):
    """524,288 rows (random fp16 codes, half/difference direction pairs in
    float64 or fp32) against the oracle's numpy frames (pinned bit-exactly
    to the reference above): every fp16 bit pattern equal."""
    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import neural
    rng = np.random.default_rng(81 + int(f64))
    from paper_2305_02678_b200.latent import LatentPyramid
    mat = neural.NeuralMaterial.create(neural.NeuralMaterialConfig(), rng)
    mat.latent = LatentPyramid(O.random_pyramid(rng, 8, 8).levels)  # unused by this entry point
    n = 1 << 19
    z = rng.standard_normal((n, 8)).astype(np.float16).astype(np.float32)
    wi, wo = O.draw_direction_pairs(rng, n)
    if not f64:
        wi, wo = wi.astype(np.float32), wo.astype(np.float32)
    om = _oracle_from(mat)
    ref = oracle_decoder_inputs(om, z, np.asarray(wi, np.float64), np.asarray(wo, np.float64))
    got = _decoder_inputs(mat, z, wi, wo)
    bad = np.flatnonzero(np.any(got != ref, axis=1))
    assert bad.size == 0, f"{bad.size} rows differ, first {bad[0]}: {got[bad[0]]} vs {ref[bad[0]]}"
    if f64:  # the float64 route is not vacuous: narrowing the directions first changes rows
        narrowed = _decoder_inputs(mat, z, wi.astype(np.float32), wo.astype(np.float32))
        assert np.any(narrowed != ref)


def test_eval_material_float64_inputs_vs_reference_golden():
    """eval_material on the reference's float64 arrays: levels bit-exact,
    colours strict (every value <= 1e-2 rel, mean <= 1e-3)."""
    from paper_2305_02678_b200 import neural
    g = load_golden("f64_inputs")
    mat = our_material(g)
    f, _, ch = neural.eval_material(mat, g["uv"], g["lod"], g["wi"], g["wo"], g["u_rr"], fp16=True)
    assert ch.dtype == np.int64 and np.array_equal(ch, g["chosen"])
    check_rel(f, g["f"], what="float64 eval_material")
    z, ch2 = mat.half()["latent"].fetch(g["uv"], g["lod"], g["u_rr"])
    assert np.array_equal(ch2, g["chosen"]) and np.array_equal(z, g["z"])
    # eval_brdf from the codes on the float64 directions (nm_eval_z_f64)
    f2, _ = neural.eval_brdf(mat, g["z"], g["wi"], g["wo"], fp16=True)
    check_rel(f2, g["f"], what="float64 eval_brdf")
    # the full query's eval part on the same float64 inputs (nm_query_f64)
    u3 = np.random.default_rng(3).random((g["uv"].shape[0], 3))
    f3, _, _ = neural.query(mat, g["uv"], g["lod"], g["u_rr"], g["wi"], g["wo"], u3)
    check_rel(f3, g["f"], what="float64 query rgb")


def test_decoder_inputs_one_frame_material():
    """One learned frame: the decoder's direction inputs are [T.wi(3), T.wo(3)]
    (x16 halves 0..5, the rest 0) — bit-exact against the oracle on float64
    directions."""
    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import neural
    from paper_2305_02678_b200.latent import LatentPyramid
    rng = np.random.default_rng(87)
    mat = neural.NeuralMaterial.create(neural.NeuralMaterialConfig(n_frames=1), rng)
    mat.latent = LatentPyramid(O.random_pyramid(rng, 8, 8).levels)
    n = 65536
    z = rng.standard_normal((n, 8)).astype(np.float16).astype(np.float32)
    wi, wo = O.draw_direction_pairs(rng, n)
    got = _decoder_inputs(mat, z, wi, wo)
    ref = oracle_decoder_inputs(_oracle_from(mat), z, wi, wo)  # (n, 6)
    assert np.array_equal(got[:, :6], ref) and not got[:, 6:].any()


def test_float64_inputs_fp32_path_and_albedo():
    """The reference's default fp16=False path and an albedo head on float64
    inputs (nm_query_f64 on the precise material): levels bit-exact, colours
    and albedo within the fp32 path's tolerance of the oracle."""
    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import neural
    from paper_2305_02678_b200.latent import LatentPyramid
    rng = np.random.default_rng(88)
    mat = neural.NeuralMaterial.create(neural.NeuralMaterialConfig(albedo_head=True), rng)
    mat.latent = LatentPyramid(O.random_pyramid(rng, 40, 24).levels)
    n = 20000
    uv = -1.0 + 3.0 * rng.random((n, 2))
    lod = rng.random(n) * (mat.latent.n_levels - 1)
    urr = rng.random(n)
    wi, wo = O.draw_direction_pairs(rng, n)
    om = _oracle_from(mat)
    for fp16 in (True, False):
        f, alb, ch = neural.eval_material(mat, uv, lod, wi, wo, urr, fp16=fp16)
        f_ref, alb_ref, ch_ref = O.eval_material(om, uv, lod, wi, wo, urr, fp16=fp16)
        assert np.array_equal(ch, ch_ref)
        tol = 1e-2 if fp16 else 1e-3
        check_rel(f, f_ref, max_tol=tol, what=f"float64 inputs fp16={fp16} rgb")
        check_rel(alb, alb_ref, max_tol=tol, what=f"float64 inputs fp16={fp16} albedo")


def test_entry_points_without_float64_reject_inexact_input():
    """spp and multi-material entry points have no float64 variant: they
    raise instead of silently narrowing (the reference computes in float64)."""
    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import neural
    from paper_2305_02678_b200.latent import LatentPyramid
    rng = np.random.default_rng(89)
    mat = neural.NeuralMaterial.create(neural.NeuralMaterialConfig(), rng)
    mat.latent = LatentPyramid(O.random_pyramid(rng, 16, 16).levels)
    n = 256
    uv = rng.random((n, 2))
    lod = np.full(n, 1.0)
    urr = rng.random(n)
    wi, wo = O.draw_direction_pairs(rng, n)
    with pytest.raises(ValueError):
        neural.eval_material_spp(mat, uv, lod, wi, wo, urr, 16)
    with pytest.raises(ValueError):
        neural.eval_material_multi([mat, mat], np.zeros(n, np.int32), uv, lod, wi, wo, urr)


def test_full_query_float64_inputs_sampled_directions():
    """The full query on float64 inputs: levels bit-exact, rgb strict, every
    sampled direction within 1e-3 of the oracle's outside the lobe-pick band
    (the reference samples from its float64 conditioning direction; the
    sampler decoder sees it narrowed to fp32 as the reference's does)."""
    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import neural
    from test_gpu_parity import check_dirs
    g = load_golden("f64_inputs")
    mat = our_material(g)
    om = _oracle_from(mat)
    u3 = np.random.default_rng(5).random((g["uv"].shape[0], 3))
    f, ws, pdf, ch = neural.query(mat, g["uv"], g["lod"], g["u_rr"], g["wi"], g["wo"], u3, return_level=True)
    f_ref, ws_ref, pdf_ref, p_ref, ch_ref = O.full_query(om, g["uv"], g["lod"], g["u_rr"], g["wi"], g["wo"], u3)
    assert np.array_equal(ch, ch_ref)
    check_rel(f, f_ref, what="float64 full query rgb")
    check_dirs(ws, ws_ref, u3, p_ref, g["wi"])
