"""Host-side logic of the product package (CPU only): fp16 quantization and
packing (the data nm_material_create consumes), file formats byte-compatible
with the reference, RNG-compatible material init, pyramid geometry.
Mirrors the reference's own tests (tests/test_mlp.py, test_latent.py,
test_neural.py) for the pieces that live on the host."""

import io
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_config, golden_nets, load_golden

from paper_2305_02678_b200 import latent, mlp, neural


def test_quantize_representable_and_rounding():
    """tests/test_mlp.py:186-194: fp16(0.1) = 0.0999755859375."""
    net = mlp.Mlp.create((2, 2), np.random.default_rng(8))
    net.layers[0].w[:] = np.array([[1.0, 0.1], [0.1, 1.0]], dtype=np.float32)
    q = mlp.quantize(net)
    w16 = q.layer_views()[0][0]
    assert w16[0, 0] == 1.0
    assert abs(w16[0, 1] - 0.0999755859375) < 1e-12


def test_quantize_clamps_and_counts():
    """tests/test_mlp.py:197-203."""
    net = mlp.Mlp.create((2, 2), np.random.default_rng(9))
    net.layers[0].w[0, 0] = 70000.0
    q = mlp.quantize(net)
    assert q.clamped == 1
    assert q.layer_views()[0][0][0, 0] == 65504.0


def test_packed_layout_access_order():
    """tests/test_mlp.py:234-241: per neuron [w_row..., bias]."""
    w = np.arange(6, dtype=np.float32).reshape(2, 3)
    net = mlp.Mlp([mlp.Layer(w, np.array([10.0, 20.0]), mlp.ACT_LINEAR)])
    q = mlp.quantize(net)
    assert np.allclose(q.packed[:4], [0, 1, 2, 10])
    assert np.allclose(q.packed[4:], [3, 4, 5, 20])


def test_quantize_matches_reference_packed_buffers():
    for name in ("c1_2x32", "vanilla", "one_frame"):
        g = load_golden(name)
        for prefix in ("brdf", "sampler", "frame"):
            if f"packed_{prefix}" not in g:
                continue
            net = mlp.Mlp([mlp.Layer(w, b, a) for w, b, a in golden_nets(g, prefix)])
            assert np.array_equal(mlp.quantize(net).packed.view(np.uint16),
                                  g[f"packed_{prefix}"].view(np.uint16))


def test_create_reproduces_reference_init():
    """NeuralMaterial.create consumes the RNG like neural.py:117-141."""
    for name in ("c1_2x32", "c1_3x64", "vanilla", "isotropic", "albedo", "one_frame"):
        g = load_golden(name)
        mat = neural.NeuralMaterial.create(neural.NeuralMaterialConfig(**golden_config(g)),
                                           np.random.default_rng(int(g["seed"])))
        for prefix, net in (("frame", mat.frame_layer), ("brdf", mat.brdf_decoder),
                            ("sampler", mat.sampler_decoder)):
            want = golden_nets(g, prefix)
            if net is None:
                assert not want
                continue
            for layer, (w, b, a) in zip(net.layers, want):
                assert np.array_equal(layer.w, w) and np.array_equal(layer.b, b) and layer.act == a


def test_blob_roundtrip_byte_identical():
    """tests/test_mlp.py:244-254."""
    net = mlp.Mlp.create((11, 32, 32, 32, 9), np.random.default_rng(12))
    data = mlp.blob_bytes(net)
    net2, q2 = mlp.blob_from_bytes(data)
    assert mlp.blob_bytes(net2) == data
    assert np.array_equal(q2.packed, mlp.quantize(net).packed)
    with pytest.raises(ValueError):
        mlp.read_blob(io.BytesIO(b"not a blob at all"))


def test_reads_reference_written_archive_byte_identically(tmp_path):
    """An NMATARC1 archive + latents written by the reference load here and
    re-save byte-identically (tests/test_neural.py:221-246)."""
    src = os.path.join(GOLDEN, "archive_albedo.nma")
    mat = neural.load_archive(src)
    assert mat.cfg.albedo_head and mat.encoder is not None
    assert mat.latent.n_levels == 5 and mat.latent.width == 16
    dst = tmp_path / "archive_albedo.nma"
    neural.save_archive(str(dst), mat, include_encoder=True)
    assert dst.read_bytes() == open(src, "rb").read()
    assert (tmp_path / "archive_albedo.latents").read_bytes() == \
        open(os.path.join(GOLDEN, "archive_albedo.latents"), "rb").read()


def test_level_shapes_halve_to_one():
    """tests/test_latent.py:17-20 plus a non-square, non-power-of-two case."""
    assert latent.level_shapes(64, 64) == [(64, 64), (32, 32), (16, 16), (8, 8), (4, 4), (2, 2), (1, 1)]
    assert latent.level_shapes(24, 20) == [(20, 24), (10, 12), (5, 6), (2, 3), (1, 1)]
    assert len(latent.level_shapes(4096, 4096)) == 13
    assert len(latent.level_shapes(15360, 15360)) == 14


def test_pyramid_file_roundtrip_equals_half_copy():
    """tests/test_latent.py:120-132."""
    rng = np.random.default_rng(7)
    pyr = latent.LatentPyramid.zeros(16, 16)
    for lvl in pyr.levels:
        lvl[:] = rng.standard_normal(lvl.shape).astype(np.float32)
    buf = io.BytesIO()
    latent.write_pyramid(buf, pyr)
    pyr2 = latent.read_pyramid(io.BytesIO(buf.getvalue()))
    buf2 = io.BytesIO()
    latent.write_pyramid(buf2, pyr2)
    assert buf.getvalue() == buf2.getvalue()
    for a, b in zip(pyr.half_copy(), pyr2.levels):
        assert np.array_equal(a.astype(np.float32), b)


def test_texel_blob_picks_fp16_only_when_exact():
    rng = np.random.default_rng(3)
    pyr = latent.LatentPyramid.zeros(8, 8)
    for lvl in pyr.levels:
        lvl[:] = rng.standard_normal(lvl.shape).astype(np.float32)
    blob, fp32 = pyr.texel_blob()
    assert fp32 and blob.dtype == np.float32
    half = latent.LatentPyramid([l.astype(np.float16).astype(np.float32) for l in pyr.levels])
    blob, fp32 = half.texel_blob()
    assert not fp32 and blob.dtype == np.float16 and blob.shape == (85, 8)


def test_fp16_false_selects_the_fp32_material_copy():
    """fp16=False (the reference's default) is served by a separate precise
    device copy — never silently by the fp16 one; without a GPU it fails loudly."""
    import inspect
    src = inspect.getsource(neural.eval_material) + inspect.getsource(neural._QueryInputs)
    assert "precise=not fp16" in src
    mat = neural.NeuralMaterial.create(neural.NeuralMaterialConfig(), np.random.default_rng(0))
    with pytest.raises(RuntimeError):  # no CUDA device here: no CPU fallback
        neural.eval_brdf(mat, np.zeros((1, 8), np.float32), [[0, 0, 1]], [[0, 0, 1]], fp16=False)

