"""KL sampler loss (reference training.py:219-273) on the GPU
against the reference's own loss and sampler-decoder gradients
(tests/golden/kl.npz, oracle/make_golden.py:make_kl_case): default material,
one frame, no frames, isotropic sampler, albedo head — fixed uniforms."""
import json

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

TAGS = ("std", "oneframe", "vanilla", "iso", "albedo", "wide")


def _mat(g, tag):
    from paper_2305_02678_b200 import mlp, neural

    def net(prefix):
        n = int(g[f"{tag}_{prefix}_n"])
        return mlp.Mlp([mlp.Layer(g[f"{tag}_{prefix}_w{i}"], g[f"{tag}_{prefix}_b{i}"],
                                  "linear" if int(g[f"{tag}_{prefix}_a{i}"]) == 0 else "leaky_relu")
                        for i in range(n)]) if n else None

    cfg = neural.NeuralMaterialConfig(**json.loads(str(g[f"{tag}_config"])))
    return neural.NeuralMaterial(cfg, None, net("frame"), net("brdf"), net("sampler"))


def _grads_close(grads, g, tag, rtol):
    i = 0
    while f"{tag}_dw{i}" in g:
        for name, a, want in (("dW", grads[i][0], g[f"{tag}_dw{i}"]), ("db", grads[i][1], g[f"{tag}_db{i}"])):
            assert a.dtype == want.dtype and a.shape == want.shape, (tag, i, name, a.dtype, want.dtype)
            # fp32 network passes in a different summation order than numpy's
            # BLAS: errors scale with the layer's gradient magnitude
            scale = np.abs(want).max()
            err = np.abs(a.astype(np.float64) - want).max()
            assert err <= rtol * scale + 1e-9, (tag, i, name, err, scale)
        i += 1
    assert len(grads) == i


@pytest.mark.parametrize("tag", TAGS)
def test_sampler_loss_and_grads_vs_reference(tag):
    from paper_2305_02678_b200 import train

    g = load_golden("kl")
    mat = _mat(g, tag)
    loss, grads = train.sampler_loss_and_grads(mat, g[f"{tag}_z"], g[f"{tag}_wi"], None,
                                               us=(g[f"{tag}_ud"], g[f"{tag}_us"]))
    assert isinstance(loss, float)
    want = float(g[f"{tag}_loss"])
    assert abs(loss - want) <= 1e-10 * max(1.0, abs(want)), (loss, want)  # measured ~1e-14
    _grads_close(grads, g, tag, rtol=2e-5)  # measured <= 5.1e-6 of the largest entry (3xTF32 dW)


def test_sampler_loss_custom_target_and_rng():
    """target_and_grad hook and the rng draw order (rng.random((b,2)) twice)."""
    from paper_2305_02678_b200 import train

    g = load_golden("kl")
    mat = _mat(g, "std")
    z, wi = g["std_z"], g["std_wi"]
    b = z.shape[0]

    def tg(wo):  # a smooth positive target: 1 + wo.z^2 and its gradient
        wo = np.asarray(wo)
        return 1.0 + wo[:, 2] ** 2, np.stack([0 * wo[:, 0], 0 * wo[:, 1], 2 * wo[:, 2]], 1)

    l1, g1 = train.sampler_loss_and_grads(mat, z, wi, None, target_and_grad=tg,
                                          us=(g["std_ud"], g["std_us"]))
    rng = np.random.default_rng(5)
    us = (rng.random((b, 2)), rng.random((b, 2)))
    l2, _ = train.sampler_loss_and_grads(mat, z, wi, np.random.default_rng(5), target_and_grad=tg)
    l3, _ = train.sampler_loss_and_grads(mat, z, wi, None, target_and_grad=tg, us=us)
    assert l2 == l3 and np.isfinite(l1)
    assert all(np.all(np.isfinite(a)) for pair in g1 for a in pair)
