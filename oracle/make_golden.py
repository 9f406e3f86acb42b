"""Generate golden vectors for the query path by running the REAL reference
implementation (/root/reference/pkg/src/neuralmat) — test infrastructure.

Writes tests/golden/*.npz (+ one reference-written archive).  The fixtures
pin (a) the numpy oracle in oracle/nm_oracle.py and (b) the CUDA kernels on
the GPU box, where /root/reference does not exist.

    python oracle/make_golden.py
"""

import json
import os
import shutil
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def _ref():
    sys.path.insert(0, REF)
    import neuralmat  # noqa: F401
    from neuralmat import geom, latent, neural, proxy
    return geom, latent, neural, proxy


def _f32(a):
    return np.asarray(a, dtype=np.float32)


def _nets(prefix, net, d):
    if net is None:
        d[prefix + "_n"] = np.int64(0)
        return
    d[prefix + "_n"] = np.int64(len(net.layers))
    for i, l in enumerate(net.layers):
        d[f"{prefix}_w{i}"] = l.w
        d[f"{prefix}_b{i}"] = l.b
        d[f"{prefix}_a{i}"] = np.int64(0 if l.act == "linear" else 1)


def make_case(name, cfg_kwargs, res=(64, 64), n=1024, seed=0, uv_lo=0.0, uv_hi=1.0,
              taps=False, fp32_path=False):
    geom, latent, neural, proxy = _ref()
    cfg = neural.NeuralMaterialConfig(**cfg_kwargs)
    mat = neural.NeuralMaterial.create(cfg, np.random.default_rng(seed))
    lrng = np.random.default_rng(seed + 1)
    pyr = latent.LatentPyramid.zeros(res[0], res[1])
    for lvl in pyr.levels:
        lvl[:] = lrng.standard_normal(lvl.shape).astype(np.float32)
    mat.latent = pyr
    q = np.random.default_rng(seed + 2)
    uv = _f32(uv_lo + (uv_hi - uv_lo) * q.random((n, 2)))
    lod = _f32(q.random(n) * (pyr.n_levels - 1))
    u_rr = _f32(q.random(n))
    wi, wo = geom.sample_half_diff(q, n)
    wi, wo = _f32(wi), _f32(wo)
    u3 = _f32(q.random((n, 3)))
    # reference fp16 path
    hl = mat.half()["latent"]
    z, chosen = hl.fetch(uv.astype(np.float64), lod.astype(np.float64), u_rr.astype(np.float64))
    f, albedo = neural.eval_brdf(mat, z, wi.astype(np.float64), wo.astype(np.float64), fp16=True)
    p = neural.infer_proxy(mat, z, wi.astype(np.float64), fp16=True)
    ws = proxy.sample(p, wi.astype(np.float64), u3.astype(np.float64))
    pdf_ws = proxy.pdf(p, wi.astype(np.float64), ws)
    pdf_wo = proxy.pdf(p, wi.astype(np.float64), wo.astype(np.float64))
    f_mat, _, chosen2 = neural.eval_material(mat, uv.astype(np.float64), lod.astype(np.float64),
                                             wi.astype(np.float64), wo.astype(np.float64),
                                             u_rr.astype(np.float64), fp16=True)
    assert np.array_equal(chosen, chosen2) and np.array_equal(f, f_mat)
    d = dict(
        config=np.array(json.dumps(cfg.to_json())), res=np.array(res), seed=np.int64(seed),
        uv=uv, lod=lod, u_rr=u_rr, wi=wi, wo=wo, u3=u3,
        z=z, chosen=chosen, f=f, ws=ws, pdf_ws=pdf_ws, pdf_wo=pdf_wo,
        params=np.concatenate([p.wd[:, None], p.ws[:, None], p.mu_d, p.alpha, p.rho[:, None],
                               p.mu_s], axis=1),
    )
    if albedo is not None:
        d["albedo"] = albedo
    for i, l in enumerate(pyr.levels):
        d[f"lat{i}"] = l
    _nets("frame", mat.frame_layer, d)
    _nets("brdf", mat.brdf_decoder, d)
    _nets("sampler", mat.sampler_decoder, d)
    hq = mat.half()
    d["packed_brdf"] = hq["brdf"].packed
    d["packed_sampler"] = hq["sampler"].packed
    if hq["frame"] is not None:
        d["packed_frame"] = hq["frame"].packed
    if taps:
        xs = np.zeros((n, 4), np.int64)
        ys = np.zeros((n, 4), np.int64)
        wts = np.zeros((n, 4))
        for lv in np.unique(chosen):
            m = chosen == lv
            a, b, c = hl._taps(int(lv), uv[m].astype(np.float64))
            xs[m], ys[m], wts[m] = a, b, c
        d.update(xs=xs, ys=ys, wts=wts)
    if fp32_path:
        f32, _ = neural.eval_brdf(mat, z, wi.astype(np.float64), wo.astype(np.float64), fp16=False)
        d["f_fp32path"] = f32
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
    print(name, {k: v.shape for k, v in d.items() if hasattr(v, "shape") and v.ndim})


def make_proxy_case(name="proxy_kat", n=2048, seed=11):
    geom, latent, neural, proxy = _ref()
    rng = np.random.default_rng(seed)
    wd = rng.uniform(0.0, 1.0, n)
    mu_d = rng.uniform(-1, 1, (n, 2)) * rng.integers(0, 2, (n, 1))
    alpha = rng.uniform(0.02, 1.0, (n, 2))
    rho = rng.uniform(-0.9, 0.9, n)
    mu_s = rng.uniform(-0.5, 0.5, (n, 2))
    blk = _f32(np.concatenate([wd[:, None], 1 - wd[:, None], mu_d, alpha, rho[:, None], mu_s], 1))
    p = proxy.ProxyParams(blk[:, 0], blk[:, 1], blk[:, 2:4], blk[:, 4:6], blk[:, 6], blk[:, 7:9])
    wi = geom.sample_uniform_hemisphere(rng.random((n, 2)))
    wi[:, 2] = np.maximum(wi[:, 2], 0.05)
    wi = _f32(geom.normalize(wi))
    u3 = _f32(rng.random((n, 3)))
    wo_any = _f32(geom.sample_uniform_sphere(rng.random((n, 2))))
    ws = proxy.sample(p, wi.astype(np.float64), u3.astype(np.float64))
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), params=blk, wi=wi, u3=u3, wo=wo_any,
                        ws=ws, pdf_ws=proxy.pdf(p, wi.astype(np.float64), ws),
                        pdf_wo=proxy.pdf(p, wi.astype(np.float64), wo_any.astype(np.float64)))
    print(name)


def make_archive(name="archive_albedo"):
    geom, latent, neural, proxy = _ref()
    rng = np.random.default_rng(12)
    mat = neural.NeuralMaterial.create(neural.NeuralMaterialConfig(albedo_head=True), rng)
    mat.latent = latent.LatentPyramid.zeros(16, 16)
    for lvl in mat.latent.levels:
        lvl[:] = rng.standard_normal(lvl.shape).astype(np.float32)
    tmp = tempfile.mkdtemp()
    neural.save_archive(os.path.join(tmp, f"{name}.nma"), mat, include_encoder=True)
    for ext in (".nma", ".latents"):
        shutil.copy(os.path.join(tmp, name + ext), os.path.join(OUT, name + ext))
    print(name)


def make_lod_case(name="lod", n=4096, seed=31):
    """LoD from ray cones through the reference renderer itself:
    render._surface_frames_and_level on a one-quad scene bound to a neural
    material, plus render.footprint_to_level on raw areas (incl. < 1 and
    beyond the top level).  Inputs are fp32-representable (the GPU takes fp32)."""
    geom, latent, neural, proxy = _ref()
    from types import SimpleNamespace
    from neuralmat import render
    rng = np.random.default_rng(seed)
    mat = neural.NeuralMaterial.create(neural.NeuralMaterialConfig(), np.random.default_rng(seed + 1))
    mat.latent = latent.LatentPyramid.zeros(512, 512)
    quad = render.Quad([-1.0, 0.0, -1.0], [2.0, 0.0, 0.0], [0.0, 0.0, 2.0], material="m",
                       uv_scale=(3.0, 2.0))
    scene = render.Scene(None, [quad], {"m": render.NeuralBinding(mat)})
    d = geom.normalize(np.stack([rng.uniform(-1, 1, n), -rng.uniform(0.02, 1, n), rng.uniform(-1, 1, n)], -1))
    d = np.asarray(_f32(d), np.float64)
    t = np.asarray(_f32(rng.uniform(0.01, 50.0, n)), np.float64)
    cone_w = np.asarray(_f32(rng.uniform(0.0, 0.05, n)), np.float64)
    cone_s = np.asarray(_f32(rng.uniform(0.0, 0.01, n)), np.float64)
    hits = SimpleNamespace(pos=np.zeros((n, 3)) + t[:, None] * d, obj=np.zeros(n, dtype=np.int64), t=t)
    frames, level = render._surface_frames_and_level(scene, SimpleNamespace(), hits, d, cone_w, cone_s)
    cos_hit = np.abs(np.sum(frames.n * d, axis=-1))
    area = np.asarray(_f32(np.exp(rng.uniform(-3.0, 30.0, n))), np.float64)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), cone_w=cone_w, cone_s=cone_s, t=t,
                        cos_hit=cos_hit, density=np.float64(quad.texel_density((512, 512))),
                        n_levels=np.int64(mat.latent.n_levels), level=level, area=area,
                        area_level=render.footprint_to_level(area, mat.latent.n_levels))
    print(name)


def make_train_case(name="train", seed=41):
    """Training-side goldens from the reference itself:
    Mlp.forward_cached / Mlp.backward on a BRDF-shaped (20-32-32-3) and a
    sampler-shaped (11-32-32-32-9) network, and LatentPyramid.
    accumulate_texel_grads on a 32x16 pyramid (incl. wrapped uv)."""
    geom, latent, neural, proxy = _ref()
    from neuralmat import mlp
    rng = np.random.default_rng(seed)
    d = {}
    for tag, sizes in (("brdf", (20, 32, 32, 3)), ("samp", (11, 32, 32, 32, 9))):
        net = mlp.Mlp.create(sizes, rng)
        for l in net.layers:  # non-zero biases so db is exercised
            l.b[:] = rng.normal(0, 0.1, l.b.shape).astype(np.float32)
        x = _f32(rng.normal(0, 1, (4099, sizes[0])))
        g = _f32(rng.normal(0, 1, (4099, sizes[-1])))
        out, cache = net.forward_cached(x)
        grads, dx = net.backward(cache, g)
        d[f"{tag}_n"] = np.int64(len(net.layers))
        for i, l in enumerate(net.layers):
            d[f"{tag}_w{i}"] = l.w
            d[f"{tag}_b{i}"] = l.b
            d[f"{tag}_a{i}"] = np.int64(0 if l.act == "linear" else 1)
            d[f"{tag}_dw{i}"] = grads[i][0]
            d[f"{tag}_db{i}"] = grads[i][1]
        d[f"{tag}_x"], d[f"{tag}_g"], d[f"{tag}_out"], d[f"{tag}_dx"] = x, g, out, dx
    # the 3x64 BRDF decoder's shape (the width-64 kernel instances) and a
    # 13-layer width-64 net whose padded / float64 weight copies exceed the
    # 200 KB SMEM budget (the unpadded forward and float-weight backward
    # fallbacks); own generator, so the cases above stay as they were
    wrng = np.random.default_rng(seed + 1)
    for tag, sizes in (("wide", (20, 64, 64, 64, 3)), ("deep", (20,) + (64,) * 12 + (3,))):
        net = mlp.Mlp.create(sizes, wrng)
        for l in net.layers:
            l.b[:] = wrng.normal(0, 0.1, l.b.shape).astype(np.float32)
        x = _f32(wrng.normal(0, 1, (2051, sizes[0])))
        g = _f32(wrng.normal(0, 1, (2051, sizes[-1])))
        out, cache = net.forward_cached(x)
        grads, dx = net.backward(cache, g)
        d[f"{tag}_n"] = np.int64(len(net.layers))
        for i, l in enumerate(net.layers):
            d[f"{tag}_w{i}"] = l.w
            d[f"{tag}_b{i}"] = l.b
            d[f"{tag}_a{i}"] = np.int64(0 if l.act == "linear" else 1)
            d[f"{tag}_dw{i}"] = grads[i][0]
            d[f"{tag}_db{i}"] = grads[i][1]
        d[f"{tag}_x"], d[f"{tag}_g"], d[f"{tag}_out"], d[f"{tag}_dx"] = x, g, out, dx
    pyr = latent.LatentPyramid.zeros(32, 16)
    for lvl in pyr.levels:
        lvl[:] = rng.standard_normal(lvl.shape).astype(np.float32)
    n = 5000
    uv = _f32(rng.uniform(-1.5, 2.5, (n, 2)))
    chosen = rng.integers(0, pyr.n_levels, n)
    zg = _f32(rng.normal(0, 1, (n, 8)))
    grads = pyr.zero_grads()
    pyr.accumulate_texel_grads(grads, uv.astype(np.float64), chosen, zg)
    d.update(tg_uv=uv, tg_level=chosen.astype(np.int64), tg_zgrad=zg, tg_w=np.int64(32), tg_h=np.int64(16))
    for i, gl in enumerate(grads):
        d[f"tg_grad{i}"] = gl
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
    print(name)


def make_vertex_case(name="vertex", n=3000, seed=51, f64=False):
    """The renderer's per-vertex shading context (render.py:340-420,
    SURVEY §8 f2) on a two-material scene: material "alpha" (2x32) bound
    fp16, "beta" (2x16) bound fp32, objects [beta, alpha, beta]; records
    eval(wi), sample(rng) -> (wi, pdf) and pdf(wi) of the reference's own
    _VertexShading, plus the inputs and both materials."""
    geom, latent, neural, proxy = _ref()
    from types import SimpleNamespace
    from neuralmat import render
    d = {}
    mats = {}
    for k, (tag, arch) in enumerate((("alpha", "2x32"), ("beta", "2x16"))):
        cfg = neural.NeuralMaterialConfig(brdf_hidden=arch)
        mat = neural.NeuralMaterial.create(cfg, np.random.default_rng(seed + 10 * k))
        lrng = np.random.default_rng(seed + 10 * k + 1)
        pyr = latent.LatentPyramid.zeros(32, 32)
        for lvl in pyr.levels:
            lvl[:] = lrng.standard_normal(lvl.shape).astype(np.float32)
        mat.latent = pyr
        mats[tag] = mat
        d[f"{tag}_config"] = np.array(json.dumps(cfg.to_json()))
        for i, l in enumerate(pyr.levels):
            d[f"{tag}_lat{i}"] = l
        _nets(f"{tag}_frame", mat.frame_layer, d)
        _nets(f"{tag}_brdf", mat.brdf_decoder, d)
        _nets(f"{tag}_sampler", mat.sampler_decoder, d)
    objects = [SimpleNamespace(material=m) for m in ("beta", "alpha", "beta")]
    materials = {"alpha": render.NeuralBinding(mats["alpha"], fp16=True),
                 "beta": render.NeuralBinding(mats["beta"], fp16=False)}
    scene = SimpleNamespace(objects=objects, materials=materials)
    q = np.random.default_rng(seed + 2)
    obj = q.integers(0, 3, n)
    uv = q.uniform(-0.5, 1.5, (n, 2))
    level = q.random(n) * 5.0
    wi, wo = geom.sample_half_diff(q, n)
    if not f64:  # fp32-representable inputs (the original case); f64: the renderer's own values
        uv, level = _f32(uv), _f32(level).astype(np.float64)
        wi, wo = _f32(wi).astype(np.float64), _f32(wo).astype(np.float64)
    hits = SimpleNamespace(obj=obj, uv=uv.astype(np.float64))
    out = {}
    for tag, cfg in (("lod", render.RenderConfig(lod=True)),
                     ("nolod", render.RenderConfig(lod=False)),
                     ("forced", render.RenderConfig(force_level=2, fp16=True))):
        rng = np.random.default_rng(seed + 3)
        ctx = render._VertexShading(scene, cfg, hits, wo, level, rng)
        f = ctx.eval(wi)
        ws, pdf_s = ctx.sample(rng)
        pb = ctx.pdf(wi)
        out.update({f"{tag}_f": f, f"{tag}_ws": ws, f"{tag}_pdf_ws": pdf_s, f"{tag}_pdf_wi": pb})
    d.update(obj=obj.astype(np.int64), uv=uv, level=level, wi=wi, wo=wo, rng_seed=np.int64(seed + 3), **out)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
    print(name)


def make_kl_case(name="kl", b=2048, seed=61):
    """KL sampler loss (training.py:219-273) from the reference:
    loss and sampler-decoder gradients with fixed uniforms, for the default
    material (2 frames), one frame, no frames (vanilla), isotropic sampler,
    the albedo head (6 decoder outputs) and the 3x64 BRDF decoder."""
    geom, latent, neural, proxy = _ref()
    from neuralmat import training
    d = {}
    variants = (("std", {}), ("oneframe", {"n_frames": 1}), ("vanilla", {"use_frames": False}),
                ("iso", {"sampler_isotropic": True}), ("albedo", {"albedo_head": True}),
                ("wide", {"brdf_hidden": "3x64"}))
    for k, (tag, kw) in enumerate(variants):
        cfg = neural.NeuralMaterialConfig(**kw)
        mat = neural.NeuralMaterial.create(cfg, np.random.default_rng(seed + k))
        rng = np.random.default_rng(seed + 100 + k)
        z = _f32(rng.normal(0, 1, (b, 8)))
        wi, _ = geom.sample_half_diff(rng, b)
        us = (rng.random((b, 2)), rng.random((b, 2)))
        loss, grads = training.sampler_loss_and_grads(mat, z, wi, None, us=us)
        d[f"{tag}_config"] = np.array(json.dumps(cfg.to_json()))
        _nets(f"{tag}_frame", mat.frame_layer, d)
        _nets(f"{tag}_brdf", mat.brdf_decoder, d)
        _nets(f"{tag}_sampler", mat.sampler_decoder, d)
        d.update({f"{tag}_z": z, f"{tag}_wi": wi, f"{tag}_ud": us[0], f"{tag}_us": us[1],
                  f"{tag}_loss": np.float64(loss)})
        for i, (dw, db) in enumerate(grads):
            d[f"{tag}_dw{i}"] = dw
            d[f"{tag}_db{i}"] = db
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
    print(name)


def make_vertex_f64_case():
    make_vertex_case("vertex_f64", f64=True)


def make_f64_case(name="f64_inputs", n=4096, seed=71):
    """The reference on genuinely float64 inputs (what its renderer passes,
    render.py:369): uv / level / u_rr / wi / wo not representable in fp32, a
    non-power-of-two pyramid.  Records eval_material's f and levels, and the
    BRDF decoder's fp16 direction inputs (neural.py:282-287:
    inp.astype(float32) -> fp16 in fused_forward) for the material's own
    frames and for two hand-set frame layers (all rows on the degenerate
    fallback tangent; a tangent 1e-8 from the normal)."""
    geom, latent, neural, proxy = _ref()
    cfg = neural.NeuralMaterialConfig()
    mat = neural.NeuralMaterial.create(cfg, np.random.default_rng(seed))
    lrng = np.random.default_rng(seed + 1)
    pyr = latent.LatentPyramid.zeros(40, 24)
    for lvl in pyr.levels:
        lvl[:] = lrng.standard_normal(lvl.shape).astype(np.float32)
    mat.latent = pyr
    q = np.random.default_rng(seed + 2)
    uv = -1.0 + 3.0 * q.random((n, 2))
    lod = q.random(n) * (pyr.n_levels - 1)
    u_rr = q.random(n)
    wi, wo = geom.sample_half_diff(q, n)
    assert not np.array_equal(wi.astype(np.float32).astype(np.float64), wi)
    f, _, chosen = neural.eval_material(mat, uv, lod, wi, wo, u_rr, fp16=True)
    z, chosen2 = mat.half()["latent"].fetch(uv, lod, u_rr)
    assert np.array_equal(chosen, chosen2)

    def dec_inputs(m):
        raw = m.half()["frame"].fused_forward(np.atleast_2d(z).astype(np.float32))
        fr = neural.frames_from_raw(raw)
        x = np.concatenate([fr.transform(wi), fr.transform(wo)], axis=-1)
        return x.astype(np.float32).astype(np.float16).view(np.uint16)

    d = dict(config=np.array(json.dumps(cfg.to_json())), uv=uv, lod=lod, u_rr=u_rr, wi=wi, wo=wo,
             z=z, chosen=chosen, f=f, x16=dec_inputs(mat))
    from neuralmat import mlp as rmlp
    for tag, bias in (("degen", [0.0, 0.0, 1.0, 0.0, 0.0, 1.0] * 2),
                      ("near", [0.0, 0.0, 1.0, 1.0, 0.0, 0.0, 0.0, 0.0, 1.0, 1e-8, 0.0, 1.0])):
        m2 = neural.NeuralMaterial.create(cfg, np.random.default_rng(seed))
        m2.frame_layer = rmlp.Mlp([rmlp.Layer(np.zeros((12, 8), np.float32), np.asarray(bias, np.float32),
                                              "linear")])
        d[f"x16_{tag}"] = dec_inputs(m2)
        d[f"bias_{tag}"] = np.asarray(bias, np.float32)
    for i, l in enumerate(pyr.levels):
        d[f"lat{i}"] = l
    _nets("frame", mat.frame_layer, d)
    _nets("brdf", mat.brdf_decoder, d)
    _nets("sampler", mat.sampler_decoder, d)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
    print(name, {k: v.shape for k, v in d.items() if hasattr(v, "shape") and v.ndim})


def main():
    os.makedirs(OUT, exist_ok=True)
    make_case("c1_2x32", {}, n=4096, taps=True, fp32_path=True)
    make_case("c1_2x16", {"brdf_hidden": "2x16"}, seed=3)
    make_case("c1_3x64", {"brdf_hidden": "3x64"}, seed=6)
    make_case("albedo", {"albedo_head": True}, res=(32, 32), seed=9)
    make_case("isotropic", {"sampler_isotropic": True}, res=(32, 32), seed=12)
    make_case("vanilla", {"use_frames": False}, res=(32, 32), seed=15)
    make_case("one_frame", {"n_frames": 1}, res=(32, 32), seed=18)
    make_case("npot_wrap", {}, res=(24, 20), seed=21, uv_lo=-2.0, uv_hi=3.0, taps=True)
    make_proxy_case()
    make_archive()
    make_lod_case()
    make_train_case()
    make_vertex_case()
    make_vertex_f64_case()
    make_kl_case()
    make_f64_case()


if __name__ == "__main__":
    if len(sys.argv) > 1:  # regenerate only the named cases, e.g. make_f64_case
        os.makedirs(OUT, exist_ok=True)
        for fn in sys.argv[1:]:
            globals()[fn]()
    else:
        main()
