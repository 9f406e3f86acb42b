"""Parity at the BASELINE.json configs' real sizes.

Every check is strict: chosen levels, tap indices and z bit-exact;
rgb / proxy parameters within rel |a-b|/(|b|+1e-2) <= 1e-2 for EVERY value
and mean <= 1e-3; sampled directions within 1e-3 outside the lobe-pick
guard band.  The batches are generated on the GPU at full size (C2: 4096^2
pyramid x 2,073,600 queries; C3: 33,177,600; C4: the five Table-1 pyramids,
8.3 GB of fp16 latents) and the oracle (the reference's algorithm restated,
pinned by test_oracle_golden.py) checks a seeded subset of >= 65,536 rows —
a stride sample over the whole batch, the partial last tile and random
rows — with the oracle's taps gathered from the device pyramid.
"""

import numpy as np
import pytest
import torch

from scaleutil import host, oracle_material, subset_rows
from test_gpu_parity import check_dirs, check_rel

pytestmark = pytest.mark.gpu

C2_N = 1920 * 1080


def _lib():
    from paper_2305_02678_b200 import _lib as L
    return L, L.load()


@pytest.mark.parametrize("arch", ["2x32", "3x64", "2x16"])
def test_c1_full_query_exact_size(arch):
    """C1 exactly: 1 random-init material, 512^2 pyramid, 65,536 queries,
    eval + sample + pdf (the reference-side recipe: numpy generator, latents
    N(0,1) per level, tests/test_latent.py:10-14)."""
    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import neural
    from paper_2305_02678_b200.latent import LatentPyramid

    rng = np.random.default_rng(0)
    mat = neural.NeuralMaterial.create(neural.NeuralMaterialConfig(brdf_hidden=arch), rng)
    mat.latent = LatentPyramid(O.random_pyramid(np.random.default_rng(0), 512, 512).levels)
    n = 65536
    qr = np.random.default_rng(1)
    uv = qr.random((n, 2)).astype(np.float32)
    lod = (qr.random(n) * (mat.latent.n_levels - 1)).astype(np.float32)
    urr = qr.random(n).astype(np.float32)
    wi, wo = O.draw_direction_pairs(qr, n)
    wi, wo = wi.astype(np.float32), wo.astype(np.float32)
    u3 = qr.random((n, 3)).astype(np.float32)

    def net(m):
        return O.Net([(l.w, l.b, l.act) for l in m.layers])

    om = O.Material(O.Config(**mat.cfg.to_json()), net(mat.frame_layer), net(mat.brdf_decoder),
                    net(mat.sampler_decoder))
    om.latent = O.Pyramid(mat.latent.levels)
    f_ref, ws_ref, pdf_ref, p_ref, ch_ref = O.full_query(om, uv, lod, urr, wi, wo, u3)
    z_ref, _ = om.half()["latent"].fetch(uv, lod, urr)

    z, ch = mat.half()["latent"].fetch(uv, lod, urr)
    assert np.array_equal(ch, ch_ref) and np.array_equal(z, z_ref)
    f, ws, pdf, ch = neural.query(mat, uv, lod, urr, wi, wo, u3, return_level=True)
    assert np.array_equal(ch, ch_ref)
    check_rel(f, f_ref, what=f"C1 {arch} query rgb")
    check_dirs(ws, ws_ref, u3, p_ref, wi)
    f2, _, _ = neural.eval_material(mat, uv, lod, wi, wo, urr, fp16=True)
    check_rel(f2, f_ref, what=f"C1 {arch} eval rgb")
    ws3, pdf3, p3 = neural.sample_pdf(mat, uv, lod, urr, wi, u3, return_params=True)
    check_rel(p3.as_array(), p_ref.as_array(), what=f"C1 {arch} params")
    check_dirs(ws3, ws_ref, u3, p_ref, wi)


def _c2_batch(seed=0):
    from paper_2305_02678_b200 import synth
    dev = torch.device("cuda", 0)
    mat = synth.material("2x32", 4096, 4096, seed=seed, device=dev)
    h = mat.device_material(dev)
    q = synth.queries(C2_N, mat.latent.n_levels, seed=1 + seed, device=dev)
    return mat, h, q


def test_c2_eval_full_batch():
    """C2: 4096^2 pyramid (13 levels), 2,073,600 coherent eval queries in one
    launch.  Levels bit-exact on every row; taps, z and rgb on the subset."""
    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import neural
    L, lib = _lib()
    mat, h, q = _c2_batch()
    n = C2_N
    f, lv = neural.eval_material(mat, q["uv"], q["lod"], q["wi"], q["wo"], q["u_rr"], fp16=True)[0::2]
    torch.cuda.synchronize()
    om = oracle_material(mat, h)
    pyr = om.half()["latent"]
    ch_all = pyr.choose_level(q["lod"].cpu().numpy(), q["u_rr"].cpu().numpy())
    assert np.array_equal(lv.cpu().numpy(), ch_all)
    rows = subset_rows(n, 65536)
    assert len(rows) >= 65536
    hq = host(q, rows)
    z_ref, ch_ref = pyr.fetch(hq["uv"], hq["lod"], hq["u_rr"])
    # taps and z through nm_fetch on the same rows
    sub = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in hq.items()}
    m = len(rows)
    z = torch.empty((m, 8), device="cuda")
    taps = torch.empty((m, 8), device="cuda", dtype=torch.int32)
    L.check(lib.nm_fetch(h.ptr, m, sub["uv"].data_ptr(), sub["lod"].data_ptr(), 1, sub["u_rr"].data_ptr(),
                         z.data_ptr(), None, taps.data_ptr(), None, torch.cuda.current_stream().cuda_stream))
    assert np.array_equal(z.cpu().numpy(), z_ref)
    t = taps.cpu().numpy().reshape(m, 4, 2)
    for lvl in np.unique(ch_ref):
        sel = ch_ref == lvl
        xs, ys, _ = pyr.taps(int(lvl), hq["uv"][sel].astype(np.float64))
        assert np.array_equal(t[sel, :, 0], xs) and np.array_equal(t[sel, :, 1], ys)
    f_ref, _ = O.eval_brdf(om, z_ref, hq["wi"], hq["wo"], fp16=True)
    check_rel(f.cpu().numpy()[rows], f_ref, what="C2 rgb")


def test_c2_exact_resolution_has_no_misses():
    """The fast kernel queues rows whose fp16 direction inputs lie within its
    error bound of a rounding midpoint.  Queuing EVERY row must give
    bit-identical output to the default bound on the full C2 batch (no row
    that needed resolution escaped it), and disabling the queue must not
    (the mechanism is what makes the strict parity hold)."""
    from paper_2305_02678_b200 import neural
    L, lib = _lib()
    mat, h, q = _c2_batch(seed=3)
    run = lambda: neural.eval_material(mat, q["uv"], q["lod"], q["wi"], q["wo"], q["u_rr"], fp16=True,  # noqa: E731
                                       return_level=False)[0].clone()
    try:
        f_default = run()
        lib.nm_set_tw_margin(1e30)
        f_all = run()
        lib.nm_set_tw_margin(1e-30)
        f_none = run()
    finally:
        lib.nm_set_tw_margin(0.0)
    torch.cuda.synchronize()
    assert torch.equal(f_default, f_all)
    n_diff = int((f_default != f_none).any(1).sum())
    assert n_diff > 0.0005 * C2_N, n_diff  # ~0.17% of rows round differently in plain fp32


def test_c3_sample_pdf_full_batch():
    """C3: 1920x1080x16 = 33,177,600 sample+pdf queries with a random lod
    per query (one launch); params, directions and pdfs on the subset."""
    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import neural, synth
    dev = torch.device("cuda", 0)
    mat = synth.material("2x32", 4096, 4096, seed=0, device=dev)
    h = mat.device_material(dev)
    n = C2_N * 16
    q = synth.queries(n, mat.latent.n_levels, seed=2, device=dev, need=("uv", "lod", "u_rr", "wi", "u3"))
    ws, pdf, p = neural.sample_pdf(mat, q["uv"], q["lod"], q["u_rr"], q["wi"], q["u3"], return_params=True)
    torch.cuda.synchronize()
    rows = subset_rows(n, 65536, seed=1)
    hq = host(q, rows)
    om = oracle_material(mat, h)
    z_ref, _ = om.half()["latent"].fetch(hq["uv"], hq["lod"], hq["u_rr"])
    p_ref = O.infer_proxy(om, z_ref, hq["wi"], fp16=True)
    ws_ref = O.sample(p_ref, hq["wi"].astype(np.float64), hq["u3"].astype(np.float64))
    ri = torch.as_tensor(rows, device=dev)
    pr = p.data[ri].cpu().numpy().astype(np.float64)
    check_rel(pr, p_ref.as_array(), what="C3 params")
    wsr = ws[ri].cpu().numpy()
    check_dirs(wsr, ws_ref, hq["u3"], p_ref, hq["wi"])
    # the kernel's pdf is the reference pdf of its own sample under the reference's params
    pdf_ref_own = O.pdf(p_ref, hq["wi"].astype(np.float64), wsr.astype(np.float64))
    from test_gpu_parity import conditioned_pdf_rows
    well, _, _ = conditioned_pdf_rows(p_ref.as_array(), hq["wi"], wsr.astype(np.float64), pdf_ref_own)
    check_rel(pdf[ri].cpu().numpy()[well], pdf_ref_own[well], what="C3 pdf")


@pytest.mark.parametrize("mode", ["binned", "divergent"])
def test_c4_multi_material_table1(mode):
    """C4: five materials with the Table-1 pyramids (15360^2 level 0 past
    2^31 bytes; npot 3712^2 / 4480^2 / 7104^2 on the float64 coordinate
    path), 1920x1080 eval queries with i.i.d. material ids."""
    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import neural, synth
    from paper_2305_02678_b200.synth import C4_RESOLUTIONS
    dev = torch.device("cuda", 0)
    mats = [synth.material("2x32", w, hh, seed=10 + k, device=dev) for k, (w, hh) in enumerate(C4_RESOLUTIONS)]
    handles = [m.device_material(dev) for m in mats]
    n = C2_N
    nl = min(m.latent.n_levels for m in mats)
    q = synth.queries(n, nl, seed=5, device=dev, need=("uv", "lod", "u_rr", "wi", "wo"))
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    ids = torch.randint(0, len(mats), (n,), device=dev, generator=g, dtype=torch.int32)
    if mode == "divergent":  # every tile decodes all five materials: a 1/8 slice keeps it quick
        n = n // 8
        q = {k: v[:n].contiguous() for k, v in q.items()}
        ids = ids[:n].contiguous()
    f = neural.eval_material_multi(mats, ids, q["uv"], q["lod"], q["wi"], q["wo"], q["u_rr"], mode=mode)
    torch.cuda.synchronize()
    rows = subset_rows(n, 65536, seed=2)
    hq = host(q, rows)
    hid = ids.cpu().numpy()[rows]
    fh = f.cpu().numpy()[rows]
    for k, (m, hk) in enumerate(zip(mats, handles)):
        sel = hid == k
        om = oracle_material(m, hk)
        z_ref, _ = om.half()["latent"].fetch(hq["uv"][sel], hq["lod"][sel], hq["u_rr"][sel])
        f_ref, _ = O.eval_brdf(om, z_ref, hq["wi"][sel], hq["wo"][sel], fp16=True)
        check_rel(fh[sel], f_ref, what=f"C4 {mode} material {k} {C4_RESOLUTIONS[k]}")
    del mats, handles
    torch.cuda.empty_cache()


def test_c4_full_query_binned_table1():
    """C4 full query (eval + sample + pdf) over the five Table-1 materials,
    binned by material id on the device (nm_query_multi)."""
    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import neural, synth
    from paper_2305_02678_b200.synth import C4_RESOLUTIONS
    dev = torch.device("cuda", 0)
    mats = [synth.material("2x32", w, hh, seed=10 + k, device=dev) for k, (w, hh) in enumerate(C4_RESOLUTIONS)]
    handles = [m.device_material(dev) for m in mats]
    n = C2_N
    nl = min(m.latent.n_levels for m in mats)
    q = synth.queries(n, nl, seed=6, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(6)
    ids = torch.randint(0, len(mats), (n,), device=dev, generator=g, dtype=torch.int32)
    f, ws, pdf = neural.query_multi(mats, ids, q["uv"], q["lod"], q["u_rr"], q["wi"], q["wo"], q["u3"])
    torch.cuda.synchronize()
    rows = subset_rows(n, 65536, seed=3)
    hq = host(q, rows)
    hid = ids.cpu().numpy()[rows]
    ri = torch.as_tensor(rows, device=dev)
    fh, wsh = f[ri].cpu().numpy(), ws[ri].cpu().numpy()
    for k, (m, hk) in enumerate(zip(mats, handles)):
        sel = hid == k
        om = oracle_material(m, hk)
        z_ref, _ = om.half()["latent"].fetch(hq["uv"][sel], hq["lod"][sel], hq["u_rr"][sel])
        f_ref, _ = O.eval_brdf(om, z_ref, hq["wi"][sel], hq["wo"][sel], fp16=True)
        p_ref = O.infer_proxy(om, z_ref, hq["wi"][sel], fp16=True)
        ws_ref = O.sample(p_ref, hq["wi"][sel].astype(np.float64), hq["u3"][sel].astype(np.float64))
        check_rel(fh[sel], f_ref, what=f"C4 query material {k}")
        check_dirs(wsh[sel], ws_ref, hq["u3"][sel], p_ref, hq["wi"][sel])
    del mats, handles
    torch.cuda.empty_cache()
