"""Multi-material eval (render.py:352-356 per-material groups): BINNED
(warp-aggregated binning + coherent kernel per segment) and DIVERGENT
(per-tile material loop) against the oracle, per query."""

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu


def _materials(rng):
    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import neural
    from paper_2305_02678_b200.latent import LatentPyramid

    specs = [({}, (64, 64)), ({"brdf_hidden": "2x16"}, (32, 32)), ({"albedo_head": True}, (24, 20)),
             ({"brdf_hidden": "3x64"}, (16, 16)), ({"use_frames": False}, (32, 16))]
    mats, omats = [], []
    for cfg, (w, h) in specs:
        m = neural.NeuralMaterial.create(neural.NeuralMaterialConfig(**cfg), rng)
        m.latent = LatentPyramid(O.random_pyramid(rng, w, h).levels)
        mats.append(m)

        def net(x):
            return None if x is None else O.Net([(l.w, l.b, l.act) for l in x.layers])

        om = O.Material(O.Config(**m.cfg.to_json()), net(m.frame_layer), net(m.brdf_decoder),
                        net(m.sampler_decoder))
        om.latent = O.Pyramid(m.latent.levels)
        omats.append(om)
    return mats, omats


def _queries(rng, n, n_levels_max=7):
    from oracle import nm_oracle as O
    uv = rng.random((n, 2)).astype(np.float32)
    lod = (rng.random(n) * n_levels_max).astype(np.float32)
    urr = rng.random(n).astype(np.float32)
    wi, wo = O.draw_direction_pairs(rng, n)
    return uv, lod, urr, wi.astype(np.float32), wo.astype(np.float32)


def _oracle_multi(omats, ids, uv, lod, urr, wi, wo):
    from oracle import nm_oracle as O
    f = np.zeros((len(ids), 3))
    for k, om in enumerate(omats):
        m = ids == k
        if m.any():
            f[m] = O.eval_material(om, uv[m], lod[m], wi[m], wo[m], urr[m], fp16=True)[0]
    return f


@pytest.mark.parametrize("mode", ["binned", "binned_async", "divergent"])
@pytest.mark.parametrize("pattern", ["random", "coherent", "blocks"])
def test_multi_material_matches_oracle(mode, pattern):
    from paper_2305_02678_b200 import neural

    rng = np.random.default_rng(42)
    mats, omats = _materials(rng)
    n = 9001
    uv, lod, urr, wi, wo = _queries(rng, n)
    if pattern == "random":
        ids = rng.integers(0, len(mats), n).astype(np.int32)
    elif pattern == "coherent":
        ids = np.full(n, 2, np.int32)
    else:
        ids = (np.arange(n) // 700 % len(mats)).astype(np.int32)
    f = neural.eval_material_multi(mats, ids, uv, lod, wi, wo, urr, mode=mode)
    ref = _oracle_multi(omats, ids, uv, lod, urr, wi, wo)
    from test_gpu_parity import check_rel
    check_rel(f, ref, what=f"{mode}/{pattern}")


def test_multi_modes_agree_and_reject_bad_ids():
    from paper_2305_02678_b200 import neural

    rng = np.random.default_rng(7)
    mats, _ = _materials(rng)
    n = 4000
    uv, lod, urr, wi, wo = _queries(rng, n)
    ids = rng.integers(0, len(mats), n).astype(np.int32)
    a = neural.eval_material_multi(mats, ids, uv, lod, wi, wo, urr, mode="binned")
    b = neural.eval_material_multi(mats, ids, uv, lod, wi, wo, urr, mode="divergent")
    np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6)
    bad = ids.copy()
    bad[17] = len(mats)
    with pytest.raises(ValueError):
        neural.eval_material_multi(mats, bad, uv, lod, wi, wo, urr, mode="binned")
    # BINNED_ASYNC never syncs: out-of-range ids (either side) are skipped by
    # the binning, every valid row is still exact
    bad[100] = -3
    c = neural.eval_material_multi(mats, bad, uv, lod, wi, wo, urr, mode="binned_async")
    ok = (bad >= 0) & (bad < len(mats))
    np.testing.assert_array_equal(c[ok], a[ok])


def test_binning_large_batch_all_rows_land():
    """Batches spanning many 1024-row scatter chunks and uneven segments:
    every query's result lands in its own row (binned == divergent)."""
    from paper_2305_02678_b200 import neural

    rng = np.random.default_rng(11)
    mats, _ = _materials(rng)
    n = 70001
    uv, lod, urr, wi, wo = _queries(rng, n)
    ids = np.minimum(rng.geometric(0.45, n) - 1, len(mats) - 1).astype(np.int32)  # skewed
    a = neural.eval_material_multi(mats, ids, uv, lod, wi, wo, urr, mode="binned_async")
    b = neural.eval_material_multi(mats, ids, uv, lod, wi, wo, urr, mode="divergent")
    np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6)


def test_binned_async_from_concurrent_host_threads():
    """Two host threads issuing BINNED_ASYNC calls on their own streams at the
    same time (shared side streams / events): each result is complete and
    exact when its call's stream is synchronized."""
    import threading
    import torch
    from paper_2305_02678_b200 import neural

    rng = np.random.default_rng(5)
    mats, _ = _materials(rng)
    n = 30000
    qs = [_queries(rng, n) for _ in range(2)]
    ids = [rng.integers(0, len(mats), n).astype(np.int32) for _ in range(2)]
    want = [neural.eval_material_multi(mats, ids[k], *qs[k][:2], qs[k][3], qs[k][4], qs[k][2],
                                       mode="binned_async") for k in range(2)]  # one thread
    dev = torch.device("cuda", 0)
    got = [None, None]

    def run(k):
        st = torch.cuda.Stream(dev)
        with torch.cuda.stream(st):
            t = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in qs[k]]
            idt = torch.from_numpy(ids[k]).to(dev)
            for _ in range(5):
                f = neural.eval_material_multi(mats, idt, t[0], t[1], t[3], t[4], t[2], mode="binned_async")
            st.synchronize()
            got[k] = f.cpu().numpy()

    th = [threading.Thread(target=run, args=(k,)) for k in range(2)]
    [x.start() for x in th]
    [x.join() for x in th]
    for k in range(2):
        np.testing.assert_array_equal(got[k], want[k])


@pytest.mark.parametrize("mode", ["binned", "binned_async"])
def test_multi_material_sample_pdf_and_query(mode):
    """The renderer's per-vertex groups on the sampler side (render.py:361-409):
    sampler + sample + pdf, and the full query, each row with its own material."""
    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import neural
    from test_gpu_parity import check_dirs, check_rel

    rng = np.random.default_rng(43)
    mats, omats = _materials(rng)
    n = 9001
    uv, lod, urr, wi, wo = _queries(rng, n)
    u3 = rng.random((n, 3)).astype(np.float32)
    ids = rng.integers(0, len(mats), n).astype(np.int32)
    ws, pdf, p = neural.sample_pdf_multi(mats, ids, uv, lod, urr, wi, u3, mode=mode, return_params=True)
    f2, ws2, pdf2 = neural.query_multi(mats, ids, uv, lod, urr, wi, wo, u3, mode=mode)
    f_ref = np.zeros((n, 3))
    ws_ref = np.zeros((n, 3))
    p_ref = np.zeros((n, 9))
    for k, om in enumerate(omats):
        m = ids == k
        fr, wsr, _, pr, _ = O.full_query(om, uv[m], lod[m], urr[m], wi[m], wo[m], u3[m])
        f_ref[m], ws_ref[m], p_ref[m] = fr, wsr, pr.as_array()
    check_rel(p.as_array(), p_ref, what=f"{mode} params")
    check_rel(f2, f_ref, what=f"{mode} query rgb")
    P = O.Proxy(p_ref[:, 0], p_ref[:, 1], p_ref[:, 2:4], p_ref[:, 4:6], p_ref[:, 6], p_ref[:, 7:9])
    check_dirs(ws, ws_ref, u3, P, wi)
    check_dirs(ws2, ws_ref, u3, P, wi)
    assert np.array_equal(ws, ws2) and np.array_equal(pdf, pdf2)  # the same kernels on the same rows
    with pytest.raises(NotImplementedError):
        neural.sample_pdf_multi(mats, ids, uv, lod, urr, wi, u3, mode="divergent")


def test_host_buffer_eval_from_threads_and_chunking():
    """The drop-in call on pageable numpy arrays (nm_eval_host_ref: pinned
    bounce pipeline, host thread pool, float64 / int64 results widened on
    the device) from two host threads at once and across many chunks equals
    the device-pointer call bit for bit."""
    import threading

    import torch

    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import _io, _lib, neural
    from paper_2305_02678_b200.latent import LatentPyramid
    rng = np.random.default_rng(91)
    mat = neural.NeuralMaterial.create(neural.NeuralMaterialConfig(albedo_head=True), rng)
    mat.latent = LatentPyramid(O.random_pyramid(rng, 64, 64).levels)
    n = 600_001  # three 256k chunks and a ragged tail
    uv = rng.random((n, 2)).astype(np.float32)
    lod = (rng.random(n) * 6).astype(np.float32)
    urr = rng.random(n).astype(np.float32)
    wi, wo = O.draw_direction_pairs(rng, n)
    wi, wo = wi.astype(np.float32), wo.astype(np.float32)
    # reference result through device pointers
    t = {k: torch.from_numpy(v).cuda() for k, v in (("uv", uv), ("lod", lod), ("urr", urr), ("wi", wi), ("wo", wo))}
    f_d, a_d, l_d = neural.eval_material(mat, t["uv"], t["lod"], t["wi"], t["wo"], t["urr"], fp16=True)
    want = (f_d.cpu().numpy().astype(np.float64), a_d.cpu().numpy().astype(np.float64),
            l_d.cpu().numpy().astype(np.int64))
    got = [None, None]

    def run(k):
        got[k] = neural.eval_material(mat, uv, lod, wi, wo, urr, fp16=True)

    th = [threading.Thread(target=run, args=(k,)) for k in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    for f, a, lv in got:
        assert f.dtype == np.float64 and a.dtype == np.float64 and lv.dtype == np.int64
        assert np.array_equal(f, want[0]) and np.array_equal(a, want[1]) and np.array_equal(lv, want[2])
    # scalar level (lod_stride 0) through the same pipeline
    f1, _, lv1 = neural.eval_material(mat, uv[:1000], np.float32(2.5), wi[:1000], wo[:1000], urr[:1000], fp16=True)
    f2, _, lv2 = neural.eval_material(mat, t["uv"][:1000], torch.tensor([2.5], device="cuda"), t["wi"][:1000],
                                      t["wo"][:1000], t["urr"][:1000], fp16=True)
    assert np.array_equal(f1, f2.cpu().numpy().astype(np.float64)) and np.array_equal(lv1, lv2.cpu().numpy())
