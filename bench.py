"""Benchmark of the neural-material query path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c3|full]

Default workload (BASELINE.json configs[1], "C2"): one random-init 2x32
material with a 4096^2 latent pyramid (13 levels, fp16), 1920x1080 =
2,073,600 coherent fused eval queries (fetch + frames + BRDF decoder) per
step per GPU.  Multi-GPU runs are weak-scaled pixel tiles (each rank owns a
1080p tile of a larger frame, replicated material, no collective on the
data path); `value` = all ranks' queries / max-over-ranks time.

One JSON line on rank 0.  `value` = device-timed throughput with inputs in
HBM (CUDA events, inputs rotating over 3 sets > L2); `e2e` = the public API
(`neural.eval_material` on pageable host numpy buffers in the reference's
call shape, H2D + kernel + D2H inside the timed region; `e2e_pinned` the
zero-copy variant); `roofline` = the fused kernel's algorithmic bytes
(fp32 I/O + 16 B per unique texel touched) / launch time vs measured HBM
peak; `cpu_baseline` = the numpy oracle (restatement of the reference,
oracle/nm_oracle.py) on the host cores for a bounded sample.
"""

import argparse
import ctypes
import json
import os
import subprocess
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # the CPU baseline forks one worker per core

import numpy as np  # noqa: E402
import torch  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C2_N = 1920 * 1080
C3_N = 1920 * 1080 * 16
RES = 4096
METRIC = "neural BRDF queries/sec (eval, sample+pdf) at 1/2/4/8 B200; % of roofline"
FLOPS_EVAL = 2 * (8 * 12 + 20 * 32 + 32 * 32 + 32 * 3)          # 3712
FLOPS_SAMPLE = 2 * (11 * 32 + 32 * 32 + 32 * 32 + 32 * 9)         # 5376


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


# ---------------------------------------------------------------------------
# distributed plumbing

def dist_init(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("NMQ_DIST_BACKEND", "nccl")  # "gloo": test the N>1 path on one GPU
        if backend == "gloo":
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    if n_gpus != world:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}")
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch.distributed as dist
    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    t = torch.tensor([x], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML, sampled from the host between launches)

class Clocks:
    REASONS = {
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
        0x2: "applications_clocks_setting",
    }

    def __init__(self, index):
        self.ok = False
        self.samples = []
        self.reasons = 0
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None

    def sample(self):
        if not self.ok:
            return
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            pass

    def start(self, period_s=0.01):
        import threading
        self._stop = threading.Event()

        def loop():
            while not self._stop.is_set():
                self.sample()
                self._stop.wait(period_s)

        self._thread = threading.Thread(target=loop, daemon=True)
        self._thread.start()

    def stop(self):
        self._stop.set()
        self._thread.join()
        self.sample()

    def report(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": [], "samples": 0}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and v != "gpu_idle"]
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max,
                "reasons": names, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# algorithmic bytes: fp32 I/O + 16 B per unique texel touched

def unique_texels(mat_handle, q):
    return int(torch.unique(texel_ids(mat_handle, q)).numel())


def texel_ids(mat_handle, q):
    """Global texel index of every tap of every query (the exact fetch taps)."""
    from paper_2305_02678_b200 import _lib
    lib = _lib.load()
    n = q["uv"].shape[0]
    taps = torch.empty((n, 8), device="cuda", dtype=torch.int32)
    lv = torch.empty((n,), device="cuda", dtype=torch.int32)
    lod_stride = 1
    _lib.check(lib.nm_fetch(mat_handle.ptr, n, q["uv"].data_ptr(), q["lod"].data_ptr(), lod_stride,
                            q["u_rr"].data_ptr(), None, lv.data_ptr(), taps.data_ptr(), None,
                            torch.cuda.current_stream().cuda_stream))
    w, h, off = mat_handle.level_table()
    w_t = torch.from_numpy(w.astype(np.int64)).cuda()
    off_t = torch.from_numpy(off).cuda()
    t = taps.view(n, 4, 2).long()
    lvl = lv.long()
    gid = off_t[lvl][:, None] + t[..., 1] * w_t[lvl][:, None] + t[..., 0]
    return gid.reshape(-1)


def hbm_roofline(bytes_per_q, n, ms, note):
    """Roofline object for workloads timed end to end on the device (several
    launches per step): achieved = algorithmic bytes / step time."""
    hbm, _, kind = peaks()
    ach = bytes_per_q * n / (ms / 1e3) / 1e9
    return {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
            "traffic": None, "peak_source": kind, "algorithmic_bytes_per_query": bytes_per_q,
            "note": note}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle restatement of the reference on host cores

_CPU = {}


def _cpu_eval_chunk(bounds):
    from oracle import nm_oracle as O
    s, e = bounds
    d = _CPU
    z, _ = d["pyr"].fetch(d["uv"][s:e], d["lod"][s:e], d["u_rr"][s:e])
    if d["kind"] == "eval":
        O.eval_brdf(d["mat"], z, d["wi"][s:e], d["wo"][s:e], fp16=True)
    elif d["kind"] == "full":
        O.eval_brdf(d["mat"], z, d["wi"][s:e], d["wo"][s:e], fp16=True)
        p = O.infer_proxy(d["mat"], z, d["wi"][s:e], fp16=True)
        ws = O.sample(p, d["wi"][s:e], d["u3"][s:e])
        O.pdf(p, d["wi"][s:e], ws)
    else:
        p = O.infer_proxy(d["mat"], z, d["wi"][s:e], fp16=True)
        ws = O.sample(p, d["wi"][s:e], d["u3"][s:e])
        O.pdf(p, d["wi"][s:e], ws)
    return e - s


def cpu_setup(mat, q, n_sample, kind):
    """Build the oracle material (same weights, same fp16 texels) and a
    host copy of the first n_sample queries."""
    from oracle import nm_oracle as O

    def net(m):
        return None if m is None else O.Net([(l.w, l.b, l.act) for l in m.layers])

    cfg = O.Config(**mat.cfg.to_json())
    om = O.Material(cfg, net(mat.frame_layer), net(mat.brdf_decoder), net(mat.sampler_decoder))
    levels = [l.astype(np.float32) for l in mat.latent.half_copy()]
    om._half = {"frame": O.quantize(om.frame) if om.frame is not None else None,
                "brdf": O.quantize(om.brdf), "sampler": O.quantize(om.sampler),
                "latent": O.Pyramid(levels)}
    _CPU.clear()
    _CPU.update(mat=om, pyr=om._half["latent"], kind=kind)
    for k in ("uv", "lod", "u_rr", "wi", "wo", "u3"):
        if k in q:
            _CPU[k] = q[k][:n_sample].double().cpu().numpy()


_POOL = {}


def cpu_pool(workers):
    """Forked worker pool created once (after cpu_setup), outside timing."""
    import multiprocessing as mp
    if workers > 1 and _POOL.get("n") != workers:
        if "pool" in _POOL:
            _POOL["pool"].terminate()
        _POOL["pool"] = mp.get_context("fork").Pool(workers)
        _POOL["n"] = workers
    return _POOL.get("pool")


def cpu_run(n_sample, workers):
    chunk = (n_sample + workers - 1) // workers
    bounds = [(s, min(n_sample, s + chunk)) for s in range(0, n_sample, chunk)]
    pool = cpu_pool(workers)
    t0 = time.perf_counter()
    if pool is None:
        done = sum(_cpu_eval_chunk(b) for b in bounds)
    else:
        done = sum(pool.map(_cpu_eval_chunk, bounds))
    return done / (time.perf_counter() - t0)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# host-side stand-ins for the no-GPU reference arm (same recipe, numpy RNG)

class HostLatent:
    """Host-side stand-in of DeviceLatent (no-GPU reference arm)."""

    def __init__(self, levels, width, height):
        self.levels16 = levels
        self.width, self.height, self.n_levels = width, height, len(levels)

    def half_copy(self):
        return self.levels16


def material_host(brdf_hidden="2x32", width=4096, height=4096, seed=0, **cfg):
    mat = _nm().NeuralMaterial.create(_nm().NeuralMaterialConfig(brdf_hidden=brdf_hidden, **cfg),
                                np.random.default_rng(seed))
    rng = np.random.default_rng(seed + 1000)
    levels = [rng.standard_normal((h, w, 8), dtype=np.float32).astype(np.float16)
              for h, w in _ls()(width, height)]
    mat.latent = HostLatent(levels, width, height)
    return mat


def queries_host(n, n_levels, seed):
    """Same recipe as queries() on the host (numpy RNG; values differ)."""
    from oracle import nm_oracle as O  # host generator only used by the CPU reference arm
    rng = np.random.default_rng(seed)
    wi, wo = O.draw_direction_pairs(rng, n)
    f = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32))  # noqa: E731
    return {"uv": f(rng.random((n, 2))), "lod": f(rng.random(n) * (n_levels - 1)),
            "u_rr": f(rng.random(n)), "wi": f(wi), "wo": f(wo), "u3": f(rng.random((n, 3)))}


def _nm():
    from paper_2305_02678_b200 import neural
    return neural


def _ls():
    from paper_2305_02678_b200.latent import level_shapes
    return level_shapes


# ---------------------------------------------------------------------------

def build_workload(args, rank, device):
    from paper_2305_02678_b200 import synth
    mat = synth.material("2x32", RES, RES, seed=0, device=device)
    n = C2_N if args.workload in ("c2", "full") else C3_N
    n *= int(os.environ.get("NMQ_BATCH_MULT", "1"))  # experiments only (scaling of fixed costs)
    n_levels = mat.latent.n_levels
    sets = [synth.queries(n, n_levels, seed=1 + 100 * rank + s, device=device)
            for s in range(args.sets)]
    return mat, n, sets


def launch(lib, h, workload, q, outs, stream):
    n = q["uv"].shape[0]
    if workload == "c2":
        return lib.nm_eval(h.ptr, n, q["uv"].data_ptr(), q["lod"].data_ptr(), 1, q["u_rr"].data_ptr(),
                           q["wi"].data_ptr(), q["wo"].data_ptr(), outs["rgb"].data_ptr(), None, None,
                           stream)
    if workload == "c3":
        return lib.nm_sample_pdf(h.ptr, n, q["uv"].data_ptr(), q["lod"].data_ptr(), 1,
                                 q["u_rr"].data_ptr(), q["wi"].data_ptr(), q["u3"].data_ptr(),
                                 outs["ws"].data_ptr(), outs["pdf"].data_ptr(), None, None, stream)
    return lib.nm_query(h.ptr, n, q["uv"].data_ptr(), q["lod"].data_ptr(), 1, q["u_rr"].data_ptr(),
                        q["wi"].data_ptr(), q["wo"].data_ptr(), q["u3"].data_ptr(),
                        outs["rgb"].data_ptr(), outs["ws"].data_ptr(), outs["pdf"].data_ptr(), None,
                        stream)


def launch_closure(lib, h, workload, q, outs, stream):
    """The C-ABI call of one step with its arguments converted once."""
    n = q["uv"].shape[0]
    P = ctypes.c_void_p
    if workload == "c2":
        fn = lib.nm_eval
        a = (P(h.ptr), ctypes.c_int64(n), P(q["uv"].data_ptr()), P(q["lod"].data_ptr()),
             ctypes.c_int32(1), P(q["u_rr"].data_ptr()), P(q["wi"].data_ptr()),
             P(q["wo"].data_ptr()), P(outs["rgb"].data_ptr()), None, None, P(stream))
    elif workload == "c3":
        fn = lib.nm_sample_pdf
        a = (P(h.ptr), ctypes.c_int64(n), P(q["uv"].data_ptr()), P(q["lod"].data_ptr()),
             ctypes.c_int32(1), P(q["u_rr"].data_ptr()), P(q["wi"].data_ptr()),
             P(q["u3"].data_ptr()), P(outs["ws"].data_ptr()), P(outs["pdf"].data_ptr()), None,
             None, P(stream))
    else:
        fn = lib.nm_query
        a = (P(h.ptr), ctypes.c_int64(n), P(q["uv"].data_ptr()), P(q["lod"].data_ptr()),
             ctypes.c_int32(1), P(q["u_rr"].data_ptr()), P(q["wi"].data_ptr()),
             P(q["wo"].data_ptr()), P(q["u3"].data_ptr()), P(outs["rgb"].data_ptr()),
             P(outs["ws"].data_ptr()), P(outs["pdf"].data_ptr()), None, P(stream))

    def go():
        rc = fn(*a)
        if rc:
            from paper_2305_02678_b200 import _lib
            _lib.check(rc)
    return go


def io_bytes(workload):
    # inputs: uv 8, lod 4, u_rr 4, wi 12 (+ wo 12) (+ u3 12); outputs rgb 12 / ws 12 + pdf 4
    return {"c2": 40 + 12, "c3": 40 + 16, "full": 52 + 28}[workload]


def _time_loop(fn, steps, warmup, stream, world):
    for i in range(warmup):
        fn(i)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(steps):
        fn(i)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    return max_over_ranks(e0.elapsed_time(e1), world) / steps


def run_c4(args):
    """C4: five materials mixed per query (Table-1-sized pyramids, 8.3 GB of
    fp16 latents), 1920x1080 eval queries with i.i.d. material ids; BINNED
    (headline) vs DIVERGENT."""
    rank, world, local = dist_init(args.gpus)
    device = torch.device("cuda", local)
    from paper_2305_02678_b200 import _lib, synth
    from paper_2305_02678_b200.synth import C4_RESOLUTIONS
    lib = _lib.load()
    mats = [synth.material("2x32", w, h, seed=10 + k, device=device)
            for k, (w, h) in enumerate(C4_RESOLUTIONS)]
    handles = [m.device_material(device) for m in mats]
    n = C2_N
    max_levels = min(m.latent.n_levels for m in mats)
    sets = [synth.queries(n, max_levels, seed=1 + 100 * rank + s, device=device)
            for s in range(args.sets)]
    g = torch.Generator(device=device)
    g.manual_seed(5 + rank)
    ids = [torch.randint(0, len(mats), (n,), device=device, generator=g, dtype=torch.int32)
           for _ in range(args.sets)]
    rgb = torch.empty((n, 3), device=device)
    ws_bytes = int(lib.nm_multi_workspace_bytes(n, len(mats)))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=device)
    ptrs = (ctypes.c_void_p * len(mats))(*[h.ptr for h in handles])
    stream = torch.cuda.current_stream(device)

    def step(mode):
        def fn(i):
            q, mid = sets[i % len(sets)], ids[i % len(sets)]
            _lib.check(lib.nm_eval_multi(ptrs, len(mats), n, mid.data_ptr(), q["uv"].data_ptr(),
                                         q["lod"].data_ptr(), 1, q["u_rr"].data_ptr(),
                                         q["wi"].data_ptr(), q["wo"].data_ptr(), rgb.data_ptr(),
                                         mode, ws.data_ptr(), ws_bytes, stream.cuda_stream))
        return fn

    steps = max(3, args.steps // 10)
    ms_b = _time_loop(step(_lib.NM_MULTI_BINNED), steps, args.warmup, stream, world)
    ms_a = _time_loop(step(_lib.NM_MULTI_BINNED_ASYNC), steps, args.warmup, stream, world)
    ms_d = _time_loop(step(_lib.NM_MULTI_DIVERGENT), max(3, steps // 4), 2, stream, world)
    # algorithmic bytes: 52 B of fp32 I/O + 16 B per unique texel touched, counted
    # exactly per material on each input set (binning traffic is overhead, not algorithm)
    tex_b = []
    for q, mid in zip(sets, ids):
        u = 0
        for k, hk in enumerate(handles):
            sel = mid == k
            u += unique_texels(hk, {key: v[sel].contiguous() for key, v in q.items()})
        tex_b.append(16.0 * u / n)
    bpq = io_bytes("c2") + float(np.mean(tex_b))
    if rank == 0:
        texels = sum(int(h.info.latent_texels) for h in handles)
        print(json.dumps({
            "metric": METRIC, "value": n * world / (ms_b / 1e3), "unit": "queries/s",
            "n_gpus": world, "steps": steps, "warmup": args.warmup, "ms_per_step": ms_b,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "fp16 x fp16 -> fp32 tensor-core (hi/lo split), fp32 SIMT",
            "data": "synthetic: 5 random-init 2x32 materials, N(0,1) fp16 latents",
            "config": {"workload": "C4 eval, 5 materials mixed per query (i.i.d. ids), 1920x1080",
                       "pyramids": [f"{w}x{h}" for w, h in C4_RESOLUTIONS],
                       "latent_gb": texels * 16 / 1e9, "mode": "binned (headline)"},
            "binned_async": {"value": n * world / (ms_a / 1e3), "ms_per_step": ms_a,
                             "note": "no host round trip (segment sizes stay on the device)"},
            "divergent": {"value": n * world / (ms_d / 1e3), "ms_per_step": ms_d},
            "binned_over_divergent": ms_d / ms_b,
            "roofline": hbm_roofline(bpq, n * world, ms_b, "binned step (histogram + scan + scatter + "
                                     "per-material launches) timed as a whole; texel bytes exact per material"),
            "roofline_binned_async": hbm_roofline(bpq, n * world, ms_a, "binned_async step"),
        }))


def run_c5(args):
    """C5: 3840x2160 x 64 spp eval (530.8M queries) sharded by pixel-row band
    across ranks (replicated material); each rank's eval kernel reduces its
    64 samples per pixel in the epilogue (nm_eval_spp: per-sample rgb never
    reaches HBM) and one gather moves the 99.5 MB image to rank 0."""
    rank, world, local = dist_init(args.gpus)
    device = torch.device("cuda", local)
    from paper_2305_02678_b200 import _lib, shard, synth
    lib = _lib.load()
    H, W, SPP = 2160, 3840, 64
    mat = synth.material("2x32", RES, RES, seed=0, device=device)
    h = mat.device_material(device)
    q0, q1 = shard.band_queries(rank, world, H, W, SPP)
    n = q1 - q0
    chunk = 1 << 24
    q = {k: torch.empty((n,) + s_, device=device) for k, s_ in
         (("uv", (2,)), ("lod", ()), ("u_rr", ()), ("wi", (3,)), ("wo", (3,)))}
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        part = synth.queries(c1 - c0, mat.latent.n_levels, seed=1000 + rank * 4096 + c0 // chunk,
                             device=device, need=tuple(q))
        for k in q:
            q[k][c0:c1] = part[k]
    img = torch.empty((n // SPP, 3), device=device)
    stream = torch.cuda.current_stream(device)

    def compute(i):
        _lib.check(lib.nm_eval_spp(h.ptr, n, q["uv"].data_ptr(), q["lod"].data_ptr(), 1, q["u_rr"].data_ptr(),
                                   q["wi"].data_ptr(), q["wo"].data_ptr(), SPP, img.data_ptr(),
                                   stream.cuda_stream))

    def frame(i):
        compute(i)
        if world > 1:
            shard.gather_bands(img.view(-1, W, 3), H, W)

    seen = torch.zeros(int(h.info.latent_texels), dtype=torch.bool, device=device)
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        seen[texel_ids(h, {k: v[c0:c1] for k, v in q.items()})] = True
    bpq = 40.0 + 12.0 / SPP + 16.0 * int(seen.sum()) / n  # inputs + the pixel's share of rgb + texels
    del seen
    steps = max(2, args.steps // 50)
    l0 = lib.nm_launch_count()
    ms_c = _time_loop(compute, steps, 2, stream, world)
    launches = int(lib.nm_launch_count() - l0)
    ms_f = _time_loop(frame, steps, 1, stream, world)
    if rank == 0:
        total = H * W * SPP
        print(json.dumps({
            "metric": METRIC, "value": total / (ms_c / 1e3), "unit": "queries/s",
            "n_gpus": world, "steps": steps, "warmup": 2, "ms_per_step": ms_c,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "fp16 x fp16 -> fp32 tensor-core (hi/lo split), fp32/fp64 SIMT",
            "data": "synthetic: random-init 2x32 material, 4096^2 N(0,1) fp16 latents",
            "config": {"workload": "C5 eval 3840x2160x64spp sharded by pixel-row band, per-pixel mean in the "
                                   "kernel epilogue", "queries_per_frame": total,
                       "parallelism": f"pixel-tile x{world}"},
            "with_gather": {"value": total / (ms_f / 1e3), "ms_per_frame": ms_f,
                            "note": "compute + one gather of the 3840x2160x3 fp32 image to rank 0"},
            "gpu_launches": launches,
            "roofline": hbm_roofline(bpq, n, ms_c, "one fused eval+spp-mean launch per rank over its band; "
                                     "bytes = 40 B inputs + 12 B / spp of image + 16 B x unique texels (exact)"),
        }))


def run_train(args):
    """SURVEY §8 f4 (training-side kernels), not the headline: one baking
    iteration's worth of network forward_cached + backward (BRDF 20-32-32-3
    and sampler 11-32-32-32-9 on 65,536 rows each, training.py batch) and the
    latent-gradient scatter of 65,536 queries into the 4096^2 pyramid; rows/s
    with the numpy oracle (the reference's algorithm) timed beside it."""
    rank, world, local = dist_init(args.gpus)
    device = torch.device("cuda", local)
    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import mlp, synth, train  # noqa: F401
    rng = np.random.default_rng(3)
    B = 65536
    nets = {"brdf": mlp.Mlp.create((20, 32, 32, 3), rng), "sampler": mlp.Mlp.create((11, 32, 32, 32, 9), rng)}
    xs = {k: torch.randn((B, n.layers[0].w.shape[1]), device=device) for k, n in nets.items()}
    gs = {k: torch.randn((B, n.layers[-1].w.shape[0]), device=device) for k, n in nets.items()}
    mat = synth.material("2x32", RES, RES, seed=0, device=device)
    q = synth.queries(B, mat.latent.n_levels, seed=1, device=device)
    lv = torch.randint(0, mat.latent.n_levels, (B,), device=device, dtype=torch.int32)
    zg = torch.randn((B, 8), device=device)
    texels = mat.latent.texels.shape[0]
    grad = torch.zeros((texels, 8), device=device)
    h = mat.device_material(device)
    from paper_2305_02678_b200 import _lib
    lib = _lib.load()
    stream = torch.cuda.current_stream(device)

    def step(i):
        for k, n in nets.items():
            _, cache = train.forward_cached(n, xs[k])
            train.backward(n, cache, gs[k])
        _lib.check(lib.nm_texel_grads(h.ptr, B, q["uv"].data_ptr(), lv.data_ptr(), zg.data_ptr(),
                                      grad.data_ptr(), stream.cuda_stream))

    steps = max(5, args.steps // 100)
    ms = _time_loop(step, steps, args.warmup, stream, world)
    # CPU: the oracle's restatement of the reference on the same shapes (1 core)
    onets = {k: O.Net([(l.w, l.b, l.act) for l in n.layers]) for k, n in nets.items()}
    xh = {k: v.cpu().numpy() for k, v in xs.items()}
    gh = {k: v.cpu().numpy() for k, v in gs.items()}
    t0 = time.perf_counter()
    for k, n in onets.items():
        _, c = O.forward_cached(n, xh[k])
        O.backward(n, c, gh[k])
    t_mlp = time.perf_counter() - t0
    if rank == 0:
        print(json.dumps({
            "metric": "training-side rows/s (forward_cached + backward of both decoders + texel-grad scatter)",
            "value": B * world / (ms / 1e3), "unit": "rows/s", "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp32 forward, fp64 backward chain / reductions",
            "data": "synthetic: random-init networks, N(0,1) inputs and gradients",
            "config": {"workload": "train (SURVEY §8 f4)", "rows": B, "latent": f"{RES}x{RES}"},
            "cpu_baseline": {"value": B / t_mlp, "unit": "rows/s", "cores": 1, "kind": "port",
                             "sample": "forward_cached + backward of both decoders (oracle, numpy, 1 core); "
                                       "texel scatter not included"},
        }))


def run_kl(args):
    """SURVEY §8 f4, not the headline: the KL sampler loss + sampler-decoder
    gradients (training.py:219-273) on 65,536 rows of the default 2x32
    material (sampler forward, BRDF forward + input backward at both lobe
    samples, the float64 heads, sampler backward) — rows/s, the loss read
    back every step; the numpy oracle (the reference's algorithm) beside it."""
    rank, world, local = dist_init(args.gpus)
    device = torch.device("cuda", local)
    from oracle import nm_oracle as O
    from paper_2305_02678_b200 import synth, train
    B = 65536
    mat = synth.material("2x32", 64, 64, seed=0, device=device)
    g = torch.Generator(device=device)
    g.manual_seed(7 + rank)
    z = torch.randn((B, 8), device=device, generator=g)
    q = synth.queries(B, 1, seed=2 + rank, device=device)
    wi = q["wi"].double()
    us = (torch.rand((B, 2), device=device, generator=g, dtype=torch.float64),
          torch.rand((B, 2), device=device, generator=g, dtype=torch.float64))
    stream = torch.cuda.current_stream(device)

    def step(i):
        train.sampler_loss_and_grads(mat, z, wi, None, us=us)

    steps = max(5, args.steps // 100)
    ms = _time_loop(step, steps, args.warmup, stream, world)
    n_cpu = 8192
    om = O.Material(O.Config(), O.Net([(l.w, l.b, l.act) for l in mat.frame_layer.layers]),
                    O.Net([(l.w, l.b, l.act) for l in mat.brdf_decoder.layers]),
                    O.Net([(l.w, l.b, l.act) for l in mat.sampler_decoder.layers]))
    zh, wih = z[:n_cpu].cpu().numpy(), wi[:n_cpu].cpu().numpy()
    ush = tuple(u[:n_cpu].cpu().numpy() for u in us)
    t0 = time.perf_counter()
    O.sampler_loss_and_grads(om, zh, wih, ush)
    t_cpu = time.perf_counter() - t0
    if rank == 0:
        print(json.dumps({
            "metric": "KL sampler-loss rows/s (loss + sampler-decoder gradients)",
            "value": B * world / (ms / 1e3), "unit": "rows/s", "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp32 networks, f64 heads / backward chains",
            "data": "synthetic: random-init 2x32 material, N(0,1) codes, half-diff directions",
            "config": {"workload": "kl (SURVEY §8 f4, training.py:219-273)", "rows": B},
            "cpu_baseline": {"value": n_cpu / t_cpu, "unit": "rows/s", "cores": 1, "kind": "port",
                             "sample": f"{n_cpu} rows, oracle.sampler_loss_and_grads (numpy, 1 core)"},
        }))


def measure(args, lib, h, workload, sets, steps, warmup, stream, world, local, clocks=None, tag=None,
            kernel=None):
    """Device-timed throughput of one workload: `steps` back-to-back launches
    of the C-ABI call with inputs resident in HBM (rotating over `sets`),
    CUDA events on the launching stream, max over ranks.  Returns a dict."""
    n = sets[0]["uv"].shape[0]
    dev = sets[0]["uv"].device
    outs = {"rgb": torch.empty((n, 3), device=dev), "ws": torch.empty((n, 3), device=dev),
            "pdf": torch.empty((n,), device=dev)}
    sp = stream.cuda_stream
    fns = [launch_closure(lib, h, workload, q, outs, sp) for q in sets]
    for i in range(warmup):
        fns[i % len(fns)]()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    l0 = lib.nm_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if clocks:
        clocks.start()  # NVML sampling on a background thread during the timed region
    ev0.record(stream)
    for i in range(steps):
        fns[i % len(fns)]()
    ev1.record(stream)
    ev1.synchronize()
    if clocks:
        clocks.stop()
    torch.cuda.synchronize()
    barrier(world)
    launches = int(lib.nm_launch_count() - l0)
    ms = ev0.elapsed_time(ev1)
    ms_max = max_over_ranks(ms, world)
    uniq = [unique_texels(h, q) for q in sets]
    texel_b = 16.0 * float(np.mean(uniq)) / n
    bpq = io_bytes(workload) + texel_b
    fpq = {"c2": FLOPS_EVAL, "c3": FLOPS_SAMPLE, "full": FLOPS_EVAL + FLOPS_SAMPLE}[workload]
    hbm, tflops, peak_kind = peaks()
    kernel_s = ms / steps / 1e3
    ach = bpq * n / kernel_s / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{tag or workload}.json")  # ncu capture of THIS kernel
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get("dram_bytes_per_launch")
    return {
        "value": n * world * steps / (ms_max / 1e3), "ms_per_step": ms_max / steps, "steps": steps,
        "queries_per_step_per_gpu": n, "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                     "traffic": traffic, "peak_source": peak_kind, "algorithmic_bytes_per_query": bpq,
                     "texel_bytes_per_query": texel_b,
                     "tensor_tflops_achieved": fpq * n / kernel_s / 1e12,
                     "tensor_frac": fpq * n / kernel_s / 1e12 / tflops,
                     "kernel": kernel or "fast_kernel<%s> (csrc/nmq_fast.cu; exact-rounding resolve in its epilogue)" % {
                         "c2": "kModeEval", "c3": "kModeSamplePdf", "full": "kModeQuery"}[workload]},
    }


def c1_case(arch="2x32"):
    """BASELINE configs[0] exactly: one random-init material, 512^2 pyramid,
    65,536 random (uv, wi, wo, lod) queries (SURVEY §8 d2/d3 recipe)."""
    from oracle import nm_oracle as O  # the host-side recipe's generator (and the CPU baseline)
    from paper_2305_02678_b200 import neural
    from paper_2305_02678_b200.latent import LatentPyramid
    rng = np.random.default_rng(0)
    mat = neural.NeuralMaterial.create(neural.NeuralMaterialConfig(brdf_hidden=arch), rng)
    mat.latent = LatentPyramid(O.random_pyramid(np.random.default_rng(0), 512, 512).levels)
    n = 65536
    qr = np.random.default_rng(1)
    q = {"uv": qr.random((n, 2)).astype(np.float32),
         "lod": (qr.random(n) * (mat.latent.n_levels - 1)).astype(np.float32),
         "u_rr": qr.random(n).astype(np.float32)}
    wi, wo = O.draw_direction_pairs(qr, n)
    q["wi"], q["wo"] = wi.astype(np.float32), wo.astype(np.float32)
    q["u3"] = qr.random((n, 3)).astype(np.float32)
    return mat, q


def c1_cpu(mat, q, workers):
    """The oracle's C1 full query (fetch + eval + proxy + sample + pdf, fp16
    path) on `workers` forked processes, OPENBLAS_NUM_THREADS=1."""
    from oracle import nm_oracle as O

    def net(m):
        return O.Net([(l.w, l.b, l.act) for l in m.layers])

    om = O.Material(O.Config(**mat.cfg.to_json()), net(mat.frame_layer), net(mat.brdf_decoder),
                    net(mat.sampler_decoder))
    om.latent = O.Pyramid(mat.latent.levels)
    om.half()
    _CPU.clear()
    _CPU.update(mat=om, pyr=om._half["latent"], kind="full", **{k: v.astype(np.float64) for k, v in q.items()})
    n = q["uv"].shape[0]
    if "pool" in _POOL:  # workers forked with other data: fork again
        _POOL["pool"].terminate()
        _POOL.clear()
    cpu_run(n, workers)  # warm (forks the pool once)
    return cpu_run(n, workers)


def run_ours(args):
    if args.workload == "c4":
        return run_c4(args)
    if args.workload == "train":
        return run_train(args)
    if args.workload == "kl":
        return run_kl(args)
    if args.workload == "c5":
        return run_c5(args)
    rank, world, local = dist_init(args.gpus)
    device = torch.device("cuda", local)
    from paper_2305_02678_b200 import _lib, neural, synth
    lib = _lib.load()
    mat, n, sets = build_workload(args, rank, device)
    h = mat.device_material(device)
    stream = torch.cuda.current_stream(device)
    clocks = Clocks(local)
    head = measure(args, lib, h, args.workload, sets, args.steps, args.warmup, stream, world, local, clocks)

    subs = {}
    if args.workload == "c2" and not args.no_subresults:
        # the rest of the metric ("eval, sample+pdf"): C3 and the full query,
        # each device-timed with its own roofline
        q3 = [synth.queries(C3_N, mat.latent.n_levels, seed=7 + 100 * rank, device=device,
                            need=("uv", "lod", "u_rr", "wi", "u3"))]
        subs["c3_sample_pdf"] = measure(args, lib, h, "c3", q3, max(5, args.steps // 50), 3, stream, world, local)
        subs["c3_sample_pdf"]["config"] = "C3: 4096^2, 1920x1080x16 = 33,177,600 sample+pdf queries per GPU, random lod"
        del q3
        subs["full_query"] = measure(args, lib, h, "full", sets, max(20, args.steps // 5), 3, stream, world, local)
        subs["full_query"]["config"] = "eval + sample + pdf, 4096^2, 1920x1080 per GPU"
        # C1 exactly (BASELINE configs[0]) on the GPU
        mat1, q1 = c1_case()
        h1 = mat1.device_material(device)
        t1 = [{k: torch.from_numpy(v).to(device) for k, v in q1.items()}]
        c1 = measure(args, lib, h1, "full", t1, max(50, args.steps // 2), 5, stream, world, local, tag="c1")
        c1["config"] = "C1: 512^2 pyramid, 65,536 full queries (inputs fit L2)"
        subs["c1_full_query"] = c1
        # the reference's default fp16=False path: fp32 master weights and pyramid
        if not args.no_fp32_path:
            from paper_2305_02678_b200.latent import LatentPyramid, level_shapes
            g = torch.Generator(device=device)
            g.manual_seed(11)
            lv = [torch.randn((hh, ww, 8), device=device, generator=g).cpu().numpy()
                  for hh, ww in level_shapes(RES, RES)]
            m32 = neural.NeuralMaterial.create(neural.NeuralMaterialConfig(), np.random.default_rng(0))
            m32.latent = LatentPyramid(lv)
            h32 = m32.device_material(device, precise=True)
            f32 = measure(args, lib, h32, "c2", sets[:1], max(10, args.steps // 20), 3, stream, world, local,
                          tag="fp32_path", kernel="fused_kernel<kModeEval> (csrc/nmq_kernels.cu, generic "
                          "tcgen05 kernel, 3 products per layer on hi/lo pairs)")
            f32["config"] = ("fp16=False (the reference default): fp32 master weights as fp16 hi/lo pairs, "
                             "fp32 4096^2 pyramid, 1920x1080 eval, generic tcgen05 kernel")
            subs["fp32_path_eval"] = f32
            del lv, m32, h32

    # ---- e2e through the drop-in call --------------------------------------------
    e2e = e2e_pinned = None
    if args.workload == "c2" and args.e2e_steps > 0:
        # the reference's own call shape (neural.py:303-309): pageable numpy
        # in, (f float64, albedo, chosen int64) out
        host = [{k: v.cpu().numpy() for k, v in q.items()} for q in sets[:2]]
        for i in range(2):
            hq = host[i % 2]
            neural.eval_material(mat, hq["uv"], hq["lod"], hq["wi"], hq["wo"], hq["u_rr"], fp16=True)
        torch.cuda.synchronize()
        barrier(world)
        t0 = time.perf_counter()
        for i in range(args.e2e_steps):
            hq = host[i % 2]
            f, _, lv = neural.eval_material(mat, hq["uv"], hq["lod"], hq["wi"], hq["wo"], hq["u_rr"], fp16=True)
        torch.cuda.synchronize()
        e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3, world)
        e2e = {"value": n * world * args.e2e_steps / (e_ms / 1e3), "unit": "queries/s",
               "h2d_bytes_per_step": int(n * 40), "d2h_bytes_per_step": int(n * 32),
               "steps": args.e2e_steps,
               "api": "paper_2305_02678_b200.neural.eval_material(mat, uv, lod, wi, wo, u_rr, fp16=True) "
                      "-> (f float64, None, chosen int64): pageable numpy in/out, the reference call shape "
                      "(neural.py:303) -> nm_eval_host_ref (pinned bounce pipeline, float64/int64 widened "
                      "on the device and copied back); H2D, kernels, D2H and the result allocation inside "
                      "the timed region"}
        # pinned host buffers and an fp32 `out`: the zero-copy launch
        pin = []
        for q in sets[:2]:
            hq = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in q.items()}
            for k in hq:
                hq[k].copy_(q[k])
            pin.append({k: v.numpy() for k, v in hq.items()})
        out_host = torch.empty((n, 3), dtype=torch.float32, pin_memory=True).numpy()
        for i in range(2):
            hq = pin[i % 2]
            neural.eval_material(mat, hq["uv"], hq["lod"], hq["wi"], hq["wo"], hq["u_rr"], fp16=True,
                                 return_level=False, out=out_host)
        torch.cuda.synchronize()
        barrier(world)
        t0 = time.perf_counter()
        for i in range(args.e2e_steps):
            hq = pin[i % 2]
            neural.eval_material(mat, hq["uv"], hq["lod"], hq["wi"], hq["wo"], hq["u_rr"], fp16=True,
                                 return_level=False, out=out_host)
        torch.cuda.synchronize()
        e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3, world)
        e2e_pinned = {"value": n * world * args.e2e_steps / (e_ms / 1e3), "unit": "queries/s",
                      "h2d_bytes_per_step": int(n * 40), "d2h_bytes_per_step": int(n * 12),
                      "api": "eval_material on pinned numpy with out= (fp32), return_level=False: one "
                             "zero-copy fused launch over PCIe"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        kind = "eval" if args.workload == "c2" else "sample_pdf"
        cpu_setup(mat, {k: v for k, v in sets[0].items()}, args.cpu_sample, kind)
        workers = os.cpu_count() or 1
        v = cpu_run(args.cpu_sample, workers)
        cpu = {"value": v, "unit": "queries/s", "cores": workers, "kind": "port",
               "sample": f"{args.cpu_sample} queries of the same {args.workload.upper()} batch "
                         f"(oracle/nm_oracle.py fp16 path, {workers} forked workers, "
                         f"OPENBLAS_NUM_THREADS=1, {cpu_model()})"}
        if args.workload == "c2":
            mat1, q1 = c1_case()
            cpu["c1_full_query_1core"] = {"value": c1_cpu(mat1, q1, 1), "unit": "queries/s", "cores": 1,
                                          "sample": "C1 exactly: 65,536 full queries, 512^2, oracle fp16 path"}
            cpu["c1_full_query_all_cores"] = {"value": c1_cpu(mat1, q1, workers), "unit": "queries/s",
                                              "cores": workers}

    if rank == 0:
        line = {
            "metric": METRIC, "value": head["value"], "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "fp16 x fp16 -> fp32 tensor-core (hi/lo split), fp32/fp64 SIMT",
            "data": "synthetic: random-init material (reference init order), N(0,1) fp16 latents, "
                    "seeded uniform queries + half/difference direction pairs",
            "config": {"workload": {"c2": "C2 coherent fused eval, 1 material, 4096^2 latent pyramid, "
                                          "1920x1080 queries per GPU",
                                    "c3": "C3 fused sample+pdf, 4096^2, 1920x1080x16 queries per GPU",
                                    "full": "full query (eval+sample+pdf), 4096^2, 1920x1080 per GPU"}[
                                        args.workload],
                       "queries_per_step_per_gpu": n, "latent": f"{RES}x{RES} 8ch fp16, 13 levels",
                       "brdf": "2x32", "sampler": "3x32", "parallelism": f"pixel-tile x{world}",
                       "parity": "exact fp16 input rounding (levels, taps, z bit-exact; strict tolerances)",
                       "l2": f"inputs rotate over {len(sets)} sets "
                             f"({len(sets) * n * io_bytes(args.workload) / 1e6:.0f} MB) > 126 MB L2"},
            "roofline": head["roofline"],
            "e2e": e2e,
            "e2e_pinned": e2e_pinned,
            "sub_results": subs or None,
            "cpu_baseline": cpu,
            "gpu_launches": head["gpu_launches"],
            "clocks": clocks.report(),
        }
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_reference(args):
    """The reference's CPU implementation of the path (the oracle port, since
    the reference is pure Python and cannot travel) on all host cores."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2305_02678_b200 import synth
    dev = torch.device("cuda", 0) if torch.cuda.is_available() else None
    n_sample = args.ref_sample
    if dev is not None:
        mat = synth.material("2x32", RES, RES, seed=0, device=dev)
        q = synth.queries(n_sample, mat.latent.n_levels, seed=1, device=dev)
    else:  # no GPU: same recipe generated on the host
        mat = material_host("2x32", RES, RES, seed=0)
        q = queries_host(n_sample, mat.latent.n_levels, seed=1)
    kind = "eval" if args.workload == "c2" else "sample_pdf"
    cpu_setup(mat, q, n_sample, kind)
    workers = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_run(n_sample, workers)
    rates = [cpu_run(n_sample, workers) for _ in range(args.steps)]
    total_s = sum(n_sample / r for r in rates)
    value = n_sample * args.steps / total_s
    sample = (f"{n_sample} queries per step of the {args.workload.upper()} workload "
              f"(oracle/nm_oracle.py, the reference's fp16 path restated in numpy; "
              f"{workers} forked workers, {cpu_model()})")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_s / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64/f32 numpy", "data": "synthetic (same recipe as ours)",
        "config": {"workload": args.workload.upper(), "latent": f"{RES}x{RES}", "brdf": "2x32"},
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": workers, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["c2", "c3", "full", "c4", "c5", "train", "kl"], default="c2")
    ap.add_argument("--sets", type=int, default=3)
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--cpu-sample", type=int, default=C2_N)
    ap.add_argument("--ref-sample", type=int, default=262144)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-subresults", action="store_true", help="headline workload only")
    ap.add_argument("--no-fp32-path", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (rank 0 prints the line)
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        raise SystemExit(subprocess.call(cmd))
    try:
        if args.impl == "reference":
            run_reference(args)
        else:
            run_ours(args)
    finally:
        if "pool" in _POOL:
            _POOL["pool"].close()
            _POOL["pool"].join()
        sys.stdout.flush()


if __name__ == "__main__":
    main()
