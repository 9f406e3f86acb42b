"""Multi-process sharding logic on CPU: world_size 2 over gloo (the GPU box
runs the same code over NCCL, one process per GPU)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2305_02678_b200 import shard


def test_row_bands_partition_the_frame():
    for world in (1, 2, 3, 4, 8):
        for h in (1, 7, 1080, 2160):
            bands = [shard.row_band(r, world, h) for r in range(world)]
            assert bands[0][0] == 0 and bands[-1][1] == h
            assert all(a[1] == b[0] for a, b in zip(bands, bands[1:]))
            sizes = [b[1] - b[0] for b in bands]
            assert max(sizes) - min(sizes) <= 1 and sizes[0] == max(sizes)


def test_band_queries_cover_all_samples():
    h, w, spp, world = 9, 5, 4, 4
    ranges = [shard.band_queries(r, world, h, w, spp) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == h * w * spp
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))


def test_reduce_spp_is_per_pixel_mean():
    x = torch.arange(24, dtype=torch.float32).view(8, 3)
    y = shard.reduce_spp(x, 4)
    assert torch.equal(y, x.view(2, 4, 3).mean(1))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, height, width, spp, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q0, q1 = shard.band_queries(rank, world, height, width, spp)
        # stand-in for the per-rank fused eval: a deterministic function of the
        # global query index, so the gathered image can be checked exactly
        idx = torch.arange(q0, q1, dtype=torch.float32)
        rgb = torch.stack([idx, idx * 2, idx * 3], dim=1)
        band = shard.reduce_spp(rgb, spp).view(-1, width, 3)
        img = shard.gather_bands(band, height, width)
        if rank == 0:
            out.put(img.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("height", [7, 8])
def test_gather_world2_gloo(height):
    world, width, spp = 2, 5, 3
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, height, width, spp, out))
             for r in range(world)]
    for p in procs:
        p.start()
    img = out.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    idx = torch.arange(height * width * spp, dtype=torch.float32)
    want = shard.reduce_spp(torch.stack([idx, idx * 2, idx * 3], 1), spp).view(height, width, 3)
    assert torch.equal(torch.from_numpy(img), want)
