"""Two ranks (gloo, both on the one GPU of the test box) each evaluate their
pixel-row band of a frame with the fused kernel — spp mean in the epilogue —
and gather the image to rank 0: equal to the single-process frame."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

H, W, SPP = 48, 40, 16


def _frame_queries(device):
    from paper_2305_02678_b200 import synth
    return synth.queries(H * W * SPP, 8, seed=77, device=device, need=("uv", "lod", "u_rr", "wi", "wo"))


def _worker(rank, world, port, out):
    import torch.distributed as dist
    from paper_2305_02678_b200 import neural, shard, synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        mat = synth.material("2x32", 256, 256, seed=9, device=dev)
        q = _frame_queries(dev)
        q0, q1 = shard.band_queries(rank, world, H, W, SPP)
        band = {k: v[q0:q1].contiguous() for k, v in q.items()}
        img = neural.eval_material_spp(mat, band["uv"], band["lod"], band["wi"], band["wo"], band["u_rr"], SPP)
        full = shard.gather_bands(img.view(-1, W, 3), H, W)
        if rank == 0:
            torch.save(full.cpu(), out)
    finally:
        dist.destroy_process_group()


def test_two_rank_band_gather_equals_single_frame(tmp_path):
    from paper_2305_02678_b200 import neural, synth
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = str(tmp_path / "frame.pt")
    mp.get_context("spawn")
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    gathered = torch.load(out).numpy()
    dev = torch.device("cuda", 0)
    mat = synth.material("2x32", 256, 256, seed=9, device=dev)
    q = _frame_queries(dev)
    ref = neural.eval_material_spp(mat, q["uv"], q["lod"], q["wi"], q["wo"], q["u_rr"], SPP)
    np.testing.assert_allclose(gathered.reshape(-1, 3), ref.cpu().numpy(), rtol=1e-6, atol=1e-7)
