"""Pixel-tile sharding of query batches across GPUs (one process per GPU).

The query path is embarrassingly parallel: queries are independent and the
material is read-only.  A frame of H x W pixels x spp samples is
split into contiguous row bands, one per rank; every rank holds a full copy
of the material (weights + latents) and runs the fused kernels on its band
with no collective on the data path.  The only exchange is the final gather
of the spp-reduced image (H x W x 3 fp32) to rank 0 — the analogue of the
reference renderer's accumulation (render.py:565) done once per frame.
"""

import torch
import torch.distributed as dist


def row_band(rank, world, height):
    """Contiguous, balanced band of image rows [y0, y1) for `rank`."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    base, extra = divmod(height, world)
    y0 = rank * base + min(rank, extra)
    return y0, y0 + base + (1 if rank < extra else 0)


def band_queries(rank, world, height, width, spp):
    """Query index range of the rank's band: pixels row-major, `spp`
    consecutive samples per pixel."""
    y0, y1 = row_band(rank, world, height)
    return y0 * width * spp, y1 * width * spp


def reduce_spp(rgb, spp):
    """(pixels*spp, 3) -> (pixels, 3) per-pixel mean."""
    return rgb.view(-1, spp, rgb.shape[-1]).mean(dim=1)


def gather_bands(band, height, width, dst=0, group=None):
    """Gather every rank's (rows, width, C) band to `dst`.  Bands are padded
    to the largest band so one gather moves equal-sized messages.  Returns
    the (height, width, C) image on `dst`, None elsewhere."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if dist.get_backend(group) == "gloo" and band.is_cuda:  # gloo gathers host tensors
        band = band.cpu()
    c = band.shape[-1]
    max_rows = row_band(0, world, height)[1]  # rank 0 holds the largest band
    buf = band.new_zeros((max_rows, width, c))
    buf[: band.shape[0]] = band
    if rank == dst:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.gather(buf, gather_list=parts, dst=dst, group=group)
        rows = [p[: row_band(r, world, height)[1] - row_band(r, world, height)[0]]
                for r, p in enumerate(parts)]
        return torch.cat(rows, dim=0)
    dist.gather(buf, gather_list=None, dst=dst, group=group)
    return None
