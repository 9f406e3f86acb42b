"""Array plumbing between the reference-style API (numpy in, numpy out) and
the device pointers the C ABI takes.  torch is used only for device memory
and streams."""

import os

import numpy as np
import torch


def cuda_device(device=None):
    if not torch.cuda.is_available():
        raise RuntimeError("the neural-material query path needs a CUDA device (no CPU fallback)")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {device!r}")
    return torch.device("cuda", d.index if d.index is not None else torch.cuda.current_device())


def is_numpy_like(x):
    return not isinstance(x, torch.Tensor)


def as_rows(x, cols, device, name="array"):
    """(B, cols) fp32 contiguous device tensor; 1-D input of length `cols` is
    promoted to one row (np.atleast_2d semantics, latent.py:90)."""
    if isinstance(x, torch.Tensor):
        t = x
        if t.dim() == 1 and cols > 1:
            t = t[None, :]
        t = t.to(device=device, dtype=torch.float32).contiguous()
    else:
        a = np.asarray(x)
        if a.ndim == 1 and cols > 1:
            a = a[None, :]
        a = np.ascontiguousarray(a, dtype=np.float32)
        t = torch.from_numpy(a).to(device, non_blocking=False)
    if cols > 1 and (t.dim() != 2 or t.shape[1] != cols):
        raise ValueError(f"{name}: expected shape (B, {cols}), got {tuple(t.shape)}")
    if cols == 1:
        t = t.reshape(-1)
    return t


def as_vec(x, n, device, name="array"):
    """(n,) fp32 device tensor; scalars broadcast (returns (tensor, stride))."""
    if isinstance(x, torch.Tensor):
        t = x.to(device=device, dtype=torch.float32).reshape(-1).contiguous()
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float32).reshape(-1))).to(device)
    if t.numel() == 1 and n != 1:
        return t, 0
    if t.numel() != n:
        raise ValueError(f"{name}: expected {n} values, got {t.numel()}")
    return t, 1


def empty(n, cols, device, dtype=torch.float32):
    shape = (n,) if cols == 1 else (n, cols)
    return torch.empty(shape, device=device, dtype=dtype)


def ptr(t):
    return None if t is None else t.data_ptr()


def stream_ptr(device):
    return torch.cuda.current_stream(device).cuda_stream


def out(t, numpy_mode, np_dtype=np.float64):
    """Return numpy (reference dtype) for numpy callers, else the tensor."""
    if not numpy_mode:
        return t
    return t.cpu().numpy().astype(np_dtype, copy=False)


# ---------------------------------------------------------------------------
# Streaming host <-> device pipeline for large host (numpy) batches: chunks of
# the batch alternate between two CUDA streams, so the H2D copy of chunk c+1,
# the kernel of chunk c and the D2H copy of chunk c-1 overlap (both copy
# engines + the SMs busy).  Host buffers should be pinned for real overlap;
# pageable memory still works (the driver stages it synchronously).

STREAM_CHUNK = int(os.environ.get("NMQ_STREAM_CHUNK", 1 << 19))  # queries per chunk
_STREAMS = {}


def _streams(dev):
    key = dev.index
    if key not in _STREAMS:
        _STREAMS[key] = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
    return _STREAMS[key]


def host_rows(x, cols, name):
    """Host fp32 (B, cols) contiguous view (no copy when already so), or None
    if x is not a plain host array of that shape."""
    a = np.asarray(x)
    if a.ndim != 2 or a.shape[1] != cols:
        return None
    return np.ascontiguousarray(a, dtype=np.float32)


def streamed(n, dev, host_in, host_out, launch, chunk=STREAM_CHUNK):
    """Run `launch(dev_in_slices, dev_out_slices, count, stream_ptr)` over
    chunks of the batch with double-buffered streams.  host_in / host_out are
    lists of host numpy arrays with n rows; outputs are complete on return."""
    d_in = [torch.empty(a.shape, device=dev, dtype=torch.float32) for a in host_in]
    d_out = [torch.empty(o.shape, device=dev, dtype=torch.from_numpy(o[:0]).dtype) for o in host_out]
    h_in = [torch.from_numpy(a) for a in host_in]
    h_out = [torch.from_numpy(o) for o in host_out]
    cur = torch.cuda.current_stream(dev)
    ss = _streams(dev)
    start = torch.cuda.Event()
    start.record(cur)
    for s in ss:
        s.wait_event(start)
    for ci, c0 in enumerate(range(0, n, chunk)):
        c1 = min(n, c0 + chunk)
        s = ss[ci & 1]
        with torch.cuda.stream(s):
            for d, h in zip(d_in, h_in):
                d[c0:c1].copy_(h[c0:c1], non_blocking=True)
            launch([d[c0:c1] for d in d_in], [o[c0:c1] for o in d_out], c1 - c0, s.cuda_stream)
            for o, h in zip(d_out, h_out):
                h[c0:c1].copy_(o[c0:c1], non_blocking=True)
    for s in ss:
        cur.wait_stream(s)
    cur.synchronize()
