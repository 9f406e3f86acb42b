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


def inexact_f64(x):
    """True if x holds float64 values fp32 cannot represent exactly (python
    float scalars included): texel coordinates, levels and roulette numbers
    select levels and taps bit for bit, so such inputs take the float64
    coordinate entry points (nm_fetch_f64 / nm_query_f64) instead of being
    narrowed (latent.py:59-82 computes them in float64)."""
    if isinstance(x, torch.Tensor):
        return x.dtype == torch.float64 and not torch.equal(x.to(torch.float32).to(torch.float64), x)
    if isinstance(x, float):
        return float(np.float32(x)) != x
    a = np.asarray(x)
    if a.dtype.kind == "f" and a.dtype.itemsize > 4:
        # one narrowing pass + one mixed comparison (NaNs count as inexact and
        # take the float64 path, which handles them like numpy)
        return not bool((a.astype(np.float32) == a).all())
    return False


def check_exact_f32(x, name):
    """Entry points without a float64 coordinate path reject float64 values
    fp32 cannot represent (see inexact_f64) instead of narrowing them."""
    if inexact_f64(x):
        raise ValueError(f"{name}: float64 values not exactly representable in fp32 (pass fp32)")


def as_rows64(x, cols, device, name="array"):
    """(B, cols) float64 contiguous device tensor (float64 coordinates)."""
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x, dtype=np.float64))
    if t.dim() == 1 and cols > 1:
        t = t[None, :]
    t = t.to(device=device, dtype=torch.float64).contiguous()
    if cols > 1 and (t.dim() != 2 or t.shape[1] != cols):
        raise ValueError(f"{name}: expected shape (B, {cols}), got {tuple(t.shape)}")
    return t


def as_vec64(x, n, device, name="array"):
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(x, np.float64)))
    t = t.to(device=device, dtype=torch.float64).reshape(-1).contiguous()
    if t.numel() == 1 and n != 1:
        return t, 0
    if t.numel() != n:
        raise ValueError(f"{name}: expected {n} values, got {t.numel()}")
    return t, 1


def as_rows(x, cols, device, name="array", exact=False):
    """(B, cols) fp32 contiguous device tensor; 1-D input of length `cols` is
    promoted to one row (np.atleast_2d semantics, latent.py:90).  exact: see
    check_exact_f32."""
    if exact:
        check_exact_f32(x, name)
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


def as_vec(x, n, device, name="array", exact=False):
    """(n,) fp32 device tensor; scalars broadcast (returns (tensor, stride))."""
    if exact:
        check_exact_f32(x, name)
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
# Large host (numpy) batches stream through the GPU inside the native library
# (nm_eval_host: chunks over staging slots, H2D / kernel / D2H on three
# internal streams, overlapped).  Host buffers should be pinned for full overlap.

STREAM_CHUNK = int(os.environ.get("NMQ_STREAM_CHUNK", 1 << 19))  # queries per chunk
REF_CHUNK = int(os.environ.get("NMQ_REF_CHUNK", 0))  # nm_eval_host_ref chunk (0 = the library's default)


def host_rows(x, cols, name):
    """Host fp32 (B, cols) contiguous view (no copy when already so), or None
    if x is not a plain host array of that shape."""
    a = np.asarray(x)
    if a.ndim != 2 or a.shape[1] != cols:
        return None
    return np.ascontiguousarray(a, dtype=np.float32)


# Result arrays of the host-buffer calls: numpy arrays backed by page-locked
# memory from torch's caching host allocator (a block returns to its cache
# when the caller drops the array and is reused by a later call), so the
# results are DMA'd straight into them — no fresh-page faults, no host copy.
# Small results stay ordinary numpy arrays.
PINNED_RESULT_MIN = int(os.environ.get("NMQ_PINNED_RESULT_MIN", 1 << 20))  # bytes


def result_array(shape, dtype):
    nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
    if nbytes < PINNED_RESULT_MIN or not torch.cuda.is_available():
        return np.empty(shape, dtype)
    tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.int64): torch.int64,
           np.dtype(np.float32): torch.float32, np.dtype(np.int32): torch.int32}[np.dtype(dtype)]
    return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()
