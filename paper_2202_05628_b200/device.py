"""Device-memory plumbing: torch owns allocations and streams; kernels see
raw pointers through the C ABI. 64-bit and 32-bit unsigned arrays travel
as same-width signed tensors (bit patterns preserved)."""

from __future__ import annotations

import numpy as np
import torch

_SIGNED = {np.dtype(np.uint64): np.int64, np.dtype(np.uint32): np.int32,
           np.dtype(np.uint8): np.uint8, np.dtype(np.bool_): np.uint8}


def device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle(stream: torch.cuda.Stream | None = None) -> int | None:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream or None


def upload(a, dtype) -> torch.Tensor:
    """numpy (any layout) -> contiguous device tensor holding dtype's bits."""
    arr = np.ascontiguousarray(a, dtype=dtype)
    view = _SIGNED.get(arr.dtype)
    if view is not None:
        arr = arr.view(view)
    return torch.from_numpy(arr).to(device(), non_blocking=False)


def empty(shape, dtype) -> torch.Tensor:
    np_dt = np.dtype(dtype)
    view = _SIGNED.get(np_dt, np_dt.type)
    t_dtype = torch.from_numpy(np.empty(0, dtype=view)).dtype
    return torch.empty(shape, dtype=t_dtype, device=device())


def download(t: torch.Tensor, dtype=None) -> np.ndarray:
    a = t.detach().cpu().numpy()
    if dtype is not None and np.dtype(dtype) != a.dtype:
        a = a.view(dtype) if np.dtype(dtype).itemsize == a.dtype.itemsize else a.astype(dtype)
    return a


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    return t.data_ptr() or None


def workspace(nbytes: int) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device())
