"""Device-array helpers shared by the API modules."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


def device() -> torch.device:
    return _lib.require_cuda()


def f64(x, dev=None) -> torch.Tensor:
    """Contiguous fp64 CUDA tensor view/copy of an array-like."""
    dev = dev or device()
    if isinstance(x, torch.Tensor):
        if x.device != dev or x.dtype != torch.float64:
            x = x.to(device=dev, dtype=torch.float64)
        return x.contiguous()
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device=dev)


def i64(x, dev=None) -> torch.Tensor:
    dev = dev or device()
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=torch.int64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.int64), device=dev)


def host(x) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def empty(shape, dev=None, dtype=torch.float64) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=dev or device())


def zeros(shape, dev=None, dtype=torch.float64) -> torch.Tensor:
    return torch.zeros(shape, dtype=dtype, device=dev or device())


def upload(a, dtype=None) -> torch.Tensor:
    """Host array -> device tensor without a stream synchronisation: staged through
    pinned memory and copied asynchronously on the current stream (the caching
    host allocator keeps the staging block alive until the copy has run)."""
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.pin_memory().to(device(), non_blocking=True)
