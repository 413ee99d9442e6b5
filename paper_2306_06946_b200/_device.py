"""Device-array helpers shared by the API modules."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


def device() -> torch.device:
    return _lib.require_cuda()


def f64(x, dev=None) -> torch.Tensor:
    """Contiguous fp64 CUDA tensor view/copy of an array-like (host data goes
    through pinned staging without a stream synchronisation, see upload)."""
    dev = dev or device()
    if isinstance(x, torch.Tensor):
        if x.device != dev or x.dtype != torch.float64:
            x = x.to(device=dev, dtype=torch.float64)
        return x.contiguous()
    return upload(np.asarray(x, dtype=np.float64), dev=dev)


def i64(x, dev=None) -> torch.Tensor:
    dev = dev or device()
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=torch.int64).contiguous()
    return upload(np.asarray(x, dtype=np.int64), dev=dev)


def host(x) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def empty(shape, dev=None, dtype=torch.float64) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=dev or device())


def zeros(shape, dev=None, dtype=torch.float64) -> torch.Tensor:
    return torch.zeros(shape, dtype=dtype, device=dev or device())


def upload(a, dtype=None, dev=None) -> torch.Tensor:
    """Host array -> device tensor without a stream synchronisation: staged through
    pinned memory (a copy taken now, so later host writes do not race) and copied
    asynchronously on the current stream (the caching host allocator keeps the
    staging block alive until the copy has run)."""
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.pin_memory().to(dev or device(), non_blocking=True)
