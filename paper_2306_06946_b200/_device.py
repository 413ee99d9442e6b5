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


def square(c: int, dev=None) -> torch.Tensor:
    """(c, c) fp64 matrix whose rows are 16-byte aligned: a view of a (c, c + c % 2)
    buffer.  Dense constraint-space operators (W) use it so the PGS kernel can
    move tiles with tensor TMA (the global row pitch must be a multiple of 16
    bytes); pass ``t.stride(0)`` as the leading dimension."""
    buf = torch.empty((c, c + (c & 1)), dtype=torch.float64, device=dev or device())
    return buf[:, :c]


def mat64(x, dev=None) -> torch.Tensor:
    """A dense operator as a row-major fp64 device matrix, keeping (or creating) the
    16-byte aligned row pitch of ``square`` for square matrices."""
    dev = dev or device()
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    if t.device != dev or t.dtype != torch.float64:
        t = t.to(device=dev, dtype=torch.float64)
    if t.dim() == 2 and t.shape[0] == t.shape[1]:
        if t.stride(1) == 1 and (t.stride(0) % 2 == 0 or t.shape[0] <= 1):
            return t
        out = square(t.shape[0], dev)
        out.copy_(t)
        return out
    return t.contiguous()


def ld(t: torch.Tensor) -> int:
    """Leading dimension (row pitch, elements) of a row-major matrix view."""
    if t.dim() != 2 or (t.shape[1] > 1 and t.stride(1) != 1):
        raise ValueError(f"expected a row-major matrix view, got shape {tuple(t.shape)} strides {t.stride()}")
    return int(t.stride(0)) if t.shape[0] > 1 else int(t.shape[1])


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
