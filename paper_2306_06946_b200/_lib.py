"""ctypes binding of the C ABI in include/cn_b200.h.

The library is built in-tree (``build.py``) for sm_100a.  There is no CPU
fallback: importing a compute entry point without the library, or without a
CUDA device, raises immediately.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcnb200.so")

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
F64 = ctypes.c_double

# name -> argtypes (restype is int status unless listed in _RESTYPES)
_SIGNATURES: dict[str, list] = {
    "cnb_abi_version": [],
    "cnb_last_error": [],
    "cnb_rebuild_w": [I64, P, P, I64, P, I64, P],
    "cnb_sandwich": [I64, I64, P, P, P, I64, P, I64, P],
    "cnb_plane_distances": [I64, P, P, F64, F64, F64, F64, P, P],
    "cnb_batch_detect_planes": [I32, I64, P, P, I64, P, P, F64, P, P, P],
    "cnb_batch_pairs": [I32, I64, I64, P, P, P, P, I64, P, P, P, P, P, P, P, P, P],
    "cnb_batch_gather_pa": [I64, P, P, P, P, I64, P, P],
    "cnb_batch_wg_gather": [I32, I64, P, P, P, P, P, P, I64, P, P],
    "cnb_gemm_dense": [I64, I64, I64, P, I64, P, I64, P, I64, P],
    "cnb_batch_rebuild_w": [I32, I64, P, P, P, P, P, P, P],
    "cnb_batch_prox": [I32, I64, P, P, P, P, F64, P, P],
    "cnb_batch_spmv": [I32, I64, P, P, P, P, I64, P, I64, P],
    "cnb_batch_rhs": [I32, I64, P, P, P, P, P, P, F64, F64, F64, P, P, P],
    "cnb_batch_scatter_acc": [I64, P, P, P, P, P, I64, P],
    "cnb_pgs_batched": [I32, P, P, P, P, P, F64, F64, I32, P, P, P, P, P, P, P],
    "cnb_violation": [I64, P, P, P, P, P],
    "cnb_scatter_add_compliance": [I64, P, I64, P, P, I64, P],
    "cnb_apply_dt": [I64, P, P, P, P, P],
    "cnb_prox_update": [I64, P, I64, P, P, P, F64, P, P, P],
    "cnb_build_frames": [I64, P, P, P, P, P, P],
    "cnb_relinearize": [I64, P, P, P, P, P, P],
    "cnb_refresh_proximity": [I64, P, P, P, P, P, P, P, P, P, P, P],
    "cnb_signed_gaps": [I64, P, P, P, P, P, P, P, P, P, P, P, P, P, P],
    "cnb_detect_work_bytes": [I64, I64],
    "cnb_detect_vertex_mesh": [I64, P, P, I64, P, P, F64, P, P, P, P],
    "cnb_pgs_profile": [P],
    "cnb_potrf_profile": [P],
    "cnb_solve_profile": [P],
    "cnb_bench_gemm": [I32, I64, I64, I64, P, I64, P, I64, P, I64, P],
    "cnb_pgs": [I64, P, I64, P, F64, F64, F64, I32, P, P, P, P, P, P, P],
    "cnb_pgs_coloured": [I64, P, I64, P, F64, F64, F64, I32, P, P, I32, F64, P, P, P, P, P, P, P],
    "cnb_local_solve": [I64, I64, P, I64, P, P, F64, F64, P, P, P],
    "cnb_gemm_naive": [I64, I64, I64, P, I64, I32, P, I64, I32, P, I64, P],
    "cnb_csr_spmv": [I64, P, P, P, P, P, F64, P],
    "cnb_fe_element": [I64, P, P, P, P, P, F64, F64, I32, P, P, P, P],
    "cnb_fe_gather": [I64, P, P, P, P, P, I64, P, P, P, P, P],
    "cnb_fe_system": [I64, P, P, P, P, P, P, F64, F64, F64, P, P, P, P, P, P, P, P],
    "cnb_chol_analyze": [I64, P, P, I32, P, I32, P],
    "cnb_chol_destroy": [P],
    "cnb_chol_info": [P, P, P],
    "cnb_chol_export_bytes": [P, ctypes.c_char_p],
    "cnb_chol_export": [P, ctypes.c_char_p, P],
    "cnb_chol_factor": [P, P, P, P],
    "cnb_chol_solve": [P, P, I64, P, I64, I64, P],
    "cnb_chol_compliance": [P, I64, P, P, P, P, I64, P, P],
    "cnb_chol_compliance_plan": [P, I64, P, P, P, I32, I32, P, P, P],
    "cnb_chol_compliance_forward": [P, P, P],
    "cnb_chol_compliance_gram": [P, P, P, P],
    "cnb_chol_compliance_finish": [P, P, P, I64, P],
    "cnb_bench_dmma": [I32, P, P],
    "cnb_bench_latency": [P, P],
    "cnb_launch_count": [],
}
_RESTYPES = {
    "cnb_launch_count": ctypes.c_longlong,
    "cnb_last_error": ctypes.c_char_p,
    "cnb_detect_work_bytes": I64,
    "cnb_chol_export_bytes": I64,
}

STATUS_ERRORS = {
    1: errors.DimensionMismatchError,
    2: errors.NotSPDError,
    3: errors.SingularBlockError,
    4: errors.DegenerateFrameError,
    5: errors.NonFiniteForceError,
    6: errors.ValidationError,
    7: errors.InvalidAttachmentError,
    8: errors.DegenerateTetError,
}

_lock = threading.Lock()
_lib = None


class LibraryMissing(RuntimeError):
    """The sm_100a library has not been built (run __graft_entry__.build())."""


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise LibraryMissing(
                    f"{LIB_PATH} is missing; build it with `python -m paper_2306_06946_b200.build`"
                )
            handle = ctypes.CDLL(LIB_PATH)
            for name, args in _SIGNATURES.items():
                fn = getattr(handle, name)
                fn.argtypes = args
                fn.restype = _RESTYPES.get(name, ctypes.c_int)
            _lib = handle
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def check(code: int, what: str = "") -> None:
    if code == 0:
        return
    msg = lib().cnb_last_error().decode(errors="replace")
    cls = STATUS_ERRORS.get(code)
    if cls is None:
        raise RuntimeError(f"{what}: native error {code}: {msg}")
    raise cls(f"{what}: {msg}" if what else msg)


# entry points whose workspaces are (re)allocated before any launch: on a
# device out-of-memory they are retried once after torch's caching allocator
# returned its unused blocks (the library's cudaMalloc competes with it)
_OOM_RETRY = {"cnb_chol_compliance", "cnb_chol_compliance_plan", "cnb_chol_solve"}


def call(name: str, *args) -> None:
    code = getattr(lib(), name)(*args)
    if code == 100 and name in _OOM_RETRY and "out of memory" in lib().cnb_last_error().decode(errors="replace"):
        torch.cuda.empty_cache()
        code = getattr(lib(), name)(*args)
    check(code, name)


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2306_06946_b200 computes on a CUDA (sm_100a) device only; none is available"
        )
    lib()
    return torch.device("cuda", torch.cuda.current_device() if device is None else device)


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


# ---- device status word (cnb_status_t) -------------------------------------

class DeviceStatus:
    """16-byte status word on the device: int32 code, int32 index, f64 value."""

    def __init__(self, device):
        self.buf = torch.zeros(2, dtype=torch.float64, device=device)

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr()

    def raise_if_set(self, what: str) -> None:
        host = self.buf.cpu()
        raw = host.numpy().view("<i4")
        code, index = int(raw[0]), int(raw[1])
        if code == 0:
            return
        value = float(host[1])
        self.buf.zero_()
        cls = STATUS_ERRORS.get(code, RuntimeError)
        if code == 3:
            raise cls(f"{what}: group {index}: singular contact block (value {value!r})")
        if code == 2:
            raise cls(f"{what}: non-positive pivot {value:.3e} at column {index}")
        if code == 4:
            raise cls(f"{what}: coincident proximity points and no element normal (pair {index})")
        raise cls(f"{what}: native status {code} at {index} ({value!r})")


_status_by_device: dict[int, DeviceStatus] = {}


def status(device: torch.device) -> DeviceStatus:
    key = device.index if device.index is not None else torch.cuda.current_device()
    st = _status_by_device.get(key)
    if st is None:
        st = DeviceStatus(device)
        _status_by_device[key] = st
    return st
