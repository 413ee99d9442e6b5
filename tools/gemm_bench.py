"""fp64 DMMA GEMM throughput of cnb_gemm_dense (batch_gemm_kernel) vs the
register-only DMMA peak, for square sizes."""
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_06946_b200 import _lib  # noqa: E402


def main():
    out = {}
    pk = (ctypes.c_double * 1)()
    _lib.call("cnb_bench_dmma", 4096, pk, _lib.stream())
    out["dmma_peak_tflops"] = round(pk[0], 2)
    for n in (1024, 2048, 4096):
        A = torch.randn(n, n, dtype=torch.float64, device="cuda")
        B = torch.randn(n, n, dtype=torch.float64, device="cuda")
        C = torch.empty_like(A)
        for _ in range(2):
            _lib.call("cnb_gemm_dense", n, n, n, A.data_ptr(), n, B.data_ptr(), n, C.data_ptr(), n, _lib.stream())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 5
        for _ in range(reps):
            _lib.call("cnb_gemm_dense", n, n, n, A.data_ptr(), n, B.data_ptr(), n, C.data_ptr(), n, _lib.stream())
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        err = (C - A @ B).abs().max().item()
        e0.record()
        for _ in range(reps):
            torch.matmul(A, B, out=C)
        e1.record()
        torch.cuda.synchronize()
        ms_cublas = e0.elapsed_time(e1) / reps
        out[n] = dict(ms=round(ms, 3), tflops=round(2 * n ** 3 / ms / 1e9, 2), err=err,
                      cublas_tflops=round(2 * n ** 3 / ms_cublas / 1e9, 2))
    n = 4096
    A = torch.randn(n, n, dtype=torch.float64, device="cuda")
    B = torch.randn(n, n, dtype=torch.float64, device="cuda")
    C = torch.empty_like(A)
    ref = A @ B
    for v in range(8):
        try:
            _lib.call("cnb_bench_gemm", v, n, n, n, A.data_ptr(), n, B.data_ptr(), n, C.data_ptr(), n, _lib.stream())
        except Exception as exc:  # noqa: BLE001
            out[f"v{v}"] = str(exc)
            continue
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            _lib.call("cnb_bench_gemm", v, n, n, n, A.data_ptr(), n, B.data_ptr(), n, C.data_ptr(), n, _lib.stream())
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        out[f"v{v}"] = dict(tflops=round(2 * n ** 3 / ms / 1e9, 2), err=(C - ref).abs().max().item())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
