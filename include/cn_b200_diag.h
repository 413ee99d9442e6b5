/* Diagnostics and measurement hooks of libcnb200.so (not part of the drop-in
 * boundary in cn_b200.h): used by bench.py and tools/ to count launches, read
 * phase profiles of the PGS / factor kernels and measure the fp64 tensor-core
 * peak the rooflines are quoted against.  Same conventions as cn_b200.h. */
#ifndef CN_B200_DIAG_H
#define CN_B200_DIAG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Number of kernels this library has launched in the process so far. */
long long cnb_launch_count(void);

/* Phase profile of the pipelined PGS kernel (env CNB_PGS_PROFILE=1): summed SM
 * cycles per slot since the last call, out[32]; slot meanings are listed at the
 * stamp() calls in csrc/pgs.cu.  CNB_E_VALIDATION when profiling is off. */
int cnb_pgs_profile(double* out);

/* Summed cycles of the 32 x 32 POTRF phases (every call, standalone or fused
 * into the SYRK; warp 0, the inverse runs beside it on warp 1) since the last
 * call: out[0] loads, [1] elimination loop, out[7] calls. */
int cnb_potrf_profile(double* out);

/* Global-timer stamps (ns, out: host, 64) of the last cooperative single-RHS
 * solve's phase ends: start, permute, then per forward level assemble and
 * panel product, per backward level, in order. */
int cnb_solve_profile(double* out);

/* fp64 DMMA GEMM tile-shape variants, C = A B (row-major; sizes multiples of
 * the variant's tile). */
int cnb_bench_gemm(int32_t variant, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                   int64_t ldb, double* C, int64_t ldc, void* stream);

/* out (host, 12): cycles per dependent op -- DFMA, DADD, fp64 div, fp64 sqrt,
 * 64-bit shuffle, FFMA, select, MUFU.RSQ64H, DMUL -- then one warp's issue
 * cost: cycles per DFMA, per broadcast LDS.64, per POTRF bulk step. */
int cnb_bench_latency(double* out /* 12 doubles */, void* stream);

/* fp64 MMA (DMMA) throughput of the whole GPU in TFLOP/s (out: host): the
 * tensor roofline denominator (not in MEASURED_PEAKS.json). */
int cnb_bench_dmma(int32_t iters, double* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CN_B200_DIAG_H */
