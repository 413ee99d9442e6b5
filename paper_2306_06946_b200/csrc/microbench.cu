// fp64 tensor-core (DMMA) peak microbenchmark: the fp64 roofline denominator
// (MEASURED_PEAKS.json carries only HBM and bf16 peaks).  Every warp issues
// long chains of independent mma.sync m8n8k4 f64 on register operands.
#include "common.cuh"

namespace cnb {

__global__ void __launch_bounds__(256) dmma_peak_kernel(int iters, double* out) {
  const int lane = threadIdx.x & 31;
  double a = 1.0 + 1e-3 * lane, b = 1.0 - 1e-3 * lane;
  double c[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma_8x8x4(c[k][0], c[k][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;  // keep the work alive
}

// Dependent-chain latencies (cycles per op) measured by one thread:
// out[0] DFMA, out[1] DADD, out[2] fp64 division, out[3] fp64 sqrt,
// out[4] 64-bit shuffle round trip, out[5] FFMA (fp32) for reference,
// out[6] fp64 compare-select + DADD, out[7] MUFU.RSQ64H + DADD, out[8] DMUL.
__global__ void latency_kernel(int n, double seed, double* out, long long* cyc) {
  double x = seed, y = 1.0000001, z = 1e-9;
  float xf = (float)seed;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, z);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x + z;
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = y / x;
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 1.0);
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + z;
  long long t5 = clock64();
  for (int i = 0; i < n; ++i) xf = fmaf(xf, 1.0000001f, 1e-9f);
  long long t6 = clock64();
  for (int i = 0; i < n; ++i) x = (x > z ? x : z) + z;  // DSETP + FSEL select, then DADD
  long long t7 = clock64();
  for (int i = 0; i < n; ++i) {
    double r;
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    x = r + 1.0;  // MUFU.RSQ64H then DADD
  }
  long long t8 = clock64();
  for (int i = 0; i < n; ++i) x = x * y;  // DMUL
  long long t9 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
    cyc[3] = t4 - t3;
    cyc[4] = t5 - t4;
    cyc[5] = t6 - t5;
    cyc[6] = t7 - t6;
    cyc[7] = t8 - t7;
    cyc[8] = t9 - t8;
    out[0] = x + xf;
  }
}

// Single-warp issue throughput (cycles per warp instruction / per bulk step):
// out[0] DFMA, 8 independent chains; out[1] LDS.64 of one broadcast address;
// out[2] the 32x32 POTRF's bulk step (31 broadcast LDS.64 + 31 DFMA, shift
// register, as chol.cu potrf_panel).
__global__ void throughput_kernel(int n, double seed, double* out, long long* cyc) {
  __shared__ double sm[128];
  const int lane = threadIdx.x & 31;
  for (int e = lane; e < 128; e += 32) sm[e] = 1.0 + 1e-9 * e;
  __syncwarp();
  double c[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k] = seed + k;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) c[k] = fma(c[k], 1.0000001, 1e-9);
  }
  long long t1 = clock64();
  double acc = 0.0;
  volatile int off = 0;
  const int o = off;
  for (int it = 0; it < n; ++it) {
    double v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = sm[(o + it + k) & 127];
#pragma unroll
    for (int k = 0; k < 32; ++k) acc += v[k] * 0.0;  // cheap consumer (DADD chain, 1 per load)
  }
  long long t2 = clock64();
  double a[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) a[k] = seed + k + lane;
  for (int it = 0; it < n; ++it) {
    const double lij = a[0] * 1e-3;
    const double* col = sm + (it & 63);
#pragma unroll
    for (int q = 0; q < 31; ++q) a[q] = fma(-lij, col[q + 1], a[q + 1]);
    a[31] = 1.0;
  }
  long long t3 = clock64();
  double s = acc;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k];
#pragma unroll
  for (int k = 0; k < 32; ++k) s += a[k];
  if (lane == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
  }
  if (s == 12345.678) out[0] = s;
}

// GEMM tile-shape experiments (C = A B, row-major, fp64 DMMA): BM x BN CTA tile,
// WM x WN warp tiles, BK-deep k chunks double-buffered with cp.async (8- or
// 16-byte copies), A staged [m][k], B staged [k][n] (both conflict-free
// fragment reads with strides == 4 mod 16 doubles); VOL: mma as asm volatile.
__device__ __forceinline__ void dmma_nv(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

template <int BM, int BN, int WM, int WN, int BK, bool V16, bool VOL>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32) gemm_var_kernel(int64_t M, int64_t N, int64_t K,
                                                                             const double* __restrict__ A,
                                                                             int64_t lda,
                                                                             const double* __restrict__ B,
                                                                             int64_t ldb, double* __restrict__ C,
                                                                             int64_t ldc) {
  constexpr int NT = (BM / WM) * (BN / WN) * 32;
  constexpr int SA = BK + 4, SB = BN + 4;
  extern __shared__ __align__(16) double gv_sm[];
  double* As = gv_sm;                 // [2][BM][SA]
  double* Bs = gv_sm + 2 * BM * SA;   // [2][BK][SB]
  const int64_t r0 = (int64_t)blockIdx.y * BM, c0 = (int64_t)blockIdx.x * BN;
  auto stage = [&](int buf, int64_t k0) {
    double* Ab = As + buf * BM * SA;
    double* Bb = Bs + buf * BK * SB;
    if (V16) {
      for (int e = threadIdx.x; e < BM * BK / 2; e += NT) {
        const int rr = e / (BK / 2), kk = 2 * (e % (BK / 2));
        const unsigned sa = (unsigned)__cvta_generic_to_shared(Ab + rr * SA + kk);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(A + (r0 + rr) * lda + k0 + kk)
                     : "memory");
      }
      for (int e = threadIdx.x; e < BK * BN / 2; e += NT) {
        const int kk = e / (BN / 2), cc = 2 * (e % (BN / 2));
        const unsigned sb = (unsigned)__cvta_generic_to_shared(Bb + kk * SB + cc);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sb), "l"(B + (k0 + kk) * ldb + c0 + cc)
                     : "memory");
      }
    } else {
      for (int e = threadIdx.x; e < BM * BK; e += NT) {
        const int rr = e / BK, kk = e % BK;
        cp_async8(Ab + rr * SA + kk, A + (r0 + rr) * lda + k0 + kk, true);
      }
      for (int e = threadIdx.x; e < BK * BN; e += NT) {
        const int kk = e / BN, cc = e % BN;
        cp_async8(Bb + kk * SB + cc, B + (k0 + kk) * ldb + c0 + cc, true);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  constexpr int WX = BN / WN;
  const int wy = (warp / WX) * WM, wx = (warp % WX) * WN;
  constexpr int FA = WM / 8, FB = WN / 8;
  double acc[FA][FB][2];
#pragma unroll
  for (int a = 0; a < FA; ++a)
#pragma unroll
    for (int b = 0; b < FB; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int nk = (int)(K / BK);  // experiment: K, M, N multiples of the tile
  stage(0, 0);
  for (int ck = 0; ck < nk; ++ck) {
    if (ck + 1 < nk) {
      stage((ck + 1) & 1, (int64_t)(ck + 1) * BK);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const double* Ab = As + (ck & 1) * BM * SA;
    const double* Bb = Bs + (ck & 1) * BK * SB;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double fa[FA], fb[FB];
#pragma unroll
      for (int a = 0; a < FA; ++a) fa[a] = Ab[(wy + 8 * a + g) * SA + kk + t];
#pragma unroll
      for (int b = 0; b < FB; ++b) fb[b] = Bb[(kk + t) * SB + wx + 8 * b + g];
#pragma unroll
      for (int a = 0; a < FA; ++a)
#pragma unroll
        for (int b = 0; b < FB; ++b) {
          if (VOL)
            dmma_8x8x4(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
          else
            dmma_nv(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < FA; ++a)
#pragma unroll
    for (int b = 0; b < FB; ++b)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int64_t r = r0 + wy + 8 * a + g, c = c0 + wx + 8 * b + 2 * t + hh;
        C[r * ldc + c] = acc[a][b][hh];
      }
}

template <int BM, int BN, int WM, int WN, int BK, bool V16, bool VOL>
static int launch_gemm_var(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                           int64_t ldb, double* C, int64_t ldc, cudaStream_t st) {
  if (M % BM || N % BN || K % BK) {
    set_error("bench_gemm: sizes must be multiples of the tile");
    return CNB_E_VALIDATION;
  }
  constexpr int NT = (BM / WM) * (BN / WN) * 32;
  const int smem = (int)(2 * (BM * (BK + 4) + BK * (BN + 4)) * sizeof(double));
  auto kern = gemm_var_kernel<BM, BN, WM, WN, BK, V16, VOL>;
  CNB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  dim3 grid((unsigned)(N / BN), (unsigned)(M / BM));
  kern<<<grid, NT, smem, st>>>(M, N, K, A, lda, B, ldb, C, ldc);
  CNB_LAUNCH_CHECK("gemm_var_kernel");
  return CNB_OK;
}

}  // namespace cnb

using namespace cnb;

extern "C" {

// out (host, 12 doubles): [0..8] cycles per dependent op, see latency_kernel;
// [9..11] single-warp issue throughput, see throughput_kernel.
int cnb_bench_latency(double* out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  double* d = nullptr;
  long long* c = nullptr;
  CNB_CUDA(cudaMalloc(&d, sizeof(double)));
  CNB_CUDA(cudaMalloc(&c, 12 * sizeof(long long)));
  const int n = 4096;
  latency_kernel<<<1, 32, 0, st>>>(n, 1.5, d, c);
  CNB_LAUNCH_CHECK("latency_kernel");
  throughput_kernel<<<1, 32, 0, st>>>(n, 1.5, d, c + 9);
  CNB_LAUNCH_CHECK("throughput_kernel");
  long long h[12];
  CNB_CUDA(cudaMemcpyAsync(h, c, sizeof(h), cudaMemcpyDeviceToHost, st));
  CNB_CUDA(cudaStreamSynchronize(st));
  for (int k = 0; k < 9; ++k) out[k] = (double)h[k] / n;
  out[9] = (double)h[9] / (n * 32.0);
  out[10] = (double)h[10] / (n * 32.0);
  out[11] = (double)h[11] / n;
  cudaFree(d);
  cudaFree(c);
  return CNB_OK;
}

// Diagnostic GEMM tile-shape variants (see gemm_var_kernel): C = A B.
int cnb_bench_gemm(int32_t variant, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                   int64_t ldb, double* C, int64_t ldc, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  switch (variant) {
    case 0: return launch_gemm_var<64, 64, 32, 32, 32, false, true>(M, N, K, A, lda, B, ldb, C, ldc, st);
    case 1: return launch_gemm_var<64, 64, 32, 32, 32, true, true>(M, N, K, A, lda, B, ldb, C, ldc, st);
    case 2: return launch_gemm_var<64, 64, 32, 32, 32, true, false>(M, N, K, A, lda, B, ldb, C, ldc, st);
    case 3: return launch_gemm_var<128, 64, 64, 32, 32, true, false>(M, N, K, A, lda, B, ldb, C, ldc, st);
    case 4: return launch_gemm_var<128, 128, 64, 32, 32, true, false>(M, N, K, A, lda, B, ldb, C, ldc, st);
    case 5: return launch_gemm_var<128, 128, 64, 32, 16, true, false>(M, N, K, A, lda, B, ldb, C, ldc, st);
    case 6: return launch_gemm_var<64, 128, 32, 64, 32, true, false>(M, N, K, A, lda, B, ldb, C, ldc, st);
    case 7: return launch_gemm_var<128, 64, 64, 32, 16, true, false>(M, N, K, A, lda, B, ldb, C, ldc, st);
    default:
      set_error("bench_gemm: unknown variant %d", variant);
      return CNB_E_VALIDATION;
  }
}

// TFLOP/s of DMMA over the whole GPU (result written to host out[0]).
int cnb_bench_dmma(int32_t iters, double* out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 0;
  CNB_CUDA(cudaGetDevice(&dev));
  CNB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* d = nullptr;
  CNB_CUDA(cudaMalloc(&d, sizeof(double)));
  const int blocks = sms * 4, threads = 256;
  dmma_peak_kernel<<<blocks, threads, 0, st>>>(iters / 8, d);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  dmma_peak_kernel<<<blocks, threads, 0, st>>>(iters, d);
  cudaEventRecord(e1, st);
  CNB_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  const double warps = (double)blocks * threads / 32.0;
  const double flops = warps * (double)iters * 8.0 * 512.0;
  out[0] = flops / (ms * 1e-3) / 1e12;
  return CNB_OK;
}

}  // extern "C"
