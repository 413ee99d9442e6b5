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

}  // namespace cnb

using namespace cnb;

extern "C" {

// out (host, 9 doubles): cycles per dependent op, see latency_kernel.
int cnb_bench_latency(double* out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  double* d = nullptr;
  long long* c = nullptr;
  CNB_CUDA(cudaMalloc(&d, sizeof(double)));
  CNB_CUDA(cudaMalloc(&c, 9 * sizeof(long long)));
  const int n = 4096;
  latency_kernel<<<1, 32, 0, st>>>(n, 1.5, d, c);
  CNB_LAUNCH_CHECK("latency_kernel");
  long long h[9];
  CNB_CUDA(cudaMemcpyAsync(h, c, sizeof(h), cudaMemcpyDeviceToHost, st));
  CNB_CUDA(cudaStreamSynchronize(st));
  for (int k = 0; k < 9; ++k) out[k] = (double)h[k] / n;
  cudaFree(d);
  cudaFree(c);
  return CNB_OK;
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
