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

}  // namespace cnb

using namespace cnb;

extern "C" {

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
