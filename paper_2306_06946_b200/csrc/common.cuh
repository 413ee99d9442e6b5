// Shared helpers for the B200 (sm_100a) contact-solver kernels.
//
// Status codes mirror the reference's exception classes
// (/root/reference/pkg/src/contactnewton/errors.py); the Python layer maps
// them back onto the same class names.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "../../include/cn_b200.h"

namespace cnb {

void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);

#define CNB_CUDA(call)                                                         \
  do {                                                                         \
    cudaError_t _e = (call);                                                   \
    if (_e != cudaSuccess) return ::cnb::cuda_status(_e, #call);               \
  } while (0)

// Every kernel launch is followed by this check; it also counts launches
// (cnb_launch_count) so benchmarks report how many of our kernels ran.
void count_launch();
void add_launches(long long n);
long long launch_count();
bool use_graphs();
#define CNB_LAUNCH_CHECK(where)                                                \
  do {                                                                         \
    ::cnb::count_launch();                                                     \
    cudaError_t _e = cudaGetLastError();                                       \
    if (_e != cudaSuccess) return ::cnb::cuda_status(_e, where);               \
  } while (0)

// IEEE round-to-nearest arithmetic without FMA contraction.  The reference
// evaluates products and sums through numpy temporaries (a*b rounded, then
// the add rounded), so kernels whose output is compared bit-for-bit use
// these instead of the contracting operators.
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// Device-side status word: kernels record the first failure here and the
// host reads it back when it synchronises for scalar outputs.
struct DevStatus {
  int code;     // CNB_OK or one of the CNB_E_* values
  int index;    // offending group / pivot / pair
  double value; // offending value (pivot, W_nn, determinant)
};

__device__ __forceinline__ void raise_status(DevStatus* st, int code, int index, double value) {
  if (st && atomicCAS(&st->code, 0, code) == 0) {
    st->index = index;
    st->value = value;
  }
}

inline int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > (1 << 30)) g = 1 << 30;
  return (int)g;
}

// fp64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col).  Lowers to
// SASS DMMA.8x8x4 on sm_100a (tcgen05 has no f64 kind).
// Fragment layout (lane = 4*g + t): a = A[g][t], b = B[t][g],
// c0,c1 = C[g][2t], C[g][2t+1].
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Asynchronous global -> shared copy of one fp64 (LDGSTS): the warp keeps
// issuing instead of waiting for each load before its shared store.
// pred == false zero-fills the destination without touching src.
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n)
               : "memory");
}
// L1-bypassing (L2-coherent) asynchronous copy of 16 bytes, for data other
// SMs rewrite while the kernel runs.  Both addresses 16-byte aligned.
__device__ __forceinline__ void cp_async16_cg(double* smem, const double* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
// n doubles gmem -> smem through L2 only (16-byte chunks + an odd tail);
// threads [0, nt) of the caller's numbering participate with index k.
__device__ __forceinline__ void copy_cg(double* smem, const double* gmem, int n, int k, int nt) {
  for (int e = k; 2 * e + 1 < n; e += nt) cp_async16_cg(smem + 2 * e, gmem + 2 * e);
  if ((n & 1) && k == 0) smem[n - 1] = __ldcg(gmem + n - 1);
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// ---- mbarrier + TMA bulk copies (cp.async.bulk, sm_90+) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// order earlier generic-proxy accesses of shared memory before later async-proxy (TMA) writes
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
// 2-D tiled tensor copy (TMA): box at (x = column, y = row) of the tensor map
// into dense shared memory (128-byte aligned), completion counted on bar.
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int x, int y, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];\n" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
// global -> shared bulk copy (TMA engine), completion counted on bar in bytes.
// dst, src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Device scratch that only grows (reused across calls on one stream).
struct GrowBuf {
  void* p = nullptr;
  size_t cap = 0;
  int ensure(size_t bytes) {
    if (bytes <= cap) return CNB_OK;
    release();
    CNB_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
    cap = std::max<size_t>(bytes, 256);
    return CNB_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Pinned host staging for per-call uploads: cudaMemcpyAsync from pageable
// memory synchronises the stream first, which would serialise the host-side
// planning of one object with the GPU work of the previous one.  `ready`
// guards reuse: the previous upload from this buffer must have executed.
struct PinnedBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaEvent_t ready = nullptr;
  int ensure(size_t bytes) {
    if (ready) CNB_CUDA(cudaEventSynchronize(ready));
    if (bytes <= cap) return CNB_OK;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    CNB_CUDA(cudaMallocHost(&p, std::max<size_t>(bytes, 4096)));
    cap = std::max<size_t>(bytes, 4096);
    return CNB_OK;
  }
  int mark(cudaStream_t st) {
    if (!ready) CNB_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    CNB_CUDA(cudaEventRecord(ready, st));
    return CNB_OK;
  }
  void release() {
    if (ready) {
      cudaEventSynchronize(ready);
      cudaEventDestroy(ready);
    }
    if (p) cudaFreeHost(p);
    p = nullptr;
    ready = nullptr;
    cap = 0;
  }
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace cnb
