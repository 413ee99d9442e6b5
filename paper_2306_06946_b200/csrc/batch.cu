// Batched independent scenes (BASELINE configs[4]: many copies of the cfg0
// beam on their own tilted planes).  All copies share the mesh, the linear
// material and therefore one system matrix A and one factorisation; what
// differs per copy is the state, the plane, the friction coefficient and the
// contact set.  These kernels process every copy in one launch:
//
//   batch_detect_planes_kernel / batch_pairs_kernel  vertex-plane detection
//       (collision.py:264-287) with per-copy compaction in canonical order;
//   batch_wg_gather_kernel   W_g of every copy gathered from the inverse of the
//       shared, constant A (a vertex-plane row of S is a unit row);
//   batch_gemm_kernel        multi-RHS solves of all copies against that
//       inverse as one DMMA GEMM (formed once from the sparse factor);
//   batch_rebuild_w_kernel   W = D W_g D^T per copy, the bit-exact order of
//       rebuild_w_kernel (constraints.py:182-191);
//   batch_prox_kernel        p_a += h^2 W_g t per copy (constraints.py:217-244);
//   batch_spmv_kernel / batch_rhs_kernel   K x and the backward-Euler right-hand
//       side of every copy (dynamics.py:183-211);
//   batch_scatter_acc_kernel S^T acc of every copy (solver.py:250-257).
// The per-pair kernels (frames, violation, D^T lambda, re-linearisation) and
// PGS (pgs_batched_kernel, one CTA per copy) work on the concatenated pairs.
#include "common.cuh"

namespace cnb {

// scene owning flattened index x given exclusive prefix offsets off[0..ns] (ascending)
__device__ __forceinline__ int scene_of(const int64_t* __restrict__ off, int ns, int64_t x) {
  int a = 0, b = ns;
  while (b - a > 1) {
    const int m = (a + b) >> 1;
    if (off[m] <= x) a = m; else b = m;
  }
  return a;
}

// numpy's 1-D dot of length 3 (n @ p), bit for bit: a fused multiply-add chain
// fma(a2, b2, fma(a1, b1, a0 b0)) (measured against numpy 2.3 on this image).
__device__ __forceinline__ double ndot3(const double* a, const double* b) {
  return fma(a[2], b[2], fma(a[1], b[1], mul(a[0], b[0])));
}

// One CTA per scene: signed distance of every candidate vertex to the scene's
// plane, ordered compaction of the vertices with s <= threshold.
__global__ void __launch_bounds__(256) batch_detect_planes_kernel(int64_t nsurf, const int64_t* __restrict__ vids,
                                                                  const double* __restrict__ Q, int64_t ldq,
                                                                  const double* __restrict__ normals,
                                                                  const double* __restrict__ offsets, double thr,
                                                                  int32_t* __restrict__ count,
                                                                  int32_t* __restrict__ kept) {
  __shared__ int wsum[32];
  __shared__ int base;
  const int s = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double n[3] = {normals[3 * s], normals[3 * s + 1], normals[3 * s + 2]};
  const double off = offsets[s];
  const double* q = Q + (int64_t)s * ldq;
  if (tid == 0) base = 0;
  __syncthreads();
  for (int64_t k0 = 0; k0 < nsurf; k0 += blockDim.x) {
    const int64_t k = k0 + tid;
    bool hit = false;
    if (k < nsurf) {
      const int64_t v = vids[k];
      const double p[3] = {q[3 * v], q[3 * v + 1], q[3 * v + 2]};
      hit = sub(ndot3(n, p), off) <= thr;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int before = base;
    for (int w = 0; w < warp; ++w) before += wsum[w];
    if (hit) kept[(int64_t)s * nsurf + before + __popc(bal & ((1u << lane) - 1))] = (int32_t)k;
    __syncthreads();
    if (tid == 0) {
      int tot = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += wsum[w];
      base += tot;
    }
    __syncthreads();
  }
  if (tid == 0) count[s] = base;
}

// Pair records of every scene at its offset: candidate index, p_a (vertex),
// p_b = foot point, reference normal (collision.py:264-287).
__global__ void batch_pairs_kernel(int ns, int64_t nsurf, const int64_t* __restrict__ poff,
                                   const int32_t* __restrict__ kept, const int64_t* __restrict__ vids,
                                   const double* __restrict__ Q, int64_t ldq, const double* __restrict__ normals,
                                   const double* __restrict__ offsets, int32_t* __restrict__ pscene,
                                   int32_t* __restrict__ pcand, double* __restrict__ pa, double* __restrict__ pb,
                                   double* __restrict__ ref, double* __restrict__ sdist) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= poff[ns]) return;
  const int s = scene_of(poff, ns, i);
  const int32_t k = kept[(int64_t)s * nsurf + (i - poff[s])];
  const int64_t v = vids[k];
  const double n[3] = {normals[3 * s], normals[3 * s + 1], normals[3 * s + 2]};
  const double* q = Q + (int64_t)s * ldq;
  const double p[3] = {q[3 * v], q[3 * v + 1], q[3 * v + 2]};
  const double d = sub(ndot3(n, p), offsets[s]);
  pscene[i] = s;
  pcand[i] = k;
  sdist[i] = d;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    pa[3 * i + a] = p[a];
    pb[3 * i + a] = sub(p[a], mul(d, n[a]));  // foot = p - signed * n
    ref[3 * i + a] = n[a];
  }
}

// p_a of every pair from the scene's node positions (vertex attachments).
__global__ void batch_gather_pa_kernel(int64_t m, const int32_t* __restrict__ pscene, const int32_t* __restrict__ pcand,
                                       const int64_t* __restrict__ vids, const double* __restrict__ Q, int64_t ldq,
                                       double* __restrict__ pa) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double* q = Q + (int64_t)pscene[i] * ldq + 3 * vids[pcand[i]];
#pragma unroll
  for (int a = 0; a < 3; ++a) pa[3 * i + a] = q[a];
}

// Signed distance of surface vertices to a plane, the reference's own float(n @ p
// - offset) (collision.py:264-270) bit for bit (ndot3 above).
__global__ void plane_distances_kernel(int64_t nv, const int64_t* __restrict__ vids, const double* __restrict__ P,
                                       double n0, double n1, double n2, double offset, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nv) return;
  const double* p = P + 3 * vids[i];
  const double n[3] = {n0, n1, n2};
  const double q[3] = {p[0], p[1], p[2]};
  out[i] = sub(ndot3(n, q), offset);
}

// W_g of every scene (packed at woff[s], c_s x c_s, c_s = 3 m_s, row stride
// c_s rounded up to even so rows are 16-byte aligned): block (I, J)
// = Ainv[3 v_I .., 3 v_J ..] (vertex rows of S are unit rows, A is shared:
// S A^-1 S^T is a gather from the inverse).  Thread per 3x3 block, flattened
// over scenes with the block prefix boff (m_s^2).
__global__ void batch_wg_gather_kernel(int ns, const int64_t* __restrict__ boff, const int64_t* __restrict__ poff,
                                       const int64_t* __restrict__ woff, const int32_t* __restrict__ pcand,
                                       const int64_t* __restrict__ vids, const double* __restrict__ C, int64_t ldc,
                                       double* __restrict__ Wg) {
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= boff[ns]) return;
  const int s = scene_of(boff, ns, x);
  const int64_t ms = poff[s + 1] - poff[s], loc = x - boff[s];
  const int64_t I = loc / ms, J = loc - I * ms;
  const int64_t ki = vids[pcand[poff[s] + I]], kj = vids[pcand[poff[s] + J]];
  const int64_t c = 3 * ms + (ms & 1);  // even row stride
  double* w = Wg + woff[s] + (3 * I) * c + 3 * J;
  const double* src = C + (3 * ki) * ldc + 3 * kj;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) w[a * c + b] = src[a * ldc + b];
}

// W = D W_g D^T per scene, same operation order as rebuild_w_kernel.
__global__ void batch_rebuild_w_kernel(int ns, const int64_t* __restrict__ boff, const int64_t* __restrict__ poff,
                                       const int64_t* __restrict__ woff, const double* __restrict__ D,
                                       const double* __restrict__ Wg, double* __restrict__ W) {
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= boff[ns]) return;
  const int s = scene_of(boff, ns, x);
  const int64_t ms = poff[s + 1] - poff[s], loc = x - boff[s];
  const int64_t I = loc / ms, J = loc - I * ms;
  const int64_t c = 3 * ms + (ms & 1);  // even row stride
  double DI[9], DJ[9], G[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) DI[e] = __ldg(D + 9 * (poff[s] + I) + e);
#pragma unroll
  for (int e = 0; e < 9; ++e) DJ[e] = __ldg(D + 9 * (poff[s] + J) + e);
  const double* src = Wg + woff[s] + (3 * I) * c + 3 * J;
#pragma unroll
  for (int l = 0; l < 3; ++l)
#pragma unroll
    for (int k = 0; k < 3; ++k) G[3 * l + k] = src[l * c + k];
  double T[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double v = mul(DI[3 * a + 0], G[0 * 3 + k]);
      v = add(v, mul(DI[3 * a + 1], G[1 * 3 + k]));
      v = add(v, mul(DI[3 * a + 2], G[2 * 3 + k]));
      T[3 * a + k] = v;
    }
  double* dst = W + woff[s] + (3 * I) * c + 3 * J;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      double v = mul(T[3 * a + 0], DJ[3 * b + 0]);
      v = add(v, mul(T[3 * a + 1], DJ[3 * b + 1]));
      v = add(v, mul(T[3 * a + 2], DJ[3 * b + 2]));
      dst[a * c + b] = v;
    }
}

// p_a += h^2 W_g t per scene (side A vertices; the plane side carries no DoFs).
// Warp per constraint row, lane-strided sums + butterfly (deterministic).
__global__ void __launch_bounds__(256) batch_prox_kernel(int ns, const int64_t* __restrict__ poff,
                                                         const int64_t* __restrict__ woff,
                                                         const double* __restrict__ Wg, const double* __restrict__ t,
                                                         double h2, double* __restrict__ pa) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= 3 * poff[ns]) return;
  const int s = scene_of(poff, ns, r / 3);
  const int64_t ms = poff[s + 1] - poff[s], c = 3 * ms, lr = r - 3 * poff[s];
  const double* row = Wg + woff[s] + lr * (c + (ms & 1));
  const double* ts = t + 3 * poff[s];
  double v = 0.0;
  for (int64_t j = lane; j < c; j += 32) v = fma(row[j], ts[j], v);
  v = warp_sum(v);
  if (lane == 0) pa[r] = add(pa[r], mul(h2, v));
}

// y[s][r] = sum_e K[r][e] x[s][col_e], the summation order of csr_spmv_kernel.
__global__ void batch_spmv_kernel(int ns, int64_t n, const int64_t* __restrict__ rp, const int64_t* __restrict__ ci,
                                  const double* __restrict__ va, const double* __restrict__ x, int64_t ldx,
                                  double* __restrict__ y, int64_t ldy) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)ns * n) return;
  const int64_t s = id / n, r = id - s * n;
  const double* xs = x + s * ldx;
  double v = 0.0;
  for (int64_t e = rp[r]; e < rp[r + 1]; ++e) v = fma(va[e], xs[ci[e]], v);
  y[s * ldy + r] = v;
}

// backward-Euler right-hand side of every scene (system_rhs_kernel per column)
__global__ void batch_rhs_kernel(int ns, int64_t n, const double* __restrict__ fel, const double* __restrict__ Kv,
                                 const double* __restrict__ m3, const double* __restrict__ v,
                                 const double* __restrict__ fext, const int8_t* __restrict__ fixed, double h,
                                 double alpha, double beta, double* __restrict__ b, DevStatus* st) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)ns * n) return;
  const int64_t r = id % n;
  const double f = fel[id] + alpha * (m3[r] * v[id]) + beta * Kv[id];
  double val = h * (fext[r] - f) - h * h * Kv[id];
  if (fixed[r]) val = 0.0;
  if (!isfinite(val)) raise_status(st, CNB_E_NONFINITE, (int)r, val);
  b[id] = val;
}

// rhs[s][3 v + a] = acc[3 i + a] for pair i of scene s (vertex v; rows of S are
// unit rows, one pair per vertex and scene): S^T acc per scene.
__global__ void batch_scatter_acc_kernel(int64_t m, const int32_t* __restrict__ pscene,
                                         const int32_t* __restrict__ pcand, const int64_t* __restrict__ vids,
                                         const double* __restrict__ acc, double* __restrict__ rhs, int64_t ldr) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double* r = rhs + (int64_t)pscene[i] * ldr + 3 * vids[pcand[i]];
#pragma unroll
  for (int a = 0; a < 3; ++a) r[a] = acc[3 * i + a];
}

// C (M x N) = A (M x K) B (K x N), row-major, fp64 tensor cores (DMMA): the
// multi-right-hand-side solves of the batched scenes against the shared
// inverse (X = B A^-1, A symmetric).  64 x 64 tiles, K staged in 32-wide
// chunks with cp.async double buffering, 4 warps x (32 x 32).
constexpr int kBT = 64, kBK = 32, kBS = kBK + 4;  // smem stride == 4 mod 16: conflict-free fragments
__global__ void __launch_bounds__(128) batch_gemm_kernel(int64_t M, int64_t N, int64_t K,
                                                         const double* __restrict__ A, int64_t lda,
                                                         const double* __restrict__ B, int64_t ldb,
                                                         double* __restrict__ C, int64_t ldc) {
  extern __shared__ __align__(16) double gsm[];
  double (*As)[kBT * kBS] = reinterpret_cast<double (*)[kBT * kBS]>(gsm);                   // [2][row][k]
  double (*Bs)[kBT * kBS] = reinterpret_cast<double (*)[kBT * kBS]>(gsm + 2 * kBT * kBS);  // [2][col][k]
  const int64_t r0 = (int64_t)blockIdx.y * kBT, c0 = (int64_t)blockIdx.x * kBT;
  auto stage = [&](int buf, int64_t k0) {
    for (int e = threadIdx.x; e < kBT * kBK; e += blockDim.x) {
      const int kk = e % kBK, rr = e / kBK;
      const int64_t r = r0 + rr, k = k0 + kk;
      cp_async8(&As[buf][rr * kBS + kk], A + r * lda + k, r < M && k < K);
    }
    for (int e = threadIdx.x; e < kBT * kBK; e += blockDim.x) {
      const int cc = e % kBT, kk = e / kBT;
      const int64_t c = c0 + cc, k = k0 + kk;
      cp_async8(&Bs[buf][cc * kBS + kk], B + k * ldb + c, c < N && k < K);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wy = (warp >> 1) * 32, wx = (warp & 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int nk = (int)((K + kBK - 1) / kBK);
  stage(0, 0);
  for (int ck = 0; ck < nk; ++ck) {
    if (ck + 1 < nk) {
      stage((ck + 1) & 1, (int64_t)(ck + 1) * kBK);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const double* Ab = As[ck & 1];
    const double* Bb = Bs[ck & 1];
#pragma unroll
    for (int kk = 0; kk < kBK; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) fa[a] = Ab[(wy + 8 * a + g) * kBS + kk + t];
#pragma unroll
      for (int b = 0; b < 4; ++b) fb[b] = Bb[(wx + 8 * b + g) * kBS + kk + t];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int64_t r = r0 + wy + 8 * a + g, c = c0 + wx + 8 * b + 2 * t + hh;
        if (r < M && c < N) C[r * ldc + c] = acc[a][b][hh];
      }
}

}  // namespace cnb

using namespace cnb;

extern "C" {

int cnb_plane_distances(int64_t nv, const int64_t* vids, const double* pts, double n0, double n1, double n2,
                        double offset, double* out, void* stream) {
  if (nv <= 0) return CNB_OK;
  plane_distances_kernel<<<grid_for(nv, 256), 256, 0, (cudaStream_t)stream>>>(nv, vids, pts, n0, n1, n2, offset, out);
  CNB_LAUNCH_CHECK("plane_distances_kernel");
  return CNB_OK;
}

int cnb_batch_detect_planes(int32_t ns, int64_t nsurf, const int64_t* vids, const double* Q, int64_t ldq,
                            const double* normals, const double* offsets, double threshold, int32_t* count,
                            int32_t* kept, void* stream) {
  if (ns <= 0 || nsurf <= 0) return CNB_OK;
  batch_detect_planes_kernel<<<ns, 256, 0, (cudaStream_t)stream>>>(nsurf, vids, Q, ldq, normals, offsets, threshold,
                                                                   count, kept);
  CNB_LAUNCH_CHECK("batch_detect_planes_kernel");
  return CNB_OK;
}

int cnb_batch_pairs(int32_t ns, int64_t m, int64_t nsurf, const int64_t* poff, const int32_t* kept,
                    const int64_t* vids, const double* Q, int64_t ldq, const double* normals, const double* offsets,
                    int32_t* pscene, int32_t* pcand, double* pa, double* pb, double* ref, double* sdist,
                    void* stream) {
  if (m <= 0) return CNB_OK;
  batch_pairs_kernel<<<grid_for(m, 128), 128, 0, (cudaStream_t)stream>>>(ns, nsurf, poff, kept, vids, Q, ldq, normals,
                                                                         offsets, pscene, pcand, pa, pb, ref, sdist);
  CNB_LAUNCH_CHECK("batch_pairs_kernel");
  return CNB_OK;
}

int cnb_batch_gather_pa(int64_t m, const int32_t* pscene, const int32_t* pcand, const int64_t* vids, const double* Q,
                        int64_t ldq, double* pa, void* stream) {
  if (m <= 0) return CNB_OK;
  batch_gather_pa_kernel<<<grid_for(m, 128), 128, 0, (cudaStream_t)stream>>>(m, pscene, pcand, vids, Q, ldq, pa);
  CNB_LAUNCH_CHECK("batch_gather_pa_kernel");
  return CNB_OK;
}

int cnb_batch_wg_gather(int32_t ns, int64_t nblocks, const int64_t* boff, const int64_t* poff, const int64_t* woff,
                        const int32_t* pcand, const int64_t* vids, const double* C, int64_t ldc, double* Wg,
                        void* stream) {
  if (nblocks <= 0) return CNB_OK;
  batch_wg_gather_kernel<<<grid_for(nblocks, 256), 256, 0, (cudaStream_t)stream>>>(ns, boff, poff, woff, pcand, vids,
                                                                                   C, ldc, Wg);
  CNB_LAUNCH_CHECK("batch_wg_gather_kernel");
  return CNB_OK;
}

int cnb_batch_rebuild_w(int32_t ns, int64_t nblocks, const int64_t* boff, const int64_t* poff, const int64_t* woff,
                        const double* D, const double* Wg, double* W, void* stream) {
  if (nblocks <= 0) return CNB_OK;
  batch_rebuild_w_kernel<<<grid_for(nblocks, 256), 256, 0, (cudaStream_t)stream>>>(ns, boff, poff, woff, D, Wg, W);
  CNB_LAUNCH_CHECK("batch_rebuild_w_kernel");
  return CNB_OK;
}

int cnb_batch_prox(int32_t ns, int64_t m, const int64_t* poff, const int64_t* woff, const double* Wg, const double* t,
                   double h, double* pa, void* stream) {
  if (m <= 0) return CNB_OK;
  batch_prox_kernel<<<grid_for(3 * m * 32, 256), 256, 0, (cudaStream_t)stream>>>(ns, poff, woff, Wg, t, h * h, pa);
  CNB_LAUNCH_CHECK("batch_prox_kernel");
  return CNB_OK;
}

int cnb_gemm_dense(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B, int64_t ldb,
                   double* C, int64_t ldc, void* stream) {
  if (M <= 0 || N <= 0) return CNB_OK;
  dim3 grid((unsigned)((N + kBT - 1) / kBT), (unsigned)((M + kBT - 1) / kBT));
  const int smem = (int)(4 * kBT * kBS * sizeof(double));
  CNB_CUDA(cudaFuncSetAttribute(batch_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  batch_gemm_kernel<<<grid, 128, smem, (cudaStream_t)stream>>>(M, N, K, A, lda, B, ldb, C, ldc);
  CNB_LAUNCH_CHECK("batch_gemm_kernel");
  return CNB_OK;
}

int cnb_batch_spmv(int32_t ns, int64_t n, const int64_t* rowptr, const int64_t* col, const double* val,
                   const double* x, int64_t ldx, double* y, int64_t ldy, void* stream) {
  if (ns <= 0 || n <= 0) return CNB_OK;
  batch_spmv_kernel<<<grid_for((int64_t)ns * n, 128), 128, 0, (cudaStream_t)stream>>>(ns, n, rowptr, col, val, x, ldx,
                                                                                      y, ldy);
  CNB_LAUNCH_CHECK("batch_spmv_kernel");
  return CNB_OK;
}

int cnb_batch_rhs(int32_t ns, int64_t n, const double* fel, const double* Kv, const double* m3, const double* v,
                  const double* fext, const int8_t* fixed, double h, double alpha, double beta, double* b,
                  cnb_status_t* d_status, void* stream) {
  if (ns <= 0 || n <= 0) return CNB_OK;
  batch_rhs_kernel<<<grid_for((int64_t)ns * n, 128), 128, 0, (cudaStream_t)stream>>>(
      ns, n, fel, Kv, m3, v, fext, fixed, h, alpha, beta, b, (DevStatus*)d_status);
  CNB_LAUNCH_CHECK("batch_rhs_kernel");
  return CNB_OK;
}

int cnb_batch_scatter_acc(int64_t m, const int32_t* pscene, const int32_t* pcand, const int64_t* vids,
                          const double* acc, double* rhs, int64_t ldr, void* stream) {
  if (m <= 0) return CNB_OK;
  batch_scatter_acc_kernel<<<grid_for(m, 128), 128, 0, (cudaStream_t)stream>>>(m, pscene, pcand, vids, acc, rhs, ldr);
  CNB_LAUNCH_CHECK("batch_scatter_acc_kernel");
  return CNB_OK;
}

}  // extern "C"
