// GPU numeric factorisation of the supernodal multifrontal Cholesky.
//
// Reference being replaced: Factorization (linalg.py:58-106) — SuperLU
// factorisation.  NotSPD is raised for a non-positive (or NaN) pivot exactly
// where the reference checks U's diagonal (linalg.py:77-84).
//
// Level by level of the supernodal tree (leaves first):
//   scatter A into the fronts (once) -> extend-add children's update blocks
//   (parent-column-owner tasks, children visited in order: deterministic, no
//   atomics) -> dense partial Cholesky of every front of the level:
//   per 32-column panel: POTRF (one CTA per front), TRSM (64-row chunks),
//   SYRK trailing update on 64x64 tiles with fp64 tensor-core MMA
//   (mma.sync m8n8k4 f64 -> SASS DMMA; tcgen05 has no f64 kind)
//   -> inversion of every diagonal block L11 (solve.cu: trinv), so that all
//   later triangular solves are GEMV / GEMM over [L11^{-1}; L21].
#include <cstdio>
#include <cstring>
#include <map>
#include <numeric>
#include <stdexcept>
#include <string>

#include "chol_dev.cuh"

// SYRK tile kernel: k depth of a staged chunk (16: a short prologue and two
// double-buffered chunks even for the rank-32 in-block updates; measured 62.6 ->
// 60.4 ms per cfg3 factor against 32) and the CTAs per SM it is compiled for
// (3: the fused POTRF's registers stay unspilled)
#ifndef SYRK_BK
#define SYRK_BK 16
#endif
#ifndef SYRK_MINB
#define SYRK_MINB 3
#endif

namespace cnb {

__global__ void scatter_kernel(int64_t nmap, const int64_t* __restrict__ src, const int64_t* __restrict__ dst,
                               const double* __restrict__ vals, double* __restrict__ front) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nmap) front[dst[k]] = vals[src[k]];
}

// extend-add: task = (parent p, parent col range [lo, hi), offset of the
// children's row ranges).  For every child c of p (ascending) and every child
// update column k whose parent column rel[k] lies in [lo, hi) -- the range
// [k0, k1) comes precomputed with the symbolic analysis (no binary searches
// on the dependent-load chain) -- F_p[rel[i], rel[k]] += U_c[i, k], i >= k.
// Rows are processed in batches of kEaBatch per thread: all loads of a batch
// are issued before its stores (the parent and child fronts live in one
// buffer, so the compiler could not reorder them otherwise).
constexpr int kEaBatch = 4;
__global__ void __launch_bounds__(256, 4) extend_add_kernel(DevSym S, const int32_t* __restrict__ tasks,
                                                         const int32_t* __restrict__ rng, double* __restrict__ front) {
  const int32_t p = tasks[4 * blockIdx.x];
  const int32_t* kr = rng + 2 * tasks[4 * blockIdx.x + 3];
  const int64_t ldp = d_ldf(S, p);
  double* Fp = front + S.front_off[p];
  for (int64_t ci = S.child_ptr[p]; ci < S.child_ptr[p + 1]; ++ci) {
    const int64_t c = S.child[ci];
    const int64_t ncc = d_nc(S, c), nrc = d_nr(S, c), ldc = d_ldf(S, c);
    const int32_t* __restrict__ rel = S.rel + S.rel_ptr[c];
    const int64_t k0 = kr[2 * (ci - S.child_ptr[p])], k1 = kr[2 * (ci - S.child_ptr[p]) + 1];
    const double* Fc = front + S.front_off[c];
    if (nrc - k0 >= (int64_t)kEaBatch * blockDim.x) {
      // long columns: one column at a time, full batches
      for (int64_t k = k0; k < k1; ++k) {
        const double* __restrict__ uc = Fc + (ncc + k) * ldc + ncc;
        double* fcol = Fp + (int64_t)rel[k] * ldp;
        for (int64_t i0 = k + threadIdx.x; i0 < nrc; i0 += (int64_t)kEaBatch * blockDim.x) {
          int32_t ri[kEaBatch];
          double u[kEaBatch], v[kEaBatch];
#pragma unroll
          for (int q = 0; q < kEaBatch; ++q) {
            const int64_t i = i0 + (int64_t)q * blockDim.x;
            ri[q] = i < nrc ? __ldg(rel + i) : -1;
            u[q] = i < nrc ? uc[i] : 0.0;
          }
#pragma unroll
          for (int q = 0; q < kEaBatch; ++q) v[q] = ri[q] >= 0 ? fcol[ri[q]] : 0.0;
#pragma unroll
          for (int q = 0; q < kEaBatch; ++q)
            if (ri[q] >= 0) fcol[ri[q]] = v[q] + u[q];
        }
      }
    } else {
      // short columns: the (column k, row i >= k) elements of the <= kEaCols
      // columns flattened, so a batch of loads spans columns
      int32_t off[kEaCols + 1];
      off[0] = 0;
#pragma unroll
      for (int q = 0; q < kEaCols; ++q) off[q + 1] = off[q] + (k0 + q < k1 ? (int32_t)(nrc - (k0 + q)) : 0);
      const int32_t tot = off[kEaCols];
      for (int32_t e0 = threadIdx.x; e0 < tot; e0 += kEaBatch * (int32_t)blockDim.x) {
        int32_t ri[kEaBatch], cj[kEaBatch];
        double u[kEaBatch], v[kEaBatch];
#pragma unroll
        for (int q = 0; q < kEaBatch; ++q) {
          const int32_t e = e0 + q * (int32_t)blockDim.x;
          int kk = 0;
          int32_t base = 0;  // (compile-time indices only: off stays in registers)
#pragma unroll
          for (int m = 1; m < kEaCols; ++m) {
            kk += e >= off[m] ? 1 : 0;
            base = e >= off[m] ? off[m] : base;
          }
          const int64_t k = k0 + kk, i = k + (e - base);
          const bool in = e < tot;
          ri[q] = in ? __ldg(rel + i) : -1;
          cj[q] = in ? __ldg(rel + k) : 0;
          u[q] = in ? Fc[(ncc + k) * ldc + ncc + i] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < kEaBatch; ++q) v[q] = ri[q] >= 0 ? Fp[(int64_t)cj[q] * ldp + ri[q]] : 0.0;
#pragma unroll
        for (int q = 0; q < kEaBatch; ++q)
          if (ri[q] >= 0) Fp[(int64_t)cj[q] * ldp + ri[q]] = v[q] + u[q];
      }
    }
    __syncthreads();
  }
}

// diagnostic: cycle sums of potrf phases (loads, factor + inverse) and calls, cnb_potrf_profile
__device__ unsigned long long g_potrf_prof[8];

// POTRF of the kw x kw diagonal block of panel k0 and the inverse of the
// resulting L_kk (kept in kkinv slot kk_off[s] + panel, 32 x 32 row-major, for
// the TRSM and the inversion of L11 (solve.cu trinv_kernel); the TRSM then is a
// plain DMMA product).  Two warps (threads 0..63 of the CTA); rows / columns
// >= kw are padded with the identity.
//
// Warp 0 factors.  Lane i keeps row i in registers as a shift register: before
// elimination step j, a[q] holds column j + q, so every step touches the same
// compile-time register names (a runtime-indexed register array would spill to
// local memory, and unrolling the 32 steps thrashes the instruction cache).
// Step j: lane i scales its l_ij, column j of L goes to shared memory, and
// a[q] <- a[q + 1] - l_ij l_(j+1+q),j for the columns that still exist (the
// steps run in four phases of decreasing width).  Only the next pivot is on
// the sequential chain, and lane j + 1 forms it from its own l_(j+1),j:
// broadcast, rsqrt, scale -- placed between the bulk multiply-adds in program
// order so that in-order issue overlaps them.  Columns are read as 16-byte
// pairs (row j of the scratch is offset so that element j + 1 is aligned).
// L goes back to the front after the loop: a global store inside it would make
// every step's release (a CTA memory barrier) wait for the store's completion.
// Warp 1 forms Y = L^{-1} (lane c owns column c, shift register u = rows j + q)
// from the published columns, one step behind (a shared-memory flag per step).
// Fused multiply-adds in the order of the step-by-step definition.
// cols: kPanel rows of 2 kPanel doubles (column j of L, rows >= 32 zero), then
// kPanel reciprocal pivots, then the step flag.
constexpr int kPotrfSmem = (2 * kPanel * kPanel + kPanel + 2) * (int)sizeof(double);
__device__ __forceinline__ double* potrf_col(double* cols, int j) { return cols + j * (2 * kPanel) + ((j + 1) & 1); }

// one elimination step with QN live columns after the pivot: returns the next
// pivot's inverse square root through (d, inv)
template <int QN>
__device__ __forceinline__ void potrf_step(double (&a)[kPanel], int j, int i, int kw, double* cols, double* rd,
                                           unsigned flag_s, double& d, double& inv, int& bad, double& bad_d) {
  double* col = potrf_col(cols, j);
  const bool fail = bad < 0 && j < kw && !(d > 0.0);
  bad = fail ? j : bad;
  bad_d = fail ? d : bad_d;
  const double lij = (i == j ? d : a[0]) * inv;  // rows above j: never read
  col[i] = lij;
  if (i == 0) rd[j] = inv;
  __syncwarp();
  if (i == 0) asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(flag_s), "r"(j + 1) : "memory");
  d = __shfl_sync(0xffffffffu, fma(-lij, lij, a[1]), (j + 1) & 31);
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  const double hd = -0.5 * d;
  const double2* c2 = reinterpret_cast<const double2*>(col + j + 1);
#pragma unroll
  for (int q0 = 0; q0 < QN; q0 += 8) {
    double lk[8];
#pragma unroll
    for (int v = 0; v < 8; v += 2)
      if (q0 + v < QN) {
        const double2 t = c2[(q0 + v) / 2];
        lk[v] = t.x;
        lk[v + 1] = t.y;
      }
#pragma unroll
    for (int v = 0; v < 8; ++v)
      if (q0 + v < QN) a[q0 + v] = fma(-lij, lk[v], a[q0 + v + 1]);
    if (q0 == 0 || q0 == (QN > 16 ? 16 : 8)) r = r * fma(hd, r * r, 1.5);
  }
  if (QN <= 8) r = r * fma(hd, r * r, 1.5);  // (one bulk chunk only)
  inv = d > 0.0 ? r : __longlong_as_double(0x7ff8000000000000LL);
}

template <int QN>
__device__ __forceinline__ void inverse_step(double (&u)[kPanel], int j, int i, const double* cols, const double* rd,
                                             unsigned flag_s, double* Y) {
  for (;;) {  // acquire: the column's stores are visible once its flag is
    int v;
    asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(flag_s) : "memory");
    if (v > j) break;
  }
  const double* col = potrf_col(const_cast<double*>(cols), j);
  const double yj = u[0] * rd[j];  // (L^{-1})[j][i]
  Y[j * kPanel + i] = yj;
  const double2* c2 = reinterpret_cast<const double2*>(col + j + 1);
#pragma unroll
  for (int q0 = 0; q0 < QN; q0 += 8) {
    double lk[8];
#pragma unroll
    for (int v = 0; v < 8; v += 2)
      if (q0 + v < QN) {
        const double2 t = c2[(q0 + v) / 2];
        lk[v] = t.x;
        lk[v + 1] = t.y;
      }
#pragma unroll
    for (int v = 0; v < 8; ++v)
      if (q0 + v < QN) u[q0 + v] = fma(-lk[v], yj, u[q0 + v + 1]);
  }
}

__device__ __noinline__ void potrf_panel(const DevSym& S, int64_t s, int k0, double* __restrict__ front,
                                         double* __restrict__ kkinv, DevStatus* st, double* __restrict__ cols) {
  const int64_t nc = d_nc(S, s), ldf = d_ldf(S, s);
  const int kw = (int)min((int64_t)kPanel, nc - k0);
  double* rd = cols + 2 * kPanel * kPanel;
  const unsigned flag_s = smem_u32(rd + kPanel);
  const int i = threadIdx.x & 31, w = (threadIdx.x >> 5) & 1;
  for (int e = threadIdx.x & 63; e < 2 * kPanel * kPanel; e += 64) cols[e] = 0.0;
  if (threadIdx.x == 0) *reinterpret_cast<int*>(rd + kPanel) = 0;
  asm volatile("bar.sync 1, 64;" ::: "memory");
  if (w == 1) {  // ---- inverse ----
    double* Y = kkinv + (S.kk_off[s] + k0 / kPanel) * (kPanel * kPanel);
    double u[kPanel];
#pragma unroll
    for (int l = 0; l < kPanel; ++l) u[l] = l == i ? 1.0 : 0.0;
    int j = 0;
    for (; j < 8; ++j) inverse_step<31>(u, j, i, cols, rd, flag_s, Y);
    for (; j < 16; ++j) inverse_step<23>(u, j, i, cols, rd, flag_s, Y);
    for (; j < 24; ++j) inverse_step<15>(u, j, i, cols, rd, flag_s, Y);
    for (; j < 32; ++j) inverse_step<7>(u, j, i, cols, rd, flag_s, Y);
    return;
  }
  // ---- factor ----
  double* F = front + S.front_off[s] + (int64_t)k0 * ldf + k0;
  long long ts[3];
  ts[0] = clock64();
  double a[kPanel];
#pragma unroll
  for (int l = 0; l < kPanel; ++l)
    a[l] = (i < kw && l < kw && l <= i) ? F[(int64_t)l * ldf + i] : (l == i ? 1.0 : 0.0);
  ts[1] = clock64();
  double d = __shfl_sync(0xffffffffu, a[0], 0);
  double inv;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(inv) : "d"(d));
  inv = inv * fma(-0.5 * d, inv * inv, 1.5);
  inv = inv * fma(-0.5 * d, inv * inv, 1.5);
  inv = d > 0.0 ? inv : __longlong_as_double(0x7ff8000000000000LL);
  int bad = -1;
  double bad_d = 0.0;
  int j = 0;
  for (; j < 8; ++j) potrf_step<31>(a, j, i, kw, cols, rd, flag_s, d, inv, bad, bad_d);
  for (; j < 16; ++j) potrf_step<23>(a, j, i, kw, cols, rd, flag_s, d, inv, bad, bad_d);
  for (; j < 24; ++j) potrf_step<15>(a, j, i, kw, cols, rd, flag_s, d, inv, bad, bad_d);
  for (; j < 32; ++j) potrf_step<7>(a, j, i, kw, cols, rd, flag_s, d, inv, bad, bad_d);
  ts[2] = clock64();
  // L back into the front (a store inside the loop would make every step's
  // release fence wait for it): lane i writes row i, column by column
#pragma unroll 1
  for (int l = 0; l < kw; ++l)
    if (i >= l && i < kw) F[(int64_t)l * ldf + i] = potrf_col(cols, l)[i];
  if (bad >= 0 && i == 0) raise_status(st, CNB_E_NOT_SPD, (int)(S.first[s] + k0 + bad), bad_d);
  if (i == 0) {
    atomicAdd(&g_potrf_prof[0], (unsigned long long)(ts[1] - ts[0]));
    atomicAdd(&g_potrf_prof[1], (unsigned long long)(ts[2] - ts[1]));
    atomicAdd(&g_potrf_prof[7], 1ull);
  }
}

// POTRF of every front's first panel (later panels are factored at the end of the
// SYRK update that last touches them, see syrk_kernel)
__global__ void __launch_bounds__(64) potrf_kernel(DevSym S, const int32_t* __restrict__ tasks, int k0,
                                                   double* __restrict__ front, double* __restrict__ kkinv,
                                                   DevStatus* st) {
  __shared__ __align__(16) double cols[kPotrfSmem / sizeof(double)];
  potrf_panel(S, tasks[blockIdx.x], k0, front, kkinv, st, cols);
}

// TRSM of the rows below the diagonal block: X = B L_kk^{-T} as a DMMA product
// with the inverse from potrf.  task = (front, 64-row chunk); 4 warps x 16 rows.
__global__ void __launch_bounds__(128) trsm_kernel(DevSym S, const int32_t* __restrict__ tasks, int k0,
                                                   double* __restrict__ front, const double* __restrict__ kkinv) {
  constexpr int LD = kPanel + 4;
  constexpr int LK = 64 + 4;  // k-major rows of the chunk (conflict-free copies and fragments)
  __shared__ double As[kPanel * LK];
  __shared__ double Is[kPanel * LD];
  const int64_t s = tasks[2 * blockIdx.x];
  const int64_t chunk = tasks[2 * blockIdx.x + 1];
  const int64_t nc = d_nc(S, s), f = nc + d_nr(S, s), ldf = d_ldf(S, s);
  const int kw = (int)min((int64_t)kPanel, nc - k0);
  double* F = front + S.front_off[s];
  const int64_t r0 = k0 + kw + chunk * 64;
  for (int e = threadIdx.x; e < 64 * kPanel; e += blockDim.x) {
    const int rr = e % 64, k = e / 64;
    const int64_t r = r0 + rr;
    cp_async8(&As[k * LK + rr], F + (int64_t)(k0 + k) * ldf + r, r < f && k < kw);
  }
  const double* Y = kkinv + (S.kk_off[s] + k0 / kPanel) * (kPanel * kPanel);
  for (int e = threadIdx.x; e < kPanel * kPanel; e += blockDim.x)
    cp_async8(&Is[(e / kPanel) * LD + (e % kPanel)], Y + e, true);
  cp_async_wait_all();
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < kPanel; kk += 4) {
    double fa[2], fb[4];
#pragma unroll
    for (int a = 0; a < 2; ++a) fa[a] = As[(kk + t) * LK + 16 * warp + 8 * a + g];
#pragma unroll
    for (int b = 0; b < 4; ++b) fb[b] = Is[(8 * b + g) * LD + kk + t];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
  }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int64_t r = r0 + 16 * warp + 8 * a + g;
        const int j = 8 * b + 2 * t + hh;
        if (r < f && j < kw) F[(int64_t)(k0 + j) * ldf + r] = acc[a][b][hh];
      }
}

// SYRK update on a 64x64 tile with DMMA, K staged through shared memory in
// kSyrkBK-deep chunks (cp.async double buffer):
//   C[rows ti, cols tj] -= P[rows ti, :] * P[rows tj, :]^T,  P = L columns [k0, k0 + kw).
// mode 0 (in-block): P = panel p (kw <= 32), target columns [t0, block end) of
//   every row below -- only the block's remaining pivot columns;
// mode 1 (trailing): P = the whole block of panel p (kw <= kBlkPanels * kPanel
//   = 512 columns: the whole supernode piece), target [block end, f).  The
//   trailing matrix is read and written once per piece, with K <= 512 (up to
//   64 flop per byte of C).
// 4 warps, each a 32x32 quadrant = 4x4 fragments of 8x8.  The staged panels
// are k-major ([k][row], as in the column-major front), so the asynchronous
// copies of consecutive rows land in consecutive banks, and the fragment loads
// are conflict-free with a row stride == 4 mod 16 doubles.
constexpr int kSK = kTile + 4;  // smem stride of one k column of a staged tile
constexpr int kSyrkBK = SYRK_BK;  // k depth of one staged chunk
constexpr size_t kSyrkSmem = 2 * 2 * kSyrkBK * kSK * sizeof(double);
static_assert(kPotrfSmem <= kSyrkSmem, "the fused POTRF reuses the SYRK staging buffers");
// TRAIL: the trailing (mode 1) launches, which never factor a panel: without
// the fused POTRF's registers they fit SYRK_TRAIL_MINB CTAs per SM
#ifndef SYRK_TRAIL_MINB
#define SYRK_TRAIL_MINB 4
#endif
constexpr unsigned kTrailMinTiles = 4 * 148;  // trailing launches of at least this many tiles take TRAIL
template <bool TRAIL>
__global__ void __launch_bounds__(128, TRAIL ? SYRK_TRAIL_MINB : SYRK_MINB)
    syrk_kernel(DevSym S, const int32_t* __restrict__ tasks, int p, int mode, double* __restrict__ front,
                double* __restrict__ kkinv, DevStatus* st) {
  extern __shared__ __align__(16) double syrk_sm[];
  double* Pi = syrk_sm;                  // [2][kSyrkBK * kSK]
  double* Pj = syrk_sm + 2 * kSyrkBK * kSK;
  const int64_t s = tasks[3 * blockIdx.x];
  const int ti = tasks[3 * blockIdx.x + 1], tj = tasks[3 * blockIdx.x + 2];
  const int64_t nc = d_nc(S, s), f = nc + d_nr(S, s), ldf = d_ldf(S, s);
  constexpr int64_t blk = (int64_t)kBlkPanels * kPanel;
  const int64_t k0p = (int64_t)p * kPanel;
  int64_t k0, kw, t0, cend;
  if (mode == 0) {
    k0 = k0p;
    kw = min((int64_t)kPanel, nc - k0);
    t0 = k0 + kw;
    cend = min((k0 / blk + 1) * blk, nc);
  } else {
    k0 = (k0p / blk) * blk;
    const int64_t bend = min(k0 + blk, nc);
    kw = bend - k0;
    t0 = bend;
    cend = f;
  }
  const int64_t r0 = t0 + (int64_t)ti * kTile, c0 = t0 + (int64_t)tj * kTile;
  double* F = front + S.front_off[s];
  // 16-byte copies of row pairs: the front columns are 16-byte aligned (even
  // stride), so a tile whose first row is odd is staged from the row before
  // (uniform shift sa / sb inside the staged tile, read back with the fragments)
  const int sa = (int)(r0 & 1), sb = (int)(c0 & 1);
  constexpr int kPairs = kTile / 2 + 1;  // 33 pairs cover 64 rows at either parity
  static_assert(2 * kPairs <= kSK, "staged tile stride too small");
  auto stage = [&](int buf, int64_t kk0) {
    double* A = Pi + buf * kSyrkBK * kSK;
    double* B = Pj + buf * kSyrkBK * kSK;
    for (int e = threadIdx.x; e < kSyrkBK * kPairs; e += blockDim.x) {
      const int kc = e / kPairs, rr = 2 * (e - kc * kPairs);
      const bool kin = kk0 + kc < kw;
      const int64_t ri = r0 - sa + rr, rj = c0 - sb + rr;
      const double* col = F + (k0 + kk0 + kc) * ldf;
      const bool va = kin && ri < f, vb = kin && rj < f;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(A + kc * kSK + rr)),
                   "l"(va ? col + ri : F), "r"(va ? 16 : 0)
                   : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(B + kc * kSK + rr)),
                   "l"(vb ? col + rj : F), "r"(vb ? 16 : 0)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wy = (warp >> 1) * 32, wx = (warp & 1) * 32;
  const bool skip = ti == tj && wx > wy;  // strictly-upper quadrant of a diagonal tile
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int nchunk = (int)((kw + kSyrkBK - 1) / kSyrkBK);
  stage(0, 0);
  for (int ck = 0; ck < nchunk; ++ck) {
    if (ck + 1 < nchunk) {
      stage((ck + 1) & 1, (int64_t)(ck + 1) * kSyrkBK);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const double* A = Pi + (ck & 1) * kSyrkBK * kSK;
    const double* B = Pj + (ck & 1) * kSyrkBK * kSK;
    const int kc = (int)min((int64_t)kSyrkBK, kw - (int64_t)ck * kSyrkBK);
    if (!skip)
      for (int kk = 0; kk < kc; kk += 4) {
        double fa[4], fb[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) fa[a] = A[(kk + t) * kSK + sa + wy + 8 * a + g];
#pragma unroll
        for (int b = 0; b < 4; ++b) fb[b] = B[(kk + t) * kSK + sb + wx + 8 * b + g];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
      }
    __syncthreads();
  }
  // epilogue (not for the strictly-upper quadrant of a diagonal tile): issue every
  // C load before the first store (F aliases itself, so
  // the compiler would otherwise serialise load -> subtract -> store)
  if (!skip) {
    // (TRAIL: in two halves of 16 values, so the accumulators plus the loaded C fit
    // the 128 registers of SYRK_TRAIL_MINB = 4 CTAs per SM)
    constexpr int kHalves = TRAIL ? 2 : 1;
  #pragma unroll
    for (int hv = 0; hv < kHalves; ++hv) {
      double cv[4 / kHalves][4][2];
  #pragma unroll
      for (int aa = 0; aa < 4 / kHalves; ++aa)
  #pragma unroll
        for (int b = 0; b < 4; ++b)
  #pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t r = r0 + wy + 8 * (hv * (4 / kHalves) + aa) + g;
            const int64_t c = c0 + wx + 8 * b + 2 * t + h;
            cv[aa][b][h] = (r < f && c < cend && r >= c) ? F[c * ldf + r] : 0.0;
          }
  #pragma unroll
      for (int aa = 0; aa < 4 / kHalves; ++aa)
  #pragma unroll
        for (int b = 0; b < 4; ++b)
  #pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int a = hv * (4 / kHalves) + aa;
            const int64_t r = r0 + wy + 8 * a + g;
            const int64_t c = c0 + wx + 8 * b + 2 * t + h;
            if (r < f && c < cend && r >= c) F[c * ldf + r] = cv[aa][b][h] - acc[a][b][h];
          }
    }
  }
  // the tile holding the next panel's diagonal block (this update is the last one
  // it receives) factors it right away: no separate POTRF launch for panels > 0
  if (!TRAIL && ti == 0 && tj == 0 && t0 < nc) {
    __syncthreads();  // the tile's stores are visible to the CTA
    if (warp < 2) potrf_panel(S, s, (int)t0, front, kkinv, st, syrk_sm);
  }
}

constexpr double kLevelEventsMaxFlops = 5e10;  // factors whose per-level M_s events are recorded
static int chol_upload(CholHandle* h) {
  if (h->uploaded) return CNB_OK;
  const Symbolic& S = h->S;
  int rc;
#define UP(d, v) \
  if ((rc = upload_vec(&h->d, S.v)) != CNB_OK) return rc;
  UP(d_first, first)
  UP(d_rows_ptr, rows_ptr)
  UP(d_rows, rows)
  UP(d_front_off, front_off)
  UP(d_child_ptr, child_ptr)
  UP(d_child, child)
  UP(d_rel_ptr, rel_ptr)
  UP(d_rel, rel)
  UP(d_map_src, map_src)
  UP(d_map_dst, map_dst)
  UP(d_perm, perm)
#undef UP
  h->m_off.assign(S.ns + 1, 0);
  for (int64_t s = 0; s < S.ns; ++s) h->m_off[s + 1] = h->m_off[s] + S.ldf(s) * S.nc(s);
  if ((rc = upload_vec(&h->d_m_off, h->m_off)) != CNB_OK) return rc;
  if ((rc = upload_vec(&h->d_ea_rng, S.ea_rng)) != CNB_OK) return rc;
  std::vector<int32_t> all;
  struct Rec {
    int64_t off, count;
  };
  std::vector<Rec> ea_rec, ti_rec, p2_rec;
  std::vector<std::vector<Rec>> po_rec, tr_rec, sy_rec, so_rec;
  for (int l = 0; l < S.n_levels; ++l) {
    const LevelTasks& T = S.tasks[l];
    ea_rec.push_back({(int64_t)all.size(), (int64_t)T.ea.size() / 4});
    all.insert(all.end(), T.ea.begin(), T.ea.end());
    po_rec.emplace_back();
    tr_rec.emplace_back();
    sy_rec.emplace_back();
    so_rec.emplace_back();
    for (size_t p = 0; p < T.potrf.size(); ++p) {
      po_rec[l].push_back({(int64_t)all.size(), (int64_t)T.potrf[p].size()});
      all.insert(all.end(), T.potrf[p].begin(), T.potrf[p].end());
      tr_rec[l].push_back({(int64_t)all.size(), (int64_t)T.trsm[p].size() / 2});
      all.insert(all.end(), T.trsm[p].begin(), T.trsm[p].end());
      sy_rec[l].push_back({(int64_t)all.size(), (int64_t)T.syrk[p].size() / 3});
      all.insert(all.end(), T.syrk[p].begin(), T.syrk[p].end());
      so_rec[l].push_back({(int64_t)all.size(), (int64_t)T.syrk_out[p].size() / 3});
      all.insert(all.end(), T.syrk_out[p].begin(), T.syrk_out[p].end());
    }
    // triangular inversion tasks: (s, 16-column chunk of L11^{-1})
    const int64_t off = (int64_t)all.size();
    for (int64_t q = S.level_ptr[l]; q < S.level_ptr[l + 1]; ++q) {
      const int64_t s = S.level_sn[q];
      for (int64_t j0 = 0; j0 < S.nc(s); j0 += kInvCols) {
        all.push_back((int32_t)s);
        all.push_back((int32_t)j0);
      }
    }
    ti_rec.push_back({off, ((int64_t)all.size() - off) / 2});
    // P21 = L21 L11^{-1} tasks: (s, 64-row block of L21)
    const int64_t off2 = (int64_t)all.size();
    for (int64_t q = S.level_ptr[l]; q < S.level_ptr[l + 1]; ++q) {
      const int64_t s = S.level_sn[q];
      for (int64_t q0 = 0; q0 < S.nr(s); q0 += 64)
        for (int64_t c0 = 0; c0 < S.nc(s); c0 += 64) {
          all.push_back((int32_t)s);
          all.push_back((int32_t)q0);
          all.push_back((int32_t)c0);
        }
    }
    p2_rec.push_back({off2, ((int64_t)all.size() - off2) / 3});
  }
  if ((rc = upload_vec(&h->d_tasks, all)) != CNB_OK) return rc;
  auto mk = [&](const Rec& r) { return DevTasks{h->d_tasks + r.off, r.count}; };
  h->ea.clear();
  h->trinv.clear();
  h->p21.clear();
  h->potrf.assign(S.n_levels, {});
  h->trsm.assign(S.n_levels, {});
  h->syrk.assign(S.n_levels, {});
  h->syrk_out.assign(S.n_levels, {});
  for (int l = 0; l < S.n_levels; ++l) {
    h->ea.push_back(mk(ea_rec[l]));
    h->trinv.push_back(mk(ti_rec[l]));
    h->p21.push_back(mk(p2_rec[l]));
    for (auto& r : po_rec[l]) h->potrf[l].push_back(mk(r));
    for (auto& r : tr_rec[l]) h->trsm[l].push_back(mk(r));
    for (auto& r : sy_rec[l]) h->syrk[l].push_back(mk(r));
    for (auto& r : so_rec[l]) h->syrk_out[l].push_back(mk(r));
  }
  CNB_CUDA(cudaMalloc((void**)&h->d_front, std::max<int64_t>(1, S.front_off[S.ns]) * sizeof(double)));
  // the padding row of an odd-f panel is read by the 16-byte tile copies: keep it finite
  CNB_CUDA(cudaMalloc((void**)&h->d_m, std::max<int64_t>(1, h->m_off[S.ns]) * sizeof(double)));
  CNB_CUDA(cudaMemset(h->d_m, 0, std::max<int64_t>(1, h->m_off[S.ns]) * sizeof(double)));
  h->kk_off.assign(S.ns + 1, 0);
  for (int64_t s = 0; s < S.ns; ++s) h->kk_off[s + 1] = h->kk_off[s] + (S.nc(s) + kPanel - 1) / kPanel;
  if ((rc = upload_vec(&h->d_kk_off, h->kk_off)) != CNB_OK) return rc;
  CNB_CUDA(cudaMalloc((void**)&h->d_kkinv, std::max<int64_t>(1, h->kk_off[S.ns]) * kPanel * kPanel * sizeof(double)));
  CNB_CUDA(cudaMalloc((void**)&h->d_vals, std::max<int64_t>(1, S.csr_nnz) * sizeof(double)));
  CNB_CUDA(cudaStreamCreateWithFlags(&h->side_stream, cudaStreamNonBlocking));
  if (S.flops < kLevelEventsMaxFlops) {  // (only small factors overlap the compliance: no extra
                                         // streams otherwise -- streams beyond the hardware queues
                                         // alias and serialise, measured +3 ms per cfg3 step)
    CNB_CUDA(cudaStreamCreateWithFlags(&h->comp_stream, cudaStreamNonBlocking));
    CNB_CUDA(cudaEventCreateWithFlags(&h->ev_pre, cudaEventDisableTiming));
    CNB_CUDA(cudaEventCreateWithFlags(&h->ev_comp, cudaEventDisableTiming));
    h->ev_level.assign(S.n_levels, nullptr);
    for (auto& e : h->ev_level) CNB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  CNB_CUDA(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
  CNB_CUDA(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  CNB_CUDA(cudaFuncSetAttribute(syrk_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSyrkSmem));
  CNB_CUDA(cudaFuncSetAttribute(syrk_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSyrkSmem));
  h->uploaded = true;
  return CNB_OK;
}

static void chol_free(CholHandle* h) {
  void* ptrs[] = {h->d_first, h->d_rows_ptr, h->d_rows, h->d_front_off, h->d_child_ptr, h->d_child,
                  h->d_rel_ptr, h->d_rel, h->d_map_src, h->d_map_dst, h->d_perm, h->d_front, h->d_tasks,
                  h->d_m, h->d_m_off, h->d_kkinv, h->d_vals, h->d_kk_off, h->d_ea_rng};
  if (h->factor_exec) cudaGraphExecDestroy(h->factor_exec);
  h->factor_exec = nullptr;
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  h->cap_stream = nullptr;
  if (h->side_stream) cudaStreamDestroy(h->side_stream);
  h->side_stream = nullptr;
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  h->ev_fork = h->ev_join = nullptr;
  if (h->comp_stream) cudaStreamDestroy(h->comp_stream);
  h->comp_stream = nullptr;
  for (cudaEvent_t e : {h->ev_pre, h->ev_comp})
    if (e) cudaEventDestroy(e);
  h->ev_pre = h->ev_comp = nullptr;
  for (auto& e : h->ev_level)
    if (e) cudaEventDestroy(e);
  h->ev_level.clear();
  h->level_events = false;
  for (void* p : ptrs)
    if (p) cudaFree(p);
  h->plan1.release();
  h->plan8.release();
  for (GrowBuf* b : {&h->bp, &h->tbuf, &h->c_int, &h->c_rhs, &h->c_val, &h->c_y}) b->release();
  h->c_pin.release();
  free_compliance_plan(h);
}

static std::map<std::string, std::pair<const void*, size_t>> export_table(const CholHandle* h) {
  const Symbolic& S = h->S;
  std::map<std::string, std::pair<const void*, size_t>> t;
  auto add = [&](const char* name, const auto& v) { t[name] = {v.data(), v.size() * sizeof(v[0])}; };
  add("perm", S.perm);
  add("iperm", S.iperm);
  add("first", S.first);
  add("rows_ptr", S.rows_ptr);
  add("rows", S.rows);
  add("parent", S.parent);
  add("level", S.level);
  add("child_ptr", S.child_ptr);
  add("child", S.child);
  add("front_off", S.front_off);
  add("rel_ptr", S.rel_ptr);
  add("rel", S.rel);
  add("map_src", S.map_src);
  add("map_dst", S.map_dst);
  add("level_ptr", S.level_ptr);
  add("level_sn", S.level_sn);
  return t;
}

static int enqueue_factor(CholHandle* h, DevStatus* d_status, cudaStream_t st) {
  const Symbolic& S = h->S;
  DevSym sym = h->sym();
  int rc;
  CNB_CUDA(cudaMemsetAsync(h->d_front, 0, std::max<int64_t>(1, S.front_off[S.ns]) * sizeof(double), st));
  const int64_t nmap = (int64_t)S.map_src.size();
  if (nmap) {
    scatter_kernel<<<grid_for(nmap, 256), 256, 0, st>>>(nmap, h->d_map_src, h->d_map_dst, h->d_vals, h->d_front);
    CNB_LAUNCH_CHECK("scatter_kernel");
  }
  for (int l = 0; l < S.n_levels; ++l) {
    if (h->ea[l].count) {
      extend_add_kernel<<<(unsigned)h->ea[l].count, 256, 0, st>>>(sym, h->ea[l].ptr, h->d_ea_rng, h->d_front);
      CNB_LAUNCH_CHECK("extend_add_kernel");
    }
    for (size_t p = 0; p < h->potrf[l].size(); ++p) {
      const int k0 = (int)(p * kPanel);
      if (p == 0 && h->potrf[l][p].count) {  // later panels: fused into the preceding SYRK
        potrf_kernel<<<(unsigned)h->potrf[l][p].count, 64, 0, st>>>(sym, h->potrf[l][p].ptr, k0, h->d_front,
                                                                       h->d_kkinv, d_status);
        CNB_LAUNCH_CHECK("potrf_kernel");
      }
      if (h->trsm[l][p].count) {
        trsm_kernel<<<(unsigned)h->trsm[l][p].count, 128, 0, st>>>(sym, h->trsm[l][p].ptr, k0, h->d_front,
                                                                   h->d_kkinv);
        CNB_LAUNCH_CHECK("trsm_kernel");
      }
      if (h->syrk[l][p].count) {
        syrk_kernel<false><<<(unsigned)h->syrk[l][p].count, 128, kSyrkSmem, st>>>(sym, h->syrk[l][p].ptr, (int)p, 0,
                                                                           h->d_front, h->d_kkinv, d_status);
        CNB_LAUNCH_CHECK("syrk_kernel");
      }
      if (h->syrk_out[l][p].count) {
        // (mode 1 factors no panel: t0 = block end = nc, pieces are <= 512 wide);
        // large launches take the 4-CTA-per-SM variant, small (latency-bound) ones
        // keep the plain epilogue
        const unsigned n1 = (unsigned)h->syrk_out[l][p].count;
        auto k1 = n1 >= kTrailMinTiles ? syrk_kernel<true> : syrk_kernel<false>;
        k1<<<n1, 128, kSyrkSmem, st>>>(sym, h->syrk_out[l][p].ptr, (int)p, 1, h->d_front, h->d_kkinv, d_status);
        CNB_LAUNCH_CHECK("syrk_kernel");
      }
    }
    // L11^{-1} and P21 of this level read L11 / L21 (columns [0, nc) of its
    // fronts) and write M_s: nothing the next levels touch, so they run on the
    // side stream, in level order, while the factorisation goes on
    CNB_CUDA(cudaEventRecord(h->ev_fork, st));
    CNB_CUDA(cudaStreamWaitEvent(h->side_stream, h->ev_fork, 0));
    if ((rc = trinv_level(h, l, h->side_stream))) return rc;
    // level l's M_s is complete: the compliance forward solve may read it (small
    // factors only: the external event nodes cost a large factor's graph ~4 ms
    // per cfg3 step, and its forward solve is not overlapped anyway)
    if (h->comp_stream) {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      CNB_CUDA(cudaStreamIsCapturing(h->side_stream, &cs));
      if (cs == cudaStreamCaptureStatusActive)
        CNB_CUDA(cudaEventRecordWithFlags(h->ev_level[l], h->side_stream, cudaEventRecordExternal));
      else
        CNB_CUDA(cudaEventRecord(h->ev_level[l], h->side_stream));
    }
  }
  CNB_CUDA(cudaEventRecord(h->ev_join, h->side_stream));
  CNB_CUDA(cudaStreamWaitEvent(st, h->ev_join, 0));
  return CNB_OK;
}

}  // namespace cnb

using namespace cnb;

extern "C" {

// diagnostic: phase end times (ns) of the last cooperative single-RHS solve
int cnb_solve_profile(double* out) { return solve_profile(out); }

// diagnostic: summed cycles of the potrf phases since the last call (loads,
// factor, store L, inverse, store Y) and the launch count in out[7]
int cnb_potrf_profile(double* out) {
  unsigned long long h[8];
  CNB_CUDA(cudaMemcpyFromSymbol(h, g_potrf_prof, sizeof(h)));
  const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  CNB_CUDA(cudaMemcpyToSymbol(g_potrf_prof, z, sizeof(z)));
  for (int k = 0; k < 8; ++k) out[k] = (double)h[k];
  return CNB_OK;
}

static CholHandle* H(cnb_chol_t h) { return reinterpret_cast<CholHandle*>(h); }

int cnb_chol_analyze(int64_t n, const int64_t* rowptr, const int64_t* col, int32_t bs, const double* coords,
                     int32_t leaf_nodes, cnb_chol_t* out) {
  *out = nullptr;
  CholHandle* h = new CholHandle();
  try {
    analyze(h->S, n, rowptr, col, bs, coords, leaf_nodes);
  } catch (const std::exception& e) {
    delete h;
    set_error("chol_analyze: %s", e.what());
    return CNB_E_INTERNAL;
  }
  *out = reinterpret_cast<cnb_chol_t>(h);
  return CNB_OK;
}

int cnb_chol_destroy(cnb_chol_t hh) {
  if (!hh) return CNB_OK;
  chol_free(H(hh));
  delete H(hh);
  return CNB_OK;
}

int cnb_chol_info(cnb_chol_t hh, int64_t* info, double* fl) {
  const Symbolic& S = H(hh)->S;
  info[0] = S.n;
  info[1] = S.ns;
  info[2] = S.nnz_L;
  info[3] = S.front_off[S.ns];
  info[4] = S.n_levels;
  info[5] = S.csr_nnz;
  info[6] = S.bs;
  int64_t fl_launch = S.map_src.empty() ? 0 : 1;
  for (const LevelTasks& T : S.tasks) {
    fl_launch += (T.ea.empty() ? 0 : 1) + 1;  // extend-add, trinv
    for (size_t p = 0; p < T.potrf.size(); ++p)
      fl_launch += (T.potrf[p].empty() ? 0 : 1) + (T.trsm[p].empty() ? 0 : 1) + (T.syrk[p].empty() ? 0 : 1) +
                   (T.syrk_out[p].empty() ? 0 : 1);
  }
  info[7] = fl_launch;
  info[8] = 2 + 4 * (int64_t)S.n_levels;
  fl[0] = S.flops;
  fl[1] = S.solve_flops_per_rhs;
  return CNB_OK;
}

int64_t cnb_chol_export_bytes(cnb_chol_t hh, const char* name) {
  auto t = export_table(H(hh));
  auto it = t.find(name);
  return it == t.end() ? -1 : (int64_t)it->second.second;
}

int cnb_chol_export(cnb_chol_t hh, const char* name, void* dst) {
  auto t = export_table(H(hh));
  auto it = t.find(name);
  if (it == t.end()) {
    set_error("chol_export: unknown array %s", name);
    return CNB_E_VALIDATION;
  }
  if (it->second.second) memcpy(dst, it->second.first, it->second.second);
  return CNB_OK;
}

int cnb_chol_factor(cnb_chol_t hh, const double* vals, cnb_status_t* d_status, void* stream) {
  CholHandle* h = H(hh);
  int rc = chol_upload(h);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const Symbolic& S = h->S;
  // values into the handle's own buffer: the captured graph reads fixed addresses
  CNB_CUDA(cudaMemcpyAsync(h->d_vals, vals, std::max<int64_t>(1, S.csr_nnz) * sizeof(double),
                           cudaMemcpyDeviceToDevice, st));
  if (h->ev_pre) CNB_CUDA(cudaEventRecord(h->ev_pre, st));  // a following compliance forward solve starts here
  if (use_graphs()) {
    if (h->factor_exec && h->factor_status != (void*)d_status) {
      cudaGraphExecDestroy(h->factor_exec);
      h->factor_exec = nullptr;
    }
    if (!h->factor_exec) {
      // capture on a private stream (the legacy default stream cannot capture)
      if (!h->cap_stream) CNB_CUDA(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
      const long long before = launch_count();
      CNB_CUDA(cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
      rc = enqueue_factor(h, (DevStatus*)d_status, h->cap_stream);
      cudaGraph_t graph = nullptr;
      cudaError_t e = cudaStreamEndCapture(h->cap_stream, &graph);
      if (rc) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
      }
      if (e != cudaSuccess) return cuda_status(e, "cudaStreamEndCapture(factor)");
      e = cudaGraphInstantiate(&h->factor_exec, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) return cuda_status(e, "cudaGraphInstantiate(factor)");
      h->factor_nodes = launch_count() - before;
      add_launches(-h->factor_nodes);  // captured, not launched
      h->factor_status = (void*)d_status;
    }
    CNB_CUDA(cudaGraphLaunch(h->factor_exec, st));
    add_launches(h->factor_nodes);
  } else {
    if ((rc = enqueue_factor(h, (DevStatus*)d_status, st))) return rc;
  }
  h->factored = true;
  h->level_events = h->comp_stream != nullptr;
  return CNB_OK;
}

int cnb_chol_solve(cnb_chol_t hh, const double* B, int64_t ldb, double* X, int64_t ldx, int64_t k, void* stream) {
  CholHandle* h = H(hh);
  if (!h->factored) {
    set_error("chol_solve: not factorised");
    return CNB_E_VALIDATION;
  }
  return solve_dense(h, B, ldb, X, ldx, k, (cudaStream_t)stream);
}

int cnb_chol_compliance(cnb_chol_t hh, int64_t ncols, const int64_t* colptr, const int64_t* rowidx,
                        const double* vals, double* U, int64_t ldu, double* flops_out, void* stream) {
  CholHandle* h = H(hh);
  if (!h->factored) {
    set_error("chol_compliance: not factorised");
    return CNB_E_VALIDATION;
  }
  return compliance(h, ncols, colptr, rowidx, vals, U, ldu, flops_out, (cudaStream_t)stream);
}

int cnb_chol_compliance_plan(cnb_chol_t hh, int64_t ncols, const int64_t* colptr, const int64_t* rowidx,
                             const double* vals, int32_t rank, int32_t world, int64_t* sizes, double* flops_out,
                             void* stream) {
  CholHandle* h = H(hh);
  if (!h->factored) {
    set_error("chol_compliance_plan: not factorised");
    return CNB_E_VALIDATION;
  }
  return compliance_split_plan(h, ncols, colptr, rowidx, vals, rank, world, sizes, flops_out, (cudaStream_t)stream);
}

int cnb_chol_compliance_forward(cnb_chol_t hh, double* ysend, void* stream) {
  return compliance_split_forward(H(hh), ysend, (cudaStream_t)stream);
}

int cnb_chol_compliance_gram(cnb_chol_t hh, const double* yall, double* tiles, void* stream) {
  return compliance_split_gram(H(hh), yall, tiles, (cudaStream_t)stream);
}

int cnb_chol_compliance_finish(cnb_chol_t hh, const double* tiles_all, double* U, int64_t ldu, void* stream) {
  return compliance_split_finish(H(hh), tiles_all, U, ldu, (cudaStream_t)stream);
}

}  // extern "C"
