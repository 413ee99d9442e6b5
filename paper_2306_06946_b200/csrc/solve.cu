// Triangular solves and the mapping compliance on the supernodal factor.
//
// Reference being replaced: Factorization.solve / solve_multi
// (linalg.py:89-106) and the multi-RHS solve + product of assemble_Wg
// (constraints.py:175-178).
//
// At factorisation time every diagonal block L11 of a supernode is inverted
// (trinv_kernel) and P21 = L21 L11^{-1} formed (p21_kernel).  A forward solve
// step of supernode s is then one matrix product over its solve panel
// M_s = [L11^{-1}; P21] (f_s x nc_s, column-major, even column stride ldf_s):
//     [y_s ; u_s] = M_s r_s,   y_s -> solution rows,  R_parent -= u_s (extend-add)
// and a backward step is two GEMVs,  x_s = L11^{-T} y_s - P21^T x_rows.
// Right-hand-side blocks R_s use the same even stride, so every tile column of
// M_s and R_s starts 16-byte aligned (16-byte asynchronous copies).
// No serial triangle chains remain on the solve path: single right-hand
// sides are coalesced GEMVs (bandwidth-bound), the compliance's many
// right-hand sides are fp64 tensor-core GEMMs (mma.sync m8n8k4 f64 = DMMA).
#include <cooperative_groups.h>

#include <cstring>
#include <numeric>

#include "chol_dev.cuh"

namespace cnb {

constexpr int kSolveThreads = 128;
constexpr int kAsmRows = 128;   // rows per assemble task
constexpr int kAsmCols = 64;    // columns per assemble task (sparse mode)
constexpr int kGemvRows = 32;   // rows per dense panel task
constexpr int kG1Rows = 16;     // rows per panel task of the cooperative single-RHS solve on levels with few
                                // tasks (kGemvRows on the others)
constexpr int kGemvJ = 256;     // staged pivot rows of the RHS per pass
constexpr int kGemvU = 16;      // panel loads in flight per thread
constexpr int kBwdRows = 4;     // pivot rows per backward task (warp per row)
constexpr int kMT = 64;         // DMMA panel tile (rows, cols)
constexpr int kMA = kMT + 4;    // k-major stride of tiles staged from column-major sources

// RHS block of supernode s: R_s = rhs + roff[s], f_s x w_s column-major with
// column stride ldf_s (d_ldf); global columns [lo_s, lo_s + w_s).
struct RhsView {
  double* rhs;
  const int64_t* roff;
  const int64_t* lo;
  const int64_t* w;
};

// ---- L11^{-1}, kInvCols columns per task -----------------------------------------
// Block forward substitution L11 X = I over 32-row blocks: the diagonal block
// of block kb is inverted already (D_kb, kept by potrf_kernel), so each block
// step is y = D_kb v (a small product, no sequential row loop) followed by the
// update of the rows below with the panel columns of L.  The task's X columns
// live in shared memory for the whole substitution (written to M_s once at the
// end), the next D block is staged with cp.async during the current step, and
// each thread's L values for the update are loaded before the step waits on D:
// a step is one shared-memory round instead of three dependent global ones.
static_assert(32 * kInvCols == 256, "trinv_kernel: one warp per column of the block (256 threads)");
constexpr size_t kTrinvSmem = (size_t)kInvCols * kMaxSnCols * sizeof(double);  // X columns (dynamic)
__global__ void __launch_bounds__(256) trinv_kernel(DevSym S, const int32_t* __restrict__ tasks,
                                                    const double* __restrict__ front, const double* __restrict__ kkinv,
                                                    double* __restrict__ panel) {
  extern __shared__ double xs[];  // [kInvCols][nc]
  __shared__ double sD[2][32][33];
  __shared__ double y[32][kInvCols];
  const int64_t s = tasks[2 * blockIdx.x], j0 = tasks[2 * blockIdx.x + 1];
  const int nc = (int)d_nc(S, s);
  const int64_t ldf = d_ldf(S, s);
  const double* F = front + S.front_off[s];
  double* X = panel + S.m_off[s];  // rows [0, nc) of M_s (stride ldf)
  const int ncols = (int)min((int64_t)kInvCols, nc - j0);
  const double* Dall = kkinv + S.kk_off[s] * (32 * 32);
  auto stage_d = [&](int kb, int buf) {  // D_kb -> sD[buf] (entries above the diagonal are never read)
    const double* D = Dall + (kb / 32) * (32 * 32);
    for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) cp_async8(&sD[buf][e >> 5][e & 31], D + e, true);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  const int kb0 = (int)(j0 / 32) * 32;
  stage_d(kb0, 0);
  for (int e = threadIdx.x; e < kInvCols * nc; e += blockDim.x) {
    const int c = e / nc, i = e - c * nc;
    xs[e] = (i == j0 + c) ? 1.0 : 0.0;
  }
  const int r = threadIdx.x & 31, cc = threadIdx.x >> 5;  // (row, column) of the 32 x kInvCols block
  int buf = 0;
  for (int kb = kb0; kb < nc; kb += 32, buf ^= 1) {
    const int bw = min(32, nc - kb);
    if (kb + 32 < nc) stage_d(kb + 32, buf ^ 1);
    // this thread's first update row: its L values in flight before the wait
    const int i0 = kb + bw + threadIdx.x;
    double l0[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) l0[j] = (i0 < nc && j < bw) ? F[(int64_t)(kb + j) * ldf + i0] : 0.0;
    if (kb + 32 < nc)
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    else
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();  // D_kb landed; the previous step's updates of xs are done
    {
      double yv = 0.0;
      if (r < bw) {  // (rows past the block: y = 0; D_kb and v are only read below the diagonal)
        const double* v = xs + cc * nc + kb;
        double a0 = 0.0, a1 = 0.0;
        for (int k = 0; k + 1 <= r; k += 2) {
          a0 = fma(sD[buf][r][k], v[k], a0);
          a1 = fma(sD[buf][r][k + 1], v[k + 1], a1);
        }
        if ((r & 1) == 0) a0 = fma(sD[buf][r][r], v[r], a0);
        yv = a0 + a1;
      }
      y[r][cc] = yv;
    }
    __syncthreads();
    if (r < bw) xs[cc * nc + kb + r] = y[r][cc];
    for (int i = i0; i < nc; i += blockDim.x) {
      double acc[kInvCols];
#pragma unroll
      for (int c = 0; c < kInvCols; ++c) acc[c] = 0.0;
      if (i == i0) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
#pragma unroll
          for (int c = 0; c < kInvCols; ++c) acc[c] = fma(l0[j], y[j][c], acc[c]);
      } else {
        for (int j = 0; j < bw; ++j) {
          const double l = F[(int64_t)(kb + j) * ldf + i];
#pragma unroll
          for (int c = 0; c < kInvCols; ++c) acc[c] = fma(l, y[j][c], acc[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < kInvCols; ++c) xs[c * nc + i] -= acc[c];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < ncols * nc; e += blockDim.x) {
    const int c = e / nc, i = e - c * nc;
    X[(j0 + c) * ldf + i] = xs[e];
  }
}

// ---- assemble front RHS blocks: init (dense) + extend-add children -----------
// task = (s, row chunk r0, column chunk c0); any block size
__device__ __forceinline__ void asm_task(const DevSym& S, const int32_t* __restrict__ task, const RhsView& R,
                                         int dense, const double* __restrict__ Bp, int64_t n) {
  const int64_t s = task[0], r0 = task[1], c0 = task[2];
  const int64_t nc = d_nc(S, s), f = nc + d_nr(S, s), ldr = d_ldf(S, s);
  const int64_t r1 = min(f, r0 + kAsmRows);
  const int64_t ws = R.w[s], los = R.lo[s];
  const int64_t c1 = min(ws, c0 + kAsmCols);
  double* Rs = R.rhs + R.roff[s];
  const int64_t first = S.first[s];
  if (dense) {
    for (int64_t c = c0; c < c1; ++c)
      for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x)
        Rs[c * ldr + i] = i < nc ? Bp[(los + c) * n + first + i] : 0.0;
    __syncthreads();
  }
  for (int64_t ci = S.child_ptr[s]; ci < S.child_ptr[s + 1]; ++ci) {
    const int64_t ch = S.child[ci];
    const int64_t wc = R.w[ch];
    if (wc == 0) continue;
    const int64_t ncc = d_nc(S, ch), nrc = d_nr(S, ch), ldc = d_ldf(S, ch);
    const int32_t* rel = S.rel + S.rel_ptr[ch];
    int64_t a = 0, b = nrc;
    while (a < b) {
      int64_t m = (a + b) >> 1;
      if (rel[m] < r0) a = m + 1; else b = m;
    }
    const int64_t k0 = a;
    b = nrc;
    while (a < b) {
      int64_t m = (a + b) >> 1;
      if (rel[m] < r1) a = m + 1; else b = m;
    }
    const int64_t k1 = a;
    const int64_t off = R.lo[ch] - los;
    const double* Rc = R.rhs + R.roff[ch];
    const int64_t cc0 = max(c0, off), cc1 = min(c1, off + wc);
    // the child's (column, row) entries flattened over the threads, 4 per thread per
    // batch: all loads of a batch are issued before its stores (the parent and child
    // windows share one buffer, so the compiler could not reorder them otherwise)
    const int nk = (int)(k1 - k0);
    const int tot = nk * (int)max((int64_t)0, cc1 - cc0);
    for (int e0 = threadIdx.x; e0 < tot; e0 += 4 * blockDim.x) {
      double u[4], v[4];
      double* d[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = e0 + q * (int)blockDim.x;
        d[q] = nullptr;
        u[q] = 0.0;
        if (e < tot) {
          const int cq = e / nk, kq = e - cq * nk;
          const int64_t c = cc0 + cq, k = k0 + kq;
          u[q] = Rc[(c - off) * ldc + ncc + k];
          d[q] = Rs + c * ldr + rel[k];
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = d[q] ? *d[q] : 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (d[q]) *d[q] = v[q] + u[q];
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kSolveThreads) asm_kernel(DevSym S, const int32_t* __restrict__ tasks, RhsView R,
                                                            int dense, const double* __restrict__ Bp, int64_t n) {
  asm_task(S, tasks + 3 * blockIdx.x, R, dense, Bp, n);
}

// ---- dense forward panel product (GEMV, NC <= 8 columns) ----------------------
// task = (s, row tile r0 of 32 rows): 8 warps split the pivot index j, lanes
// take consecutive rows (coalesced column reads of M_s), partial sums reduced
// through shared memory.  y -> Bp pivot rows, u subtracted from R_s.
template <int NC>
__device__ __forceinline__ void gemv_task(const DevSym& S, const int32_t* __restrict__ task, const RhsView& R,
                                          const double* __restrict__ panel, double* Bp, int64_t n,
                                          double (*rt)[NC], double (*red)[32][NC]) {
  const int64_t s = task[0], r0 = task[1];
  const int64_t nc = d_nc(S, s), f = nc + d_nr(S, s), ldm = d_ldf(S, s);
  const int64_t ws = R.w[s], los = R.lo[s];
  const int ncols = (int)min((int64_t)NC, ws);
  double* Rs = R.rhs + R.roff[s];
  const double* M = panel + S.m_off[s];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int64_t i = r0 + lane;
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0;
  for (int64_t jb = 0; jb < nc; jb += kGemvJ) {
    const int jn = (int)min((int64_t)kGemvJ, nc - jb);
    __syncthreads();
    for (int e = threadIdx.x; e < jn * NC; e += blockDim.x) {
      const int j = e % jn, c = e / jn;
      cp_async8(&rt[j][c], Rs + c * ldm + jb + j, c < ncols);
    }
    cp_async_wait_all();
    __syncthreads();
    if (i < f) {
      // every row runs over all jn pivots (the upper triangle of L11^{-1} in M_s is
      // zero): kGemvU loads in flight per thread before their multiply-adds, the
      // chain per thread stays j = grp, grp + 8, ... in order
      const double* pc = M + jb * ldm + i;
      for (int j0 = grp; j0 < jn; j0 += 8 * kGemvU) {
        double mv[kGemvU];
#pragma unroll
        for (int u = 0; u < kGemvU; ++u) mv[u] = j0 + 8 * u < jn ? pc[(int64_t)(j0 + 8 * u) * ldm] : 0.0;
#pragma unroll
        for (int u = 0; u < kGemvU; ++u)
          if (j0 + 8 * u < jn)
#pragma unroll
            for (int c = 0; c < NC; ++c) acc[c] = fma(mv[u], rt[j0 + 8 * u][c], acc[c]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) red[grp][lane][c] = acc[c];
  __syncthreads();
  if (grp == 0 && i < f) {
    const int64_t first = S.first[s];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      if (c >= ncols) break;
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) v += red[q][lane][c];
      if (i < nc)
        Bp[(los + c) * n + first + i] = v;
      else
        Rs[c * ldm + i] -= v;
    }
  }
}

template <int NC>
__global__ void __launch_bounds__(256) panel_gemv_kernel(DevSym S, const int32_t* __restrict__ tasks, RhsView R,
                                                         const double* __restrict__ panel, double* Bp,
                                                         int64_t n) {
  __shared__ double rt[kGemvJ][NC];
  __shared__ double red[8][32][NC];
  gemv_task<NC>(S, tasks + 3 * blockIdx.x, R, panel, Bp, n, rt, red);
}

// ---- sparse-mode forward panel product on DMMA tiles --------------------------
// task = (s, r0, c0): 64 x 64 tile of M_s (f x nc) x R_s[0:nc, c0:c0+64];
// rows < nc -> Y_s (nc x w, ld nc + (nc & 1)), rows >= nc: R_s -= .
// Both operands are staged with 16-byte copies (M_s and R_s columns are 16-byte
// aligned): a copy that straddles the end of a column reads the padding row of
// M_s (zero) or, for R_s, row nc -- whose product is with a zero-filled column
// of the A tile.
__global__ void __launch_bounds__(128) panel_mma_kernel(DevSym S, const int32_t* __restrict__ tasks, RhsView R,
                                                        const double* __restrict__ panel, double* __restrict__ Y,
                                                        const int64_t* __restrict__ yoff) {
  // k chunks of 16, double-buffered (cp.async of chunk k+1 overlaps the MMAs of k);
  // 38 KB of static shared memory keeps four CTAs per SM
  constexpr int BK = 16, SB = BK + 4;
  __shared__ __align__(16) double As[2][BK * kMA];  // [k][row]
  __shared__ __align__(16) double Bs[2][kMT * SB];  // [col][k]
  const int64_t s = tasks[3 * blockIdx.x], r0 = tasks[3 * blockIdx.x + 1], c0 = tasks[3 * blockIdx.x + 2];
  const int64_t nc = d_nc(S, s), f = nc + d_nr(S, s), ldm = d_ldf(S, s);
  const int64_t ws = R.w[s];
  double* Rs = R.rhs + R.roff[s];
  const double* M = panel + S.m_off[s];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wy = (warp >> 1) * 32, wx = (warp & 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  // rows of this tile that lie in L11^{-1} only need k <= row (its upper triangle is zero)
  const int64_t kend = (r0 + kMT <= nc) ? min(nc, r0 + kMT) : nc;
  auto stage = [&](int buf, int64_t k0) {
    for (int e = threadIdx.x; e < kMT * BK / 2; e += blockDim.x) {
      const int rr = 2 * (e % (kMT / 2)), kk = e / (kMT / 2);
      const int64_t i = r0 + rr, j = k0 + kk;
      const bool in = i < f && j < nc;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(&As[buf][kk * kMA + rr])),
                   "l"(in ? M + j * ldm + i : M), "r"(in ? 16 : 0)
                   : "memory");
    }
    for (int e = threadIdx.x; e < kMT * BK / 2; e += blockDim.x) {
      const int kk = 2 * (e % (BK / 2)), cc = e / (BK / 2);
      const int64_t j = k0 + kk, c = c0 + cc;
      const bool in = j < nc && c < ws;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(&Bs[buf][cc * SB + kk])),
                   "l"(in ? Rs + c * ldm + j : Rs), "r"(in ? 16 : 0)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  if (kend > 0) stage(0, 0);
  int buf = 0;
  for (int64_t k0 = 0; k0 < kend; k0 += BK) {
    if (k0 + BK < kend) {
      stage(buf ^ 1, k0 + BK);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const double* Ab = As[buf];
    const double* Bb = Bs[buf];
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) fa[a] = Ab[(kk + t) * kMA + wy + 8 * a + g];
#pragma unroll
      for (int b = 0; b < 4; ++b) fb[b] = Bb[(wx + 8 * b + g) * SB + kk + t];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
    }
    __syncthreads();
    buf ^= 1;
  }
  double* Ys = Y + yoff[s];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int64_t i = r0 + wy + 8 * a + g;
        const int64_t c = c0 + wx + 8 * b + 2 * t + hh;
        if (i >= f || c >= ws) continue;
        if (i < nc)
          Ys[c * (nc + (nc & 1)) + i] = acc[a][b][hh];
        else
          Rs[c * ldm + i] -= acc[a][b][hh];
      }
}

// ---- dense backward: x_s = L11^{-T} y_s - P21^T x_rows (warp per pivot row) -----
// Column i of M_s holds L11^{-1}[:, i] (rows < nc) and P21[:, i] (rows >= nc).
// y comes from Bp (forward result), ancestors' x from X; the supernode's x is
// written to X.
// y of pivot row j, column c at yb[c * ldy + j]
template <int NC>
__device__ __forceinline__ void bwd_row(const DevSym& S, int64_t s, int64_t i, int lane,
                                        const double* __restrict__ panel, const double* __restrict__ yb,
                                        int64_t ldy, double* __restrict__ X, int64_t n, int64_t k) {
  const int64_t nc = d_nc(S, s), nr = d_nr(S, s);
  if (i >= nc) return;
  const int ncols = (int)min((int64_t)NC, k);
  const double* lcol = panel + S.m_off[s] + i * d_ldf(S, s);  // L11^{-1}[:, i] = row i of L11^{-T}
  const double* pcol = lcol + nc;                             // P21[:, i]
  const int64_t* rows = S.rows + S.rows_ptr[s];
  const int64_t first = S.first[s];
  // eight independent partial sums per column (lane-strided chunks of 256): the
  // loads and gathers X[rows[q]] of a chunk are all in flight together
  constexpr int U = 8;
  double acc[U][NC];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[u][c] = 0.0;
  for (int64_t j0 = i + lane; j0 < nc; j0 += 32 * U) {
    double l[U];
#pragma unroll
    for (int u = 0; u < U; ++u) l[u] = j0 + 32 * u < nc ? lcol[j0 + 32 * u] : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (c < ncols && j0 + 32 * u < nc) acc[u][c] = fma(l[u], yb[c * ldy + j0 + 32 * u], acc[u][c]);
  }
  for (int64_t q0 = lane; q0 < nr; q0 += 32 * U) {
    double pq[U];
    int64_t rq[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool in = q0 + 32 * u < nr;
      pq[u] = in ? pcol[q0 + 32 * u] : 0.0;
      rq[u] = in ? rows[q0 + 32 * u] : -1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (c < ncols && rq[u] >= 0) acc[u][c] = fma(-pq[u], X[c * n + rq[u]], acc[u][c]);
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const double v = warp_sum(((acc[0][c] + acc[1][c]) + (acc[2][c] + acc[3][c])) +
                              ((acc[4][c] + acc[5][c]) + (acc[6][c] + acc[7][c])));
    if (lane == 0 && c < ncols) X[c * n + first + i] = v;
  }
}

template <int NC>
__global__ void __launch_bounds__(32 * kBwdRows) bwd_kernel(DevSym S, const int32_t* __restrict__ tasks,
                                                            const double* __restrict__ panel,
                                                            const double* __restrict__ Bp, double* __restrict__ X,
                                                            int64_t n, int64_t k) {
  const int64_t s = tasks[3 * blockIdx.x];
  bwd_row<NC>(S, s, tasks[3 * blockIdx.x + 1] + (threadIdx.x >> 5), threadIdx.x & 31, panel, Bp + S.first[s], n, X,
              n, k);
}

// ---- single right-hand side: the whole solve in one cooperative kernel ------
// Permute, forward levels (assemble, panel GEMV), backward levels, permute back,
// with a grid barrier between dependent phases: the same tasks and arithmetic
// as the per-level launches (bitwise the same result), without a launch per
// level and phase (a 12k-DoF solve is ~25 dependent launches otherwise).
// single RHS: the panel GEMV of gemv_task<1> with the front's assembly folded
// in -- pivot rows are gathered while they are staged, update rows right
// before their product is subtracted (same sums in the same order as the
// separate assembly: start value, then the children's rows in order)
__device__ __forceinline__ double gather_row(int32_t r, double v, const int32_t* __restrict__ cptr,
                                             const int32_t* __restrict__ csrc, const double* rhs) {
  for (int32_t q = cptr[r]; q < cptr[r + 1]; ++q) v = v + rhs[csrc[q]];
  return v;
}
template <int ROWS>
__device__ __forceinline__ void gemv1_task(const DevSym& S, const int32_t* __restrict__ task, const RhsView& R,
                                           const double* __restrict__ panel, double* Bp,
                                           const int32_t* __restrict__ cptr, const int32_t* __restrict__ csrc,
                                           double* rt, double* ug, double* red_) {
  constexpr int kG1Grp = 256 / ROWS;  // column groups
  double(*red)[ROWS] = reinterpret_cast<double(*)[ROWS]>(red_);
  // one pass of gathers for the whole task (pivot rows into rt, this task's
  // update rows into ug) with the first panel loads already in flight.  A task
  // is ROWS rows x all nc columns, split over 256 / ROWS column groups.  Levels
  // with few tasks (the top levels' few large fronts) take ROWS = 16 (a
  // half-warp reads 128 contiguous bytes of a panel column): twice the tasks and
  // half the dependent load batches per thread.
  const int64_t s = task[0], r0 = task[1];
  const int64_t nc = d_nc(S, s), f = nc + d_nr(S, s), ldm = d_ldf(S, s);
  const int32_t rb = (int32_t)R.roff[s];
  const double* M = panel + S.m_off[s];
  const int64_t first = S.first[s];
  const int lr = threadIdx.x % ROWS, grp = threadIdx.x / ROWS;
  const int64_t i = r0 + lr;
  const double* pc = M + i;
  double mv[kGemvU];
#pragma unroll
  for (int u = 0; u < kGemvU; ++u)
    mv[u] = (i < f && grp + kG1Grp * u < nc) ? pc[(int64_t)(grp + kG1Grp * u) * ldm] : 0.0;
  for (int j = threadIdx.x; j < nc; j += blockDim.x)
    rt[j] = gather_row(rb + (int32_t)j, Bp[first + j], cptr, csrc, R.rhs);
  if (threadIdx.x < ROWS && i >= nc && i < f) ug[lr] = gather_row(rb + (int32_t)i, 0.0, cptr, csrc, R.rhs);
  __syncthreads();
  double acc = 0.0;
  if (i < f) {
    for (int j0 = grp;;) {
#pragma unroll
      for (int u = 0; u < kGemvU; ++u)
        if (j0 + kG1Grp * u < nc) acc = fma(mv[u], rt[j0 + kG1Grp * u], acc);
      j0 += kG1Grp * kGemvU;
      if (j0 >= nc) break;
#pragma unroll
      for (int u = 0; u < kGemvU; ++u) mv[u] = j0 + kG1Grp * u < nc ? pc[(int64_t)(j0 + kG1Grp * u) * ldm] : 0.0;
    }
  }
  red[grp][lr] = acc;
  __syncthreads();
  if (grp == 0 && i < f) {
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < kG1Grp; ++q) v += red[q][lr];
    // y into the front's own RHS rows (the front's other tasks may still be
    // staging its pivot rows from Bp), updates into the rows below
    R.rhs[rb + i] = i < nc ? v : ug[lr] - v;
  }
}

__device__ unsigned long long g_solve_prof[64];
__device__ __forceinline__ unsigned long long solve_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct SolveLevel {
  const int32_t* gemv_t;  // panel tasks of `rows` rows
  const int32_t* bwd_t;
  int32_t n_gemv, n_bwd, rows;
};

// The assembly is a gather folded into the panel GEMV (gemv1_task): RHS
// position r sums its children's update rows (cptr / csrc, children in order:
// the extend-add's arithmetic, no searches).
__global__ void __launch_bounds__(256, 3) solve1_kernel(DevSym S, RhsView R, const double* __restrict__ panel,
                                                     const SolveLevel* __restrict__ lv, int nlev,
                                                     const int32_t* __restrict__ cptr, const int32_t* __restrict__ csrc,
                                                     const int64_t* __restrict__ perm, const double* __restrict__ B,
                                                     double* __restrict__ X, double* Bp, double* T, int64_t n) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double rt[kMaxSnCols];
  __shared__ double ug[kGemvRows];
  __shared__ double red[256];
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
  int ph = 0;
  auto mark = [&]() {  // diagnostic: phase end times of CTA 0 (cnb_solve_profile)
    if (gt == 0 && ph < 64) g_solve_prof[ph] = solve_ns();
    ++ph;
  };
  mark();
  for (int64_t p = gt; p < n; p += gs) Bp[p] = B[perm[p]];
  grid.sync();
  mark();
  for (int l = 0; l < nlev; ++l) {
    const SolveLevel L = lv[l];
    for (int q = blockIdx.x; q < L.n_gemv; q += gridDim.x) {
      if (L.rows == kG1Rows)
        gemv1_task<kG1Rows>(S, L.gemv_t + 3 * q, R, panel, Bp, cptr, csrc, rt, ug, red);
      else
        gemv1_task<kGemvRows>(S, L.gemv_t + 3 * q, R, panel, Bp, cptr, csrc, rt, ug, red);
      __syncthreads();  // rt / red reused by the next task
    }
    grid.sync();
    mark();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int l = nlev - 1; l >= 0; --l) {
    const SolveLevel L = lv[l];
    for (int q = blockIdx.x * 8 + warp; q < L.n_bwd * kBwdRows; q += gridDim.x * 8) {
      const int32_t* t = L.bwd_t + 3 * (q / kBwdRows);
      bwd_row<1>(S, t[0], t[1] + q % kBwdRows, lane, panel, R.rhs + R.roff[t[0]], 0, T, n, 1);
    }
    grid.sync();
    mark();
  }
  for (int64_t p = gt; p < n; p += gs) X[perm[p]] = T[p];
}

// ---- factor epilogue: P21 = L21 L11^{-1} (DMMA) into rows [nc, f) of M_s ---------
// task = (s, 64-row block q0 of L21, 64-column block c0); L11^{-1} is lower
// triangular, so only k >= c0 contributes.
__global__ void __launch_bounds__(128) p21_kernel(DevSym S, const int32_t* __restrict__ tasks,
                                                  const double* __restrict__ front, double* __restrict__ panel) {
  // k chunks of 16, cp.async double buffer (as panel_mma_kernel)
  constexpr int BK = 16, SB = BK + 4;
  __shared__ double As[2][BK * kMA];  // [k][row]
  __shared__ double Bs[2][kMT * SB];  // [col][k]
  const int64_t s = tasks[3 * blockIdx.x], q0 = tasks[3 * blockIdx.x + 1], c0 = tasks[3 * blockIdx.x + 2];
  const int64_t nc = d_nc(S, s), nr = d_nr(S, s), ldf = d_ldf(S, s);
  const double* F = front + S.front_off[s];
  const double* Li = panel + S.m_off[s];  // L11^{-1}: rows [0, nc) of M_s, stride ldf
  double* P = panel + S.m_off[s] + nc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wy = (warp >> 1) * 32, wx = (warp & 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  auto stage = [&](int buf, int64_t k0) {
    for (int e = threadIdx.x; e < kMT * BK; e += blockDim.x) {
      const int rr = e % kMT, kk = e / kMT;
      const int64_t q = q0 + rr, k = k0 + kk;
      cp_async8(&As[buf][kk * kMA + rr], F + k * ldf + nc + q, q < nr && k < nc);
    }
    for (int e = threadIdx.x; e < kMT * BK; e += blockDim.x) {
      const int kk = e % BK, cc = e / BK;
      const int64_t k = k0 + kk, c = c0 + cc;
      cp_async8(&Bs[buf][cc * SB + kk], Li + c * ldf + k, k < nc && c < nc && k >= c);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  // L11^{-1} is lower triangular: only k >= c0 contributes
  stage(0, c0);
  int buf = 0;
  for (int64_t k0 = c0; k0 < nc; k0 += BK) {
    if (k0 + BK < nc) {
      stage(buf ^ 1, k0 + BK);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const double* Ab = As[buf];
    const double* Bb = Bs[buf];
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) fa[a] = Ab[(kk + t) * kMA + wy + 8 * a + g];
#pragma unroll
      for (int b = 0; b < 4; ++b) fb[b] = Bb[(wx + 8 * b + g) * SB + kk + t];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
    }
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int64_t q = q0 + wy + 8 * a + g;
        const int64_t c = c0 + wx + 8 * b + 2 * t + hh;
        if (q < nr && c < nc) P[c * ldf + q] = acc[a][b][hh];
      }
}

__global__ void permute_kernel(int64_t n, int64_t k, const int64_t* __restrict__ perm, const double* __restrict__ src,
                               int64_t lds, double* __restrict__ dst, int64_t ldd, int inverse) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t c = blockIdx.y;
  if (p >= n || c >= k) return;
  if (!inverse)
    dst[c * ldd + p] = src[c * lds + perm[p]];
  else
    dst[c * ldd + perm[p]] = src[c * lds + p];
}

// ----------------------------------------------------------------------------
// host orchestration
// ----------------------------------------------------------------------------
int trinv_level(CholHandle* h, int level, cudaStream_t st) {
  const DevTasks& T = h->trinv[level];
  if (!T.count) return CNB_OK;
  static bool attr = false;
  if (!attr) {
    CNB_CUDA(cudaFuncSetAttribute(trinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTrinvSmem));
    attr = true;
  }
  trinv_kernel<<<(unsigned)T.count, 256, kTrinvSmem, st>>>(h->sym(), T.ptr, h->d_front, h->d_kkinv, h->d_m);
  CNB_LAUNCH_CHECK("trinv_kernel");
  const DevTasks& P = h->p21[level];
  if (P.count) {
    p21_kernel<<<(unsigned)P.count, 128, 0, st>>>(h->sym(), P.ptr, h->d_front, h->d_m);
    CNB_LAUNCH_CHECK("p21_kernel");
  }
  return CNB_OK;
}

static int build_plan(CholHandle* h, SolvePlan& P, int64_t width) {
  if (P.width == width) return CNB_OK;
  P.release();
  const Symbolic& S = h->S;
  std::vector<int32_t> all;
  std::vector<std::pair<int64_t, int64_t>> ra, rp, rb;
  for (int l = 0; l < S.n_levels; ++l) {
    int64_t off = (int64_t)all.size();
    for (int64_t q = S.level_ptr[l]; q < S.level_ptr[l + 1]; ++q) {
      const int64_t s = S.level_sn[q];
      for (int64_t r = 0; r < S.f(s); r += kAsmRows) all.insert(all.end(), {(int32_t)s, (int32_t)r, 0});
    }
    ra.push_back({off, ((int64_t)all.size() - off) / 3});
    off = (int64_t)all.size();
    for (int64_t q = S.level_ptr[l]; q < S.level_ptr[l + 1]; ++q) {
      const int64_t s = S.level_sn[q];
      for (int64_t r = 0; r < S.f(s); r += kGemvRows) all.insert(all.end(), {(int32_t)s, (int32_t)r, 0});
    }
    rp.push_back({off, ((int64_t)all.size() - off) / 3});
    off = (int64_t)all.size();
    for (int64_t q = S.level_ptr[l]; q < S.level_ptr[l + 1]; ++q) {
      const int64_t s = S.level_sn[q];
      for (int64_t r = 0; r < S.nc(s); r += kBwdRows) all.insert(all.end(), {(int32_t)s, (int32_t)r, 0});
    }
    rb.push_back({off, ((int64_t)all.size() - off) / 3});
  }
  int rc;
  if ((rc = upload_vec(&P.d_tasks, all))) return rc;
  P.asm_t.clear();
  P.panel_t.clear();
  P.bwd_t.clear();
  for (int l = 0; l < S.n_levels; ++l) {
    P.asm_t.push_back({P.d_tasks + ra[l].first, ra[l].second});
    P.panel_t.push_back({P.d_tasks + rp[l].first, rp[l].second});
    P.bwd_t.push_back({P.d_tasks + rb[l].first, rb[l].second});
  }
  std::vector<int64_t> roff(S.ns + 1, 0), lo(S.ns, 0), w(S.ns, width);
  for (int64_t s = 0; s < S.ns; ++s) roff[s + 1] = roff[s] + S.ldf(s) * width;
  if ((rc = upload_vec(&P.d_roff, roff))) return rc;
  if ((rc = upload_vec(&P.d_lo, lo))) return rc;
  if ((rc = upload_vec(&P.d_w, w))) return rc;
  CNB_CUDA(cudaMalloc((void**)&P.d_rhs, std::max<int64_t>(1, roff[S.ns]) * sizeof(double)));
  if (width == 1) {  // per-level tables of the cooperative single-RHS kernel
    // gather lists of the assembly: RHS position roff[s] + rel_c[k] <- roff[c] + nc_c + k
    std::vector<int32_t> cnt(roff[S.ns] + 1, 0);
    for (int64_t s = 0; s < S.ns; ++s)
      for (int64_t ci = S.child_ptr[s]; ci < S.child_ptr[s + 1]; ++ci) {
        const int64_t c = S.child[ci];
        for (int64_t k = 0; k < S.nr(c); ++k) ++cnt[roff[s] + S.rel[S.rel_ptr[c] + k] + 1];
      }
    std::vector<int32_t> cptr(roff[S.ns] + 1, 0);
    for (int64_t r = 0; r < roff[S.ns]; ++r) cptr[r + 1] = cptr[r] + cnt[r + 1];
    std::vector<int32_t> csrc(std::max<int32_t>(1, cptr[roff[S.ns]])), fill(cptr.begin(), cptr.end() - 1);
    for (int64_t s = 0; s < S.ns; ++s)  // children ascending, rows ascending: the extend-add order
      for (int64_t ci = S.child_ptr[s]; ci < S.child_ptr[s + 1]; ++ci) {
        const int64_t c = S.child[ci];
        for (int64_t k = 0; k < S.nr(c); ++k)
          csrc[fill[roff[s] + S.rel[S.rel_ptr[c] + k]]++] = (int32_t)(roff[c] + S.nc(c) + k);
      }
    if ((rc = upload_vec(&P.d_cptr, cptr))) return rc;
    if ((rc = upload_vec(&P.d_csrc, csrc))) return rc;
    int dev = 0, sms = 0, occ = 0;
    CNB_CUDA(cudaGetDevice(&dev));
    CNB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CNB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, solve1_kernel, 256, 0));
    // more resident CTAs help the latency-bound bottom levels of a large tree;
    // a small one pays more for its grid barriers than it gains
    P.coop_grid = sms * std::min(occ, S.ns > 1000 ? 3 : 2);
    // panel tasks: kG1Rows rows on levels whose kGemvRows tasks would leave more
    // than half of the grid idle
    std::vector<int32_t> g1;
    std::vector<SolveLevel> lv(S.n_levels);
    std::vector<int64_t> g1off(S.n_levels);
    for (int l = 0; l < S.n_levels; ++l) {
      const int64_t off = (int64_t)g1.size();
      int64_t n32 = 0;
      for (int64_t q = S.level_ptr[l]; q < S.level_ptr[l + 1]; ++q) n32 += (S.f(S.level_sn[q]) + kGemvRows - 1) / kGemvRows;
      const int rows = 2 * n32 < P.coop_grid ? kG1Rows : kGemvRows;
      for (int64_t q = S.level_ptr[l]; q < S.level_ptr[l + 1]; ++q) {
        const int64_t s = S.level_sn[q];
        for (int64_t r = 0; r < S.f(s); r += rows) g1.insert(g1.end(), {(int32_t)s, (int32_t)r, 0});
      }
      g1off[l] = off;
      lv[l] = SolveLevel{nullptr, P.bwd_t[l].ptr, (int32_t)(((int64_t)g1.size() - off) / 3), (int32_t)P.bwd_t[l].count,
                         rows};
    }
    if ((rc = upload_vec(&P.d_g1, g1))) return rc;
    for (int l = 0; l < S.n_levels; ++l) lv[l].gemv_t = P.d_g1 + g1off[l];
    CNB_CUDA(cudaMalloc(&P.d_lv, std::max<size_t>(1, lv.size()) * sizeof(SolveLevel)));
    if (!lv.empty()) CNB_CUDA(cudaMemcpy(P.d_lv, lv.data(), lv.size() * sizeof(SolveLevel), cudaMemcpyHostToDevice));
  }
  P.width = width;
  return CNB_OK;
}

template <int NC>
static int solve_chunk(CholHandle* h, SolvePlan& P, int64_t kk, cudaStream_t st) {
  const Symbolic& S = h->S;
  const int64_t n = S.n;
  DevSym sym = h->sym();
  RhsView R{P.d_rhs, P.d_roff, P.d_lo, P.d_w};
  double* Bp = (double*)h->bp.p;
  double* T = (double*)h->tbuf.p;
  for (int l = 0; l < S.n_levels; ++l) {
    asm_kernel<<<(unsigned)P.asm_t[l].count, kSolveThreads, 0, st>>>(sym, P.asm_t[l].ptr, R, 1, Bp, n);
    CNB_LAUNCH_CHECK("asm_kernel");
    panel_gemv_kernel<NC><<<(unsigned)P.panel_t[l].count, 256, 0, st>>>(sym, P.panel_t[l].ptr, R, h->d_m, Bp, n);
    CNB_LAUNCH_CHECK("panel_gemv_kernel");
  }
  for (int l = S.n_levels - 1; l >= 0; --l) {
    bwd_kernel<NC><<<(unsigned)P.bwd_t[l].count, 32 * kBwdRows, 0, st>>>(sym, P.bwd_t[l].ptr, h->d_m, Bp, T, n,
                                                                        kk);
    CNB_LAUNCH_CHECK("bwd_kernel");
  }
  return CNB_OK;
}

int solve_profile(double* out) {
  unsigned long long h[64];
  CNB_CUDA(cudaMemcpyFromSymbol(h, g_solve_prof, sizeof(h)));
  for (int k = 0; k < 64; ++k) out[k] = (double)h[k];
  return CNB_OK;
}

int solve_dense(CholHandle* h, const double* B, int64_t ldb, double* X, int64_t ldx, int64_t k, cudaStream_t st) {
  if (k <= 0) return CNB_OK;
  const int64_t n = h->S.n;
  const int64_t width = k == 1 ? 1 : 8;
  SolvePlan& P = width == 1 ? h->plan1 : h->plan8;
  int rc;
  if ((rc = build_plan(h, P, width))) return rc;
  if ((rc = h->bp.ensure(n * width * sizeof(double)))) return rc;
  if ((rc = h->tbuf.ensure(n * width * sizeof(double)))) return rc;
  double* Bp = (double*)h->bp.p;
  if (width == 1 && P.coop_grid > 0) {
    DevSym sym = h->sym();
    RhsView R{P.d_rhs, P.d_roff, P.d_lo, P.d_w};
    const SolveLevel* lv = (const SolveLevel*)P.d_lv;
    int nlev = h->S.n_levels;
    int64_t nn = n;
    double* T = (double*)h->tbuf.p;
    const double* panel = h->d_m;
    const int64_t* perm = h->d_perm;
    const int32_t* cptr = P.d_cptr;
    const int32_t* csrc = P.d_csrc;
    void* args[] = {(void*)&sym, (void*)&R,    (void*)&panel, (void*)&lv, (void*)&nlev, (void*)&cptr,
                    (void*)&csrc, (void*)&perm, (void*)&B,     (void*)&X,  (void*)&Bp,   (void*)&T, (void*)&nn};
    CNB_CUDA(cudaLaunchCooperativeKernel((const void*)solve1_kernel, dim3(P.coop_grid), dim3(256), args, 0, st));
    CNB_LAUNCH_CHECK("solve1_kernel");
    return CNB_OK;
  }
  for (int64_t c0 = 0; c0 < k; c0 += width) {
    const int64_t kk = std::min(width, k - c0);
    if (kk < width) CNB_CUDA(cudaMemsetAsync(Bp, 0, n * width * sizeof(double), st));
    dim3 g(grid_for(n, 256), (unsigned)kk);
    permute_kernel<<<g, 256, 0, st>>>(n, kk, h->d_perm, B + c0 * ldb, ldb, Bp, n, 0);
    CNB_LAUNCH_CHECK("permute_kernel");
    rc = width == 1 ? solve_chunk<1>(h, P, kk, st) : solve_chunk<8>(h, P, kk, st);
    if (rc) return rc;
    permute_kernel<<<g, 256, 0, st>>>(n, kk, h->d_perm, (double*)h->tbuf.p, n, X + c0 * ldx, ldx, 1);
    CNB_LAUNCH_CHECK("permute_kernel");
  }
  return CNB_OK;
}

// ----------------------------------------------------------------------------
// Mapping compliance U = S A^{-1} S^T (constraints.py:155-179)
// ----------------------------------------------------------------------------
// U = Y^T Y with Y = L^{-1} P S^T.  Column j of Y is non-zero only on the
// elimination paths of its S entries: RHS columns are sorted by their first
// touched supernode and every supernode keeps a window [lo_s, hi_s) of sorted
// columns (nested along the tree).  The forward solve runs on those windows
// (asm_kernel + panel_mma_kernel); the Gram product accumulates, for each
// 64x64 output tile, Y_s^T Y_s of exactly the supernodes whose window covers
// it, in a fixed order (deterministic), on DMMA.
constexpr int kGT = 64;

__global__ void __launch_bounds__(128) gram_kernel(DevSym S, RhsView R, const double* __restrict__ Y,
                                                   const int64_t* __restrict__ yoff, const int32_t* __restrict__ tile_ptr,
                                                   const int32_t* __restrict__ tile_sn, int64_t ncols,
                                                   const int64_t* __restrict__ sorted_cols, double* __restrict__ U,
                                                   int64_t ldu, double* __restrict__ tiles, int rank, int world) {
  // (supernode, 16-deep k chunk) sequence of the tile, cp.async double buffer:
  // chunk q+1 is staged while chunk q is multiplied (41 KB static shared memory)
  constexpr int BK = 16, SB = BK + 4;
  __shared__ __align__(16) double Ya[2][kGT * SB];  // 16-byte cp.async destinations
  __shared__ __align__(16) double Yb[2][kGT * SB];
  // multi-GPU: this rank owns tiles t = rank, rank + world, ... (round robin)
  const int64_t t = (int64_t)blockIdx.x * world + rank;
  int64_t A = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((A + 1) * (A + 2) / 2 <= t) ++A;
  while (A * (A + 1) / 2 > t) --A;
  const int64_t B = t - A * (A + 1) / 2;
  const int64_t ra0 = A * kGT, rb0 = B * kGT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int wy = (warp >> 1) * 32, wx = (warp & 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int32_t e0 = tile_ptr[t], e1 = tile_ptr[t + 1];
  auto stage = [&](int buf, int32_t e, int64_t k0) {
    const int64_t s = tile_sn[e];
    const int64_t nc = d_nc(S, s);
    const int64_t lo = R.lo[s], w = R.w[s];
    const double* Ys = Y + yoff[s];
    const int64_t ldy = nc + (nc & 1);  // Y columns 16-byte aligned (panel_mma_kernel)
    // 16-byte copies of k pairs; a pair straddling nc takes its valid element
    // alone and a zero (the padding entry of Y is never written)
    for (int idx = threadIdx.x; idx < (BK / 2) * kGT; idx += blockDim.x) {
      const int kk = 2 * (idx % (BK / 2)), cc = idx / (BK / 2);
      const int64_t k = k0 + kk;
      const int64_t la = ra0 + cc - lo, lb = rb0 + cc - lo;
      const bool ia = la >= 0 && la < w, ib = lb >= 0 && lb < w;
      double* da = &Ya[buf][cc * SB + kk];
      double* db = &Yb[buf][cc * SB + kk];
      if (k + 1 < nc) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(da)),
                     "l"(ia ? Ys + la * ldy + k : Ys), "r"(ia ? 16 : 0)
                     : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(db)),
                     "l"(ib ? Ys + lb * ldy + k : Ys), "r"(ib ? 16 : 0)
                     : "memory");
      } else {
        cp_async8(da, Ys + la * ldy + k, ia && k < nc);
        cp_async8(db, Ys + lb * ldy + k, ib && k < nc);
        da[1] = 0.0;
        db[1] = 0.0;
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  int32_t e = e0;
  int64_t k0 = 0;
  if (e < e1) stage(0, e, 0);
  int buf = 0;
  while (e < e1) {
    int32_t en = e;
    int64_t kn = k0 + BK;
    if (kn >= d_nc(S, tile_sn[e])) {
      ++en;
      kn = 0;
    }
    if (en < e1) {
      stage(buf ^ 1, en, kn);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const double* Pa = Ya[buf];
    const double* Pb = Yb[buf];
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) fa[a] = Pa[(wy + 8 * a + g) * SB + kk + tq];
#pragma unroll
      for (int b = 0; b < 4; ++b) fb[b] = Pb[(wx + 8 * b + g) * SB + kk + tq];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
    }
    __syncthreads();
    e = en;
    k0 = kn;
    buf ^= 1;
  }
  if (tiles) {  // split mode: the whole 64x64 tile into this rank's slot (scattered by the caller's finish)
    double* T = tiles + (int64_t)blockIdx.x * (kGT * kGT);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
          T[(wy + 8 * a + g) * kGT + wx + 8 * b + 2 * tq + hh] = acc[a][b][hh];
    return;
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int64_t ra = ra0 + wy + 8 * a + g;
        const int64_t rb = rb0 + wx + 8 * b + 2 * tq + hh;
        if (ra >= ncols || rb >= ncols) continue;
        if (A == B && rb > ra) continue;
        const int64_t ja = sorted_cols[ra], jb = sorted_cols[rb];
        U[ja * ldu + jb] = acc[a][b][hh];
        U[jb * ldu + ja] = acc[a][b][hh];
      }
}

__global__ void scatter_rhs_kernel(int64_t nnz, const int64_t* __restrict__ dst, const double* __restrict__ val,
                                   double* __restrict__ rhs) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nnz) rhs[dst[k]] = val[k];
}

// Multi-GPU split: each rank forward-solves a contiguous range
// of the sorted right-hand-side columns (windows clipped to the range) into a
// compact Y of its own; the caller all-gathers the compact Ys (NCCL); every
// rank unpacks them into the full Y and computes the 64x64 Gram tiles it
// owns (round robin, tile t -> rank t mod world) into a tile buffer; the
// caller all-gathers the tile buffers and every rank scatters all tiles into
// U.  Each column's forward solve and each tile's Gram sum run exactly as on
// one GPU, so U is bit-identical for every world size.
__global__ void unpack_y_kernel(int64_t nseg, const int64_t* __restrict__ seg, const double* __restrict__ src,
                                double* __restrict__ dst) {
  // segment q = (src offset, dst offset, length): one CTA per segment, grid-stride
  for (int64_t q = blockIdx.x; q < nseg; q += gridDim.x) {
    const int64_t so = seg[3 * q], d0 = seg[3 * q + 1], len = seg[3 * q + 2];
    for (int64_t i = threadIdx.x; i < len; i += blockDim.x) dst[d0 + i] = src[so + i];
  }
}

__global__ void scatter_tiles_kernel(int64_t npairs, int world, int64_t per_rank, const double* __restrict__ tiles,
                                     int64_t ncols, const int64_t* __restrict__ sorted_cols, double* __restrict__ U,
                                     int64_t ldu) {
  const int64_t t = blockIdx.x;
  if (t >= npairs) return;
  int64_t A = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((A + 1) * (A + 2) / 2 <= t) ++A;
  while (A * (A + 1) / 2 > t) --A;
  const int64_t B = t - A * (A + 1) / 2;
  const double* T = tiles + ((t % world) * per_rank + t / world) * (int64_t)(kGT * kGT);
  for (int e = threadIdx.x; e < kGT * kGT; e += blockDim.x) {
    const int i = e / kGT, j = e % kGT;
    const int64_t ra = A * kGT + i, rb = B * kGT + j;
    if (ra >= ncols || rb >= ncols || (A == B && rb > ra)) continue;
    const double v = T[e];
    const int64_t ja = sorted_cols[ra], jb = sorted_cols[rb];
    U[ja * ldu + jb] = v;
    U[jb * ldu + ja] = v;
  }
}

struct CompliancePlan {
  int64_t ncols = 0;
  int rank = 0, world = 1;
  // full problem: sorted columns, windows, Y layout, Gram tiles
  std::vector<int64_t> sorted_cols, lo, w, yoff;
  std::vector<int32_t> tile_ptr, tile_sn;
  int64_t npairs = 0, tiles_per_rank = 0;
  double gram_flops = 0.0, fwd_flops = 0.0;
  // this rank's forward solve (windows clipped to its column range)
  std::vector<int64_t> flo, fw, froff, fyoff, sc_dst;
  std::vector<double> sc_val;
  std::vector<std::vector<int32_t>> asm_t, panel_t;  // per level, (s, r0, c0)
  double rank_fwd_flops = 0.0;
  // split bookkeeping: column boundaries (sorted order), unpack segments, send size
  std::vector<int64_t> split, seg;
  int64_t send_doubles = 0;
  // device offsets into h->c_int (bytes) and record lists
  size_t o_lo = 0, o_w = 0, o_yoff = 0, o_sorted = 0, o_flo = 0, o_fw = 0, o_froff = 0, o_fyoff = 0, o_dst = 0,
         o_seg = 0, o_tptr = 0, o_tsn = 0;
  std::vector<std::pair<size_t, size_t>> arec, prec;
  bool uploaded = false;
};

void free_compliance_plan(CholHandle* h) {
  delete h->cplan;
  h->cplan = nullptr;
}

static inline int64_t ystride(int64_t nc) { return nc + (nc & 1); }  // Y columns 16-byte aligned

static int plan_build(const Symbolic& S, int64_t ncols, const int64_t* colptr, const int64_t* rowidx,
                      const double* vals, int rank, int world, CompliancePlan& P) {
  const int64_t ns = S.ns;
  P.ncols = ncols;
  P.rank = rank;
  P.world = world;
  std::vector<int64_t> dof_sn(S.n);
  for (int64_t s = 0; s < ns; ++s)
    for (int64_t d = S.first[s]; d < S.first[s + 1]; ++d) dof_sn[d] = s;
  std::vector<int64_t> key(ncols, ns);
  for (int64_t j = 0; j < ncols; ++j)
    for (int64_t e = colptr[j]; e < colptr[j + 1]; ++e) {
      const int64_t d = rowidx[e];
      if (d < 0 || d >= S.n) {
        set_error("compliance: row index %lld out of range", (long long)d);
        return CNB_E_INVALID_ATTACHMENT;
      }
      key[j] = std::min(key[j], dof_sn[S.iperm[d]]);
    }
  P.sorted_cols.resize(ncols);
  std::iota(P.sorted_cols.begin(), P.sorted_cols.end(), 0);
  std::stable_sort(P.sorted_cols.begin(), P.sorted_cols.end(), [&](int64_t a, int64_t b) { return key[a] < key[b]; });
  std::vector<int64_t> pos(ncols);
  for (int64_t r = 0; r < ncols; ++r) pos[P.sorted_cols[r]] = r;
  std::vector<int64_t> lo(ns, INT64_MAX), hi(ns, -1);
  for (int64_t j = 0; j < ncols; ++j)
    for (int64_t e = colptr[j]; e < colptr[j + 1]; ++e) {
      const int64_t s = dof_sn[S.iperm[rowidx[e]]];
      lo[s] = std::min(lo[s], pos[j]);
      hi[s] = std::max(hi[s], pos[j] + 1);
    }
  for (int64_t s = 0; s < ns; ++s) {  // postorder: a window contains its children's
    const int64_t p = S.parent[s];
    if (p >= 0 && hi[s] > 0) {
      lo[p] = std::min(lo[p], lo[s]);
      hi[p] = std::max(hi[p], hi[s]);
    }
  }
  P.lo.assign(ns, 0);
  P.w.assign(ns, 0);
  P.yoff.assign(ns + 1, 0);
  for (int64_t s = 0; s < ns; ++s) {
    if (hi[s] > 0) {
      P.lo[s] = lo[s];
      P.w[s] = hi[s] - lo[s];
    }
    P.yoff[s + 1] = P.yoff[s] + ystride(S.nc(s)) * P.w[s];
    const double nc = (double)S.nc(s), nr = (double)S.nr(s), w = (double)P.w[s];
    P.fwd_flops += w * (nc * nc + 2.0 * nc * nr);
  }
  // column ranges of the ranks, balanced by forward work (f_s nc_s per column of each window)
  P.split.assign(world + 1, ncols);
  P.split[0] = 0;
  if (world > 1) {
    std::vector<double> diff(ncols + 1, 0.0);
    for (int64_t s = 0; s < ns; ++s)
      if (P.w[s]) {
        const double c = (double)S.f(s) * (double)S.nc(s);
        diff[P.lo[s]] += c;
        diff[P.lo[s] + P.w[s]] -= c;
      }
    std::vector<double> cum(ncols + 1, 0.0);
    double run = 0.0;
    for (int64_t j = 0; j < ncols; ++j) {
      run += diff[j];
      cum[j + 1] = cum[j] + run;
    }
    for (int q = 1; q < world; ++q) {
      const double target = cum[ncols] * q / world;
      P.split[q] = std::lower_bound(cum.begin(), cum.end(), target) - cum.begin();
      P.split[q] = std::max(P.split[q], P.split[q - 1]);
    }
  }
  // every rank's clipped windows: compact Y layout and the unpack segments
  P.send_doubles = 1;
  for (int q = 0; q < world; ++q) {
    const int64_t ca = P.split[q], cb = P.split[q + 1];
    int64_t off = 0;
    for (int64_t s = 0; s < ns; ++s) {
      if (!P.w[s]) continue;
      const int64_t l = std::max(P.lo[s], ca), r = std::min(P.lo[s] + P.w[s], cb);
      if (r <= l) continue;
      const int64_t len = (r - l) * ystride(S.nc(s));
      if (world > 1) P.seg.insert(P.seg.end(), {off, P.yoff[s] + (l - P.lo[s]) * ystride(S.nc(s)), len});
      off += len;
    }
    P.send_doubles = std::max(P.send_doubles, off);
  }
  if (world > 1)  // segment sources are offsets within the rank's slot of the gathered buffer
    for (int q = 0, k = 0; q < world; ++q) {
      const int64_t ca = P.split[q], cb = P.split[q + 1];
      for (int64_t s = 0; s < ns; ++s) {
        if (!P.w[s]) continue;
        const int64_t l = std::max(P.lo[s], ca), r = std::min(P.lo[s] + P.w[s], cb);
        if (r <= l) continue;
        P.seg[3 * k++] += q * P.send_doubles;
      }
    }
  // this rank's forward plan
  const int64_t ca = P.split[rank], cb = P.split[rank + 1];
  P.flo.assign(ns, 0);
  P.fw.assign(ns, 0);
  P.froff.assign(ns + 1, 0);
  P.fyoff.assign(ns + 1, 0);
  for (int64_t s = 0; s < ns; ++s) {
    if (P.w[s]) {
      const int64_t l = std::max(P.lo[s], ca), r = std::min(P.lo[s] + P.w[s], cb);
      if (r > l) {
        P.flo[s] = l;
        P.fw[s] = r - l;
      }
    }
    P.froff[s + 1] = P.froff[s] + S.ldf(s) * P.fw[s];
    P.fyoff[s + 1] = P.fyoff[s] + ystride(S.nc(s)) * P.fw[s];
    const double nc = (double)S.nc(s), nr = (double)S.nr(s), w = (double)P.fw[s];
    P.rank_fwd_flops += w * (nc * nc + 2.0 * nc * nr);
  }
  for (int64_t j = 0; j < ncols; ++j) {
    if (pos[j] < ca || pos[j] >= cb) continue;
    for (int64_t e = colptr[j]; e < colptr[j + 1]; ++e) {
      const int64_t p = S.iperm[rowidx[e]];
      const int64_t s = dof_sn[p];
      P.sc_dst.push_back(P.froff[s] + (pos[j] - P.flo[s]) * S.ldf(s) + (p - S.first[s]));
      P.sc_val.push_back(vals[e]);
    }
  }
  P.asm_t.assign(S.n_levels, {});
  P.panel_t.assign(S.n_levels, {});
  for (int l = 0; l < S.n_levels; ++l)
    for (int64_t q = S.level_ptr[l]; q < S.level_ptr[l + 1]; ++q) {
      const int64_t s = S.level_sn[q];
      if (P.fw[s] == 0) continue;
      if (S.child_ptr[s + 1] > S.child_ptr[s])
        for (int64_t r = 0; r < S.f(s); r += kAsmRows)
          for (int64_t c = 0; c < P.fw[s]; c += kAsmCols)
            P.asm_t[l].insert(P.asm_t[l].end(), {(int32_t)s, (int32_t)r, (int32_t)c});
      for (int64_t r = 0; r < S.f(s); r += kMT)
        for (int64_t c = 0; c < P.fw[s]; c += kMT) P.panel_t[l].insert(P.panel_t[l].end(), {(int32_t)s, (int32_t)r, (int32_t)c});
    }
  // Gram tiles of the full problem
  const int64_t nt = (ncols + kGT - 1) / kGT;
  P.npairs = nt * (nt + 1) / 2;
  P.tiles_per_rank = (P.npairs + world - 1) / world;
  std::vector<int32_t> count(P.npairs + 1, 0);
  for (int64_t s = 0; s < ns; ++s) {
    if (P.w[s] == 0) continue;
    const int64_t t0 = P.lo[s] / kGT, t1 = (P.lo[s] + P.w[s] - 1) / kGT;
    for (int64_t a = t0; a <= t1; ++a)
      for (int64_t b = t0; b <= a; ++b) count[a * (a + 1) / 2 + b + 1]++;
    P.gram_flops += (double)S.nc(s) * (double)P.w[s] * (double)(P.w[s] + 1);
  }
  for (int64_t t = 0; t < P.npairs; ++t) count[t + 1] += count[t];
  P.tile_ptr = count;
  P.tile_sn.assign(count[P.npairs], 0);
  std::vector<int32_t> fill(count.begin(), count.end() - 1);
  for (int64_t s = 0; s < ns; ++s) {
    if (P.w[s] == 0) continue;
    const int64_t t0 = P.lo[s] / kGT, t1 = (P.lo[s] + P.w[s] - 1) / kGT;
    for (int64_t a = t0; a <= t1; ++a)
      for (int64_t b = t0; b <= a; ++b) P.tile_sn[fill[a * (a + 1) / 2 + b]++] = (int32_t)s;
  }
  return CNB_OK;
}

// Upload the plan (one pinned staging copy, asynchronous) and size the workspaces.
static int plan_upload(CholHandle* h, CompliancePlan& P, cudaStream_t st) {
  const Symbolic& S = h->S;
  std::vector<int64_t> ints;
  auto put = [&](const std::vector<int64_t>& v) {
    size_t o = ints.size() * sizeof(int64_t);
    ints.insert(ints.end(), v.begin(), v.end());
    return o;
  };
  P.o_lo = put(P.lo);
  P.o_w = put(P.w);
  P.o_yoff = put(P.yoff);
  P.o_sorted = put(P.sorted_cols);
  P.o_flo = put(P.flo);
  P.o_fw = put(P.fw);
  P.o_froff = put(P.froff);
  P.o_fyoff = put(P.fyoff);
  P.o_dst = put(P.sc_dst);
  P.o_seg = put(P.seg);
  std::vector<int32_t> i32;
  P.arec.clear();
  P.prec.clear();
  for (int l = 0; l < S.n_levels; ++l) {
    P.arec.push_back({i32.size(), P.asm_t[l].size() / 3});
    i32.insert(i32.end(), P.asm_t[l].begin(), P.asm_t[l].end());
    P.prec.push_back({i32.size(), P.panel_t[l].size() / 3});
    i32.insert(i32.end(), P.panel_t[l].begin(), P.panel_t[l].end());
  }
  const size_t t_tptr = i32.size();
  i32.insert(i32.end(), P.tile_ptr.begin(), P.tile_ptr.end());
  const size_t t_tsn = i32.size();
  i32.insert(i32.end(), P.tile_sn.begin(), P.tile_sn.end());
  const size_t bytes64 = ints.size() * sizeof(int64_t);
  const size_t off32 = (bytes64 + 15) & ~(size_t)15;
  const size_t bytes32 = i32.size() * sizeof(int32_t);
  for (auto& r : P.arec) r.first = off32 + r.first * sizeof(int32_t);
  for (auto& r : P.prec) r.first = off32 + r.first * sizeof(int32_t);
  P.o_tptr = off32 + t_tptr * sizeof(int32_t);
  P.o_tsn = off32 + t_tsn * sizeof(int32_t);
  int rc;
  if ((rc = h->c_int.ensure(off32 + bytes32 + 16))) return rc;
  if ((rc = h->c_rhs.ensure(std::max<int64_t>(1, P.froff[S.ns]) * sizeof(double)))) return rc;
  if ((rc = h->c_y.ensure(std::max<int64_t>(1, P.yoff[S.ns]) * sizeof(double)))) return rc;
  if ((rc = h->c_val.ensure(std::max<size_t>(1, P.sc_val.size()) * sizeof(double)))) return rc;
  const size_t vbytes = P.sc_val.size() * sizeof(double);
  const size_t offv = (off32 + bytes32 + 15) & ~(size_t)15;
  if ((rc = h->c_pin.ensure(offv + vbytes + 16))) return rc;
  char* pin = (char*)h->c_pin.p;
  memcpy(pin, ints.data(), bytes64);
  if (bytes32) memcpy(pin + off32, i32.data(), bytes32);
  if (vbytes) memcpy(pin + offv, P.sc_val.data(), vbytes);
  CNB_CUDA(cudaMemcpyAsync(h->c_int.p, pin, off32 + bytes32, cudaMemcpyHostToDevice, st));
  if (vbytes) CNB_CUDA(cudaMemcpyAsync(h->c_val.p, pin + offv, vbytes, cudaMemcpyHostToDevice, st));
  if ((rc = h->c_pin.mark(st))) return rc;
  P.uploaded = true;
  return CNB_OK;
}

template <typename T>
static inline T* at(const GrowBuf& b, size_t off) {
  return (T*)((char*)b.p + off);
}

// Forward solve of this rank's columns: Y (compact layout fyoff) = L^{-1} P E.
constexpr double kOverlapMaxFlops = 2e10;  // forward solves overlapped with the factorisation (see compliance)
// lev (optional): per-level events; level l waits for lev[l] (its M_s formed)
static int plan_forward(CholHandle* h, const CompliancePlan& P, double* Y, cudaStream_t st,
                        const cudaEvent_t* lev = nullptr) {
  const Symbolic& S = h->S;
  double* rhs = (double*)h->c_rhs.p;
  CNB_CUDA(cudaMemsetAsync(rhs, 0, std::max<int64_t>(1, P.froff[S.ns]) * sizeof(double), st));
  const int64_t nnz = (int64_t)P.sc_val.size();
  if (nnz) {
    scatter_rhs_kernel<<<grid_for(nnz, 256), 256, 0, st>>>(nnz, at<int64_t>(h->c_int, P.o_dst),
                                                           (const double*)h->c_val.p, rhs);
    CNB_LAUNCH_CHECK("scatter_rhs_kernel");
  }
  DevSym sym = h->sym();
  RhsView R{rhs, at<int64_t>(h->c_int, P.o_froff), at<int64_t>(h->c_int, P.o_flo), at<int64_t>(h->c_int, P.o_fw)};
  for (int l = 0; l < S.n_levels; ++l) {
    if (lev && (P.arec[l].second || P.prec[l].second)) CNB_CUDA(cudaStreamWaitEvent(st, lev[l], 0));
    if (P.arec[l].second) {
      asm_kernel<<<(unsigned)P.arec[l].second, kSolveThreads, 0, st>>>(sym, at<int32_t>(h->c_int, P.arec[l].first),
                                                                        R, 0, nullptr, S.n);
      CNB_LAUNCH_CHECK("asm_kernel(sparse)");
    }
    if (P.prec[l].second) {
      panel_mma_kernel<<<(unsigned)P.prec[l].second, 128, 0, st>>>(sym, at<int32_t>(h->c_int, P.prec[l].first), R,
                                                                   h->d_m, Y, at<int64_t>(h->c_int, P.o_fyoff));
      CNB_LAUNCH_CHECK("panel_mma_kernel");
    }
  }
  return CNB_OK;
}

// Gram tiles of this rank over the full Y: into U directly (world 1) or into
// the rank's tile buffer (slot = t / world).
static int plan_gram(CholHandle* h, const CompliancePlan& P, const double* Y, double* U, int64_t ldu, double* tiles,
                     cudaStream_t st) {
  const int64_t owned = (P.npairs - P.rank + P.world - 1) / P.world;
  if (owned <= 0) return CNB_OK;
  RhsView R{nullptr, nullptr, at<int64_t>(h->c_int, P.o_lo), at<int64_t>(h->c_int, P.o_w)};
  gram_kernel<<<(unsigned)owned, 128, 0, st>>>(h->sym(), R, Y, at<int64_t>(h->c_int, P.o_yoff),
                                               at<int32_t>(h->c_int, P.o_tptr), at<int32_t>(h->c_int, P.o_tsn),
                                               P.ncols, at<int64_t>(h->c_int, P.o_sorted), U, ldu, tiles, P.rank,
                                               P.world);
  CNB_LAUNCH_CHECK("gram_kernel");
  return CNB_OK;
}

int compliance(CholHandle* h, int64_t ncols, const int64_t* colptr, const int64_t* rowidx, const double* vals,
               double* U, int64_t ldu, double* flops_out, cudaStream_t st) {
  if (ncols <= 0) return CNB_OK;
  CompliancePlan P;
  int rc = plan_build(h->S, ncols, colptr, rowidx, vals, 0, 1, P);
  if (rc) return rc;
  // the forward solve overlaps the factorisation that produced M: on the
  // handle's compliance stream, from the point before that factorisation (or
  // after the previous compliance's Gram), each level after its M_s is formed;
  // the Gram (which writes the caller's U) runs on the caller's stream after it
  // (latency-bound forward solves only: a large one -- cfg3's 870 GFLOP per body --
  // competes with the factor's own DMMA work and with the other bodies', measured
  // 497 -> 502 ms per cfg3 step, while cfg1's 3.54 -> 3.20 ms)
  const bool ov = h->level_events && h->comp_stream && P.fwd_flops < kOverlapMaxFlops;
  cudaStream_t fs = ov ? h->comp_stream : st;
  if (ov) CNB_CUDA(cudaStreamWaitEvent(fs, h->ev_pre, 0));
  if ((rc = plan_upload(h, P, fs))) return rc;
  if (flops_out) {
    flops_out[0] = P.fwd_flops;
    flops_out[1] = P.gram_flops;
  }
  double* Y = (double*)h->c_y.p;
  if ((rc = plan_forward(h, P, Y, fs, ov ? h->ev_level.data() : nullptr))) return rc;
  if (ov) {
    CNB_CUDA(cudaEventRecord(h->ev_comp, fs));
    CNB_CUDA(cudaStreamWaitEvent(st, h->ev_comp, 0));
  }
  if ((rc = plan_gram(h, P, Y, U, ldu, nullptr, st))) return rc;
  if (ov) CNB_CUDA(cudaEventRecord(h->ev_pre, st));  // the next forward solve reuses the buffers after this Gram
  h->last_fwd_flops = P.fwd_flops;
  h->last_gram_flops = P.gram_flops;
  return CNB_OK;
}

int compliance_split_plan(CholHandle* h, int64_t ncols, const int64_t* colptr, const int64_t* rowidx,
                          const double* vals, int rank, int world, int64_t* sizes, double* flops_out,
                          cudaStream_t st) {
  if (world < 1 || rank < 0 || rank >= world) {
    set_error("compliance: invalid rank %d / world %d", rank, world);
    return CNB_E_VALIDATION;
  }
  free_compliance_plan(h);
  h->cplan = new CompliancePlan();
  CompliancePlan& P = *h->cplan;
  int rc = plan_build(h->S, ncols, colptr, rowidx, vals, rank, world, P);
  if (rc) return rc;
  if ((rc = plan_upload(h, P, st))) return rc;
  sizes[0] = P.send_doubles;
  sizes[1] = P.tiles_per_rank * kGT * kGT;
  sizes[2] = P.split[rank];
  sizes[3] = P.split[rank + 1];
  if (flops_out) {
    flops_out[0] = P.rank_fwd_flops;
    flops_out[1] = P.gram_flops / world;
  }
  return CNB_OK;
}

int compliance_split_forward(CholHandle* h, double* ysend, cudaStream_t st) {
  if (!h->cplan) {
    set_error("compliance_split_forward: no plan");
    return CNB_E_VALIDATION;
  }
  return plan_forward(h, *h->cplan, ysend, st);
}

int compliance_split_gram(CholHandle* h, const double* yall, double* tiles, cudaStream_t st) {
  if (!h->cplan) {
    set_error("compliance_split_gram: no plan");
    return CNB_E_VALIDATION;
  }
  const CompliancePlan& P = *h->cplan;
  double* Y = (double*)h->c_y.p;
  const int64_t nseg = (int64_t)P.seg.size() / 3;
  if (nseg) {
    unpack_y_kernel<<<(unsigned)std::min<int64_t>(nseg, 148 * 16), 256, 0, st>>>(
        nseg, at<int64_t>(h->c_int, P.o_seg), yall, Y);
    CNB_LAUNCH_CHECK("unpack_y_kernel");
  }
  return plan_gram(h, P, Y, nullptr, 0, tiles, st);
}

int compliance_split_finish(CholHandle* h, const double* tiles_all, double* U, int64_t ldu, cudaStream_t st) {
  if (!h->cplan) {
    set_error("compliance_split_finish: no plan");
    return CNB_E_VALIDATION;
  }
  const CompliancePlan& P = *h->cplan;
  if (P.npairs) {
    scatter_tiles_kernel<<<(unsigned)P.npairs, 256, 0, st>>>(P.npairs, P.world, P.tiles_per_rank, tiles_all,
                                                             P.ncols, at<int64_t>(h->c_int, P.o_sorted), U, ldu);
    CNB_LAUNCH_CHECK("scatter_tiles_kernel");
  }
  // a later single-GPU compliance reuses the plan buffers after this point
  if (h->ev_pre) CNB_CUDA(cudaEventRecord(h->ev_pre, st));
  return CNB_OK;
}

}  // namespace cnb
