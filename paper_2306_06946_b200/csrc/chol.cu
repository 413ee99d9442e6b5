// GPU numeric phases of the supernodal multifrontal Cholesky.
//
// Reference being replaced: Factorization (linalg.py:58-106) — SuperLU
// factorisation, solve, solve_multi.  NotSPD is raised for a non-positive
// (or NaN) pivot exactly where the reference checks U's diagonal
// (linalg.py:77-84).
//
// Factorisation, level by level of the supernodal tree (leaves first):
//   scatter A into the fronts (once) -> extend-add children's update blocks
//   (parent-column-owner tasks, children visited in order: deterministic, no
//   atomics) -> dense partial Cholesky of every front of the level:
//   per 32-column panel: POTRF (one CTA per front), TRSM (64-row chunks),
//   SYRK trailing update on 64x64 tiles with fp64 tensor-core MMA
//   (mma.sync m8n8k4 f64 -> SASS DMMA; tcgen05 has no f64 kind).
//
// Solves (forward L, backward L^T) run over the same fronts with per-front
// right-hand-side blocks R_s (f_s x w columns, column-major) so that child
// contributions are pulled by the parent, again deterministically.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <numeric>
#include <stdexcept>
#include <string>

#include "chol.h"
#include "common.cuh"

namespace cnb {

// ----------------------------------------------------------------------------
// device views of the symbolic structure
// ----------------------------------------------------------------------------
struct DevSym {
  const int64_t* first;
  const int64_t* rows_ptr;
  const int64_t* rows;
  const int64_t* front_off;
  const int64_t* child_ptr;
  const int64_t* child;
  const int64_t* rel_ptr;
  const int32_t* rel;
};

__device__ __forceinline__ int64_t d_nc(const DevSym& S, int64_t s) { return S.first[s + 1] - S.first[s]; }
__device__ __forceinline__ int64_t d_nr(const DevSym& S, int64_t s) { return S.rows_ptr[s + 1] - S.rows_ptr[s]; }

// ---- scatter A values into the fronts --------------------------------------
__global__ void scatter_kernel(int64_t nmap, const int64_t* __restrict__ src, const int64_t* __restrict__ dst,
                               const double* __restrict__ vals, double* __restrict__ front) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nmap) front[dst[k]] = vals[src[k]];
}

// ---- extend-add: task = (parent p, parent col range [lo, hi)) ---------------
// For every child c of p (ascending), every child update column k whose
// parent column rel[k] lies in [lo, hi): F_p[rel[i], rel[k]] += U_c[i, k], i >= k.
__global__ void __launch_bounds__(256) extend_add_kernel(DevSym S, const int32_t* __restrict__ tasks,
                                                         double* __restrict__ front) {
  const int32_t p = tasks[3 * blockIdx.x], lo = tasks[3 * blockIdx.x + 1], hi = tasks[3 * blockIdx.x + 2];
  const int64_t fp = d_nc(S, p) + d_nr(S, p);
  double* Fp = front + S.front_off[p];
  for (int64_t ci = S.child_ptr[p]; ci < S.child_ptr[p + 1]; ++ci) {
    const int64_t c = S.child[ci];
    const int64_t ncc = d_nc(S, c), nrc = d_nr(S, c), fc = ncc + nrc;
    const int32_t* rel = S.rel + S.rel_ptr[c];
    // child columns mapping into [lo, hi): rel is increasing
    int64_t k0 = 0, k1 = nrc;
    {
      int64_t a = 0, b = nrc;
      while (a < b) {
        int64_t m = (a + b) >> 1;
        if (rel[m] < lo) a = m + 1; else b = m;
      }
      k0 = a;
      a = k0;
      b = nrc;
      while (a < b) {
        int64_t m = (a + b) >> 1;
        if (rel[m] < hi) a = m + 1; else b = m;
      }
      k1 = a;
    }
    const double* Fc = front + S.front_off[c];
    for (int64_t k = k0; k < k1; ++k) {
      const double* uc = Fc + (ncc + k) * fc + ncc;  // column k of U_c
      double* fcol = Fp + (int64_t)rel[k] * fp;
      for (int64_t i = k + threadIdx.x; i < nrc; i += blockDim.x) fcol[rel[i]] += uc[i];
    }
    __syncthreads();
  }
}

// ---- POTRF of the kw x kw diagonal block of panel k0 (one CTA per front) ----
__global__ void __launch_bounds__(256) potrf_kernel(DevSym S, const int32_t* __restrict__ tasks, int k0,
                                                    double* __restrict__ front, DevStatus* st) {
  __shared__ double a[kPanel][kPanel + 1];
  const int64_t s = tasks[blockIdx.x];
  const int64_t nc = d_nc(S, s), f = nc + d_nr(S, s);
  const int kw = (int)min((int64_t)kPanel, nc - k0);
  double* F = front + S.front_off[s];
  for (int e = threadIdx.x; e < kw * kw; e += blockDim.x) {
    int i = e % kw, j = e / kw;
    a[i][j] = (i >= j) ? F[(int64_t)(k0 + j) * f + k0 + i] : 0.0;
  }
  __syncthreads();
  for (int j = 0; j < kw; ++j) {
    if (threadIdx.x == 0) {
      double d = a[j][j];
      if (!(d > 0.0)) {
        raise_status(st, CNB_E_NOT_SPD, (int)(S.first[s] + k0 + j), d);
        d = nan("");
      }
      a[j][j] = sqrt(d);
    }
    __syncthreads();
    const double piv = a[j][j];
    for (int i = j + 1 + threadIdx.x; i < kw; i += blockDim.x) a[i][j] /= piv;
    __syncthreads();
    const int rem = kw - j - 1;
    for (int e = threadIdx.x; e < rem * rem; e += blockDim.x) {
      int i = j + 1 + e % rem, l = j + 1 + e / rem;
      if (i >= l) a[i][l] -= a[i][j] * a[l][j];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < kw * kw; e += blockDim.x) {
    int i = e % kw, j = e / kw;
    if (i >= j) F[(int64_t)(k0 + j) * f + k0 + i] = a[i][j];
  }
}

// ---- TRSM: rows below the diagonal block, X L_kk^T = B (task = front, chunk) -
__global__ void __launch_bounds__(kTile) trsm_kernel(DevSym S, const int32_t* __restrict__ tasks, int k0,
                                                     double* __restrict__ front) {
  __shared__ double L[kPanel][kPanel + 1];
  const int64_t s = tasks[2 * blockIdx.x];
  const int64_t chunk = tasks[2 * blockIdx.x + 1];
  const int64_t nc = d_nc(S, s), f = nc + d_nr(S, s);
  const int kw = (int)min((int64_t)kPanel, nc - k0);
  double* F = front + S.front_off[s];
  for (int e = threadIdx.x; e < kw * kw; e += blockDim.x) {
    int i = e % kw, j = e / kw;
    L[i][j] = (i >= j) ? F[(int64_t)(k0 + j) * f + k0 + i] : 0.0;
  }
  __syncthreads();
  const int64_t r = k0 + kw + chunk * kTile + threadIdx.x;
  if (r >= f) return;
  double x[kPanel];
#pragma unroll
  for (int j = 0; j < kPanel; ++j) x[j] = j < kw ? F[(int64_t)(k0 + j) * f + r] : 0.0;
#pragma unroll
  for (int j = 0; j < kPanel; ++j) {
    if (j < kw) {
      double v = x[j];
#pragma unroll
      for (int l = 0; l < j; ++l) v = fma(-x[l], L[j][l], v);
      x[j] = v / L[j][j];
    }
  }
#pragma unroll
  for (int j = 0; j < kPanel; ++j)
    if (j < kw) F[(int64_t)(k0 + j) * f + r] = x[j];
}

// ---- SYRK trailing update on a 64x64 tile with DMMA --------------------------
// C[rows ti, cols tj] -= P[rows ti, :] * P[rows tj, :]^T, P = panel columns.
// 4 warps, each a 32x32 quadrant = 4x4 fragments of 8x8.
constexpr int kSP = kPanel + 4;  // smem row stride (== 4 mod 16 doubles: conflict-free fragments)
__global__ void __launch_bounds__(128) syrk_kernel(DevSym S, const int32_t* __restrict__ tasks, int k0,
                                                   double* __restrict__ front) {
  __shared__ double Pi[kTile * kSP];
  __shared__ double Pj[kTile * kSP];
  const int64_t s = tasks[3 * blockIdx.x];
  const int ti = tasks[3 * blockIdx.x + 1], tj = tasks[3 * blockIdx.x + 2];
  const int64_t nc = d_nc(S, s), f = nc + d_nr(S, s);
  const int kw = (int)min((int64_t)kPanel, nc - k0);
  const int64_t t0 = k0 + kw;
  const int64_t r0 = t0 + (int64_t)ti * kTile, c0 = t0 + (int64_t)tj * kTile;
  double* F = front + S.front_off[s];
  for (int e = threadIdx.x; e < kTile * kPanel; e += blockDim.x) {
    const int rr = e % kTile, kk = e / kTile;
    const bool kin = kk < kw;
    const int64_t ri = r0 + rr, rj = c0 + rr;
    Pi[rr * kSP + kk] = (kin && ri < f) ? F[(int64_t)(k0 + kk) * f + ri] : 0.0;
    Pj[rr * kSP + kk] = (kin && rj < f) ? F[(int64_t)(k0 + kk) * f + rj] : 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wy = (warp >> 1) * 32, wx = (warp & 1) * 32;
  if (ti == tj && wx > wy) return;  // strictly-upper quadrant of a diagonal tile
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int kk = 0; kk < kw; kk += 4) {
    double fa[4], fb[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) fa[a] = Pi[(wy + 8 * a + g) * kSP + kk + t];
#pragma unroll
    for (int b = 0; b < 4; ++b) fb[b] = Pj[(wx + 8 * b + g) * kSP + kk + t];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t r = r0 + wy + 8 * a + g;
        const int64_t c = c0 + wx + 8 * b + 2 * t + h;
        if (r < f && c < f && r >= c) F[c * f + r] -= acc[a][b][h];
      }
}

// ----------------------------------------------------------------------------
// forward / backward substitution over front RHS blocks
// ----------------------------------------------------------------------------
// RHS block of supernode s: R_s = rhs + roff[s], f_s rows x w_s columns,
// column-major (ld = f_s); window [lo_s, lo_s + w_s) of the global columns.
struct RhsView {
  double* rhs;
  const int64_t* roff;  // per supernode
  const int64_t* lo;    // per supernode (global column of R_s column 0)
  const int64_t* w;     // per supernode
};

// Dense-mode task: (s, global column chunk c0).  Init from Bp (permuted,
// column-major n x k), extend-add children, then forward-solve the front.
constexpr int kFwdCols = 8;
__global__ void __launch_bounds__(128) fwd_kernel(DevSym S, const int32_t* __restrict__ tasks, int dense,
                                                  const double* __restrict__ front, RhsView R, double* Bp,
                                                  int64_t n) {
  const int64_t s = tasks[2 * blockIdx.x];
  const int64_t cb = tasks[2 * blockIdx.x + 1];  // local column chunk start within s's window
  const int64_t nc = d_nc(S, s), nr = d_nr(S, s), f = nc + nr;
  const int64_t ws = R.w[s], los = R.lo[s];
  const int ncols = (int)min((int64_t)kFwdCols, ws - cb);
  double* Rs = R.rhs + R.roff[s];
  const double* F = front + S.front_off[s];
  const int64_t first = S.first[s];
  if (dense) {
    for (int cc = 0; cc < ncols; ++cc) {
      const int64_t gc = los + cb + cc;
      double* col = Rs + (cb + cc) * f;
      for (int64_t i = threadIdx.x; i < f; i += blockDim.x) col[i] = i < nc ? Bp[gc * n + first + i] : 0.0;
    }
    __syncthreads();
  }
  // extend-add children
  for (int64_t ci = S.child_ptr[s]; ci < S.child_ptr[s + 1]; ++ci) {
    const int64_t c = S.child[ci];
    const int64_t ncc = d_nc(S, c), nrc = d_nr(S, c), fc = ncc + nrc;
    const int64_t off = R.lo[c] - los;  // child's window start inside s's window
    const int32_t* rel = S.rel + S.rel_ptr[c];
    const double* Rc = R.rhs + R.roff[c];
    for (int cc = 0; cc < ncols; ++cc) {
      const int64_t lc = cb + cc - off;  // child's local column
      if (lc < 0 || lc >= R.w[c]) continue;
      const double* src = Rc + lc * fc + ncc;
      double* dst = Rs + (cb + cc) * f;
      for (int64_t i = threadIdx.x; i < nrc; i += blockDim.x) dst[rel[i]] += src[i];
    }
    __syncthreads();
  }
  // forward solve: blocks of 32 pivot columns; warp 0 solves the triangle,
  // every thread then updates the rows below with the block's solution.
  __shared__ double y[32][kFwdCols];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t kb = 0; kb < nc; kb += 32) {
    const int bw = (int)min((int64_t)32, nc - kb);
    if (warp == 0) {
      for (int cc = 0; cc < ncols; ++cc) {
        double* col = Rs + (cb + cc) * f;
        double v = lane < bw ? col[kb + lane] : 0.0;
        for (int j = 0; j < bw; ++j) {
          double yj = 0.0;
          if (lane == j) yj = v / F[(kb + j) * f + kb + j];
          yj = __shfl_sync(0xffffffffu, yj, j);
          if (lane > j && lane < bw) v = fma(-F[(kb + j) * f + kb + lane], yj, v);
          if (lane == j) v = yj;
        }
        if (lane < bw) {
          col[kb + lane] = v;
          y[lane][cc] = v;
        }
      }
    }
    __syncthreads();
    for (int64_t i = kb + bw + threadIdx.x; i < f; i += blockDim.x) {
      double acc[kFwdCols];
#pragma unroll
      for (int cc = 0; cc < kFwdCols; ++cc) acc[cc] = 0.0;
      for (int j = 0; j < bw; ++j) {
        const double l = F[(kb + j) * f + i];
#pragma unroll
        for (int cc = 0; cc < kFwdCols; ++cc) acc[cc] = fma(l, y[j][cc], acc[cc]);
      }
      for (int cc = 0; cc < ncols; ++cc) Rs[(cb + cc) * f + i] -= acc[cc];
    }
    __syncthreads();
  }
  if (dense) {
    for (int cc = 0; cc < ncols; ++cc) {
      const int64_t gc = los + cb + cc;
      const double* col = Rs + (cb + cc) * f;
      for (int64_t i = threadIdx.x; i < nc; i += blockDim.x) Bp[gc * n + first + i] = col[i];
    }
  }
}

// Backward solve (dense mode): X_s = L11^{-T} (Y_s - L21^T X[rows_s]).
// Bp holds Y on entry for not-yet-processed supernodes and X for ancestors.
__global__ void __launch_bounds__(128) bwd_kernel(DevSym S, const int32_t* __restrict__ tasks,
                                                  const double* __restrict__ front, double* Bp, int64_t n,
                                                  int64_t k) {
  const int64_t s = tasks[2 * blockIdx.x];
  const int64_t c0 = tasks[2 * blockIdx.x + 1];
  const int ncols = (int)min((int64_t)kFwdCols, k - c0);
  const int64_t nc = d_nc(S, s), nr = d_nr(S, s), f = nc + nr;
  const double* F = front + S.front_off[s];
  const int64_t first = S.first[s];
  const int64_t* rows = S.rows + S.rows_ptr[s];
  // r_i = Y_i - sum_q L[nc+q][i] X[rows[q]]
  for (int64_t i = threadIdx.x; i < nc; i += blockDim.x) {
    double acc[kFwdCols];
#pragma unroll
    for (int cc = 0; cc < kFwdCols; ++cc) acc[cc] = 0.0;
    const double* lcol = F + i * f + nc;
    for (int64_t q = 0; q < nr; ++q) {
      const double l = lcol[q];
      const int64_t rq = rows[q];
#pragma unroll
      for (int cc = 0; cc < kFwdCols; ++cc)
        if (cc < ncols) acc[cc] = fma(l, Bp[(c0 + cc) * n + rq], acc[cc]);
    }
    for (int cc = 0; cc < ncols; ++cc) Bp[(c0 + cc) * n + first + i] -= acc[cc];
  }
  __syncthreads();
  // L11^T x = r, blocks of 32 from the bottom
  __shared__ double xs[32][kFwdCols];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nblk = (nc + 31) / 32;
  for (int64_t bi = nblk - 1; bi >= 0; --bi) {
    const int64_t kb = bi * 32;
    const int bw = (int)min((int64_t)32, nc - kb);
    if (warp == 0) {
      for (int cc = 0; cc < ncols; ++cc) {
        double* col = Bp + (c0 + cc) * n + first;
        double v = lane < bw ? col[kb + lane] : 0.0;
        for (int j = bw - 1; j >= 0; --j) {
          double xj = 0.0;
          if (lane == j) xj = v / F[(kb + j) * f + kb + j];
          xj = __shfl_sync(0xffffffffu, xj, j);
          // row lane (< j) of L^T: L[j][lane]
          if (lane < j) v = fma(-F[(kb + lane) * f + kb + j], xj, v);
          if (lane == j) v = xj;
        }
        if (lane < bw) {
          col[kb + lane] = v;
          xs[lane][cc] = v;
        }
      }
    }
    __syncthreads();
    // rows above the block: r_i -= sum_j L[kb+j][i] x_j   (i < kb)
    for (int64_t i = threadIdx.x; i < kb; i += blockDim.x) {
      double acc[kFwdCols];
#pragma unroll
      for (int cc = 0; cc < kFwdCols; ++cc) acc[cc] = 0.0;
      const double* lcol = F + i * f + kb;
      for (int j = 0; j < bw; ++j) {
        const double l = lcol[j];
#pragma unroll
        for (int cc = 0; cc < kFwdCols; ++cc) acc[cc] = fma(l, xs[j][cc], acc[cc]);
      }
      for (int cc = 0; cc < ncols; ++cc) Bp[(c0 + cc) * n + first + i] -= acc[cc];
    }
    __syncthreads();
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
// handle
// ----------------------------------------------------------------------------
struct DevTasks {
  int32_t* ptr = nullptr;
  int64_t count = 0;  // number of tasks
};

// Device workspace grown on demand (owned by a handle).
struct GrowBuf {
  void* p = nullptr;
  size_t cap = 0;
  int ensure(size_t bytes) {
    if (bytes <= cap) return CNB_OK;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
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

struct CholHandle {
  Symbolic S;
  bool uploaded = false;
  bool factored = false;
  // device symbolic
  int64_t *d_first = nullptr, *d_rows_ptr = nullptr, *d_rows = nullptr, *d_front_off = nullptr;
  int64_t *d_child_ptr = nullptr, *d_child = nullptr, *d_rel_ptr = nullptr, *d_perm = nullptr;
  int32_t* d_rel = nullptr;
  int64_t *d_map_src = nullptr, *d_map_dst = nullptr;
  double* d_front = nullptr;
  int32_t* d_tasks = nullptr;  // all task lists concatenated
  std::vector<DevTasks> ea;                       // per level
  std::vector<std::vector<DevTasks>> potrf, trsm, syrk;  // per level, per panel
  // dense-solve plan: per level (s, col chunk) tasks, built lazily per k
  int64_t solve_k = -1;
  int32_t* d_solve_tasks = nullptr;
  std::vector<DevTasks> solve_tasks;  // per level
  int64_t *d_roff = nullptr, *d_lo = nullptr, *d_w = nullptr;
  double* d_rhs = nullptr;
  double* d_bp = nullptr;
  int64_t bp_cap = 0;
  // compliance workspace
  GrowBuf c_int, c_rhs, c_val;
  double last_gram_flops = 0.0, last_fwd_flops = 0.0;

  DevSym sym() const {
    return DevSym{d_first, d_rows_ptr, d_rows, d_front_off, d_child_ptr, d_child, d_rel_ptr, d_rel};
  }
};

template <typename T>
static int upload(T** dptr, const std::vector<T>& v) {
  size_t bytes = std::max<size_t>(1, v.size()) * sizeof(T);
  CNB_CUDA(cudaMalloc((void**)dptr, bytes));
  if (!v.empty()) CNB_CUDA(cudaMemcpy(*dptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return CNB_OK;
}

static int chol_upload(CholHandle* h) {
  if (h->uploaded) return CNB_OK;
  const Symbolic& S = h->S;
  int rc;
#define UP(d, v) \
  if ((rc = upload(&h->d, S.v)) != CNB_OK) return rc;
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
  // concatenate task lists
  std::vector<int32_t> all;
  struct Rec {
    int64_t off, count;
  };
  std::vector<Rec> ea_rec;
  std::vector<std::vector<Rec>> po_rec, tr_rec, sy_rec;
  for (int l = 0; l < S.n_levels; ++l) {
    const LevelTasks& T = S.tasks[l];
    ea_rec.push_back({(int64_t)all.size(), (int64_t)T.ea.size() / 3});
    all.insert(all.end(), T.ea.begin(), T.ea.end());
    po_rec.emplace_back();
    tr_rec.emplace_back();
    sy_rec.emplace_back();
    for (size_t p = 0; p < T.potrf.size(); ++p) {
      po_rec[l].push_back({(int64_t)all.size(), (int64_t)T.potrf[p].size()});
      all.insert(all.end(), T.potrf[p].begin(), T.potrf[p].end());
      tr_rec[l].push_back({(int64_t)all.size(), (int64_t)T.trsm[p].size() / 2});
      all.insert(all.end(), T.trsm[p].begin(), T.trsm[p].end());
      sy_rec[l].push_back({(int64_t)all.size(), (int64_t)T.syrk[p].size() / 3});
      all.insert(all.end(), T.syrk[p].begin(), T.syrk[p].end());
    }
  }
  if ((rc = upload(&h->d_tasks, all)) != CNB_OK) return rc;
  auto mk = [&](const Rec& r) { return DevTasks{h->d_tasks + r.off, r.count}; };
  h->ea.clear();
  h->potrf.assign(S.n_levels, {});
  h->trsm.assign(S.n_levels, {});
  h->syrk.assign(S.n_levels, {});
  for (int l = 0; l < S.n_levels; ++l) {
    h->ea.push_back(mk(ea_rec[l]));
    for (auto& r : po_rec[l]) h->potrf[l].push_back(mk(r));
    for (auto& r : tr_rec[l]) h->trsm[l].push_back(mk(r));
    for (auto& r : sy_rec[l]) h->syrk[l].push_back(mk(r));
  }
  CNB_CUDA(cudaMalloc((void**)&h->d_front, std::max<int64_t>(1, S.front_off[S.ns]) * sizeof(double)));
  h->uploaded = true;
  return CNB_OK;
}

static void chol_free(CholHandle* h) {
  void* ptrs[] = {h->d_first, h->d_rows_ptr, h->d_rows, h->d_front_off, h->d_child_ptr, h->d_child,
                  h->d_rel_ptr, h->d_rel, h->d_map_src, h->d_map_dst, h->d_perm, h->d_front, h->d_tasks,
                  h->d_solve_tasks, h->d_roff, h->d_lo, h->d_w, h->d_rhs, h->d_bp};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  h->c_int.release();
  h->c_rhs.release();
  h->c_val.release();
}

// dense-solve plan for column chunks of width kc
static int ensure_solve_plan(CholHandle* h, int64_t kc) {
  if (h->solve_k == kc) return CNB_OK;
  const Symbolic& S = h->S;
  for (void* p : {(void*)h->d_solve_tasks, (void*)h->d_roff, (void*)h->d_lo, (void*)h->d_w, (void*)h->d_rhs})
    if (p) cudaFree(p);
  std::vector<int32_t> all;
  std::vector<std::pair<int64_t, int64_t>> rec;
  for (int l = 0; l < S.n_levels; ++l) {
    int64_t off = (int64_t)all.size();
    for (int64_t q = S.level_ptr[l]; q < S.level_ptr[l + 1]; ++q) {
      const int64_t s = S.level_sn[q];
      for (int64_t c = 0; c < kc; c += kFwdCols) {
        all.push_back((int32_t)s);
        all.push_back((int32_t)c);
      }
    }
    rec.push_back({off, ((int64_t)all.size() - off) / 2});
  }
  int rc;
  if ((rc = upload(&h->d_solve_tasks, all)) != CNB_OK) return rc;
  h->solve_tasks.clear();
  for (auto& r : rec) h->solve_tasks.push_back(DevTasks{h->d_solve_tasks + r.first, r.second});
  std::vector<int64_t> roff(S.ns + 1, 0), lo(S.ns, 0), w(S.ns, kc);
  for (int64_t s = 0; s < S.ns; ++s) roff[s + 1] = roff[s] + S.f(s) * kc;
  if ((rc = upload(&h->d_roff, roff)) != CNB_OK) return rc;
  if ((rc = upload(&h->d_lo, lo)) != CNB_OK) return rc;
  if ((rc = upload(&h->d_w, w)) != CNB_OK) return rc;
  CNB_CUDA(cudaMalloc((void**)&h->d_rhs, std::max<int64_t>(1, roff[S.ns]) * sizeof(double)));
  h->solve_k = kc;
  return CNB_OK;
}

// ----------------------------------------------------------------------------
// Mapping compliance U = S A^{-1} S^T (constraints.py:155-179)
// ----------------------------------------------------------------------------
// With P A P^T = L L^T:  U = Y^T Y,  Y = L^{-1} P S^T.  Column j of Y is
// non-zero only on the elimination paths of its S entries, so RHS columns are
// sorted by their first touched supernode and every supernode s keeps a
// window [lo_s, hi_s) of sorted columns (nested along the tree).  The
// forward solve runs over the fronts on those windows (fwd_kernel, sparse
// mode); the Gram product accumulates, for each 64x64 output tile, the
// contributions Y_s^T Y_s of exactly the supernodes whose window covers it,
// in a fixed order (deterministic), on fp64 MMA.
constexpr int kGT = 64;        // Gram tile
constexpr int kGK = 32;        // k-chunk
constexpr int kGS = kGT + 4;   // smem stride (== 4 mod 16)

__global__ void __launch_bounds__(128) gram_kernel(DevSym S, RhsView R, const int32_t* __restrict__ tile_ptr,
                                                   const int32_t* __restrict__ tile_sn, int64_t ncols,
                                                   const int64_t* __restrict__ sorted_cols, double* __restrict__ U,
                                                   int64_t ldu) {
  __shared__ double Ya[kGK * kGS];
  __shared__ double Yb[kGK * kGS];
  // tile pair index -> (A, B), B <= A
  const int64_t t = blockIdx.x;
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
  for (int32_t e = tile_ptr[t]; e < tile_ptr[t + 1]; ++e) {
    const int64_t s = tile_sn[e];
    const int64_t nc = d_nc(S, s), f = nc + d_nr(S, s);
    const int64_t lo = R.lo[s], w = R.w[s];
    const double* Ys = R.rhs + R.roff[s];
    for (int64_t k0 = 0; k0 < nc; k0 += kGK) {
      __syncthreads();
      for (int idx = threadIdx.x; idx < kGK * kGT; idx += blockDim.x) {
        const int kk = idx % kGK, cc = idx / kGK;
        const int64_t k = k0 + kk;
        const int64_t la = ra0 + cc - lo, lb = rb0 + cc - lo;
        Ya[kk * kGS + cc] = (k < nc && la >= 0 && la < w) ? Ys[la * f + k] : 0.0;
        Yb[kk * kGS + cc] = (k < nc && lb >= 0 && lb < w) ? Ys[lb * f + k] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < kGK; kk += 4) {
        double fa[4], fb[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) fa[a] = Ya[(kk + tq) * kGS + wy + 8 * a + g];
#pragma unroll
        for (int b = 0; b < 4; ++b) fb[b] = Yb[(kk + tq) * kGS + wx + 8 * b + g];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
      }
    }
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

struct CompliancePlan {
  int64_t ncols = 0;
  std::vector<int64_t> sorted_cols, lo, w, roff;
  std::vector<int64_t> sc_dst;
  std::vector<double> sc_val;
  std::vector<std::vector<int32_t>> fwd;  // per level (s, col chunk)
  std::vector<int32_t> tile_ptr, tile_sn;
  double gram_flops = 0.0, fwd_flops = 0.0;
};

static int build_compliance_plan(const Symbolic& S, int64_t ncols, const int64_t* colptr, const int64_t* rowidx,
                                 const double* vals, CompliancePlan& P) {
  P = CompliancePlan();
  P.ncols = ncols;
  const int64_t ns = S.ns;
  std::vector<int64_t> dof_sn(S.n);
  for (int64_t s = 0; s < ns; ++s)
    for (int64_t d = S.first[s]; d < S.first[s + 1]; ++d) dof_sn[d] = s;
  // key = earliest supernode touched; empty columns go last
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
  std::vector<int64_t> rank(ncols);
  for (int64_t r = 0; r < ncols; ++r) rank[P.sorted_cols[r]] = r;
  std::vector<int64_t> lo(ns, INT64_MAX), hi(ns, -1);
  for (int64_t j = 0; j < ncols; ++j)
    for (int64_t e = colptr[j]; e < colptr[j + 1]; ++e) {
      const int64_t s = dof_sn[S.iperm[rowidx[e]]];
      lo[s] = std::min(lo[s], rank[j]);
      hi[s] = std::max(hi[s], rank[j] + 1);
    }
  for (int64_t s = 0; s < ns; ++s) {  // postorder: children before parents
    const int64_t p = S.parent[s];
    if (p >= 0 && hi[s] > 0) {
      lo[p] = std::min(lo[p], lo[s]);
      hi[p] = std::max(hi[p], hi[s]);
    }
  }
  P.lo.assign(ns, 0);
  P.w.assign(ns, 0);
  P.roff.assign(ns + 1, 0);
  for (int64_t s = 0; s < ns; ++s) {
    if (hi[s] > 0) {
      P.lo[s] = lo[s];
      P.w[s] = hi[s] - lo[s];
    }
    P.roff[s + 1] = P.roff[s] + S.f(s) * P.w[s];
    const double nc = (double)S.nc(s), nr = (double)S.nr(s), w = (double)P.w[s];
    P.fwd_flops += w * (nc * nc + 2.0 * nc * nr);
  }
  for (int64_t j = 0; j < ncols; ++j)
    for (int64_t e = colptr[j]; e < colptr[j + 1]; ++e) {
      const int64_t p = S.iperm[rowidx[e]];
      const int64_t s = dof_sn[p];
      P.sc_dst.push_back(P.roff[s] + (rank[j] - P.lo[s]) * S.f(s) + (p - S.first[s]));
      P.sc_val.push_back(vals[e]);
    }
  P.fwd.assign(S.n_levels, {});
  for (int l = 0; l < S.n_levels; ++l)
    for (int64_t q = S.level_ptr[l]; q < S.level_ptr[l + 1]; ++q) {
      const int64_t s = S.level_sn[q];
      for (int64_t c = 0; c < P.w[s]; c += kFwdCols) {
        P.fwd[l].push_back((int32_t)s);
        P.fwd[l].push_back((int32_t)c);
      }
    }
  // Gram tile lists
  const int64_t nt = (ncols + kGT - 1) / kGT;
  const int64_t npairs = nt * (nt + 1) / 2;
  std::vector<int32_t> count(npairs + 1, 0);
  for (int64_t s = 0; s < ns; ++s) {
    if (P.w[s] == 0) continue;
    const int64_t t0 = P.lo[s] / kGT, t1 = (P.lo[s] + P.w[s] - 1) / kGT;
    for (int64_t a = t0; a <= t1; ++a)
      for (int64_t b = t0; b <= a; ++b) count[a * (a + 1) / 2 + b + 1]++;
    P.gram_flops += (double)S.nc(s) * (double)P.w[s] * (double)(P.w[s] + 1);
  }
  for (int64_t t = 0; t < npairs; ++t) count[t + 1] += count[t];
  P.tile_ptr = count;
  P.tile_sn.assign(count[npairs], 0);
  std::vector<int32_t> fill(count.begin(), count.end() - 1);
  for (int64_t s = 0; s < ns; ++s) {
    if (P.w[s] == 0) continue;
    const int64_t t0 = P.lo[s] / kGT, t1 = (P.lo[s] + P.w[s] - 1) / kGT;
    for (int64_t a = t0; a <= t1; ++a)
      for (int64_t b = t0; b <= a; ++b) P.tile_sn[fill[a * (a + 1) / 2 + b]++] = (int32_t)s;
  }
  return CNB_OK;
}

static std::map<std::string, std::pair<const void*, size_t>> export_table(const CholHandle* h) {
  const Symbolic& S = h->S;
  std::map<std::string, std::pair<const void*, size_t>> t;
  auto add = [&](const char* name, const auto& v) {
    t[name] = {v.data(), v.size() * sizeof(v[0])};
  };
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

}  // namespace cnb

using namespace cnb;

extern "C" {



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
  CholHandle* h = reinterpret_cast<CholHandle*>(hh);
  if (!h) return CNB_OK;
  chol_free(h);
  delete h;
  return CNB_OK;
}

// info: [n, ns, nnz_L, front_doubles, n_levels, csr_nnz, bs]; fl: [flops, solve_flops_per_rhs]
int cnb_chol_info(cnb_chol_t hh, int64_t* info, double* fl) {
  CholHandle* h = reinterpret_cast<CholHandle*>(hh);
  const Symbolic& S = h->S;
  info[0] = S.n;
  info[1] = S.ns;
  info[2] = S.nnz_L;
  info[3] = S.front_off[S.ns];
  info[4] = S.n_levels;
  info[5] = S.csr_nnz;
  info[6] = S.bs;
  // kernel launches of one numeric factorisation and of one solve (k <= 64)
  int64_t fl_launch = 1 + (S.map_src.empty() ? 0 : 1);
  for (const LevelTasks& T : S.tasks) {
    fl_launch += T.ea.empty() ? 0 : 1;
    for (size_t p = 0; p < T.potrf.size(); ++p)
      fl_launch += (T.potrf[p].empty() ? 0 : 1) + (T.trsm[p].empty() ? 0 : 1) + (T.syrk[p].empty() ? 0 : 1);
  }
  info[7] = fl_launch;
  info[8] = 2 + 2 * (int64_t)S.n_levels;
  fl[0] = S.flops;
  fl[1] = S.solve_flops_per_rhs;
  return CNB_OK;
}

int64_t cnb_chol_export_bytes(cnb_chol_t hh, const char* name) {
  CholHandle* h = reinterpret_cast<CholHandle*>(hh);
  auto t = export_table(h);
  auto it = t.find(name);
  return it == t.end() ? -1 : (int64_t)it->second.second;
}

int cnb_chol_export(cnb_chol_t hh, const char* name, void* dst) {
  CholHandle* h = reinterpret_cast<CholHandle*>(hh);
  auto t = export_table(h);
  auto it = t.find(name);
  if (it == t.end()) {
    set_error("chol_export: unknown array %s", name);
    return CNB_E_VALIDATION;
  }
  if (it->second.second) memcpy(dst, it->second.first, it->second.second);
  return CNB_OK;
}

int cnb_chol_factor(cnb_chol_t hh, const double* vals, cnb_status_t* d_status, void* stream) {
  CholHandle* h = reinterpret_cast<CholHandle*>(hh);
  int rc = chol_upload(h);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const Symbolic& S = h->S;
  DevSym sym = h->sym();
  CNB_CUDA(cudaMemsetAsync(h->d_front, 0, std::max<int64_t>(1, S.front_off[S.ns]) * sizeof(double), st));
  const int64_t nmap = (int64_t)S.map_src.size();
  if (nmap) {
    scatter_kernel<<<grid_for(nmap, 256), 256, 0, st>>>(nmap, h->d_map_src, h->d_map_dst, vals, h->d_front);
    CNB_LAUNCH_CHECK("scatter_kernel");
  }
  for (int l = 0; l < S.n_levels; ++l) {
    if (h->ea[l].count) {
      extend_add_kernel<<<(unsigned)h->ea[l].count, 256, 0, st>>>(sym, h->ea[l].ptr, h->d_front);
      CNB_LAUNCH_CHECK("extend_add_kernel");
    }
    for (size_t p = 0; p < h->potrf[l].size(); ++p) {
      const int k0 = (int)(p * kPanel);
      if (h->potrf[l][p].count) {
        potrf_kernel<<<(unsigned)h->potrf[l][p].count, 256, 0, st>>>(sym, h->potrf[l][p].ptr, k0, h->d_front,
                                                                      (DevStatus*)d_status);
        CNB_LAUNCH_CHECK("potrf_kernel");
      }
      if (h->trsm[l][p].count) {
        trsm_kernel<<<(unsigned)h->trsm[l][p].count, kTile, 0, st>>>(sym, h->trsm[l][p].ptr, k0, h->d_front);
        CNB_LAUNCH_CHECK("trsm_kernel");
      }
      if (h->syrk[l][p].count) {
        syrk_kernel<<<(unsigned)h->syrk[l][p].count, 128, 0, st>>>(sym, h->syrk[l][p].ptr, k0, h->d_front);
        CNB_LAUNCH_CHECK("syrk_kernel");
      }
    }
  }
  h->factored = true;
  return CNB_OK;
}

// X = A^{-1} B for k right-hand sides stored as k contiguous vectors of
// length n (column-major n x k, leading dimension ldb / ldx); X may alias B.
int cnb_chol_solve(cnb_chol_t hh, const double* B, int64_t ldb, double* X, int64_t ldx, int64_t k, void* stream) {
  CholHandle* h = reinterpret_cast<CholHandle*>(hh);
  if (!h->factored) {
    set_error("chol_solve: not factorised");
    return CNB_E_VALIDATION;
  }
  if (k <= 0) return CNB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const Symbolic& S = h->S;
  const int64_t n = S.n;
  const int64_t kc = std::min<int64_t>(k, 64);
  int rc = ensure_solve_plan(h, (kc + kFwdCols - 1) / kFwdCols * kFwdCols);
  if (rc) return rc;
  if (h->bp_cap < n * h->solve_k) {
    if (h->d_bp) cudaFree(h->d_bp);
    CNB_CUDA(cudaMalloc((void**)&h->d_bp, n * h->solve_k * sizeof(double)));
    h->bp_cap = n * h->solve_k;
  }
  DevSym sym = h->sym();
  RhsView R{h->d_rhs, h->d_roff, h->d_lo, h->d_w};
  for (int64_t c0 = 0; c0 < k; c0 += kc) {
    const int64_t kk = std::min(kc, k - c0);
    if (kk < h->solve_k) CNB_CUDA(cudaMemsetAsync(h->d_bp, 0, n * h->solve_k * sizeof(double), st));
    dim3 g(grid_for(n, 256), (unsigned)kk);
    permute_kernel<<<g, 256, 0, st>>>(n, kk, h->d_perm, B + c0 * ldb, ldb, h->d_bp, n, 0);
    CNB_LAUNCH_CHECK("permute_kernel");
    for (int l = 0; l < S.n_levels; ++l) {
      fwd_kernel<<<(unsigned)h->solve_tasks[l].count, 128, 0, st>>>(sym, h->solve_tasks[l].ptr, 1, h->d_front, R,
                                                                    h->d_bp, n);
      CNB_LAUNCH_CHECK("fwd_kernel");
    }
    for (int l = S.n_levels - 1; l >= 0; --l) {
      bwd_kernel<<<(unsigned)h->solve_tasks[l].count, 128, 0, st>>>(sym, h->solve_tasks[l].ptr, h->d_front,
                                                                    h->d_bp, n, h->solve_k);
      CNB_LAUNCH_CHECK("bwd_kernel");
    }
    permute_kernel<<<g, 256, 0, st>>>(n, kk, h->d_perm, h->d_bp, n, X + c0 * ldx, ldx, 1);
    CNB_LAUNCH_CHECK("permute_kernel");
  }
  return CNB_OK;
}

// U (ncols x ncols, row-major, device) = S A^{-1} S^T for the RHS columns of
// S^T given in host CSC form (colptr, rowidx = DoF ids in the original
// numbering, vals).  flops_out (host, may be NULL) receives {forward, gram}
// algorithmic flops.
int cnb_chol_compliance(cnb_chol_t hh, int64_t ncols, const int64_t* colptr, const int64_t* rowidx,
                        const double* vals, double* U, int64_t ldu, double* flops_out, void* stream) {
  CholHandle* h = reinterpret_cast<CholHandle*>(hh);
  if (!h->factored) {
    set_error("chol_compliance: not factorised");
    return CNB_E_VALIDATION;
  }
  if (ncols <= 0) return CNB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const Symbolic& S = h->S;
  CompliancePlan P;
  int rc = build_compliance_plan(S, ncols, colptr, rowidx, vals, P);
  if (rc) return rc;
  if (flops_out) {
    flops_out[0] = P.fwd_flops;
    flops_out[1] = P.gram_flops;
  }
  // pack integer arrays into one upload
  std::vector<int64_t> ints;
  auto put = [&](const std::vector<int64_t>& v) {
    size_t o = ints.size();
    ints.insert(ints.end(), v.begin(), v.end());
    return o;
  };
  const size_t o_lo = put(P.lo), o_w = put(P.w), o_roff = put(P.roff), o_sorted = put(P.sorted_cols),
               o_dst = put(P.sc_dst);
  std::vector<int32_t> i32;
  std::vector<std::pair<size_t, size_t>> fwd_rec;
  for (auto& v : P.fwd) {
    fwd_rec.push_back({i32.size(), v.size() / 2});
    i32.insert(i32.end(), v.begin(), v.end());
  }
  const size_t o_tptr = i32.size();
  i32.insert(i32.end(), P.tile_ptr.begin(), P.tile_ptr.end());
  const size_t o_tsn = i32.size();
  i32.insert(i32.end(), P.tile_sn.begin(), P.tile_sn.end());
  const size_t bytes64 = ints.size() * sizeof(int64_t);
  const size_t bytes32 = i32.size() * sizeof(int32_t);
  if ((rc = h->c_int.ensure(bytes64 + bytes32 + 16))) return rc;
  if ((rc = h->c_rhs.ensure(std::max<int64_t>(1, P.roff[S.ns]) * sizeof(double)))) return rc;
  if ((rc = h->c_val.ensure(std::max<size_t>(1, P.sc_val.size()) * sizeof(double)))) return rc;
  char* base = (char*)h->c_int.p;
  int64_t* d64 = (int64_t*)base;
  int32_t* d32 = (int32_t*)(base + ((bytes64 + 15) & ~(size_t)15));
  CNB_CUDA(cudaMemcpyAsync(d64, ints.data(), bytes64, cudaMemcpyHostToDevice, st));
  if (bytes32) CNB_CUDA(cudaMemcpyAsync(d32, i32.data(), bytes32, cudaMemcpyHostToDevice, st));
  if (!P.sc_val.empty())
    CNB_CUDA(cudaMemcpyAsync(h->c_val.p, P.sc_val.data(), P.sc_val.size() * sizeof(double),
                             cudaMemcpyHostToDevice, st));
  double* rhs = (double*)h->c_rhs.p;
  CNB_CUDA(cudaMemsetAsync(rhs, 0, std::max<int64_t>(1, P.roff[S.ns]) * sizeof(double), st));
  const int64_t nnz = (int64_t)P.sc_val.size();
  if (nnz) {
    scatter_rhs_kernel<<<grid_for(nnz, 256), 256, 0, st>>>(nnz, d64 + o_dst, (const double*)h->c_val.p, rhs);
    CNB_LAUNCH_CHECK("scatter_rhs_kernel");
  }
  DevSym sym = h->sym();
  RhsView R{rhs, d64 + o_roff, d64 + o_lo, d64 + o_w};
  for (int l = 0; l < S.n_levels; ++l) {
    if (fwd_rec[l].second == 0) continue;
    fwd_kernel<<<(unsigned)fwd_rec[l].second, 128, 0, st>>>(sym, d32 + fwd_rec[l].first, 0, h->d_front, R, nullptr,
                                                            S.n);
    CNB_LAUNCH_CHECK("fwd_kernel(sparse)");
  }
  const int64_t nt = (ncols + kGT - 1) / kGT;
  const int64_t npairs = nt * (nt + 1) / 2;
  gram_kernel<<<(unsigned)npairs, 128, 0, st>>>(sym, R, d32 + o_tptr, d32 + o_tsn, ncols, d64 + o_sorted, U, ldu);
  CNB_LAUNCH_CHECK("gram_kernel");
  h->last_fwd_flops = P.fwd_flops;
  h->last_gram_flops = P.gram_flops;
  return CNB_OK;
}

}  // extern "C"
