// Constraint-space kernels of the fast scheme: W rebuild (3x3 block
// congruence), violation, D^T lambda, proximity update, contact frames.
//
// Reference semantics (all paths relative to /root/reference/pkg/src/contactnewton):
//   rebuild_W_fast      constraints.py:182-191, gemm linalg.py:121-147
//   compute_violation   constraints.py:208-214
//   apply_transposed    constraints.py:62-64
//   fast_update_proximity constraints.py:217-244
//   build_frames / _frame_from_direction / _tangents  collision.py:351-375
//   relinearize / max_frame_rotation                 collision.py:381-414
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>

#include <algorithm>

#include "common.cuh"

namespace cnb {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void add_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(); }
// CUDA graphs replay static launch sequences (factorisation); CNB_NO_GRAPHS=1 disables
bool use_graphs() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("CNB_NO_GRAPHS");
    v = (e && e[0] && e[0] != '0') ? 0 : 1;
  }
  return v == 1;
}

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

int cuda_status(cudaError_t e, const char* where) {
  set_error("CUDA error %d (%s) at %s", (int)e, cudaGetErrorString(e), where);
  return CNB_E_CUDA;
}

// ---------------------------------------------------------------------------
// W = D Wg D^T, one thread per 3x3 output block.
//
// The reference multiplies dense c x c matrices with a rank-1 loop over the
// inner index (linalg.py:145-146).  For a block-diagonal D the only non-zero
// terms of row i are the three of its own block, summed in ascending order
// from +0; products and sums are rounded separately (numpy temporaries).
// So per block (I, J):
//   T[a][k] = ((D_I[a][0] Wg[3I][3J+k] + D_I[a][1] Wg[3I+1][3J+k]) + D_I[a][2] Wg[3I+2][3J+k])
//   W[a][b] = ((T[a][0] D_J[b][0] + T[a][1] D_J[b][1]) + T[a][2] D_J[b][2])
// which is what this kernel evaluates, bit for bit.
// Threads of a warp take consecutive J so the 24-byte row segments of Wg and
// W they touch are contiguous across the warp (coalesced).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) rebuild_w_kernel(int64_t groups, const double* __restrict__ D,
                                                        const double* __restrict__ Wg, int64_t ldwg,
                                                        double* __restrict__ W, int64_t ldw) {
  const int64_t J = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t I = blockIdx.y + (int64_t)gridDim.y * blockIdx.z;
  if (J >= groups || I >= groups) return;
  double DI[9], DJ[9], G[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) DI[e] = __ldg(D + 9 * I + e);
#pragma unroll
  for (int e = 0; e < 9; ++e) DJ[e] = __ldg(D + 9 * J + e);
  const double* src = Wg + (3 * I) * ldwg + 3 * J;
#pragma unroll
  for (int l = 0; l < 3; ++l) {
#pragma unroll
    for (int k = 0; k < 3; ++k) G[3 * l + k] = __ldcs(src + l * ldwg + k);
  }
  double T[9];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double s = mul(DI[3 * a + 0], G[0 * 3 + k]);
      s = add(s, mul(DI[3 * a + 1], G[1 * 3 + k]));
      s = add(s, mul(DI[3 * a + 2], G[2 * 3 + k]));
      T[3 * a + k] = s;
    }
  }
  double* dst = W + (3 * I) * ldw + 3 * J;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      double s = mul(T[3 * a + 0], DJ[3 * b + 0]);
      s = add(s, mul(T[3 * a + 1], DJ[3 * b + 1]));
      s = add(s, mul(T[3 * a + 2], DJ[3 * b + 2]));
      __stcs(dst + a * ldw + b, s);
    }
  }
}

// delta_g = D_g (p_a[g] - p_b[g])   (einsum "gij,gj->gi", constraints.py:58-60).
// numpy's einsum contracts a contiguous length-3 index as (x0 y0 + x2 y2) + x1 y1
// (checked bit-for-bit against the reference's outputs, tests/golden).
__global__ void violation_kernel(int64_t groups, const double* __restrict__ D,
                                 const double* __restrict__ pa, const double* __restrict__ pb,
                                 double* __restrict__ delta) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= groups) return;
  double r0 = sub(pa[3 * g + 0], pb[3 * g + 0]);
  double r1 = sub(pa[3 * g + 1], pb[3 * g + 1]);
  double r2 = sub(pa[3 * g + 2], pb[3 * g + 2]);
  const double* d = D + 9 * g;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double s = add(mul(d[3 * i + 0], r0), mul(d[3 * i + 2], r2));
    s = add(s, mul(d[3 * i + 1], r1));
    delta[3 * g + i] = s;
  }
}

// t_g = D_g^T lam_g (einsum "gji,gj->gi"); optional running impulse sum.
__global__ void apply_dt_kernel(int64_t groups, const double* __restrict__ D,
                                const double* __restrict__ lam, double* __restrict__ t,
                                double* __restrict__ acc) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= groups) return;
  const double* d = D + 9 * g;
  double l0 = lam[3 * g], l1 = lam[3 * g + 1], l2 = lam[3 * g + 2];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double s = mul(d[0 * 3 + i], l0);
    s = add(s, mul(d[1 * 3 + i], l1));
    s = add(s, mul(d[2 * 3 + i], l2));
    if (t) t[3 * g + i] = s;
    if (acc) acc[3 * g + i] = add(acc[3 * g + i], s);
  }
}

// Proximity update of one object: one warp per row of the compact U_o.
// y_r = sum_c U[r][c] t[3 idx[c/3] + c%3]; move = h^2 y; side A adds, B subtracts
// (constraints.py:238-243).  Lane-strided partial sums + butterfly reduction:
// a fixed summation order, so results are run-to-run deterministic.
__global__ void __launch_bounds__(256) prox_update_kernel(int64_t mo, const double* __restrict__ U,
                                                          int64_t ldu, const int64_t* __restrict__ idx,
                                                          const int8_t* __restrict__ side,
                                                          const double* __restrict__ t, double h2,
                                                          double* __restrict__ pa, double* __restrict__ pb) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t rows = 3 * mo;
  if (r >= rows) return;
  const double* row = U + r * ldu;
  // t is contiguous here (gathered by prox_gather_kernel when the object uses a
  // subset of the pairs); four independent accumulators, streaming loads
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int64_t c = lane;
  for (; c + 96 < rows; c += 128) {
    s0 = fma(__ldcs(row + c), t[c], s0);
    s1 = fma(__ldcs(row + c + 32), t[c + 32], s1);
    s2 = fma(__ldcs(row + c + 64), t[c + 64], s2);
    s3 = fma(__ldcs(row + c + 96), t[c + 96], s3);
  }
  for (; c < rows; c += 32) s0 = fma(__ldcs(row + c), t[c], s0);
  double s = (s0 + s1) + (s2 + s3);
  s = warp_sum(s);
  if (lane == 0) {
    const int64_t k = r / 3;
    const int d = (int)(r - 3 * k);
    const int64_t pair = idx ? idx[k] : k;
    const double move = mul(h2, s);
    if (side[k] > 0)
      pa[3 * pair + d] = add(pa[3 * pair + d], move);
    else
      pb[3 * pair + d] = sub(pb[3 * pair + d], move);
  }
}

// Large objects: U_o is symmetric, so y = U t reads only its lower triangle.
// One CTA per 128 x 128 tile (I, J), I >= J, all 16 rows of a warp loaded up
// front: the row products U_IJ t_J go to part[I][J], and (I > J) the column
// products U_IJ^T t_I to part[J][I].  Every slot is written exactly once and
// prox_sym_sum_kernel adds each row's nt slots in J order: deterministic, and
// 8 n^2 / 2 bytes of U per update instead of 8 n^2.
constexpr int kPT = 128;
constexpr int64_t kProxSymMinTiles = 8;  // below ~1 000 rows the warp-per-row GEMV is one short launch
__global__ void __launch_bounds__(256, 2) prox_sym_tile_kernel(int64_t n, int64_t nt, const double* __restrict__ U,
                                                            int64_t ldu, const double* __restrict__ t,
                                                            double* __restrict__ part) {
  const int64_t b = blockIdx.x;
  int64_t I = (int64_t)((sqrt(8.0 * (double)b + 1.0) - 1.0) * 0.5);
  while (I * (I + 1) / 2 > b) --I;
  while ((I + 1) * (I + 2) / 2 <= b) ++I;
  const int64_t J = b - I * (I + 1) / 2;
  __shared__ double tI[kPT], tJ[kPT];
  __shared__ double colp[8][kPT];
  const int64_t r0 = I * kPT, c0 = J * kPT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < kPT) {
    const int e = threadIdx.x;
    tI[e] = r0 + e < n ? t[r0 + e] : 0.0;
    tJ[e] = c0 + e < n ? t[c0 + e] : 0.0;
  }
  __syncthreads();
  // the warp's 16 rows in two halves of 8 (64 KB of U in flight per CTA, two CTAs per SM)
  double rs = 0.0;
  double ca[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int hf = 0; hf < 2; ++hf) {
    double v[8][4];
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      const int64_t r = r0 + warp * 16 + 8 * hf + rr;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t c = c0 + lane + 32 * q;
        v[rr][q] = (r < n && c < n) ? __ldcs(U + r * ldu + c) : 0.0;
      }
    }
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      double s = fma(v[rr][0], tJ[lane], v[rr][1] * tJ[lane + 32]) + fma(v[rr][2], tJ[lane + 64], v[rr][3] * tJ[lane + 96]);
      s = warp_sum(s);
      if (lane == 8 * hf + rr) rs = s;
    }
    if (I != J) {
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) {
        const double ti = tI[warp * 16 + 8 * hf + rr];
#pragma unroll
        for (int q = 0; q < 4; ++q) ca[q] = fma(v[rr][q], ti, ca[q]);
      }
    }
  }
  if (lane < 16) part[(I * nt + J) * kPT + warp * 16 + lane] = rs;
  if (I == J) return;
#pragma unroll
  for (int q = 0; q < 4; ++q) colp[warp][lane + 32 * q] = ca[q];
  __syncthreads();
  if (threadIdx.x < kPT) {
    const int e = threadIdx.x;
    double s = colp[0][e];
#pragma unroll
    for (int w = 1; w < 8; ++w) s += colp[w][e];
    part[(J * nt + I) * kPT + e] = s;
  }
}

__global__ void prox_sym_sum_kernel(int64_t mo, int64_t nt, const double* __restrict__ part,
                                    const int64_t* __restrict__ idx, const int8_t* __restrict__ side, double h2,
                                    double* __restrict__ pa, double* __restrict__ pb) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= 3 * mo) return;
  const int64_t I = r / kPT, i = r - I * kPT;
  const double* p = part + I * nt * kPT + i;
  double s = 0.0;
  for (int64_t J = 0; J < nt; ++J) s += p[J * kPT];
  const int64_t k = r / 3;
  const int d = (int)(r - 3 * k);
  const int64_t pair = idx ? idx[k] : k;
  const double move = mul(h2, s);
  if (side[k] > 0)
    pa[3 * pair + d] = add(pa[3 * pair + d], move);
  else
    pb[3 * pair + d] = sub(pb[3 * pair + d], move);
}

// tg[c] = t[3 idx[c / 3] + c % 3]: the object's rows of D^T lambda, contiguous
__global__ void prox_gather_kernel(int64_t mo, const int64_t* __restrict__ idx, const double* __restrict__ t,
                                   double* __restrict__ tg) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= 3 * mo) return;
  const int64_t k = c / 3;
  tg[c] = t[3 * idx[k] + (c - 3 * k)];
}

// total[3 idx[I] + a][3 idx[J] + b] += U[3 I + a][3 J + b]: one object's compact
// compliance added into W_g (constraints.py:175-179, objects in ascending id
// order).  Warp per U row: the row is read contiguously, the destination
// columns ascend with J (idx is sorted).
__global__ void __launch_bounds__(256) scatter_add_compliance_kernel(int64_t mo, const double* __restrict__ U,
                                                                     int64_t ldu, const int64_t* __restrict__ idx,
                                                                     double* __restrict__ total, int64_t ldt) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= 3 * mo) return;
  const int64_t I = r / 3;
  double* dst = total + (3 * idx[I] + (r - 3 * I)) * ldt;
  const double* src = U + r * ldu;
  for (int64_t c = lane; c < 3 * mo; c += 32) {
    const int64_t J = c / 3;
    const int64_t col = 3 * __ldg(idx + J) + (c - 3 * J);
    dst[col] = add(dst[col], __ldcs(src + c));
  }
}

// ---- frames ---------------------------------------------------------------

__device__ __forceinline__ double dot3(const double* a, const double* b) {
  return add(add(mul(a[0], b[0]), mul(a[1], b[1])), mul(a[2], b[2]));
}

// _tangents collision.py:351-356: t1 = e_x - (e_x.n) n, fallback e_z when
// |t1| < 1e-6, normalised; t2 = n x t1.
__device__ void tangents(const double* n, double* t1, double* t2) {
  double c = n[0];  // e_x . n
  t1[0] = sub(1.0, mul(c, n[0]));
  t1[1] = sub(0.0, mul(c, n[1]));
  t1[2] = sub(0.0, mul(c, n[2]));
  double nrm = sqrt(dot3(t1, t1));
  if (nrm < 1e-6) {
    c = n[2];  // e_z . n
    t1[0] = sub(0.0, mul(c, n[0]));
    t1[1] = sub(0.0, mul(c, n[1]));
    t1[2] = sub(1.0, mul(c, n[2]));
    nrm = sqrt(dot3(t1, t1));
  }
  t1[0] = __ddiv_rn(t1[0], nrm);
  t1[1] = __ddiv_rn(t1[1], nrm);
  t1[2] = __ddiv_rn(t1[2], nrm);
  t2[0] = sub(mul(n[1], t1[2]), mul(n[2], t1[1]));
  t2[1] = sub(mul(n[2], t1[0]), mul(n[0], t1[2]));
  t2[2] = sub(mul(n[0], t1[1]), mul(n[1], t1[0]));
}

__device__ __forceinline__ void store_frame(double* f, const double* n, const double* t1,
                                            const double* t2) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    f[i] = n[i];
    f[3 + i] = t1[i];
    f[6 + i] = t2[i];
  }
}

#define CNB_COINCIDENT_EPS 1e-9  // collision.py:24
#define CNB_MAX_TILT_COS 0.5     // collision.py:378

__global__ void build_frames_kernel(int64_t pairs, const double* __restrict__ pa,
                                    const double* __restrict__ pb, const double* __restrict__ ref,
                                    double* __restrict__ frames, DevStatus* st) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= pairs) return;
  double d[3] = {sub(pa[3 * i], pb[3 * i]), sub(pa[3 * i + 1], pb[3 * i + 1]),
                 sub(pa[3 * i + 2], pb[3 * i + 2])};
  const double r[3] = {ref[3 * i], ref[3 * i + 1], ref[3 * i + 2]};
  double n[3];
  double nrm = sqrt(dot3(d, d));
  if (nrm > CNB_COINCIDENT_EPS) {
    for (int k = 0; k < 3; ++k) n[k] = __ddiv_rn(d[k], nrm);
    if (dot3(n, r) < 0.0)
      for (int k = 0; k < 3; ++k) n[k] = -n[k];
  } else {
    double rn = sqrt(dot3(r, r));
    if (rn > 0.5) {
      for (int k = 0; k < 3; ++k) n[k] = __ddiv_rn(r[k], rn);
    } else {
      raise_status(st, CNB_E_DEGENERATE_FRAME, (int)i, nrm);
      for (int k = 0; k < 3; ++k) n[k] = 0.0;
      store_frame(frames + 9 * i, n, n, n);
      return;
    }
  }
  double t1[3], t2[3];
  tangents(n, t1, t2);
  store_frame(frames + 9 * i, n, t1, t2);
}

// Re-linearisation (collision.py:381-405) fused with the rotation reduction
// (collision.py:408-414).  Angles are non-negative, so their IEEE bit
// patterns order like unsigned integers and atomicMax on the bits is exact.
__global__ void relinearize_kernel(int64_t pairs, const double* __restrict__ pa,
                                   const double* __restrict__ pb, const double* __restrict__ prev,
                                   double* __restrict__ frames, unsigned long long* rot_bits) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double angle = 0.0;
  if (i < pairs) {
    const double* pf = prev + 9 * i;
    double* of = frames + 9 * i;
    double d[3] = {sub(pa[3 * i], pb[3 * i]), sub(pa[3 * i + 1], pb[3 * i + 1]),
                   sub(pa[3 * i + 2], pb[3 * i + 2])};
    const double np_[3] = {pf[0], pf[1], pf[2]};
    double nrm = sqrt(dot3(d, d));
    bool keep = !(nrm > CNB_COINCIDENT_EPS);
    double n[3];
    if (!keep) {
      for (int k = 0; k < 3; ++k) n[k] = __ddiv_rn(d[k], nrm);
      if (dot3(n, np_) < 0.0)
        for (int k = 0; k < 3; ++k) n[k] = -n[k];
      if (dot3(n, np_) < CNB_MAX_TILT_COS) keep = true;
    }
    if (keep) {
      for (int e = 0; e < 9; ++e) of[e] = pf[e];
      // arccos(clip(n.n)) of a frame with itself: the reference still
      // evaluates it (tiny non-zero angles from rounding are possible).
      double c = fmin(1.0, fmax(-1.0, dot3(np_, np_)));
      angle = acos(c);
    } else {
      double t1[3], t2[3];
      tangents(n, t1, t2);
      store_frame(of, n, t1, t2);
      double c = fmin(1.0, fmax(-1.0, dot3(np_, n)));
      angle = acos(c);
    }
  }
  // block-level max, then one atomic per block
  angle = warp_max(angle);
  __shared__ double wmax[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) wmax[wid] = angle;
  __syncthreads();
  if (wid == 0) {
    double v = lane < (blockDim.x >> 5) ? wmax[lane] : 0.0;
    v = warp_max(v);
    if (lane == 0 && v > 0.0) atomicMax(rot_bits, (unsigned long long)__double_as_longlong(v));
  }
}

// Naive-order dense product, one thread per output (linalg.py:121-147).
__global__ void gemm_naive_kernel(int64_t m, int64_t n, int64_t k, const double* __restrict__ A,
                                  int64_t lda, int ta, const double* __restrict__ B, int64_t ldb,
                                  int tb, double* __restrict__ C, int64_t ldc) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = blockIdx.y + (int64_t)gridDim.y * blockIdx.z;
  if (i >= m || j >= n) return;
  double s = 0.0;
  for (int64_t p = 0; p < k; ++p) {
    double a = ta ? A[p * lda + i] : A[i * lda + p];
    double b = tb ? B[j * ldb + p] : B[p * ldb + j];
    s = add(s, mul(a, b));
  }
  C[i * ldc + j] = s;
}

// y = alpha * A x for a CSR matrix, one thread per row, entries summed in
// column order (deterministic).  Used for S^T t of the mechanical correction
// (solver.py:250-257) and the stiffness products of the RHS assembly.
__global__ void csr_spmv_kernel(int64_t rows, const int64_t* __restrict__ rp, const int64_t* __restrict__ ci,
                                const double* __restrict__ va, const double* __restrict__ x,
                                double* __restrict__ y, double alpha) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double s = 0.0;
  for (int64_t e = rp[r]; e < rp[r + 1]; ++e) s = fma(va[e], x[ci[e]], s);
  y[r] = alpha == 1.0 ? s : alpha * s;
}

// U = S C S^T for a sparse S (m x k) stored as ELL rows of width 4 (col, val;
// padding val = 0) and a dense symmetric C (k x k).  One CTA per output row j:
// t = C^T s_j (<= 4 contiguous rows of C combined, in shared memory), then
// U[j][i] = sum_e s_ie t[col_ie] for every i (gathers from shared memory),
// fixed summation order.  Used for the mapping compliance of contact DoFs:
// U_o = S_o (E^T A^-1 E) S_o^T with E the unit columns of the DoFs S_o touches.
constexpr int kEll = 4;
__global__ void __launch_bounds__(1024) sandwich_kernel(int64_t m, int64_t k, const int32_t* __restrict__ ecol,
                                                       const double* __restrict__ eval, const double* __restrict__ C,
                                                       int64_t ldc, double* __restrict__ U, int64_t ldu) {
  extern __shared__ double tsm[];
  const int64_t j = blockIdx.x;
  int32_t cj[kEll];
  double vj[kEll];
#pragma unroll
  for (int e = 0; e < kEll; ++e) {
    cj[e] = ecol[kEll * j + e];
    vj[e] = eval[kEll * j + e];
  }
  for (int64_t a = threadIdx.x; a < k; a += blockDim.x) {
    double t = 0.0;
#pragma unroll
    for (int e = 0; e < kEll; ++e) t = fma(vj[e], C[(int64_t)cj[e] * ldc + a], t);
    tsm[a] = t;
  }
  __syncthreads();
  double* urow = U + j * ldu;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const int4 ci = *reinterpret_cast<const int4*>(ecol + kEll * i);
    const double2 v01 = *reinterpret_cast<const double2*>(eval + kEll * i);
    const double2 v23 = *reinterpret_cast<const double2*>(eval + kEll * i + 2);
    double u = v01.x * tsm[ci.x];
    u = fma(v01.y, tsm[ci.y], u);
    u = fma(v23.x, tsm[ci.z], u);
    u = fma(v23.y, tsm[ci.w], u);
    urow[i] = u;
  }
}

static void split_rows(int64_t rows, dim3& grid, int64_t cols_blocks) {
  // rows across y (<= 65535) and z
  int64_t gy = rows < 65535 ? rows : 65535;
  int64_t gz = (rows + gy - 1) / gy;
  grid = dim3((unsigned)cols_blocks, (unsigned)(gy > 0 ? gy : 1), (unsigned)(gz > 0 ? gz : 1));
}

}  // namespace cnb

using namespace cnb;

extern "C" {

int cnb_abi_version(void) { return 2; }

int cnb_sandwich(int64_t m, int64_t k, const int32_t* ell_col, const double* ell_val, const double* C, int64_t ldc,
                 double* U, int64_t ldu, void* stream) {
  if (m < 0 || k < 0 || ldc < k || ldu < m) {
    set_error("sandwich: invalid sizes (m=%lld, k=%lld)", (long long)m, (long long)k);
    return CNB_E_DIMENSION;
  }
  if (m == 0) return CNB_OK;
  const size_t smem = sizeof(double) * (size_t)std::max<int64_t>(k, 1);
  int dev = 0, maxs = 0;
  CNB_CUDA(cudaGetDevice(&dev));
  CNB_CUDA(cudaDeviceGetAttribute(&maxs, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (smem > (size_t)maxs) {
    set_error("sandwich: k=%lld exceeds the shared-memory row buffer", (long long)k);
    return CNB_E_VALIDATION;
  }
  CNB_CUDA(cudaFuncSetAttribute(sandwich_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  sandwich_kernel<<<(unsigned)m, 1024, smem, (cudaStream_t)stream>>>(m, k, ell_col, ell_val, C, ldc, U, ldu);
  CNB_LAUNCH_CHECK("sandwich_kernel");
  return CNB_OK;
}

long long cnb_launch_count(void) { return g_launches.load(); }

const char* cnb_last_error(void) { return g_last_error.c_str(); }

int cnb_rebuild_w(int64_t groups, const double* D, const double* Wg, int64_t ldwg, double* W,
                  int64_t ldw, void* stream) {
  if (groups < 0) {
    set_error("rebuild_w: negative group count");
    return CNB_E_DIMENSION;
  }
  if (groups == 0) return CNB_OK;
  dim3 grid;
  const int block = groups >= 256 ? 256 : (groups >= 64 ? 64 : 32);
  split_rows(groups, grid, (groups + block - 1) / block);
  rebuild_w_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(groups, D, Wg, ldwg, W, ldw);
  CNB_LAUNCH_CHECK("rebuild_w_kernel");
  return CNB_OK;
}

int cnb_violation(int64_t groups, const double* D, const double* p_a, const double* p_b,
                  double* delta, void* stream) {
  if (groups <= 0) return CNB_OK;
  violation_kernel<<<grid_for(groups, 128), 128, 0, (cudaStream_t)stream>>>(groups, D, p_a, p_b, delta);
  CNB_LAUNCH_CHECK("violation_kernel");
  return CNB_OK;
}

int cnb_apply_dt(int64_t groups, const double* D, const double* lam, double* t, double* accumulated,
                 void* stream) {
  if (groups <= 0) return CNB_OK;
  apply_dt_kernel<<<grid_for(groups, 128), 128, 0, (cudaStream_t)stream>>>(groups, D, lam, t, accumulated);
  CNB_LAUNCH_CHECK("apply_dt_kernel");
  return CNB_OK;
}

int cnb_prox_update(int64_t mo, const double* U, int64_t ldu, const int64_t* idx, const int8_t* side,
                    const double* t, double h, double* p_a, double* p_b, void* stream) {
  if (mo <= 0) return CNB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const double* tv = t;
  if (idx) {  // gather the object's rows of t once (the GEMV then streams U against a contiguous vector)
    static GrowBuf tg;
    int rc = tg.ensure((size_t)(3 * mo) * sizeof(double));
    if (rc) return rc;
    prox_gather_kernel<<<grid_for(3 * mo, 256), 256, 0, st>>>(mo, idx, t, (double*)tg.p);
    CNB_LAUNCH_CHECK("prox_gather_kernel");
    tv = (const double*)tg.p;
  }
  const int64_t n = 3 * mo, nt = (n + kPT - 1) / kPT;
  static const bool sym_off = [] {
    const char* e = getenv("CNB_PROX_SYM");
    return e && e[0] == '0';
  }();
  if (nt >= kProxSymMinTiles && !sym_off) {
    static GrowBuf part;
    int rc = part.ensure((size_t)(nt * nt * kPT) * sizeof(double));
    if (rc) return rc;
    prox_sym_tile_kernel<<<(unsigned)(nt * (nt + 1) / 2), 256, 0, st>>>(n, nt, U, ldu, tv, (double*)part.p);
    CNB_LAUNCH_CHECK("prox_sym_tile_kernel");
    prox_sym_sum_kernel<<<grid_for(n, 256), 256, 0, st>>>(mo, nt, (const double*)part.p, idx, side, h * h, p_a, p_b);
    CNB_LAUNCH_CHECK("prox_sym_sum_kernel");
    return CNB_OK;
  }
  const int64_t threads = 3 * mo * 32;
  prox_update_kernel<<<grid_for(threads, 256), 256, 0, st>>>(mo, U, ldu, idx, side, tv, h * h, p_a, p_b);
  CNB_LAUNCH_CHECK("prox_update_kernel");
  return CNB_OK;
}

int cnb_scatter_add_compliance(int64_t mo, const double* U, int64_t ldu, const int64_t* idx, double* total,
                               int64_t ldt, void* stream) {
  if (mo <= 0) return CNB_OK;
  scatter_add_compliance_kernel<<<grid_for(3 * mo * 32, 256), 256, 0, (cudaStream_t)stream>>>(mo, U, ldu, idx, total,
                                                                                             ldt);
  CNB_LAUNCH_CHECK("scatter_add_compliance_kernel");
  return CNB_OK;
}

int cnb_build_frames(int64_t pairs, const double* p_a, const double* p_b, const double* ref_normal,
                     double* frames, cnb_status_t* d_status, void* stream) {
  if (pairs <= 0) return CNB_OK;
  build_frames_kernel<<<grid_for(pairs, 128), 128, 0, (cudaStream_t)stream>>>(
      pairs, p_a, p_b, ref_normal, frames, (DevStatus*)d_status);
  CNB_LAUNCH_CHECK("build_frames_kernel");
  return CNB_OK;
}

int cnb_relinearize(int64_t pairs, const double* p_a, const double* p_b, const double* prev,
                    double* frames, double* rotation, void* stream) {
  CNB_CUDA(cudaMemsetAsync(rotation, 0, sizeof(double), (cudaStream_t)stream));
  if (pairs <= 0) return CNB_OK;
  relinearize_kernel<<<grid_for(pairs, 128), 128, 0, (cudaStream_t)stream>>>(
      pairs, p_a, p_b, prev, frames, (unsigned long long*)rotation);
  CNB_LAUNCH_CHECK("relinearize_kernel");
  return CNB_OK;
}

int cnb_csr_spmv(int64_t rows, const int64_t* rowptr, const int64_t* col, const double* val, const double* x,
                 double* y, double alpha, void* stream) {
  if (rows <= 0) return CNB_OK;
  csr_spmv_kernel<<<grid_for(rows, 128), 128, 0, (cudaStream_t)stream>>>(rows, rowptr, col, val, x, y, alpha);
  CNB_LAUNCH_CHECK("csr_spmv_kernel");
  return CNB_OK;
}

int cnb_gemm_naive(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, int32_t trans_a,
                   const double* B, int64_t ldb, int32_t trans_b, double* C, int64_t ldc, void* stream) {
  if (m <= 0 || n <= 0) return CNB_OK;
  dim3 grid;
  split_rows(m, grid, (n + 127) / 128);
  gemm_naive_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(m, n, k, A, lda, trans_a, B, ldb, trans_b, C, ldc);
  CNB_LAUNCH_CHECK("gemm_naive_kernel");
  return CNB_OK;
}

}  // extern "C"
