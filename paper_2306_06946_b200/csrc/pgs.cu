// Projected Gauss-Seidel with Signorini + isotropic Coulomb friction, in the
// reference's exact canonical group order.
//
// Reference: pgs solver.py:168-202, local_solve solver.py:124-165,
// regularize solver.py:99-121 (paths under /root/reference/pkg/src/contactnewton).
//
// Gauss-Seidel over a dense W is sequential in the group index: group g's
// local solve needs  delta_g = delta_base_g + h^2 W[g,:] lam  with every
// earlier group of the sweep already updated.  The reference keeps delta for
// all rows current by a rank-3 update after every group (8 c^2 bytes of W per
// sweep).  Here the sweep is blocked, 32 groups per block:
//
//   * one SOLVER warp owns the block being solved, lane l <-> group l; the
//     block's diagonal W tile sits in shared memory and the in-block rank-3
//     updates are warp-synchronous (shuffles, no barriers);
//   * while it solves block b, the HELPER warps evaluate, for the rows of the
//     next block b', the lazy row products  P = W[b', not b] lam  — every
//     lambda they read is final for this point of the sweep;
//   * after the barrier all warps add the cross term W[b', b] lam_b and stage
//     block b''s diagonal tile, and the solver continues.
//
// The iterate is mathematically the reference's; only the association of
// the floating-point sums of delta differs (the per-group arithmetic of
// local_solve is reproduced operation by operation).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace cnb {

constexpr int kBG = 32;         // groups per block (one per solver lane)
constexpr int kBR = 3 * kBG;    // rows per block
constexpr int kLDT = kBR + 1;   // shared tile row stride: odd, so lane l's rows 3l.. fall in distinct banks
constexpr int kPgsThreads = 256;

struct PgsScene {
  int64_t groups;
  const double* W;
  int64_t ldw;
  const double* delta_base;
  double h2, mu, tol;
  int max_iter;
  double* lam;
  double* delta_end;
  double* eps_hist;
  int* iters_conv;
  DevStatus* status;
  double* shift_out;  // per-group regularisation shift (may be null)
};

// eigenvalues of a symmetric 3x3 by cyclic Jacobi (converges to rounding)
__device__ void sym3_eigs(double a[3][3], double out[3]) {
  for (int sweep = 0; sweep < 12; ++sweep) {
    double off = fabs(a[0][1]) + fabs(a[0][2]) + fabs(a[1][2]);
    if (off == 0.0) break;
    for (int p = 0; p < 2; ++p) {
      for (int q = p + 1; q < 3; ++q) {
        double apq = a[p][q];
        if (apq == 0.0) continue;
        double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 3; ++k) {  // columns p, q
          double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {  // rows p, q
          double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
        a[p][q] = a[q][p] = 0.0;
      }
    }
  }
  out[0] = a[0][0];
  out[1] = a[1][1];
  out[2] = a[2][2];
}

// local_solve solver.py:124-165 on one group; Wd = regularised diagonal
// block (row-major).  Returns 0, or CNB_E_SINGULAR_BLOCK.
__device__ __forceinline__ int local_solve_dev(const double d[3], const double l[3], const double Wd[9],
                                               double mu, double h2, double out[3]) {
  const double Wnn = Wd[0];
  if (!(Wnn > 0.0)) return CNB_E_SINGULAR_BLOCK;
  const double ln_old = l[0];
  const double x = sub(ln_old, __ddiv_rn(d[0], mul(h2, Wnn)));
  const double ln = x > 0.0 ? x : 0.0;  // Python max(0.0, x)
  if (ln == 0.0) {
    out[0] = out[1] = out[2] = 0.0;
    return 0;
  }
  if (mu == 0.0) {
    out[0] = ln;
    out[1] = out[2] = 0.0;
    return 0;
  }
  const double dln = sub(ln, ln_old);
  const double dt0 = add(d[1], mul(mul(h2, Wd[3]), dln));
  const double dt1 = add(d[2], mul(mul(h2, Wd[6]), dln));
  const double T00 = mul(h2, Wd[4]), T01 = mul(h2, Wd[5]);
  const double T10 = mul(h2, Wd[7]), T11 = mul(h2, Wd[8]);
  const double det = sub(mul(T00, T11), mul(T01, T10));
  if (!(det > 0.0)) return CNB_E_SINGULAR_BLOCK;
  const double r0 = -dt0, r1 = -dt1;
  const double dl0 = __ddiv_rn(sub(mul(T11, r0), mul(T01, r1)), det);
  const double dl1 = __ddiv_rn(sub(mul(T00, r1), mul(T10, r0)), det);
  double lt0 = add(l[1], dl0), lt1 = add(l[2], dl1);
  const double radius = mul(mu, ln);
  const double nt = hypot(lt0, lt1);
  if (nt > radius) {
    const double s = __ddiv_rn(radius, nt);
    lt0 = mul(lt0, s);
    lt1 = mul(lt1, s);
  }
  out[0] = ln;
  out[1] = lt0;
  out[2] = lt1;
  return 0;
}

// Per-group constants of local_solve that depend only on W (and h): computed
// once per block load, in parallel over the solver lanes, so the sequential
// per-group chain is a handful of multiply-adds instead of four divisions
// and a hypot (dependent fp64 operations cost ~30+ cycles each on sm_100a).
struct GroupConst {
  double ihw;        // 1 / (h^2 W_nn)
  double htn0, htn1; // h^2 W_tn
  double it00, it01, it10, it11;  // (h^2 W_tt)^{-1}
  double b0, b1;     // (h^2 W_tt)^{-1} h^2 W_tn: tangential response to a normal change
  double hwnn;       // h^2 W_nn (= 1 / ihw up to rounding)
  int bad;           // bit 0: W_nn <= 0, bit 1: det(h^2 W_tt) <= 0
};

__device__ __forceinline__ void group_const(const double Wd[9], double h2, GroupConst& k) {
  k.bad = 0;
  const double Wnn = Wd[0];
  if (!(Wnn > 0.0)) k.bad |= 1;
  k.hwnn = mul(h2, Wnn);
  k.ihw = 1.0 / k.hwnn;
  k.htn0 = mul(h2, Wd[3]);
  k.htn1 = mul(h2, Wd[6]);
  const double T00 = mul(h2, Wd[4]), T01 = mul(h2, Wd[5]);
  const double T10 = mul(h2, Wd[7]), T11 = mul(h2, Wd[8]);
  const double det = sub(mul(T00, T11), mul(T01, T10));
  if (!(det > 0.0)) k.bad |= 2;
  const double idet = 1.0 / det;
  k.it00 = T11 * idet;
  k.it01 = -T01 * idet;
  k.it10 = -T10 * idet;
  k.it11 = T00 * idet;
  k.b0 = fma(k.it00, k.htn0, k.it01 * k.htn1);
  k.b1 = fma(k.it10, k.htn0, k.it11 * k.htn1);
}

// fp64 1/sqrt(x) for x > 0 without the library's special-case branch: the
// hardware approximation (rsqrt.approx.f64) refined by two Newton steps.
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-0.5 * x, y * y, 1.5);
  y = y * fma(-0.5 * x, y * y, 1.5);
  return y;
}

// Branch-free local_solve (solver.py:124-165) with the precomputed constants
// (divisions by loop-invariant quantities become multiplications by
// reciprocals): every lane evaluates its own group with the same instruction
// stream (no divergence in the sequential chain); the caller keeps only the
// result of the lane whose turn it is (the unprojected branch multiplies by
// exactly 1.0).
template <int V = 0>
__device__ __forceinline__ int local_solve_sel(const double d[3], const double l[3], const GroupConst& k,
                                               double mu, double out[3]) {
  const double ln_old = l[0];
  const double x = fma(-d[0], k.ihw, ln_old);
  const double ln = x > 0.0 ? x : 0.0;
  const double dln = ln - ln_old;
  const double dt0 = fma(k.htn0, dln, d[1]);
  const double dt1 = fma(k.htn1, dln, d[2]);
  double lt0 = l[1] - fma(k.it00, dt0, k.it01 * dt1);
  double lt1 = l[2] - fma(k.it10, dt0, k.it11 * dt1);
  const double radius = mu * ln;
  const double n2 = fma(lt0, lt0, lt1 * lt1);
  double sc;
  if (V & 2) {  // branch-free: evaluate the projection scale unconditionally
    const double rs = radius * rsqrt_nr(fmax(n2, 1e-300));
    sc = n2 > radius * radius ? rs : 1.0;
  } else {
    sc = n2 > radius * radius ? radius * rsqrt(n2) : 1.0;
  }
  lt0 *= sc;
  lt1 *= sc;
  const bool zero = ln == 0.0, nofric = mu == 0.0;
  out[0] = ln;
  out[1] = (zero || nofric) ? 0.0 : lt0;
  out[2] = (zero || nofric) ? 0.0 : lt1;
  return ((k.bad & 1) || (!zero && !nofric && (k.bad & 2))) ? 1 : 0;
}

// Sequential Gauss-Seidel over one block of ng <= 32 groups by one warp,
// lane l <-> group l.  Wt: the block's regularised diagonal tile (row stride
// kLDT).  Per group: all lanes run local_solve_sel, lane g's change is
// broadcast (3 shuffles) and every lane applies the rank-3 update of its
// delta; W entries are loaded ahead of the chain.  EXACT selects the
// reference's unfused association (a*b rounded, then the add) for the
// update, otherwise fused multiply-adds.  err: lane-local flag for the
// group the lane owns; dsq: sum of squared lambda changes of the lane.
// V bit 0: the tile holds h^2 W (the update is three fused multiply-adds);
// V bit 1: branch-free projection scale (rsqrt_nr).
template <bool EXACT, int V = 0>
__device__ __forceinline__ void block_solve(const double* __restrict__ Wt, int ng, int lane, double dl_[3],
                                            double lm[3], const GroupConst& kc, double mu, double h2, double& dsq,
                                            int& err) {
  const double* wrow = Wt + 3 * lane * kLDT;
#pragma unroll 2
  for (int g = 0; g < ng; ++g) {
    double w[9];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) w[3 * a + c] = wrow[a * kLDT + 3 * g + c];
    double nw[3];
    const int e = local_solve_sel<V>(dl_, lm, kc, mu, nw);
    const bool me = lane == g;
    double d0 = nw[0] - lm[0], d1 = nw[1] - lm[1], d2 = nw[2] - lm[2];
    if (me) {
      err |= e;
      dsq += d0 * d0 + d1 * d1 + d2 * d2;
      lm[0] = nw[0];
      lm[1] = nw[1];
      lm[2] = nw[2];
    }
    d0 = __shfl_sync(0xffffffffu, d0, g);
    d1 = __shfl_sync(0xffffffffu, d1, g);
    d2 = __shfl_sync(0xffffffffu, d2, g);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (EXACT) {
        const double tmp = add(add(mul(w[3 * a], d0), mul(w[3 * a + 1], d1)), mul(w[3 * a + 2], d2));
        dl_[a] = add(dl_[a], mul(h2, tmp));
      } else if (V & 1) {
        dl_[a] = fma(w[3 * a + 2], d2, fma(w[3 * a + 1], d1, fma(w[3 * a], d0, dl_[a])));
      } else {
        const double tmp = fma(w[3 * a + 2], d2, fma(w[3 * a + 1], d1, w[3 * a] * d0));
        dl_[a] = fma(h2, tmp, dl_[a]);
      }
    }
  }
}

template <bool CG>
__device__ __forceinline__ double lane_dot(const double* __restrict__ w, const double* __restrict__ x, int64_t lo,
                                           int64_t hi, int lane) {
  double a[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) a[u] = 0.0;
  int64_t j = lo + lane;
  for (; j + 224 < hi; j += 256) {
    double wv[8], xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) wv[u] = w[j + 32 * u];
#pragma unroll
    for (int u = 0; u < 8; ++u) xv[u] = CG ? __ldcg(x + j + 32 * u) : x[j + 32 * u];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = fma(wv[u], xv[u], a[u]);
  }
  for (; j < hi; j += 32) a[0] = fma(w[j], CG ? __ldcg(x + j) : x[j], a[0]);
  return ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
}

// eight per-lane partial sums reduced across the warp at once (9 shuffles): lane
// L returns the total of value 4 ((L >> 4) & 1) + 2 ((L >> 3) & 1) + ((L >> 2) & 1)
__device__ __forceinline__ double warp_sum8(const double v[8], int lane) {
  double a[4], b[2];
  const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
#pragma unroll
  for (int k = 0; k < 4; ++k) a[k] = (h16 ? v[k + 4] : v[k]) + __shfl_xor_sync(0xffffffffu, h16 ? v[k] : v[k + 4], 16);
#pragma unroll
  for (int k = 0; k < 2; ++k) b[k] = (h8 ? a[k + 2] : a[k]) + __shfl_xor_sync(0xffffffffu, h8 ? a[k] : a[k + 2], 8);
  double c = (h4 ? b[1] : b[0]) + __shfl_xor_sync(0xffffffffu, h4 ? b[0] : b[1], 4);
  c += __shfl_xor_sync(0xffffffffu, c, 2);
  c += __shfl_xor_sync(0xffffffffu, c, 1);
  return c;
}
// Shared-memory layout of one scene's PGS.
struct PgsSmem {
  double* lam;     // c
  double* dshift;  // groups (regularisation shift per group, 0 if none)
  double* Wbb;     // kBR x kBR diagonal tile of the block being solved
  double* P;       // kBR lazy row products for the next block (helpers)
  double* dnext;   // kBR delta of the next block (read by the solver)
  double* red;     // 32 reduction slots
  int* flags;      // [0] abort code, [1] converged
};

__device__ __forceinline__ double w_reg(const PgsScene& s, const PgsSmem& sm, int64_t r, int64_t c) {
  double w = s.W[r * s.ldw + c];
  if (r == c) w = add(w, sm.dshift[r / 3]);
  return w;
}

__device__ void pgs_cta(const PgsScene& s, PgsSmem sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  const int64_t G = s.groups, c = 3 * G;
  const int nb = (int)((G + kBG - 1) / kBG);

  // ---- regularize (solver.py:99-121) ----
  double tr = 0.0;
  for (int64_t i = tid; i < c; i += blockDim.x) tr += s.W[i * s.ldw + i];
  tr = warp_sum(tr);
  if (lane == 0) sm.red[warp] = tr;
  if (tid == 0) sm.flags[0] = sm.flags[1] = 0;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < nwarps; ++w) t += sm.red[w];
    sm.red[31] = t;
  }
  __syncthreads();
  double shift = 1e-10 * sm.red[31] / (double)c;
  if (shift <= 0.0) shift = 1e-30;
  for (int64_t g = tid; g < G; g += blockDim.x) {
    double a[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        a[i][j] = 0.5 * (s.W[(3 * g + i) * s.ldw + 3 * g + j] + s.W[(3 * g + j) * s.ldw + 3 * g + i]);
    double e[3];
    sym3_eigs(a, e);
    double mn = fmin(e[0], fmin(e[1], e[2]));
    double scale = fmax(fmax(fabs(e[0]), fmax(fabs(e[1]), fabs(e[2]))), 1e-300);
    sm.dshift[g] = (mn <= 1e-12 * scale) ? shift : 0.0;
    if (s.shift_out) s.shift_out[g] = sm.dshift[g];
  }
  for (int64_t i = tid; i < c; i += blockDim.x) sm.lam[i] = 0.0;
  __syncthreads();

  // stage block 0: delta = delta_base (lambda = 0), diagonal tile
  // asynchronous copy (LDGSTS) of the block's diagonal tile, then the
  // regularisation shift on its diagonal (solver.py:119-120)
  auto stage_tile = [&](int b) {
    const int64_t r0 = (int64_t)b * kBR;
    const int rows = (int)min((int64_t)kBR, c - r0);
    for (int e = tid; e < rows * rows; e += blockDim.x) {
      int i = e / rows, j = e - i * rows;
      cp_async8(&sm.Wbb[i * kLDT + j], s.W + (r0 + i) * s.ldw + r0 + j, true);
    }
    cp_async_wait_all();
    __syncthreads();
    for (int i = tid; i < rows; i += blockDim.x) sm.Wbb[i * kLDT + i] = add(sm.Wbb[i * kLDT + i], sm.dshift[(r0 + i) / 3]);
  };
  stage_tile(0);
  for (int i = tid; i < (int)min((int64_t)kBR, c); i += blockDim.x) sm.dnext[i] = s.delta_base[i];
  // solver lane state
  double dl_[3] = {0, 0, 0}, lm[3] = {0, 0, 0};
  __syncthreads();

  const double h2 = s.h2;
  int iterations = 0;
  bool converged = false;
  for (int sweep = 0; sweep < s.max_iter; ++sweep) {
    iterations = sweep + 1;
    double dsq = 0.0;  // solver lanes: sum of squared lambda changes
    for (int b = 0; b < nb; ++b) {
      const int64_t g0 = (int64_t)b * kBG;
      const int ng = (int)min((int64_t)kBG, G - g0);
      const int bn = (b + 1 == nb) ? 0 : b + 1;  // next block (wraps to the next sweep)
      const int64_t gn0 = (int64_t)bn * kBG;
      const int ngn = (int)min((int64_t)kBG, G - gn0);
      if (warp == 0) {
        // ---- sequential block solve ----
        const bool mine = lane < ng;
        GroupConst kc{};
        if (mine) {
          for (int a = 0; a < 3; ++a) {
            lm[a] = sm.lam[3 * (g0 + lane) + a];
            dl_[a] = sm.dnext[3 * lane + a];
          }
          double Wd[9];
          for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) Wd[3 * i + j] = sm.Wbb[(3 * lane + i) * kLDT + 3 * lane + j];
          group_const(Wd, h2, kc);
        }
        int err = 0;
        block_solve<true>(sm.Wbb, ng, lane, dl_, lm, kc, s.mu, h2, dsq, err);
        const unsigned bad = __ballot_sync(0xffffffffu, mine && err);
        if (bad) {
          const int g = __ffs(bad) - 1;  // first failing group in Gauss-Seidel order
          if (lane == g) raise_status(s.status, CNB_E_SINGULAR_BLOCK, (int)(g0 + g), 1.0 / kc.ihw);
          if (lane == 0) sm.flags[0] = CNB_E_SINGULAR_BLOCK;
        } else if (mine) {
          for (int a = 0; a < 3; ++a) sm.lam[3 * (g0 + lane) + a] = lm[a];
        }
      } else if (nb > 1) {
        // ---- helpers: P[r] = W[r, not block b] lam for rows of block bn ----
        const int64_t rn0 = gn0 * 3;
        const int rows = 3 * ngn;
        const int64_t cb0 = g0 * 3, cb1 = cb0 + 3 * ng;
        for (int i = warp - 1; i < rows; i += nwarps - 1) {
          const int64_t r = rn0 + i;
          const double* wr = s.W + r * s.ldw;
          double acc = lane_dot<false>(wr, sm.lam, 0, cb0, lane) + lane_dot<false>(wr, sm.lam, cb1, c, lane);
          acc = warp_sum(acc);
          if (lane == 0) {
            // regularised diagonal of row r (inside block bn, never block b
            // unless nb == 1, which has no helpers)
            sm.P[i] = fma(sm.dshift[r / 3], sm.lam[r], acc);
          }
        }
      }
      __syncthreads();
      if (sm.flags[0]) break;
      if (b + 1 == nb) {
        // ---- end of sweep: epsilon (solver.py:194-199) ----
        if (warp == 0) {
          double v = warp_sum(dsq);
          if (lane == 0) sm.red[0] = v;
        }
        double nl = 0.0;
        for (int64_t i = tid; i < c; i += blockDim.x) nl += sm.lam[i] * sm.lam[i];
        nl = warp_sum(nl);
        if (lane == 0) sm.red[1 + warp] = nl;
        __syncthreads();
        if (tid == 0) {
          double den2 = 0.0;
          for (int w = 0; w < nwarps; ++w) den2 += sm.red[1 + w];
          const double num = sqrt(sm.red[0]), den = sqrt(den2);
          const double eps = (num == 0.0) ? 0.0 : (den == 0.0 ? INFINITY : num / den);
          s.eps_hist[sweep] = eps;
          sm.flags[1] = (eps <= s.tol) ? 1 : 0;
        }
        __syncthreads();
        if (sm.flags[1]) {
          converged = true;
          break;
        }
      }
      // ---- delta for the next block, its diagonal tile ----
      {
        const int64_t rn0 = gn0 * 3;
        const int rows = 3 * ngn;
        const int64_t cb0 = g0 * 3;
        const int cols = 3 * ng;
        for (int i = warp; i < rows; i += nwarps) {
          const int64_t r = rn0 + i;
          double acc = 0.0;
          if (nb > 1) {
            acc = lane_dot<false>(s.W + r * s.ldw + cb0, sm.lam + cb0, 0, cols, lane);
          } else {
            for (int j = lane; j < cols; j += 32) acc = fma(w_reg(s, sm, r, cb0 + j), sm.lam[cb0 + j], acc);
          }
          acc = warp_sum(acc);
          if (lane == 0) sm.dnext[i] = add(s.delta_base[r], mul(h2, (nb > 1 ? sm.P[i] : 0.0) + acc));
        }
        if (nb > 1) stage_tile(bn);
      }
      __syncthreads();
    }
    if (sm.flags[0] || converged) break;
  }
  __syncthreads();
  // ---- delta_end = delta_base + h^2 W_reg lam (solver.py:201); skipped when not wanted ----
  for (int64_t r = warp; s.delta_end && r < c; r += nwarps) {
    const double* wr = s.W + r * s.ldw;
    double acc = lane_dot<false>(wr, sm.lam, 0, c, lane);
    acc = warp_sum(acc);
    if (lane == 0) {
      acc = fma(sm.dshift[r / 3], sm.lam[r], acc);
      s.delta_end[r] = add(s.delta_base[r], mul(h2, acc));
    }
  }
  for (int64_t i = tid; i < c; i += blockDim.x) s.lam[i] = sm.lam[i];
  if (tid == 0) {
    s.iters_conv[0] = iterations;
    s.iters_conv[1] = converged ? 1 : 0;
  }
}

__host__ __device__ inline size_t pgs_smem_bytes(int64_t groups) {
  return sizeof(double) * (size_t)(3 * groups + groups + kBR * kLDT + 2 * kBR + 32) + 2 * sizeof(int) + 16;
}

__device__ __forceinline__ PgsSmem carve(char* base, int64_t groups) {
  PgsSmem sm;
  double* p = (double*)base;
  sm.lam = p;
  p += 3 * groups;
  sm.dshift = p;
  p += groups;
  sm.Wbb = p;
  p += kBR * kLDT;
  sm.P = p;
  p += kBR;
  sm.dnext = p;
  p += kBR;
  sm.red = p;
  p += 32;
  sm.flags = (int*)p;
  return sm;
}

__global__ void __launch_bounds__(kPgsThreads) pgs_single_kernel(PgsScene s) {
  extern __shared__ __align__(16) char smem[];
  pgs_cta(s, carve(smem, s.groups));
}

__global__ void __launch_bounds__(kPgsThreads) pgs_batched_kernel(const PgsScene* scenes) {
  extern __shared__ __align__(16) char smem[];
  PgsScene s = scenes[blockIdx.x];
  pgs_cta(s, carve(smem, s.groups));
}

__global__ void local_solve_kernel(int64_t alpha, const double* W, int64_t ldw, const double* dc,
                                   const double* lam, double mu, double h2, double* out,
                                   DevStatus* st) {
  const int64_t i = 3 * alpha;
  double Wd[9], d[3], l[3], o[3];
  for (int a = 0; a < 3; ++a) {
    d[a] = dc[i + a];
    l[a] = lam[i + a];
    for (int b = 0; b < 3; ++b) Wd[3 * a + b] = W[(i + a) * ldw + i + b];
  }
  if (local_solve_dev(d, l, Wd, mu, h2, o)) {
    raise_status(st, CNB_E_SINGULAR_BLOCK, (int)alpha, Wd[0]);
    o[0] = o[1] = o[2] = 0.0;
  }
  for (int a = 0; a < 3; ++a) out[a] = o[a];
}

size_t pgs_max_smem() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  return (size_t)v;
}

// ============================================================================
// Grid-scale PGS (thousands of groups: cfg2 / cfg3)
// ============================================================================
// Same iterate as pgs_cta.  One persistent cooperative kernel, one CTA per SM:
// CTA 0 is the solver (warp 0 runs the sequential block solve exactly as
// above); every other CTA is a helper that computes, for the rows of the next
// block, the lazy row products over all columns except the block being solved,
// split in column chunks (partial[buf][row][chunk], summed in fixed order by
// the solver: deterministic).  Hand-off through global counters:
//   solved = completed block steps (release by the solver, acquire by helpers)
//   ready  = helper CTAs done (cumulative; acquire by the solver)
// A device-clock watchdog turns a stuck wait into an error instead of a hang.
struct GridCtl {
  unsigned solved, ready, stop, timeout;
  unsigned ready4[4];  // pipelined kernel: helper completions of steps t = s (mod 4), per slot s
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// spin until *p >= target (or stop / watchdog); returns false on timeout
// Regularisation shift (solver.py:99-121) and the per-group constants of the
// regularised diagonal blocks, once per PGS call; lambda <- 0.
constexpr int kKC = 11;  // doubles per packed GroupConst
constexpr int kKCP = 9;  // leading doubles of the record the pipelined kernel stages
// Regularisation (solver.py:99-121) and the per-group constants of the grid
// kernels, grid-wide in two passes (a single CTA is latency-bound on the strided
// diagonal loads): pass 1, one thread per group,
// reads the group's diagonal block once, keeps the eigenvalue test (independent
// of the shift) in dshift as 0 / 1 and the CTA's trace partial in part[];
// pass 2: every CTA sums the partials in the same fixed order (the same shift
// everywhere) and writes the shifts, the group constants and lambda = 0.
constexpr int kPrepThreads = 128;
__global__ void __launch_bounds__(kPrepThreads) pgs_prep1_kernel(PgsScene s, double* dshift, double* part) {
  __shared__ double red[kPrepThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t g = (int64_t)blockIdx.x * kPrepThreads + tid;
  double tr = 0.0;
  if (g < s.groups) {
    double a[3][3], Wd[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) Wd[3 * i + j] = s.W[(3 * g + i) * s.ldw + 3 * g + j];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) a[i][j] = 0.5 * (Wd[3 * i + j] + Wd[3 * j + i]);
    tr = (Wd[0] + Wd[4]) + Wd[8];
    double e[3];
    sym3_eigs(a, e);
    const double mn = fmin(e[0], fmin(e[1], e[2]));
    const double scale = fmax(fmax(fabs(e[0]), fmax(fabs(e[1]), fabs(e[2]))), 1e-300);
    dshift[g] = (mn <= 1e-12 * scale) ? 1.0 : 0.0;
  }
  tr = warp_sum(tr);
  if (lane == 0) red[warp] = tr;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < kPrepThreads / 32; ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kPrepThreads) pgs_prep2_kernel(PgsScene s, double* dshift, double* kconst,
                                                                 const double* part, int nparts, GridCtl* ctl) {
  __shared__ double shs;
  const int tid = threadIdx.x;
  if (tid == 0) {
    double t = 0.0;
    for (int k = 0; k < nparts; ++k) t += part[k];
    double shift = 1e-10 * t / (double)(3 * s.groups);
    if (shift <= 0.0) shift = 1e-30;
    shs = shift;
    if (blockIdx.x == 0) {
      ctl->solved = ctl->ready = ctl->stop = ctl->timeout = 0;
      ctl->ready4[0] = ctl->ready4[1] = ctl->ready4[2] = ctl->ready4[3] = 0;
    }
  }
  __syncthreads();
  const int64_t g = (int64_t)blockIdx.x * kPrepThreads + tid;
  if (g < s.groups) {
    double Wd[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) Wd[3 * i + j] = s.W[(3 * g + i) * s.ldw + 3 * g + j];
    const double sh = dshift[g] != 0.0 ? shs : 0.0;
    dshift[g] = sh;
    for (int i = 0; i < 3; ++i) Wd[4 * i] = add(Wd[4 * i], sh);
    GroupConst kc;
    group_const(Wd, s.h2, kc);
    double* o = kconst + kKC * g;  // packed record, see load_group_const
    o[0] = kc.ihw;
    o[1] = kc.it00;
    o[2] = kc.it01;
    o[3] = kc.it10;
    o[4] = kc.it11;
    o[5] = kc.b0;
    o[6] = kc.b1;
    o[7] = (double)kc.bad;
    o[8] = kc.hwnn;
    o[9] = kc.htn0;
    o[10] = kc.htn1;
    for (int a = 0; a < 3; ++a) s.lam[3 * g + a] = 0.0;
  }
}

constexpr int kHelpPre = 32;  // W values per lane a helper warp holds in registers (32 x 32 columns)
// the pipelined kernel's chain reads its diagonal tile transposed (W symmetric:
// conflict-free shared loads), measured 1.347 -> 1.328 ms/sweep at cfg3
#ifndef PGS_TRANS
#define PGS_TRANS true
#endif
constexpr int kPipeThreads = 512;
constexpr int kPG = 26;             // groups per block
constexpr int kPR = 3 * kPG;        // rows per block
constexpr int kPS = kPR;            // dense tile rows (TMA box); 78 = 14 mod 16: at most 2-way bank conflicts
constexpr int kTileBytes = (kPR * kPS * 8 + 127) / 128 * 128;  // 128-byte aligned tiles
constexpr int kTileD = kTileBytes / 8;
constexpr int kXW = 9;              // X2 warps
constexpr int kXRows = (kPR + kXW - 1) / kXW;
constexpr int kPartBufs = 3;
constexpr int kHelpWarps = kPipeThreads / 32;         // warps per helper CTA
constexpr int kSeg = 4;                                // partial slots per row (helper CTAs a row can span)

__device__ __forceinline__ int x2_index(int warp) {  // warps 5,6,7,9,10,11,13,14,15 -> 0..8
  return (warp >= 5 && (warp & 3) != 0) ? ((warp >> 2) - 1) * 3 + (warp & 3) - 1 : -1;
}

struct PipeSmem {
  double *T0, *T1, *Wt, *X, *dcur, *lamx, *lamn, *kcn, *sv, *dbs, *dsh, *red;
  unsigned long long* bar;  // [0] T + Wt, [1] X
  int* flags;
};

__host__ __device__ inline size_t pipe_smem_bytes() {
  return 128 + sizeof(double) * (size_t)(4 * kTileD + kPR + 2 * kPR + 2 * kPR + kKCP * kPG + 4 * kPG + kPR + kPG + 8) +
         16 + 8 * sizeof(int);
}


__device__ __forceinline__ PipeSmem pipe_carve(char* base) {
  PipeSmem g;
  double* p = (double*)base;
  g.T0 = p;
  p += kTileD;
  g.T1 = p;
  p += kTileD;
  g.Wt = p;
  p += kTileD;
  g.X = p;
  p += kTileD;
  g.dcur = p;
  p += kPR;
  g.lamx = p;
  p += 2 * kPR;
  g.lamn = p;  // old lambda of the block being solved / of the next one, by step parity
  p += 2 * kPR;
  g.kcn = p;
  p += kKCP * kPG;
  g.sv = p;
  p += 4 * kPG;
  g.dbs = p;
  p += kPR;
  g.dsh = p;
  p += kPG;
  g.red = p;
  p += 8;
  g.bar = (unsigned long long*)p;
  p += 2;
  g.flags = (int*)p;
  return g;
}

// group constants of one group from a packed record (global or shared):
// [ihw, it00, it01, it10, it11, b0, b1, bad, hwnn, htn0, htn1]; the pipelined
// kernel stages only the first kKCP (what block_solve_v4 reads)
__device__ __forceinline__ void load_group_const(GroupConst& k, const double* kk, bool valid, int stride = kKC) {
  if (valid) {
    k.ihw = kk[0];
    k.it00 = kk[1];
    k.it01 = kk[2];
    k.it10 = kk[3];
    k.it11 = kk[4];
    k.b0 = kk[5];
    k.b1 = kk[6];
    k.bad = (int)kk[7];
    k.hwnn = kk[8];
    k.htn0 = stride > 9 ? kk[9] : 0.0;
    k.htn1 = stride > 10 ? kk[10] : 0.0;
  } else {
    k.ihw = k.hwnn = 1.0;
    k.htn0 = k.htn1 = k.it00 = k.it01 = k.it10 = k.it11 = k.b0 = k.b1 = 0.0;
    k.bad = 0;
  }
}

// Sequential Gauss-Seidel over one block, minimal per-group chain: every lane
// evaluates local_solve for its own group from the current delta (only the
// lane whose turn it is matters), broadcasts the h^2-scaled lambda change
// and all lanes apply the rank-3 delta update.  Nothing else happens per
// group: lane g only records (x, dh_t1, dh_t2, open) of its own group in sv,
// and block_commit turns the records into lambda after the block (a lane's
// lambda is read by the chain only at its own step).  Same branches as
// local_solve (solver.py:124-165): normal clamp at zero, frictionless,
// tangential stick solve, projection onto the cone.
// CHUNKS: after the groups ending at e1 and e2 and after the last group the
// warp arrives at named barriers 7, 8 and 9 (with the phase-B warp, 64
// threads): the records of those groups are final, and the phase-B warp folds
// them into the next block's delta while the chain continues.
template <bool FRIC, bool CHUNKS = false, bool TRANS = false>
__device__ __forceinline__ void block_solve_v4(const double* __restrict__ Wt, int ld, int ng, int lane,
                                               double dl_[3], const double lm[3], const GroupConst& kc, double mu,
                                               double h2, double* __restrict__ sv, int e1 = 0, int e2 = 0) {
  // TRANS: read W[g, l] instead of W[l, g] (W is symmetric): at step g the lanes
  // read consecutive columns of the same three rows (no bank conflicts)
  const int lr = (TRANS && lane >= 32 - 4) ? 0 : lane;
  const double* wrow = Wt + 3 * lr * ld;
  const double* wcol = Wt + 3 * lr;
  const double h2l1 = h2 * lm[1], h2l2 = h2 * lm[2];
  const double nl0 = -lm[0], lhw = lm[0] * kc.hwnn, nihw = -kc.ihw;
#pragma unroll 2
  for (int g = 0; g < ng; ++g) {
    double w[9];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) w[3 * a + c] = TRANS ? wcol[(3 * g + c) * ld + a] : wrow[a * ld + 3 * g + c];
    const double d0 = dl_[0], d1 = dl_[1], d2 = dl_[2];
    const bool open = d0 < lhw;                        // l_n - d_n/(h^2 W_nn) > 0
    const double x = fma(nihw, d0, lm[0]);
    const double dln = open ? d0 * nihw : nl0;         // max(0, x) - l_n
    double dh0 = h2 * dln, dh1, dh2;
    if (FRIC) {
      const double a0 = fma(-kc.it00, d1, fma(-kc.it01, d2, lm[1]));
      const double a1 = fma(-kc.it10, d1, fma(-kc.it11, d2, lm[2]));
      const double lt0 = fma(-kc.b0, dln, a0), lt1 = fma(-kc.b1, dln, a1);
      const double radius = mu * x;
      const double n2 = fma(lt0, lt0, lt1 * lt1);
      const bool proj = n2 > radius * radius;
      double y;
      asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(n2));
      const double e = fma(-0.5 * n2, y * y, 1.5);   // rsqrt(n2) = y e (one Newton step)
      const double ry = radius * y;
      const double hl0 = h2 * lt0, hl1 = h2 * lt1;
      const double p0 = fma(hl0 * ry, e, -h2l1), p1 = fma(hl1 * ry, e, -h2l2);
      const double u0 = hl0 - h2l1, u1 = hl1 - h2l2;
      dh1 = open ? (proj ? p0 : u0) : -h2l1;
      dh2 = open ? (proj ? p1 : u1) : -h2l2;
    } else {
      dh1 = -h2l1;
      dh2 = -h2l2;
    }
    const double s0 = __shfl_sync(0xffffffffu, dh0, g);
    const double s1 = __shfl_sync(0xffffffffu, dh1, g);
    const double s2 = __shfl_sync(0xffffffffu, dh2, g);
    // the owning lane records its group (predicated stores: no divergent branch)
    asm volatile(
        "{\n .reg .pred p;\n setp.eq.s32 p, %0, %1;\n"
        " @p st.shared.v2.f64 [%2], {%3, %4};\n @p st.shared.v2.f64 [%2+16], {%5, %6};\n}\n" ::"r"(lane),
        "r"(g), "r"(smem_u32(sv + 4 * g)), "d"(x), "d"(dh1), "d"(dh2), "d"(open ? 1.0 : 0.0)
        : "memory");
#pragma unroll
    for (int a = 0; a < 3; ++a) dl_[a] = fma(w[3 * a + 2], s2, fma(w[3 * a + 1], s1, fma(w[3 * a], s0, dl_[a])));
    if (CHUNKS) {
      if (g == e1 - 1) asm volatile("bar.arrive 7, 64;" ::: "memory");
      if (g == e2 - 1) asm volatile("bar.arrive 8, 64;" ::: "memory");
    }
  }
  if (CHUNKS) asm volatile("bar.arrive 9, 64;" ::: "memory");
}

// lambda of the lane's group from its block_solve_v4 record; dsq += |change|^2;
// returns the error flag (W_nn <= 0, or a singular tangential block when used)
__device__ __forceinline__ int block_commit(const double* sv, int lane, double lm[3], const GroupConst& kc,
                                            double mu, double ih2, double& dsq) {
  const double x = sv[4 * lane], dh1 = sv[4 * lane + 1], dh2 = sv[4 * lane + 2];
  const bool open = sv[4 * lane + 3] != 0.0;
  const bool fric = open && mu != 0.0;
  const double n0 = open ? fmax(x, 0.0) : 0.0;
  const double n1 = fric ? fma(dh1, ih2, lm[1]) : 0.0;
  const double n2 = fric ? fma(dh2, ih2, lm[2]) : 0.0;
  const double q0 = n0 - lm[0], q1 = n1 - lm[1], q2 = n2 - lm[2];
  dsq += q0 * q0 + q1 * q1 + q2 * q2;
  lm[0] = n0;
  lm[1] = n1;
  lm[2] = n2;
  return ((kc.bad & 1) || (fric && (kc.bad & 2))) ? 1 : 0;
}

__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_gpu_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// spin (acquire) until *p >= target, or stop / watchdog; false on timeout
__device__ bool wait_acq(const unsigned* p, unsigned target, const unsigned* stop, GridCtl* ctl) {
  const unsigned long long t0 = global_ns();
  while (ld_acquire_gpu(p) < target) {
    if (stop && ld_acquire_gpu(stop)) return true;
    if (global_ns() - t0 > 20000000000ull) {  // 20 s
      atomicExch(&ctl->timeout, 1u);
      atomicExch(&ctl->stop, 1u);
      return false;
    }
  }
  return true;
}

// Tagged records ("LL" style): a double split into two 8-byte words, each
// carrying 32 data bits and the 32-bit tag of the step that wrote it.  An
// 8-byte store is single-copy atomic, so a word whose tag matches carries that
// step's data: the consumer polls the record itself, no fence or counter.
__device__ __forceinline__ void ll_store(double* slot, double v, unsigned tag) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const unsigned long long w0 = (b & 0xffffffffull) | ((unsigned long long)tag << 32);
  const unsigned long long w1 = (b >> 32) | ((unsigned long long)tag << 32);
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};\n" ::"l"(slot), "l"(w0), "l"(w1) : "memory");
}
__device__ __forceinline__ double ll_load(const double* slot, unsigned tag, GridCtl* ctl) {
  unsigned long long w0, w1;
  unsigned long long t0 = 0;
  for (unsigned n = 0;; ++n) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(w0), "=l"(w1) : "l"(slot) : "memory");
    if ((unsigned)(w0 >> 32) == tag && (unsigned)(w1 >> 32) == tag) break;
    __nanosleep(64);  // polling loads share the SM's memory pipe with the solver warp
    if ((n & 1023) == 0) {  // watchdog
      const unsigned long long now = global_ns();
      if (n == 0) t0 = now;
      else if (now - t0 > 20000000000ull) {
        atomicExch(&ctl->timeout, 1u);
        atomicExch(&ctl->stop, 1u);
        return 0.0;
      }
    }
  }
  return __longlong_as_double((long long)((w0 & 0xffffffffull) | (w1 << 32)));
}

__global__ void __launch_bounds__(kPipeThreads) pgs_pipe_kernel(PgsScene s, const double* __restrict__ dshift,
                                                                const double* __restrict__ kconst, double* partial,
                                                                GridCtl* ctl, int nch, int lam_in_smem, int tma,
                                                                unsigned long long* prof, unsigned tag0,
                                                                const __grid_constant__ CUtensorMap tmap) {
  const int dbg = tma & ~1;
  tma = (dbg & 2) ? 0 : (tma & 1);
  extern __shared__ __align__(16) char smem_dyn[];
  // 128-byte aligned base for the TMA tiles; offsetting the shared array (not
  // an integer round trip) keeps the accesses LDS/STS instead of generic loads
  char* smem_raw = smem_dyn + ((128u - (smem_u32(smem_dyn) & 127u)) & 127u);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t G = s.groups, c = 3 * G;
  const int nb = (int)((G + kPG - 1) / kPG);
  const double h2 = s.h2;
  double* lamg = s.lam;
  unsigned* psolved = &ctl->solved;
  unsigned* pstop = &ctl->stop;
  const size_t pstride = (size_t)kPR * kSeg;  // one partial buffer: kSeg row sums per row
  auto rows_of = [&](int blk) { return 3 * (int)min((int64_t)kPG, G - (int64_t)blk * kPG); };
  auto wrap = [&](int blk) { return blk >= nb ? blk - nb : blk; };
  // CNB_PGS_PROFILE=1 (SM cycles per phase, summed; clock64, the global timer is
  // too coarse for sub-microsecond phases): tid 0: [0] idle at B1, [1] phase B,
  // [2] block solve; tid 32+64*.. see stamp() calls; helpers (CTA 1, tid 0): [4] wait, [5] work
  unsigned long long tp = 0;
  const bool stamper = prof && (tid == 0 || tid == 32 || tid == 64 || tid == 96 || tid == 160) && blockIdx.x <= 1;
  auto stamp = [&](int k) {
    if (stamper) {
      const unsigned long long now = (unsigned long long)clock64();
      if (k >= 0) atomicAdd(prof + k, now - tp);  // fire-and-forget RED
      tp = now;
    }
  };

  if (blockIdx.x == 0) {
    // ---- solver CTA.  Step t solves block b; meanwhile, for block b+1:
    //   warp 2: tensor TMA of T(b+1) and Wt = W[b, b+1] (the transpose of
    //           W[b+1, b] by symmetry: its rows are W[b+1, b]'s columns), then
    //           X = W[b+2, b] for the next step's X2, then the regularisation
    //           shift of T(b+1)'s diagonal;
    //   warp 3: lambda(b+1) (previous sweep), group constants, delta_base and
    //           shifts of b+1; then phase B: W[b+1, b] (lambda_b new) folded in
    //           chunk by chunk as the solver releases its groups (named
    //           barriers 7-9), so only the last chunk follows the chain;
    //   X2 warps: W[b+1, b-1] lambda_{b-1} and the helpers' row partials;
    //   warp 1: publisher of each solved block's lambda.
    // One CTA barrier per step (B2); the other hand-offs are named barriers
    // between the warps involved.
    PipeSmem sm = pipe_carve(smem_raw);
    const int xi = x2_index(warp);
    constexpr int kC1 = 9, kC2 = 18;  // phase-B chunk ends (groups)
    if (tid == 0) {
      sm.flags[0] = sm.flags[1] = 0;
      mbar_init(sm.bar, 1);
      mbar_init(sm.bar + 1, 1);
    }
    // prologue: T(0), delta(0); X = W[2, 0] for step 1 is fetched in step 0
    {
      const int r0 = rows_of(0);
      for (int i = warp; i < r0; i += kPipeThreads / 32)
        for (int j = lane; j < r0; j += 32) cp_async8(&sm.T0[i * kPS + j], s.W + i * s.ldw + j, true);
      cp_async_wait_all();
    }
    for (int i = tid; i < kPR; i += blockDim.x) {
      sm.dcur[i] = i < rows_of(0) ? s.delta_base[i] : 0.0;
      sm.lamn[i] = sm.lamn[kPR + i] = 0.0;  // lambda starts at zero (prep zeroed the global copy)
      sm.lamx[i] = sm.lamx[kPR + i] = 0.0;
    }
    __syncthreads();
    for (int i = tid; i < rows_of(0); i += blockDim.x)
      sm.T0[i * kPS + i] = add(sm.T0[i * kPS + i], dshift[i / 3]);
    GroupConst kc{};
    double dsq = 0.0;
    const double ih2 = 1.0 / h2;
    if (warp == 0) load_group_const(kc, kconst + kKC * lane, lane < rows_of(0) / 3);
    volatile unsigned* vcnt = (volatile unsigned*)(sm.flags + 4);  // [0] lambda in smem, [1] published (steps)
    if (tid == 0) {
      sm.flags[2] = 0;
      vcnt[0] = vcnt[1] = 0;
    }
    __syncthreads();
    stamp(-1);
    int iterations = 0;
    bool converged = false;
    if (warp != 1) {
    for (unsigned t = 0;; ++t) {
      const int b = (int)(t % nb), sweep = (int)(t / nb);
      const int b1 = wrap(b + 1), b2 = wrap(b + 2), bm = (b == 0) ? nb - 1 : b - 1;
      const int rows = rows_of(b), rows1 = rows_of(b1), rowsm = rows_of(bm);
      const int slot = (int)(t & 1);
      double* Tc = slot ? sm.T1 : sm.T0;
      double* Tn = slot ? sm.T0 : sm.T1;
      double* lamc = sm.lamx + slot * kPR;         // lambda_b (this solve)
      double* lamp = sm.lamx + (slot ^ 1) * kPR;   // lambda_{b-1}
      const double* lold = sm.lamn + slot * kPR;   // lambda_b before this solve
      double* lnext = sm.lamn + (slot ^ 1) * kPR;  // lambda_{b+1} before its solve
      const int64_t rb = 3 * (int64_t)b * kPG, rb1 = 3 * (int64_t)b1 * kPG;
      const int ng = rows / 3;
      const int e1 = min(ng, kC1), e2 = min(ng, kC2);
      if (warp == 0) {
        // ---- sequential block solve ----
        const bool mine = lane < ng;
        double lm[3], dl[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          lm[a] = mine ? lold[3 * lane + a] : 0.0;
          dl[a] = mine ? sm.dcur[3 * lane + a] : 0.0;
        }
        asm volatile("bar.arrive 2, %0;" ::"n"(32 + 32 * kXW));  // dcur consumed
        stamp(13);
        if (s.mu != 0.0)
          block_solve_v4<true, true, PGS_TRANS>(Tc, kPS, ng, lane, dl, lm, kc, s.mu, h2, sm.sv, e1, e2);
        else
          block_solve_v4<false, true, PGS_TRANS>(Tc, kPS, ng, lane, dl, lm, kc, s.mu, h2, sm.sv, e1, e2);
        __syncwarp();
        stamp(14);
        const int err = mine ? block_commit(sm.sv, lane, lm, kc, s.mu, ih2, dsq) : 0;
        const unsigned bad = __ballot_sync(0xffffffffu, err);
        if (bad) {
          const int g = __ffs(bad) - 1;  // first failing group in Gauss-Seidel order
          if (lane == g) raise_status(s.status, CNB_E_SINGULAR_BLOCK, (int)(rb / 3 + g), 1.0 / kc.ihw);
          if (lane == 0) sm.flags[0] = 1;
        }
        if (t >= 2)  // the publisher has read this slot's previous lambda (step t-2)
          while (vcnt[1] + 1 < t) {
          }
        if (mine)
#pragma unroll
          for (int a = 0; a < 3; ++a) lamc[3 * lane + a] = lm[a];
        __syncwarp();
        if (lane == 0)  // lambda_b in shared memory: the publisher takes it (release: no full fence)
          asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(smem_u32((const void*)&vcnt[0])), "r"(t + 1)
                       : "memory");
        if (b == nb - 1) {  // end of sweep: ||dlam||^2 and this block's ||lambda||^2
          const double l2 = mine ? (lm[0] * lm[0] + lm[1] * lm[1]) + lm[2] * lm[2] : 0.0;
          const double sl = warp_sum(l2), sd = warp_sum(dsq);
          if (lane == 0) {
            sm.red[0] = sd;
            sm.red[1] = sl;
          }
          dsq = 0.0;
        }
        stamp(2);
        // next block's group constants (warp 3 staged them: barrier 10)
        asm volatile("bar.sync 10, 64;" ::: "memory");
        load_group_const(kc, sm.kcn + kKCP * lane, lane < rows1 / 3, kKCP);
        if (b == nb - 1 && lane == 0 && !sm.flags[0]) {
          while (vcnt[1] < t) {  // the publisher's sum of blocks 0..nb-2 (step t-1) is in red[2]
          }
          const double num = sqrt(sm.red[0]), den = sqrt(sm.red[1] + sm.red[2]);
          const double eps = (num == 0.0) ? 0.0 : (den == 0.0 ? INFINITY : num / den);
          s.eps_hist[sweep] = eps;
          sm.flags[1] = (eps <= s.tol) ? 1 : ((sweep + 1 >= s.max_iter) ? 2 : 0);
        }
        stamp(0);
      } else if (warp == 2) {
        // T(b+1) and Wt = W[b, b+1]: one tensor-TMA box each (out-of-range rows and
        // columns of a ragged last block arrive as zeros)
        if (tma) {
          if (lane == 0) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(sm.bar, 2u * kPR * kPS * 8);
            tma_load_2d(Tn, &tmap, (int)rb1, (int)rb1, sm.bar);
            tma_load_2d(sm.Wt, &tmap, (int)rb1, (int)rb, sm.bar);
          }
        } else {
          for (int i = 0; i < rows1; ++i) {
            const double* src = s.W + (rb1 + i) * s.ldw;
            for (int j = lane; j < rows1; j += 32) cp_async8(&Tn[i * kPS + j], src + rb1 + j, true);
          }
          for (int i = 0; i < rows; ++i) {
            const double* src = s.W + (rb + i) * s.ldw;
            for (int j = lane; j < rows1; j += 32) cp_async8(&sm.Wt[i * kPS + j], src + rb1 + j, true);
          }
          cp_async_wait_all();
          __syncwarp();
        }
        stamp(10);
        // X = W[b+2, b] for the next step's X2, once this step's X2 has read the tile
        asm volatile("bar.sync 3, %0;" ::"n"(32 + 32 * kXW));
        stamp(11);
        const int rows2 = rows_of(b2);
        const int64_t rb2 = 3 * (int64_t)b2 * kPG;
        if (tma) {
          if (lane == 0) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(sm.bar + 1, 1u * kPR * kPS * 8);
            tma_load_2d(sm.X, &tmap, (int)rb, (int)rb2, sm.bar + 1);
          }
        } else {
          for (int i = 0; i < rows2; ++i)
            for (int j = lane; j < rows; j += 32) cp_async8(&sm.X[i * kPS + j], s.W + (rb2 + i) * s.ldw + rb + j, true);
          cp_async_wait_all();
        }
        stamp(12);
        // regularisation shift of T(b+1)'s diagonal (shifts staged by warp 3: barrier 11)
        if (tma) mbar_wait(sm.bar, t & 1);
        asm volatile("bar.sync 11, 64;" ::: "memory");
        for (int i = lane; i < rows1; i += 32) Tn[i * kPS + i] = add(Tn[i * kPS + i], sm.dsh[i / 3]);
      } else if (warp == 3) {
        double lv[3];
#pragma unroll
        for (int u = 0; u < 3; ++u) {
          const int j = lane + 32 * u;
          lv[u] = j < rows1 ? __ldcg(lamg + rb1 + j) : 0.0;
        }
        for (int e = lane; e < kKCP * rows1 / 3; e += 32) {
          const int g = e / kKCP, k = e - g * kKCP;
          cp_async8(&sm.kcn[e], kconst + kKC * (rb1 / 3 + g) + k, true);
        }
        // delta_base and the regularisation shifts of block b+1
        for (int j = lane; j < rows1; j += 32) cp_async8(&sm.dbs[j], s.delta_base + rb1 + j, true);
        if (lane < rows1 / 3) cp_async8(&sm.dsh[lane], dshift + rb1 / 3 + lane, true);
#pragma unroll
        for (int u = 0; u < 3; ++u) {
          const int j = lane + 32 * u;
          if (j < kPR) lnext[j] = lv[u];
        }
        cp_async_wait_all();
        __syncwarp();
        asm volatile("bar.arrive 10, 64;" ::: "memory");  // constants of b+1 -> warp 0
        asm volatile("bar.arrive 11, 64;" ::: "memory");  // shifts of b+1 -> warp 2
        // ---- phase B: v = W[b+1, b] lambda_b, lane <-> rows lane, lane+32, lane+64 of
        // block b+1; lambda_b of a group from the solver's record (block_commit's
        // arithmetic), the column of W[b+1, b] from row 3g+a of Wt (contiguous)
        if (tma) mbar_wait(sm.bar, t & 1);
        double v[3] = {0.0, 0.0, 0.0};
        const bool fr = s.mu != 0.0;
        auto fold = [&](int gs, int ge) {
          for (int g = gs; g < ge; ++g) {
            const double2 ra = *reinterpret_cast<const double2*>(sm.sv + 4 * g);      // x, dh1
            const double2 rc = *reinterpret_cast<const double2*>(sm.sv + 4 * g + 2);  // dh2, open
            const bool open = rc.y != 0.0, fric = open && fr;
            const double n0 = open ? fmax(ra.x, 0.0) : 0.0;
            const double n1 = fric ? fma(ra.y, ih2, lold[3 * g + 1]) : 0.0;
            const double n2 = fric ? fma(rc.x, ih2, lold[3 * g + 2]) : 0.0;
            const double* w0 = sm.Wt + (3 * g) * kPS;
#pragma unroll
            for (int u = 0; u < 3; ++u) {
              const int r = lane + 32 * u;
              if (r < kPR)
                v[u] = fma(w0[2 * kPS + r], n2, fma(w0[kPS + r], n1, fma(w0[r], n0, v[u])));
            }
          }
        };
        asm volatile("bar.sync 7, 64;" ::: "memory");
        fold(0, e1);
        asm volatile("bar.sync 8, 64;" ::: "memory");
        fold(e1, e2);
        asm volatile("bar.sync 9, 64;" ::: "memory");
        fold(e2, ng);
        stamp(9);
        // the X2 warps' part of delta(b+1) is in dcur (barrier 12)
        asm volatile("bar.sync 12, %0;" ::"n"(32 + 32 * kXW) : "memory");
#pragma unroll
        for (int u = 0; u < 3; ++u) {
          const int r = lane + 32 * u;
          if (r < rows1) sm.dcur[r] = add(sm.dbs[r], mul(h2, sm.dcur[r] + v[u]));
        }
      } else if (xi >= 0) {
        // X2 = W[b+1, b-1] lambda_{b-1} from the X tile (fetched last step)
        if (tma && t > 0) mbar_wait(sm.bar + 1, (t - 1) & 1);
        // lanes 3k..3k+2 share row xi + kXW*k (k < 9), a third of its columns each
        double x2v = 0.0;
        {
          const int k = lane / 3, part = lane - 3 * k;
          const int i = xi + kXW * k;
          if (t > 0 && lane < 3 * kXRows && i < rows1) {
            const double* xr = sm.X + i * kPS;
            const int j0 = part * (kPR / 3), j1 = min(j0 + kPR / 3, rowsm);
            double a0 = 0.0, a1 = 0.0;
            int j = j0;
            for (; j + 1 < j1; j += 2) {
              a0 = fma(xr[j], lamp[j], a0);
              a1 = fma(xr[j + 1], lamp[j + 1], a1);
            }
            if (j < j1) a0 = fma(xr[j], lamp[j], a0);
            x2v = a0 + a1;
          }
          const double n1 = __shfl_down_sync(0xffffffffu, x2v, 1), n2 = __shfl_down_sync(0xffffffffu, x2v, 2);
          x2v = (x2v + n1) + n2;  // valid in lanes 3k
        }
        asm volatile("bar.arrive 3, %0;" ::"n"(32 + 32 * kXW));  // X tile free for the next fetch
        if (xi == 0) stamp(6);
        // partials of block b+1 (helpers, step t-1): the tagged row sums, one per
        // helper CTA the row spans, added in fixed order; lane k <-> row xi + kXW k
        if (xi == 0) stamp(3);
        const double* part = partial + 2 * (size_t)((t + kPartBufs - 1) % kPartBufs) * pstride;
        double pvl = 0.0;
        {
          const int i = xi + kXW * lane;
          if (t > 0 && lane < kXRows && i < rows1) {
            const int nseg = ((i + 1) * nch - 1) / kHelpWarps - (i * nch) / kHelpWarps + 1;
            for (int sg = 0; sg < nseg; ++sg) pvl += ll_load(part + 2 * ((size_t)i * kSeg + sg), tag0 + t - 1, ctl);
          }
        }
        asm volatile("bar.sync 2, %0;" ::"n"(32 + 32 * kXW));  // warp 0 has read dcur
        const double pk = __shfl_sync(0xffffffffu, pvl, lane / 3);  // lane 3k picks up row k's sum
        {
          const int k = lane / 3, i = xi + kXW * k;
          if (lane == 3 * k && k < kXRows && i < rows1) sm.dcur[i] = x2v + pk;  // partial sums of block b+1
        }
        __syncwarp();
        asm volatile("bar.arrive 12, %0;" ::"n"(32 + 32 * kXW) : "memory");  // -> warp 3 (phase B)
        if (xi == 0) stamp(7);
      }
      asm volatile("bar.sync 6, %0;" ::"n"(kPipeThreads - 32) : "memory");  // B2 (all but the publisher)
      if (warp == 0 || warp == 5) stamp(1); else stamp(-1);
      if (b == nb - 1) {
        iterations = sweep + 1;
        converged = sm.flags[1] == 1;
      }
      if (sm.flags[0] || sm.flags[1]) {
        if (tma && warp == 2) mbar_wait(sm.bar + 1, t & 1);  // drain the X fetch in flight
        if (tid == 0) sm.flags[2] = 1;                       // the publisher stops after this step
        break;
      }
    }
    } else {
      // ---- warp 1: publisher.  Copies each solved block's lambda to global
      // memory and releases the helpers (psolved = steps published), keeps
      // ||lambda||^2 of the sweep; decoupled from the step barriers, so the
      // release fence never delays the solver.
      double sumsq = 0.0;
      for (unsigned t = 0;; ++t) {
        if (lane == 0) {
          while (vcnt[0] < t + 1 && !*(volatile int*)&sm.flags[2]) __nanosleep(20);
          if (*(volatile unsigned*)&ctl->timeout) sm.flags[0] = 1;  // watchdog fired elsewhere
        }
        unsigned seen;
        asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(seen) : "r"(smem_u32((const void*)&vcnt[0])) : "memory");
        const unsigned go = __shfl_sync(0xffffffffu, seen >= t + 1 ? 1u : 0u, 0);
        if (!go) break;
        const int b = (int)(t % nb), rows = rows_of(b);
        const int64_t rb = 3 * (int64_t)b * kPG;
        const double* lamc = sm.lamx + (t & 1) * kPR;
        double v = 0.0;
        for (int j = lane; j < rows; j += 32) {
          const double l = lamc[j];
          __stcg(lamg + rb + j, l);
          v = fma(l, l, v);
        }
        __syncwarp();
        if (lane == 0) st_release_gpu(psolved, t + 1);
        // ||lambda||^2 of blocks 0..nb-2 of this sweep (fixed order); warp 0 adds the last
        if (b == 0) sumsq = 0.0;
        if (b < nb - 1) sumsq += warp_sum(v);
        if (b == nb - 2 && lane == 0) sm.red[2] = sumsq;
        __syncwarp();
        if (lane == 0)
          asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(smem_u32((const void*)&vcnt[1])), "r"(t + 1)
                       : "memory");
      }
    }
    // everyone (publisher included): last lambda block is in global memory; release the grid
    __syncthreads();
    if (tid == 0) {
      st_release_gpu(pstop, 1u);
      s.iters_conv[0] = iterations;
      s.iters_conv[1] = converged ? 1 : 0;
    }
  } else {
    // ---- helpers ----
    // Each helper warp owns one (row, column chunk) item per step; the chunk
    // index is fixed, the row moves with the step.  Step t: wait for
    // lambda_{b-1}, refresh it in shared memory, dot products from registers,
    // then at once issue the loads of step t+1's W slice (hidden behind the
    // reduction and the next wait), and warp 0 reduces the CTA's items per row
    // and stores the sums as tagged records (no fence, no counter).
    double* lams = (double*)smem_raw;
    __shared__ unsigned hflag;
    __shared__ double hp[kHelpWarps];
    const unsigned hw = (blockIdx.x - 1) * kHelpWarps + warp;
    const int64_t csz = (((c + nch - 1) / nch) + 1) & ~(int64_t)1;  // even: 16-byte column pairs
    struct Item {
      bool has;
      int i, rows2;
      int64_t r, c0, c1, e0, e1, f0, f1;
    };
    auto item_of = [&](unsigned tt) {
      Item it;
      const int b = (int)(tt % nb), b1 = wrap(b + 1), b2 = wrap(b + 2);
      it.rows2 = rows_of(b2);
      it.has = hw < (unsigned)(it.rows2 * nch);
      it.i = it.has ? (int)(hw / nch) : 0;
      const int ch = it.has ? (int)(hw % nch) : 0;
      it.r = 3 * (int64_t)b2 * kPG + it.i;
      it.c0 = (int64_t)ch * csz;
      it.c1 = min(c, it.c0 + csz);
      it.e0 = 3 * (int64_t)b * kPG;  // excluded: block b
      it.e1 = it.e0 + rows_of(b);
      it.f0 = 3 * (int64_t)b1 * kPG;  // excluded: block b+1
      it.f1 = it.f0 + rows_of(b1);
      return it;
    };
    // W slice in registers: lane holds column pairs (c0 + 2 lane + 64 u, +1); the
    // pipelined kernel requires an even row pitch, so every pair is 16-byte aligned,
    // and block boundaries (multiples of 78) never split a pair
    double2 wv[kHelpPre / 2];
    auto preload = [&](const Item& it) {
      const double* wr = s.W + it.r * s.ldw;
#pragma unroll
      for (int u = 0; u < kHelpPre / 2; ++u) {
        const int64_t j = it.c0 + 2 * lane + 64 * u;
        const bool ok = it.has && j < it.c1 && (j < it.e0 || j >= it.e1) && (j < it.f0 || j >= it.f1);
        if (ok && j + 1 < it.c1) {
          wv[u] = *reinterpret_cast<const double2*>(wr + j);
        } else {
          wv[u].x = ok ? wr[j] : 0.0;
          wv[u].y = 0.0;
        }
      }
    };
    // L2 prefetch, about two steps ahead, of what the solver CTA will fetch for
    // block q = b+4: W[q, b+2] (its X tile at step t+2), W[q, b+3] (its Wx tile
    // at step t+3), lambda(q), delta_base(q), group constants(q)
    auto l2_prefetch = [&](unsigned tt) {
      const int b = (int)(tt % nb), q = (b + 4) % nb, qa = (b + 2) % nb, qb = (b + 3) % nb;
      const int rq = rows_of(q);
      const int64_t q0 = 3 * (int64_t)q * kPG;
      if (hw < (unsigned)rq) {
        const double* qr = s.W + (q0 + hw) * s.ldw;
        const int64_t cb = 3 * (int64_t)((lane < 8) ? qa : qb) * kPG;
        const int64_t j = cb + 16 * (lane & 7);
        if (lane < 16 && 16 * (lane & 7) < kPR + 15 && j < c) asm volatile("prefetch.global.L2 [%0];" ::"l"(qr + j));
      } else if (hw == (unsigned)rq) {
        const int64_t g0 = q0 / 3;
        const int64_t jl = q0 + 16 * lane, jd = q0 + 16 * (lane - 6), jk = kKC * g0 + 16 * (lane - 12);
        if (lane < 6) {
          if (jl < c) asm volatile("prefetch.global.L2 [%0];" ::"l"(lamg + jl));
        } else if (lane < 12) {
          if (jd < c) asm volatile("prefetch.global.L2 [%0];" ::"l"(s.delta_base + jd));
        } else if (lane < 30 && jk < kKC * G) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(kconst + jk));
        }
      }
    };
    if (stamper) tp = (unsigned long long)clock64();
    long long hc = clock64();
    auto hstamp = [&](int k) {  // CNB_PGS_PROFILE: cycles per helper phase (CTA 1, thread 0), slots 16..21
      if (prof && blockIdx.x == 1 && tid == 0) {
        const long long n = clock64();
        atomicAdd(prof + k, (unsigned long long)(n - hc));
        hc = n;
      }
    };
    Item it = item_of(0);
    preload(it);
    l2_prefetch(0);
    for (unsigned t = 0;; ++t) {
      const int b = (int)(t % nb), bm = (b == 0) ? nb - 1 : b - 1;
      stamp(5);
      // one thread decides stop and broadcasts it (threads reading the flag
      // themselves could disagree and split the CTA at the next barrier)
      if (tid == 0) {
        wait_acq(psolved, t, pstop, ctl);
        hflag = ld_acquire_gpu(pstop);
      }
      __syncthreads();
      const unsigned hstop = hflag;
      hstamp(16);  // wait for the solver
      stamp(4);
      if (hstop) break;
      if (lam_in_smem) {
        if (t == 0) {
          for (int64_t j = tid; j < c; j += blockDim.x) lams[j] = 0.0;
        } else {
          const int64_t pb0 = 3 * (int64_t)bm * kPG;
          const int pcols = rows_of(bm);
          for (int j = tid; j < pcols; j += blockDim.x) lams[pb0 + j] = __ldcg(lamg + pb0 + j);
        }
        __syncthreads();
      }
      hstamp(17);  // lambda refresh
      if (it.has) {
        const double* wr = s.W + it.r * s.ldw;
        double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int u = 0; u < kHelpPre / 2; ++u) {
          const int64_t j = min(it.c0 + 2 * lane + 64 * u, (c - 1) & ~(int64_t)1);
          double2 l;
          if (lam_in_smem) {
            l = *reinterpret_cast<const double2*>(lams + j);
          } else {
            l.x = __ldcg(lamg + j);
            l.y = j + 1 < c ? __ldcg(lamg + j + 1) : 0.0;
          }
          a[(2 * u) & 3] = fma(wv[u].x, l.x, a[(2 * u) & 3]);
          a[(2 * u + 1) & 3] = fma(wv[u].y, l.y, a[(2 * u + 1) & 3]);
        }
        for (int64_t j0 = it.c0 + 32 * kHelpPre; j0 < it.c1; j0 += 32 * kHelpPre) {  // slices wider than the registers
#pragma unroll 8
          for (int u = 0; u < kHelpPre; ++u) {
            const int64_t j = j0 + lane + 32 * u;
            if (j < it.c1 && (j < it.e0 || j >= it.e1) && (j < it.f0 || j >= it.f1))
              a[u & 3] = fma(wr[j], lam_in_smem ? lams[j] : __ldcg(lamg + j), a[u & 3]);
          }
        }
        double acc = warp_sum((a[0] + a[1]) + (a[2] + a[3]));
        if (lane == 0) {
          if (it.r >= it.c0 && it.r < it.c1)
            acc = fma(dshift[it.r / 3], lam_in_smem ? lams[it.r] : __ldcg(lamg + it.r), acc);
          hp[warp] = acc;
        }
      }
      hstamp(20);  // dot products (waits for the preloaded slice)
      const Item cur = it;
      it = item_of(t + 1);  // next step's slice: loads in flight during the reduction and the wait
      preload(it);
      l2_prefetch(t + 1);
      {
        // the slice of step t+2 into L2 now, so next step's register preload hits L2
        // (the HBM stream of all helpers is ~14 MB per step at cfg3)
        const Item it2 = item_of(t + 2);
        if (it2.has) {
          const double* wr2 = s.W + it2.r * s.ldw;
          for (int64_t j = it2.c0 + 16 * lane; j < it2.c1; j += 16 * 32)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(wr2 + j));
        }
      }
      __syncthreads();
      hstamp(18);  // next preload issue + prefetches + barrier
      // one sum per (row, CTA): segmented reduction over the CTA's warps in
      // warp order (fixed tree: deterministic), first warp of a row stores it
      if (warp == 0) {
        const unsigned hw0 = (blockIdx.x - 1) * kHelpWarps, hwl = hw0 + lane;
        const unsigned nitems = (unsigned)(cur.rows2 * nch);
        const bool valid = lane < kHelpWarps && hwl < nitems;
        const int ir = valid ? (int)(hwl / nch) : -1 - lane;
        double v = valid ? hp[lane] : 0.0;
#pragma unroll
        for (int off = 1; off < kHelpWarps; off <<= 1) {
          const double u = __shfl_down_sync(0xffffffffu, v, off);
          const int iu = __shfl_down_sync(0xffffffffu, ir, off);
          if (lane + off < kHelpWarps && iu == ir) v += u;
        }
        if (valid && (lane == 0 || (hwl - 1) / nch != (unsigned)ir)) {
          const int seg = (int)(blockIdx.x - 1) - (int)(((unsigned)ir * nch) / kHelpWarps);
          ll_store(partial + 2 * ((size_t)(t % kPartBufs) * pstride + (size_t)ir * kSeg + seg), v, tag0 + t);
        }
      }
      hstamp(19);  // row sums
    }
  }
  // ---- everyone: wait for the final lambda, then delta_end = delta_base + h^2 W_reg lam
  cp_async_wait_all();
  if (tid == 0) wait_acq(pstop, 1u, nullptr, ctl);
  __syncthreads();
  const unsigned gw = blockIdx.x * (kPipeThreads / 32) + warp, ngw = gridDim.x * (kPipeThreads / 32);
  for (int64_t r = gw; s.delta_end && r < c; r += ngw) {
    const double* wr = s.W + r * s.ldw;
    double acc = lane_dot<true>(wr, lamg, 0, c, lane);
    acc = warp_sum(acc);
    if (lane == 0) {
      acc = fma(dshift[r / 3], __ldcg(lamg + r), acc);
      s.delta_end[r] = add(s.delta_base[r], mul(h2, acc));
    }
  }
  if (blockIdx.x == 0 && tid == 0 && ctl->timeout) raise_status(s.status, CNB_E_INTERNAL, 0, 0.0);
}

// ============================================================================
// Batched PGS, one CTA per independent scene (cfg4 copies)
// ============================================================================
// The iterate of pgs_cta with the pipelined kernel's per-group chain
// (block_solve_v4 + block_commit) and warp specialisation inside the CTA,
// blocks of kCG = 16 groups:
//   warp 0     : sequential solve of block b from its diagonal tile T(b);
//   warps 1..7 : meanwhile, cp.async of T(b+1) and Wx = W[b+1, b] into shared
//                memory, and the lazy row products P = W[b+1, not b] lambda
//                (+ the regularisation shift) from global memory / L2, all rows
//                of a warp interleaved so their loads are in flight together;
//   all        : delta(b+1) = delta_base + h^2 (P + Wx lambda_b) from shared
//                memory (4 threads per row); two barriers per block.
// eps = ||dlambda|| / ||lambda|| is accumulated by the solver lanes (every
// group is visited once per sweep), so a sweep ends without an extra pass.
constexpr int kCG = 16, kCR = 3 * kCG, kCS = kCR + 2;  // tile stride 50: at most 2-way bank conflicts
constexpr int kCopyThreads = 256;
constexpr int kCHelp = kCopyThreads / 32 - 2;       // helper warps: all but the solver and warp 4
constexpr int kCRW = (kCR + kCHelp - 1) / kCHelp;   // rows per helper warp
constexpr int kCU = 2;                              // column chunks per load batch

__host__ __device__ inline size_t copy_smem_bytes(int64_t G) {
  return sizeof(double) * (size_t)(3 * kCR * kCS + 4 * kCG + 8 + 3 * kCR + 3 * G + kKCP * G + G + 1) + 16;
}

// rows [r0, r0+nr) x cols [c0, c0+nc) of W -> dst (row stride kCS), 16-byte
// copies (W rows 16-byte aligned, c0 even; an odd nc copies one padding column
// that nothing reads), zero-filled outside; threads k of nt participate
__device__ __forceinline__ void copy_stage(double* dst, const double* W, int64_t ld, int64_t r0, int nr, int64_t c0,
                                           int nc, int k, int nt) {
  constexpr int kH = kCR / 2;
  for (int e = k; e < kCR * kH; e += nt) {
    const int i = e / kH, j = 2 * (e - i * kH);
    const bool v = i < nr && j < nc;
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + i * kCS + j);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(v ? W + (r0 + i) * ld + c0 + j : W),
                 "r"(v ? 16 : 0)
                 : "memory");
  }
}

// the next block's diagonal tile T and Wx = W[rows, cols of block b] by TMA bulk
// copies, one row per thread (k < 2 rows), completion on bar; an odd column
// count copies one padding column more (rows are 16-byte aligned, ld even)
__device__ __forceinline__ void copy_stage_bulk(double* T, double* X, const double* W, int64_t ld, int64_t rn0,
                                                int rows, int64_t cb0, int xcols, int k, unsigned long long* bar) {
  const unsigned bt = (unsigned)((rows + 1) & ~1) * 8u, bx = (unsigned)((xcols + 1) & ~1) * 8u;
  if (k == 0) mbar_arrive_expect_tx(bar, (unsigned)rows * (bt + bx));
  if (k < 2 * rows) {
    fence_proxy_async_smem();  // earlier generic reads / writes of the buffers before the async writes
    if (k < rows)
      bulk_g2s(T + k * kCS, W + (rn0 + k) * ld + rn0, bt, bar);
    else
      bulk_g2s(X + (k - rows) * kCS, W + (rn0 + k - rows) * ld + cb0, bx, bar);
  }
}

static_assert(kCRW == 8, "helper rows per warp must match warp_sum8");

__global__ void __launch_bounds__(kCopyThreads, 2) pgs_copy_kernel(const PgsScene* scenes, unsigned long long* prof, int exper) {
  extern __shared__ __align__(16) double pcsm[];
  const PgsScene s = scenes[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t G = s.groups, c = 3 * G;
  if (G == 0) {
    if (tid == 0) {
      s.iters_conv[0] = 0;
      s.iters_conv[1] = 1;
    }
    return;
  }
  double* p = pcsm;
  double* T0 = p;
  p += kCR * kCS;
  double* T1 = p;
  p += kCR * kCS;
  double* Wx = p;
  p += kCR * kCS;
  double* sv = p;
  p += 4 * kCG;
  double* red = p;
  p += 8;
  double* dn = p;
  p += kCR;
  double* P = p;
  p += kCR;
  double* dbn = p;  // delta_base of the next block
  p += kCR;
  double* lam = p;
  p += 3 * G;
  double* rec = p;
  p += kKCP * G;
  double* dsh = p;
  p += G;
  unsigned long long* tbar = (unsigned long long*)p;  // 8-byte aligned (every block above is whole doubles)
  p += 1;
  int* flags = (int*)p;
  const int nb = (int)((G + kCG - 1) / kCG);
  const double h2 = s.h2, ih2 = 1.0 / h2, mu = s.mu;
  const double* __restrict__ W = s.W;
  const int64_t ld = s.ldw;

  // ---- regularize (solver.py:99-121) and the per-group constants ----
  double tr = 0.0;
  for (int64_t i = tid; i < c; i += blockDim.x) tr += W[i * ld + i];
  tr = warp_sum(tr);
  if (lane == 0) red[warp] = tr;
  if (tid == 0) {
    flags[0] = flags[1] = 0;
    mbar_init(tbar, 1);
  }
  __syncthreads();
  double shift = 0.0;
  for (int w = 0; w < kCopyThreads / 32; ++w) shift += red[w];
  shift = 1e-10 * shift / (double)c;
  if (shift <= 0.0) shift = 1e-30;
  for (int64_t g = tid; g < G; g += blockDim.x) {
    double a[3][3], Wd[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        Wd[3 * i + j] = W[(3 * g + i) * ld + 3 * g + j];
        a[i][j] = 0.5 * (W[(3 * g + i) * ld + 3 * g + j] + W[(3 * g + j) * ld + 3 * g + i]);
      }
    double e[3];
    sym3_eigs(a, e);
    const double mn = fmin(e[0], fmin(e[1], e[2]));
    const double scale = fmax(fmax(fabs(e[0]), fmax(fabs(e[1]), fabs(e[2]))), 1e-300);
    const double sh = (mn <= 1e-12 * scale) ? shift : 0.0;
    dsh[g] = sh;
    for (int i = 0; i < 3; ++i) Wd[4 * i] = add(Wd[4 * i], sh);
    GroupConst kc;
    group_const(Wd, h2, kc);
    double* o = rec + kKCP * g;  // record layout: load_group_const
    o[0] = kc.ihw;
    o[1] = kc.it00;
    o[2] = kc.it01;
    o[3] = kc.it10;
    o[4] = kc.it11;
    o[5] = kc.b0;
    o[6] = kc.b1;
    o[7] = (double)kc.bad;
    o[8] = kc.hwnn;
  }
  for (int64_t i = tid; i < c; i += blockDim.x) lam[i] = 0.0;
  {
    const int r0n = 3 * (int)min((int64_t)kCG, G);
    copy_stage(T0, W, ld, 0, r0n, 0, r0n, tid, blockDim.x);
    for (int i = tid; i < r0n; i += blockDim.x) dn[i] = s.delta_base[i];
    cp_async_wait_all();
    __syncthreads();
    for (int i = tid; i < r0n; i += blockDim.x) T0[i * kCS + i] = add(T0[i * kCS + i], dsh[i / 3]);
    __syncthreads();
  }

  double dl[3] = {0, 0, 0}, lm[3] = {0, 0, 0}, dsq = 0.0, nl = 0.0;
  GroupConst kc;
  double* Tc = T0;
  double* Tn = T1;
  int iterations = 0;
  bool converged = false;
  // CNB_PGS_PROFILE=1: cycle sums of CTA 0 (solver solve / solver wait / helper
  // products / helper tile wait / delta phase / blocks)
  const bool stamp = prof && blockIdx.x == 0 && (tid == 0 || tid == 32);
  unsigned long long pf[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long t0 = 0, t1 = 0;
  unsigned tph = 0;  // phase of tbar (helper thread 0 only)
  for (int sweep = 0; sweep < s.max_iter; ++sweep) {
    iterations = sweep + 1;
    for (int b = 0; b < nb; ++b) {
      const int64_t g0 = (int64_t)b * kCG;
      const int ng = (int)min((int64_t)kCG, G - g0);
      const int bn = (b + 1 == nb) ? 0 : b + 1;
      const int64_t gn0 = (int64_t)bn * kCG;
      const int ngn = (int)min((int64_t)kCG, G - gn0);
      const int64_t cb0 = 3 * g0, cb1 = cb0 + 3 * ng, rn0 = 3 * gn0;
      const int rows = 3 * ngn;
      if (stamp) t0 = clock64();
      if (warp == 0) {
        // ---- sequential block solve ----
        const bool mine = lane < ng;
        load_group_const(kc, rec + kKCP * (g0 + (mine ? lane : 0)), mine, kKCP);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          lm[a] = mine ? lam[3 * (g0 + lane) + a] : 0.0;
          dl[a] = mine ? dn[3 * lane + a] : 0.0;
        }
        if (mu != 0.0)
          block_solve_v4<true>(Tc, kCS, ng, lane, dl, lm, kc, mu, h2, sv);
        else
          block_solve_v4<false>(Tc, kCS, ng, lane, dl, lm, kc, mu, h2, sv);
        __syncwarp();
        int err = 0;
        if (mine) {
          err = block_commit(sv, lane, lm, kc, mu, ih2, dsq);
#pragma unroll
          for (int a = 0; a < 3; ++a) lam[3 * (g0 + lane) + a] = lm[a];
          nl = fma(lm[0], lm[0], fma(lm[1], lm[1], fma(lm[2], lm[2], nl)));
        }
        const unsigned bad = __ballot_sync(0xffffffffu, err);
        if (bad) {
          const int g = __ffs(bad) - 1;  // first failing group in Gauss-Seidel order
          if (lane == g) raise_status(s.status, CNB_E_SINGULAR_BLOCK, (int)(g0 + g), 1.0 / kc.ihw);
          if (lane == 0) flags[0] = CNB_E_SINGULAR_BLOCK;
        }
        if (stamp) {
          t1 = clock64();
          pf[0] += t1 - t0;
        }
        if (b + 1 == nb) {
          // ---- end of sweep: epsilon (solver.py:194-199) ----
          const double num2 = warp_sum(dsq), den2 = warp_sum(nl);
          dsq = nl = 0.0;
          if (lane == 0) {
            const double num = sqrt(num2), den = sqrt(den2);
            const double eps = (num == 0.0) ? 0.0 : (den == 0.0 ? INFINITY : num / den);
            s.eps_hist[sweep] = eps;
            flags[1] = (eps <= s.tol) ? 1 : 0;
          }
        }
      } else if (nb > 1 && warp != 4) {
        // ---- helpers: next block's tiles, lazy products over every column but block b ----
        // (warp 4 shares the solver's SM sub-partition and stays idle)
        const int hw = warp < 4 ? warp - 1 : warp - 2;
        const int k = 32 * hw + lane, nt = 32 * kCHelp;
        if (!(exper & 2)) copy_stage_bulk(Tn, Wx, W, ld, rn0, rows, cb0, 3 * ng, k, tbar);
        if (!(exper & 4)) {
          // L2 prefetch of the row panel the helpers read in the next step
          const int bn2 = (bn + 1 == nb) ? 0 : bn + 1;
          const int64_t r2 = 3 * (int64_t)bn2 * kCG;
          const int rows2 = 3 * (int)min((int64_t)kCG, G - (int64_t)bn2 * kCG);
          const int i = k - 2 * kCR;  // threads past the bulk-copy issuers
          if (i >= 0 && i < rows2)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(W + (r2 + i) * ld),
                         "r"((unsigned)(((c + 1) & ~1LL) * 8)));
        }
        for (int i = k; i < rows; i += nt) cp_async8(dbn + i, s.delta_base + rn0 + i, true);
        if (stamp) pf[6] += clock64() - t0;
        double acc[kCRW];
#pragma unroll
        for (int r = 0; r < kCRW; ++r) acc[r] = 0.0;
        // unconditional loads (rows clamped, excluded / padding columns masked through
        // lambda = 0) so a batch of kCU x kCRW loads is in flight together
        const double* rp[kCRW];
#pragma unroll
        for (int r = 0; r < kCRW; ++r) rp[r] = W + (rn0 + min(hw + kCHelp * r, rows - 1)) * ld;
        const int64_t cend = (exper & 1) ? 0 : c;  // diagnostic: skip the products
        for (int64_t j0 = 0; j0 < cend; j0 += 32 * kCU) {
          double w[kCU][kCRW], lj[kCU];
#pragma unroll
          for (int u = 0; u < kCU; ++u) {
            const int64_t j = j0 + 32 * u + lane;
            const int64_t jj = min(j, c - 1);
            lj[u] = (j < c && (j < cb0 || j >= cb1)) ? lam[jj] : 0.0;
#pragma unroll
            for (int r = 0; r < kCRW; ++r) w[u][r] = __ldg(rp[r] + jj);
          }
#pragma unroll
          for (int u = 0; u < kCU; ++u)
#pragma unroll
            for (int r = 0; r < kCRW; ++r) acc[r] = fma(w[u][r], lj[u], acc[r]);
        }
        if (stamp) pf[7] += clock64() - t0;
        {
          const double v = warp_sum8(acc, lane);
          const int i = hw + kCHelp * (4 * ((lane >> 4) & 1) + 2 * ((lane >> 3) & 1) + ((lane >> 2) & 1));
          if ((lane & 3) == 0 && i < rows) P[i] = fma(dsh[(rn0 + i) / 3], lam[rn0 + i], v);
        }
        if (stamp) {
          t1 = clock64();
          pf[2] += t1 - t0;
        }
        cp_async_wait_all();
        if (k == 0 && !(exper & 2)) {
          mbar_wait(tbar, tph);
          tph ^= 1u;
        }
        if (stamp) pf[3] += clock64() - t1;
      }
      __syncthreads();
      if (stamp) {
        const long long t2 = clock64();
        if (tid == 0) pf[1] += t2 - t1;
        t1 = t2;
      }
      if (flags[0]) break;
      if (b + 1 == nb && flags[1]) {
        converged = true;
        break;
      }
      // ---- delta of the next block (4 threads per row) ----
      {
        const double* X = nb > 1 ? Wx : Tc;  // one block: its own regularised tile, all columns
        const int ncol = 3 * ng;
        const int i = tid >> 2, q = tid & 3;
        double acc = 0.0;
        if (i < rows)
          for (int j = q; j < ncol; j += 4) acc = fma(X[i * kCS + j], lam[cb0 + j], acc);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        if (q == 0 && i < rows) dn[i] = add(nb > 1 ? dbn[i] : s.delta_base[rn0 + i], mul(h2, (nb > 1 ? P[i] : 0.0) + acc));
        if (nb > 1)
          for (int r = tid; r < rows; r += blockDim.x) Tn[r * kCS + r] = add(Tn[r * kCS + r], dsh[(rn0 + r) / 3]);
      }
      __syncthreads();
      if (stamp && tid == 0) {
        pf[4] += clock64() - t1;
        pf[5] += 1;
      }
      if (nb > 1) {
        double* t = Tc;
        Tc = Tn;
        Tn = t;
      }
    }
    if (flags[0] || converged) break;
  }
  __syncthreads();
  // ---- delta_end = delta_base + h^2 W_reg lam (solver.py:201); skipped when not wanted ----
  for (int64_t r = warp; s.delta_end && r < c; r += kCopyThreads / 32) {
    double acc = lane_dot<false>(W + r * ld, lam, 0, c, lane);
    acc = warp_sum(acc);
    if (lane == 0) {
      acc = fma(dsh[r / 3], lam[r], acc);
      s.delta_end[r] = add(s.delta_base[r], mul(h2, acc));
    }
  }
  for (int64_t i = tid; i < c; i += blockDim.x) s.lam[i] = lam[i];
  if (tid == 0) {
    s.iters_conv[0] = iterations;
    s.iters_conv[1] = converged ? 1 : 0;
  }
  if (stamp)
    for (int k = 0; k < 8; ++k)
      if (pf[k]) atomicAdd(prof + 8 + k, pf[k]);
}

static unsigned long long* pgs_profile_buffer() {
  static unsigned long long* buf = nullptr;
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("CNB_PGS_PROFILE");
    on = (e && e[0] == '1') ? 1 : 0;
    if (on && cudaMalloc(&buf, 32 * sizeof(unsigned long long)) == cudaSuccess)
      cudaMemset(buf, 0, 32 * sizeof(unsigned long long));
    else
      buf = nullptr;
  }
  return buf;
}

// Grid-scale PGS: the pipelined lookahead-2 kernel (pgs_pipe_kernel), one CTA
// per SM.  Its tiles move by tensor TMA and 16-byte row pairs, so W must have a
// 16-byte aligned base and an even row pitch; other layouts are first copied
// into an aligned scratch matrix (the Python layer always allocates aligned W).
static int launch_pgs_grid(PgsScene s, cudaStream_t st) {
  int dev = 0, sms = 0;
  CNB_CUDA(cudaGetDevice(&dev));
  CNB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if ((s.ldw & 1) || ((uintptr_t)s.W & 15)) {
    static GrowBuf aligned;
    const int64_t c = 3 * s.groups, ld = c + (c & 1);
    int rc = aligned.ensure((size_t)c * ld * sizeof(double));
    if (rc) return rc;
    CNB_CUDA(cudaMemcpy2DAsync(aligned.p, ld * sizeof(double), s.W, s.ldw * sizeof(double), c * sizeof(double), c,
                               cudaMemcpyDeviceToDevice, st));
    s.W = (const double*)aligned.p;
    s.ldw = ld;
  }
  int tma = 1;
  int dbg = 0;
  {
    const char* e = getenv("CNB_PGS_TMA");
    if (e && e[0] == '0') tma = 0;  // cp.async staging of the tiles instead of tensor TMA
    const char* d = getenv("CNB_PGS_DEBUG");
    if (d) dbg = atoi(d) & ~1;
  }
  const void* kfn = (const void*)pgs_pipe_kernel;
  const int nthreads = kPipeThreads;
  const size_t tiles = pipe_smem_bytes();
  const size_t lam_bytes = sizeof(double) * (size_t)(3 * s.groups) + 128;  // + alignment slack
  const int lam_in_smem = lam_bytes <= pgs_max_smem() ? 1 : 0;
  const size_t smem = std::max(tiles, lam_in_smem ? lam_bytes : (size_t)0);
  if (smem > pgs_max_smem()) {
    set_error("pgs: grid kernel needs %zu bytes of shared memory", smem);
    return CNB_E_INTERNAL;
  }
  CNB_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  CNB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, nthreads, smem));
  if (per_sm < 1) {
    set_error("pgs: grid kernel does not fit on an SM");
    return CNB_E_INTERNAL;
  }
  const int grid = sms;  // one CTA per SM: all co-resident (cooperative launch)
  const int nwarps = nthreads / 32;
  // one (row, column-slice) item per helper warp; the partials of a block are
  // staged in a kBR x kLDT tile by the solver
  // pipe: a row spans at most kSeg helper CTAs, so nch <= (kSeg - 1) * kHelpWarps
  const int nch = std::max(1, std::min(((grid - 1) * nwarps) / kPR, (kSeg - 1) * kHelpWarps));
  const size_t bytes =
      64 + sizeof(double) * ((size_t)s.groups * (1 + kKC) + 1 + kPartBufs * (size_t)kBR * std::max(nch, kSeg));
  static void* ws_p = nullptr;
  static size_t ws_cap = 0;
  if (bytes > ws_cap) {
    if (ws_p) cudaFree(ws_p);
    ws_p = nullptr;
    CNB_CUDA(cudaMalloc(&ws_p, bytes));
    ws_cap = bytes;
  }
  GridCtl* ctl = (GridCtl*)ws_p;
  double* dshift = (double*)((char*)ws_p + 64);
  double* kconst = dshift + s.groups;
  double* partial = kconst + kKC * s.groups + (((1 + kKC) * s.groups) & 1);  // 16-byte aligned (copy_cg)
  {
    // regularisation shifts + group constants, grid-wide (two passes)
    const int nparts = (int)((s.groups + kPrepThreads - 1) / kPrepThreads);
    static GrowBuf prep_part;
    int rc = prep_part.ensure((size_t)nparts * sizeof(double));
    if (rc) return rc;
    double* part = (double*)prep_part.p;
    pgs_prep1_kernel<<<nparts, kPrepThreads, 0, st>>>(s, dshift, part);
    CNB_LAUNCH_CHECK("pgs_prep1_kernel");
    pgs_prep2_kernel<<<nparts, kPrepThreads, 0, st>>>(s, dshift, kconst, part, nparts, ctl);
    CNB_LAUNCH_CHECK("pgs_prep2_kernel");
  }
  PgsScene sc = s;
  int lis = lam_in_smem;
  int nchv = nch;
  unsigned long long* prof = pgs_profile_buffer();
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  if (tma) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
      cudaDriverEntryPointQueryResult q;
      void* fn = nullptr;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }
    const cuuint64_t dims[2] = {(cuuint64_t)(3 * s.groups), (cuuint64_t)(3 * s.groups)};  // {columns, rows}
    const cuuint64_t pitch[1] = {(cuuint64_t)s.ldw * sizeof(double)};
    const cuuint32_t box[2] = {(cuuint32_t)kPR, (cuuint32_t)kPR};
    const cuuint32_t estr[2] = {1, 1};
    if (!encode || encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)s.W, dims, pitch, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      tma = 0;  // fall back to cp.async staging
  }
  int tma_arg = tma | dbg;
  // record tags: unique across launches (a record left by an earlier call never matches)
  static unsigned tag_base = 1;
  const unsigned long long steps = (unsigned long long)((s.groups + kPG - 1) / kPG) * (unsigned)s.max_iter + 8;
  if ((unsigned long long)tag_base + steps >= 0xffffffffull) tag_base = 1;  // wrap (records are rewritten each call)
  unsigned tag0 = tag_base;
  tag_base += (unsigned)steps;
  void* args_pipe[] = {(void*)&sc, (void*)&dshift, (void*)&kconst, (void*)&partial, (void*)&ctl,
                       (void*)&nchv, (void*)&lis, (void*)&tma_arg, (void*)&prof, (void*)&tag0, (void*)&tmap};
  CNB_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(grid), dim3(nthreads), args_pipe, smem, st));
  CNB_LAUNCH_CHECK("pgs_pipe_kernel");
  if (s.shift_out)
    CNB_CUDA(cudaMemcpyAsync(s.shift_out, dshift, s.groups * sizeof(double), cudaMemcpyDeviceToDevice, st));
  return CNB_OK;
}


// ============================================================================
// Graph-coloured PGS (north star option; NOT the reference's iterate)
// ============================================================================
// The groups are coloured on the host so that two groups sharing a DoF of any
// object (the sparsified coupling graph of S) never share a colour.  A sweep
// visits the colours in order; all groups of a colour are updated at once from
// the lambda at the start of the colour (Jacobi inside a colour, Gauss-Seidel
// across colours), one CTA per group: the CTA streams the group's three rows
// of W against lambda (HBM-bound, every SM busy), thread 0 runs local_solve
// (solver.py:124-165 branches) on the regularised diagonal block.  The iterate
// differs from the reference's exact order (W is dense: the coloured graph is
// a sparsification), so this is a measured option validated on the converged
// lambda only.  Deterministic: fixed reduction trees, values committed after a
// grid barrier.
constexpr int kColThreads = 256;

__global__ void __launch_bounds__(kColThreads) pgs_colour_kernel(PgsScene s, const double* __restrict__ dshift,
                                                                 const double* __restrict__ kconst,
                                                                 const int64_t* __restrict__ cptr,
                                                                 const int64_t* __restrict__ cgrp, int ncol,
                                                                 double* __restrict__ stage, double* __restrict__ gsq,
                                                                 GridCtl* ctl, double omega) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[3][kColThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t G = s.groups, c = 3 * G;
  const double h2 = s.h2;
  double* lam = s.lam;
  int iterations = 0;
  bool converged = false;
  for (int sweep = 0; sweep < s.max_iter; ++sweep) {
    for (int k = 0; k < ncol; ++k) {
      for (int64_t q = cptr[k] + blockIdx.x; q < cptr[k + 1]; q += gridDim.x) {
        const int64_t g = cgrp[q];
        const double* w0 = s.W + 3 * g * s.ldw;
        const double* w1 = w0 + s.ldw;
        const double* w2 = w1 + s.ldw;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        // 16-byte column pairs: W rows and lambda are 16-byte aligned (even pitch)
        for (int64_t j = 2 * tid; j < c; j += 2 * kColThreads) {
          if (j + 1 < c) {
            const double2 l = __ldcg(reinterpret_cast<const double2*>(lam + j));
            const double2 x0 = __ldcs(reinterpret_cast<const double2*>(w0 + j));
            const double2 x1 = __ldcs(reinterpret_cast<const double2*>(w1 + j));
            const double2 x2 = __ldcs(reinterpret_cast<const double2*>(w2 + j));
            a0 = fma(x0.y, l.y, fma(x0.x, l.x, a0));
            a1 = fma(x1.y, l.y, fma(x1.x, l.x, a1));
            a2 = fma(x2.y, l.y, fma(x2.x, l.x, a2));
          } else {
            const double l = __ldcg(lam + j);
            a0 = fma(w0[j], l, a0);
            a1 = fma(w1[j], l, a1);
            a2 = fma(w2[j], l, a2);
          }
        }
        a0 = warp_sum(a0);
        a1 = warp_sum(a1);
        a2 = warp_sum(a2);
        if (lane == 0) {
          red[0][warp] = a0;
          red[1][warp] = a1;
          red[2][warp] = a2;
        }
        __syncthreads();
        if (tid == 0) {
          double l[3], d[3], nw[3];
          for (int a = 0; a < 3; ++a) {
            double acc = 0.0;
            for (int w = 0; w < kColThreads / 32; ++w) acc += red[a][w];
            l[a] = __ldcg(lam + 3 * g + a);
            acc = fma(dshift[g], l[a], acc);  // the regularisation shift of the block
            d[a] = add(s.delta_base[3 * g + a], mul(h2, acc));
          }
          GroupConst kc;
          load_group_const(kc, kconst + kKC * g, true);
          if (local_solve_sel(d, l, kc, s.mu, nw)) raise_status(s.status, CNB_E_SINGULAR_BLOCK, (int)g, kc.hwnn);
          if (omega != 1.0)  // under-relaxation: a convex combination stays in the friction cone
            for (int a = 0; a < 3; ++a) nw[a] = fma(omega, nw[a] - l[a], l[a]);
          const double q0 = nw[0] - l[0], q1 = nw[1] - l[1], q2 = nw[2] - l[2];
          for (int a = 0; a < 3; ++a) stage[3 * g + a] = nw[a];
          gsq[2 * g] = q0 * q0 + q1 * q1 + q2 * q2;
          gsq[2 * g + 1] = (nw[0] * nw[0] + nw[1] * nw[1]) + nw[2] * nw[2];
        }
        __syncthreads();
      }
      grid.sync();
      // commit the colour's lambda (every CTA of the colour read the old values)
      const int64_t n = cptr[k + 1] - cptr[k];
      for (int64_t e = (int64_t)blockIdx.x * kColThreads + tid; e < 3 * n; e += (int64_t)gridDim.x * kColThreads) {
        const int64_t g = cgrp[cptr[k] + e / 3];
        lam[3 * g + e % 3] = stage[3 * g + e % 3];
      }
      grid.sync();
    }
    // epsilon = |d lambda| / |lambda| (solver.py:194-199), one CTA, fixed order
    if (blockIdx.x == 0) {
      double sd = 0.0, sl = 0.0;
      for (int64_t g = tid; g < G; g += kColThreads) {
        sd += gsq[2 * g];
        sl += gsq[2 * g + 1];
      }
      sd = warp_sum(sd);
      sl = warp_sum(sl);
      if (lane == 0) {
        red[0][warp] = sd;
        red[1][warp] = sl;
      }
      __syncthreads();
      if (tid == 0) {
        double td = 0.0, tl = 0.0;
        for (int w = 0; w < kColThreads / 32; ++w) {
          td += red[0][w];
          tl += red[1][w];
        }
        const double num = sqrt(td), den = sqrt(tl);
        const double eps = (num == 0.0) ? 0.0 : (den == 0.0 ? INFINITY : num / den);
        s.eps_hist[sweep] = eps;
        ctl->stop = (eps <= s.tol) ? 1u : ((sweep + 1 >= s.max_iter) ? 2u : 0u);
      }
    }
    grid.sync();
    const unsigned st = *(volatile unsigned*)&ctl->stop;
    if (st) {
      iterations = sweep + 1;
      converged = st == 1u;
      break;
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    s.iters_conv[0] = iterations;
    s.iters_conv[1] = converged ? 1 : 0;
  }
  // delta_end = delta_base + h^2 W_reg lam (solver.py:201)
  const unsigned gw = blockIdx.x * (kColThreads / 32) + warp, ngw = gridDim.x * (kColThreads / 32);
  for (int64_t r = gw; s.delta_end && r < c; r += ngw) {
    double acc = lane_dot<true>(s.W + r * s.ldw, lam, 0, c, lane);
    acc = warp_sum(acc);
    if (lane == 0) {
      acc = fma(dshift[r / 3], __ldcg(lam + r), acc);
      s.delta_end[r] = add(s.delta_base[r], mul(h2, acc));
    }
  }
}

static int launch_pgs_coloured(PgsScene s, const int64_t* colour_ptr, const int64_t* colour_groups, int ncol,
                               double omega, cudaStream_t st) {
  if ((s.ldw & 1) || ((uintptr_t)s.W & 15) || ((uintptr_t)s.lam & 15)) {
    set_error("pgs_coloured: W and lambda need 16-byte aligned rows (even ldw)");
    return CNB_E_VALIDATION;
  }
  int dev = 0, sms = 0, per_sm = 0;
  CNB_CUDA(cudaGetDevice(&dev));
  CNB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CNB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pgs_colour_kernel, kColThreads, 0));
  if (per_sm < 1) {
    set_error("pgs_coloured: kernel does not fit on an SM");
    return CNB_E_INTERNAL;
  }
  const int64_t G = s.groups;
  static GrowBuf ws;
  const size_t nd = (size_t)G * (1 + kKC + 3 + 2) + (size_t)(ncol + 1) + (size_t)G;  // doubles / int64 slots
  int rc = ws.ensure(64 + 8 * nd);
  if (rc) return rc;
  GridCtl* ctl = (GridCtl*)ws.p;
  double* dshift = (double*)((char*)ws.p + 64);
  double* kconst = dshift + G;
  double* stage = kconst + kKC * G;
  double* gsq = stage + 3 * G;
  int64_t* d_cptr = (int64_t*)(gsq + 2 * G);
  int64_t* d_cgrp = d_cptr + ncol + 1;
  CNB_CUDA(cudaMemcpyAsync(d_cptr, colour_ptr, (ncol + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  CNB_CUDA(cudaMemcpyAsync(d_cgrp, colour_groups, G * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  const int nparts = (int)((G + kPrepThreads - 1) / kPrepThreads);
  static GrowBuf prep_part;
  if ((rc = prep_part.ensure((size_t)nparts * sizeof(double)))) return rc;
  pgs_prep1_kernel<<<nparts, kPrepThreads, 0, st>>>(s, dshift, (double*)prep_part.p);
  CNB_LAUNCH_CHECK("pgs_prep1_kernel");
  pgs_prep2_kernel<<<nparts, kPrepThreads, 0, st>>>(s, dshift, kconst, (double*)prep_part.p, nparts, ctl);
  CNB_LAUNCH_CHECK("pgs_prep2_kernel");
  PgsScene sc = s;
  void* args[] = {(void*)&sc, (void*)&dshift, (void*)&kconst, (void*)&d_cptr, (void*)&d_cgrp, (void*)&ncol,
                  (void*)&stage, (void*)&gsq, (void*)&ctl, (void*)&omega};
  CNB_CUDA(cudaLaunchCooperativeKernel((const void*)pgs_colour_kernel, dim3(sms * per_sm), dim3(kColThreads), args,
                                       0, st));
  CNB_LAUNCH_CHECK("pgs_colour_kernel");
  if (s.shift_out) CNB_CUDA(cudaMemcpyAsync(s.shift_out, dshift, G * sizeof(double), cudaMemcpyDeviceToDevice, st));
  return CNB_OK;
}

// CNB_PGS_GRID=1 forces the grid-scale kernel, =0 the single-CTA kernel
// whenever its shared-memory footprint fits; unset: by size.
static int pgs_grid_override() {
  const char* e = getenv("CNB_PGS_GRID");
  if (!e || !e[0]) return -1;
  return e[0] == '1' ? 1 : 0;
}

}  // namespace cnb

using namespace cnb;

extern "C" {

// Phase sums (ns) of the grid PGS kernel since the last call (CNB_PGS_PROFILE=1):
// out[0] solver wait, [1] delta, [2] solves, [3] epilogue, [4] helper wait,
// [5] helper partials, [6] helper hand-off, [7] the sequential group loop.
// Returns CNB_E_VALIDATION if off.
int cnb_pgs_profile(double* out) {
  unsigned long long* b = pgs_profile_buffer();
  if (!b) {
    set_error("pgs profile: set CNB_PGS_PROFILE=1");
    return CNB_E_VALIDATION;
  }
  unsigned long long h[32];
  CNB_CUDA(cudaMemcpy(h, b, sizeof(h), cudaMemcpyDeviceToHost));
  CNB_CUDA(cudaMemset(b, 0, sizeof(h)));
  for (int k = 0; k < 32; ++k) out[k] = (double)h[k];
  return CNB_OK;
}

int cnb_pgs(int64_t groups, const double* W, int64_t ldw, const double* delta_base, double h, double mu,
            double tol, int32_t max_iter, double* lam, double* delta_end, double* eps_hist,
            int32_t* iters_conv, double* shift_out, cnb_status_t* d_status, void* stream) {
  if (groups < 0 || max_iter < 1) {
    set_error("pgs: invalid arguments (groups=%lld, max_iter=%d)", (long long)groups, max_iter);
    return CNB_E_VALIDATION;
  }
  if (groups == 0) return CNB_OK;
  PgsScene s;
  s.groups = groups;
  s.W = W;
  s.ldw = ldw;
  s.delta_base = delta_base;
  s.h2 = h * h;
  s.mu = mu;
  s.tol = tol;
  s.max_iter = max_iter;
  s.lam = lam;
  s.delta_end = delta_end;
  s.eps_hist = eps_hist;
  s.iters_conv = iters_conv;
  s.status = (DevStatus*)d_status;
  s.shift_out = shift_out;
  const size_t smem = pgs_smem_bytes(groups);
  // large scenes: the grid-scale kernel (helpers on every SM); small ones stay
  // on one CTA with lambda in shared memory
  const int ov = pgs_grid_override();
  // the pipelined kernel needs at least four blocks of kPG groups
  const bool grid = groups >= 4 * kPG && (smem > pgs_max_smem() || (ov < 0 ? groups > 512 : ov == 1));
  if (grid) return launch_pgs_grid(s, (cudaStream_t)stream);
  CNB_CUDA(cudaFuncSetAttribute(pgs_single_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  pgs_single_kernel<<<1, kPgsThreads, smem, (cudaStream_t)stream>>>(s);
  CNB_LAUNCH_CHECK("pgs_single_kernel");
  return CNB_OK;
}

// Independent scenes (BASELINE configs[4]): one CTA per scene runs pgs_cta on
// its own W (packed at w_off[s], c_s x c_s), violation, lambda and outputs at
// the scene's group offset g_off[s].  Host arrays describe the scenes.
int cnb_pgs_batched(int32_t nscenes, const int64_t* g_off, const int64_t* w_off, const double* mu, const double* W,
                    const double* delta_base, double h, double tol, int32_t max_iter, double* lam, double* delta_end,
                    double* eps_hist, int32_t* iters_conv, const int32_t* order, cnb_status_t* d_status,
                    void* stream) {
  if (nscenes <= 0) return CNB_OK;
  if (max_iter < 1) {
    set_error("pgs_batched: max_iter must be positive");
    return CNB_E_VALIDATION;
  }
  static PgsScene* d_sc = nullptr;
  static size_t cap = 0;
  static PinnedBuf pin;
  const size_t bytes = sizeof(PgsScene) * (size_t)nscenes;
  if (bytes > cap) {
    if (d_sc) cudaFree(d_sc);
    d_sc = nullptr;
    CNB_CUDA(cudaMalloc(&d_sc, bytes));
    cap = bytes;
  }
  int rc = pin.ensure(bytes);
  if (rc) return rc;
  PgsScene* hs = (PgsScene*)pin.p;
  int64_t gmax = 0;
  for (int k = 0; k < nscenes; ++k) {
    // launch order: CTA k solves scene order[k] (heaviest expected first, so the
    // longest solves do not start in the last wave); identity without order
    const int i = order ? order[k] : k;
    if (i < 0 || i >= nscenes) {
      set_error("pgs_batched: order[%d] = %d out of range", k, i);
      return CNB_E_VALIDATION;
    }
    const int64_t G = g_off[i + 1] - g_off[i];
    gmax = std::max(gmax, G);
    PgsScene& sc = hs[k];
    sc.groups = G;
    sc.W = W + w_off[i];
    sc.ldw = 3 * G + (G & 1);  // even row stride (16-byte aligned rows)
    sc.delta_base = delta_base + 3 * g_off[i];
    sc.h2 = h * h;
    sc.mu = mu[i];
    sc.tol = tol;
    sc.max_iter = max_iter;
    sc.lam = lam + 3 * g_off[i];
    sc.delta_end = delta_end ? delta_end + 3 * g_off[i] : nullptr;
    sc.eps_hist = eps_hist + (int64_t)i * max_iter;
    sc.iters_conv = iters_conv + 2 * i;
    sc.status = (DevStatus*)d_status;
    sc.shift_out = nullptr;
  }
  // per-copy pipelined kernel unless CNB_PGS_BATCHED=cta asks for the plain single-CTA iterate
  static const bool plain = [] {
    const char* e = getenv("CNB_PGS_BATCHED");
    return e && !strcmp(e, "cta");
  }();
  const size_t smem = plain ? pgs_smem_bytes(std::max<int64_t>(gmax, 1)) : copy_smem_bytes(std::max<int64_t>(gmax, 1));
  if (smem > pgs_max_smem()) {
    set_error("pgs_batched: %lld groups in one scene exceed the single-CTA kernel", (long long)gmax);
    return CNB_E_VALIDATION;
  }
  cudaStream_t st = (cudaStream_t)stream;
  CNB_CUDA(cudaMemcpyAsync(d_sc, hs, bytes, cudaMemcpyHostToDevice, st));
  if ((rc = pin.mark(st))) return rc;
  if (plain) {
    CNB_CUDA(cudaFuncSetAttribute(pgs_batched_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    pgs_batched_kernel<<<nscenes, kPgsThreads, smem, st>>>(d_sc);
    CNB_LAUNCH_CHECK("pgs_batched_kernel");
  } else {
    CNB_CUDA(cudaFuncSetAttribute(pgs_copy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const char* ee = getenv("CNB_PGS_COPY_EXP");  // diagnostic switches (results invalid when set)
    const int exper = ee ? atoi(ee) : 0;
    pgs_copy_kernel<<<nscenes, kCopyThreads, smem, st>>>(d_sc, pgs_profile_buffer(), exper);
    CNB_LAUNCH_CHECK("pgs_copy_kernel");
  }
  return CNB_OK;
}

int cnb_pgs_coloured(int64_t groups, const double* W, int64_t ldw, const double* delta_base, double h, double mu,
                     double tol, int32_t max_iter, const int64_t* colour_ptr, const int64_t* colour_groups,
                     int32_t ncolours, double omega, double* lam, double* delta_end, double* eps_hist,
                     int32_t* iters_conv, double* shift_out, cnb_status_t* d_status, void* stream) {
  if (groups < 0 || max_iter < 1 || ncolours < 0 || (groups > 0 && ncolours < 1) || !(omega > 0.0 && omega <= 1.0)) {
    set_error("pgs_coloured: invalid arguments (groups=%lld, max_iter=%d, colours=%d)", (long long)groups, max_iter,
              ncolours);
    return CNB_E_VALIDATION;
  }
  if (groups == 0) return CNB_OK;
  if (colour_ptr[0] != 0 || colour_ptr[ncolours] != groups) {
    set_error("pgs_coloured: the colour classes must partition the %lld groups", (long long)groups);
    return CNB_E_VALIDATION;
  }
  PgsScene s;
  s.groups = groups;
  s.W = W;
  s.ldw = ldw;
  s.delta_base = delta_base;
  s.h2 = h * h;
  s.mu = mu;
  s.tol = tol;
  s.max_iter = max_iter;
  s.lam = lam;
  s.delta_end = delta_end;
  s.eps_hist = eps_hist;
  s.iters_conv = iters_conv;
  s.status = (DevStatus*)d_status;
  s.shift_out = shift_out;
  return launch_pgs_coloured(s, colour_ptr, colour_groups, ncolours, omega, (cudaStream_t)stream);
}

int cnb_local_solve(int64_t alpha, int64_t groups, const double* W, int64_t ldw, const double* delta_cur,
                    const double* lam, double mu, double h2, double* out, cnb_status_t* d_status,
                    void* stream) {
  if (alpha < 0 || alpha >= groups) {
    set_error("local_solve: group %lld out of range", (long long)alpha);
    return CNB_E_DIMENSION;
  }
  local_solve_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(alpha, W, ldw, delta_cur, lam, mu, h2, out,
                                                         (DevStatus*)d_status);
  CNB_LAUNCH_CHECK("local_solve_kernel");
  return CNB_OK;
}

}  // extern "C"
