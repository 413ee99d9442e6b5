// Tetrahedral FE assembly of the implicit-Euler system on the device.
//
// Reference: dynamics.py — assemble_stiffness 81-99 (constant-strain tet
// blocks V(lam g_a g_b^T + mu g_b g_a^T + mu (g_a.g_b) I)), internal_force
// 172-177, SoftBody.assemble 183-211:
//   A = (1 + h alpha) M + (h beta + h^2) K,  fixed rows/cols -> identity,
//   b = h (f_ext - f(q, v)) - h^2 K v,  b[fixed] = 0,
//   f(q, v) = f_el(q) + alpha M v + beta K v.
// The reference material is linear (K constant, f_el = K (q - q0)).  The
// corotational material (north star; not in the reference)
// uses per-tet rotations R_e from the polar decomposition of
// F = sum_a x_a g_a^T:  K(q) = sum_e R_e K_e R_e^T,
// f_el = sum_e R_e K_e (R_e^T x_e - x0_e); it reduces exactly to the linear
// material when every R_e = I.
//
// Two passes, no fp64 atomics (bitwise repeatable):
//   element_kernel: one thread per tet -> 16 rotated 3x3 blocks + 4 forces;
//   gather kernels: one thread per global 3x3 block / node sums its
//   contributions in ascending (tet, a, b) order.
#include "common.cuh"

namespace cnb {

// Rotation maximising tr(R^T F) over SO(3) for any F (Horn's quaternion
// form): tr(R(q)^T F) = q^T N q for a unit quaternion q, with N the symmetric
// 4x4 matrix below, so the maximiser is N's top eigenvector (cyclic Jacobi,
// fp64).  It equals the polar factor when det F > 0 and
// U diag(1, 1, -1) V^T (F = U S V^T) for inverted elements — the oracle's
// rotation_factor (oracle/cn_oracle.py).
__device__ void max_trace_rotation(const double F[9], double R[9]) {
  // S = F^T in Horn's notation (S_ab = sum over points of a_a b_b)
  const double Sxx = F[0], Sxy = F[3], Sxz = F[6];
  const double Syx = F[1], Syy = F[4], Syz = F[7];
  const double Szx = F[2], Szy = F[5], Szz = F[8];
  double A[4][4] = {{Sxx + Syy + Szz, Syz - Szy, Szx - Sxz, Sxy - Syx},
                    {Syz - Szy, Sxx - Syy - Szz, Sxy + Syx, Szx + Sxz},
                    {Szx - Sxz, Sxy + Syx, -Sxx + Syy - Szz, Syz + Szy},
                    {Sxy - Syx, Szx + Sxz, Syz + Szy, -Sxx - Syy + Szz}};
  double V[4][4] = {{1, 0, 0, 0}, {0, 1, 0, 0}, {0, 0, 1, 0}, {0, 0, 0, 1}};
  for (int sweep = 0; sweep < 50; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < 3; ++p)
      for (int q = p + 1; q < 4; ++q) off += fabs(A[p][q]);
    if (off == 0.0) break;
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int q = p + 1; q < 4; ++q) {
        const double apq = A[p][q];
        const double g = 100.0 * fabs(apq);
        if (sweep > 3 && fabs(A[p][p]) + g == fabs(A[p][p]) && fabs(A[q][q]) + g == fabs(A[q][q])) {
          A[p][q] = A[q][p] = 0.0;
          continue;
        }
        if (apq == 0.0) continue;
        const double theta = (A[q][q] - A[p][p]) / (2.0 * apq);
        double t;
        if (fabs(theta) > 1e150) {
          t = 0.5 / theta;
        } else {
          t = 1.0 / (fabs(theta) + sqrt(theta * theta + 1.0));
          if (theta < 0.0) t = -t;
        }
        const double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
        for (int k = 0; k < 4; ++k) {  // columns p, q
          const double akp = A[k][p], akq = A[k][q];
          A[k][p] = c * akp - sn * akq;
          A[k][q] = sn * akp + c * akq;
        }
        for (int k = 0; k < 4; ++k) {  // rows p, q
          const double apk = A[p][k], aqk = A[q][k];
          A[p][k] = c * apk - sn * aqk;
          A[q][k] = sn * apk + c * aqk;
        }
        for (int k = 0; k < 4; ++k) {
          const double vkp = V[k][p], vkq = V[k][q];
          V[k][p] = c * vkp - sn * vkq;
          V[k][q] = sn * vkp + c * vkq;
        }
      }
  }
  int best = 0;
  for (int k = 1; k < 4; ++k)
    if (A[k][k] > A[best][best]) best = k;
  double w = V[0][best], x = V[1][best], y = V[2][best], z = V[3][best];
  const double inv = 1.0 / sqrt(w * w + x * x + y * y + z * z);
  w *= inv;
  x *= inv;
  y *= inv;
  z *= inv;
  R[0] = w * w + x * x - y * y - z * z;
  R[1] = 2.0 * (x * y - w * z);
  R[2] = 2.0 * (x * z + w * y);
  R[3] = 2.0 * (x * y + w * z);
  R[4] = w * w - x * x + y * y - z * z;
  R[5] = 2.0 * (y * z - w * x);
  R[6] = 2.0 * (x * z - w * y);
  R[7] = 2.0 * (y * z + w * x);
  R[8] = w * w - x * x - y * y + z * z;
}

// Orthogonal polar factor by Newton iteration R <- (R + R^{-T}) / 2 from F
// (quadratic convergence, exact to rounding for det F > 0).  Inverted or
// degenerate elements (det F <= 1e-12) take the rotation maximising
// tr(R^T F) instead (max_trace_rotation).
__device__ void polar_rotation(const double F[9], double R[9]) {
  const double det = F[0] * (F[4] * F[8] - F[5] * F[7]) - F[1] * (F[3] * F[8] - F[5] * F[6]) +
                     F[2] * (F[3] * F[7] - F[4] * F[6]);
  if (det > 1e-12) {
    for (int e = 0; e < 9; ++e) R[e] = F[e];
    for (int it = 0; it < 30; ++it) {
      // inverse transpose = cofactor / det
      double C[9];
      C[0] = R[4] * R[8] - R[5] * R[7];
      C[1] = R[5] * R[6] - R[3] * R[8];
      C[2] = R[3] * R[7] - R[4] * R[6];
      C[3] = R[2] * R[7] - R[1] * R[8];
      C[4] = R[0] * R[8] - R[2] * R[6];
      C[5] = R[1] * R[6] - R[0] * R[7];
      C[6] = R[1] * R[5] - R[2] * R[4];
      C[7] = R[2] * R[3] - R[0] * R[5];
      C[8] = R[0] * R[4] - R[1] * R[3];
      const double d = R[0] * C[0] + R[1] * C[1] + R[2] * C[2];
      double diff = 0.0;
      for (int e = 0; e < 9; ++e) {
        const double nr = 0.5 * (R[e] + C[e] / d);
        diff = fmax(diff, fabs(nr - R[e]));
        R[e] = nr;
      }
      if (diff <= 1e-15) break;
    }
    return;
  }
  max_trace_rotation(F, R);
}

// One thread per tet.  grads: (tets, 4, 3) rest shape-function gradients;
// vol: rest volumes.  Outputs: Kb (tets, 4, 4, 3, 3) rotated blocks,
// fe (tets, 4, 3) element elastic forces, Rout (tets, 9) if non-null.
__global__ void __launch_bounds__(128) element_kernel(int64_t ntets, const int64_t* __restrict__ tets,
                                                      const double* __restrict__ grads, const double* __restrict__ vol,
                                                      const double* __restrict__ x, const double* __restrict__ x0,
                                                      double lam, double mu, int corot, double* __restrict__ Kb,
                                                      double* __restrict__ fe, double* __restrict__ Rout) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ntets) return;
  int64_t nd[4];
  double g[4][3], xe[4][3], x0e[4][3];
  for (int a = 0; a < 4; ++a) {
    nd[a] = tets[4 * e + a];
    for (int d = 0; d < 3; ++d) {
      g[a][d] = grads[12 * e + 3 * a + d];
      xe[a][d] = x[3 * nd[a] + d];
      x0e[a][d] = x0[3 * nd[a] + d];
    }
  }
  const double V = vol[e];
  double R[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  if (corot) {
    double F[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double s = 0.0;
        for (int a = 0; a < 4; ++a) s += xe[a][i] * g[a][j];
        F[3 * i + j] = s;
      }
    polar_rotation(F, R);
  }
  if (Rout)
    for (int k = 0; k < 9; ++k) Rout[9 * e + k] = R[k];
  // local displacement u_b = R^T x_b - x0_b (linear: x_b - x0_b)
  double u[4][3];
  for (int b = 0; b < 4; ++b)
    for (int d = 0; d < 3; ++d) {
      const double rx = corot ? (R[0 * 3 + d] * xe[b][0] + R[1 * 3 + d] * xe[b][1] + R[2 * 3 + d] * xe[b][2]) : xe[b][d];
      u[b][d] = rx - x0e[b][d];
    }
  for (int a = 0; a < 4; ++a) {
    double fl[3] = {0, 0, 0};
    for (int b = 0; b < 4; ++b) {
      // unrotated block K_ab = V (lam g_a g_b^T + mu g_b g_a^T + mu (g_a.g_b) I)
      const double dab = g[a][0] * g[b][0] + g[a][1] * g[b][1] + g[a][2] * g[b][2];
      double K[9];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
          K[3 * i + j] = V * (lam * g[a][i] * g[b][j] + mu * g[b][i] * g[a][j] + (i == j ? mu * dab : 0.0));
      for (int i = 0; i < 3; ++i) fl[i] += K[3 * i] * u[b][0] + K[3 * i + 1] * u[b][1] + K[3 * i + 2] * u[b][2];
      double* out = Kb + ((e * 4 + a) * 4 + b) * 9;
      if (corot) {
        double T[9];  // R K
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) T[3 * i + j] = R[3 * i] * K[j] + R[3 * i + 1] * K[3 + j] + R[3 * i + 2] * K[6 + j];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j)
            out[3 * i + j] = T[3 * i] * R[3 * j] + T[3 * i + 1] * R[3 * j + 1] + T[3 * i + 2] * R[3 * j + 2];
      } else {
        for (int k = 0; k < 9; ++k) out[k] = K[k];
      }
    }
    double* fo = fe + (e * 4 + a) * 3;
    if (corot) {
      for (int i = 0; i < 3; ++i) fo[i] = R[3 * i] * fl[0] + R[3 * i + 1] * fl[1] + R[3 * i + 2] * fl[2];
    } else {
      for (int i = 0; i < 3; ++i) fo[i] = fl[i];
    }
  }
}

// One thread per global 3x3 block: sum contributions (tet*16 + a*4 + b) in
// order into the DoF-level CSR values (dst = value index of the block's
// (row 3i, col 3j) entry; rows of the block are ld apart in CSR: given by
// rowstride[3] offsets).
__global__ void gather_blocks_kernel(int64_t nblocks, const int64_t* __restrict__ cptr,
                                     const int64_t* __restrict__ contrib, const double* __restrict__ Kb,
                                     const int64_t* __restrict__ dst, double* __restrict__ vals) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nblocks) return;
  double s[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t c = cptr[k]; c < cptr[k + 1]; ++c) {
    const double* b = Kb + contrib[c] * 9;
    for (int e = 0; e < 9; ++e) s[e] += b[e];
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) vals[dst[3 * k + i] + j] = s[3 * i + j];
}

// One thread per node: f_el[node] = sum of element forces (tet*4 + a) in order.
__global__ void gather_forces_kernel(int64_t nnodes, const int64_t* __restrict__ fptr, const int64_t* __restrict__ fidx,
                                     const double* __restrict__ fe, double* __restrict__ f) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnodes) return;
  double s[3] = {0, 0, 0};
  for (int64_t c = fptr[i]; c < fptr[i + 1]; ++c)
    for (int d = 0; d < 3; ++d) s[d] += fe[fidx[c] * 3 + d];
  for (int d = 0; d < 3; ++d) f[3 * i + d] = s[d];
}

// A = k_scale K + diag((1 + h alpha) m) with fixed rows/cols -> identity.
// A has its own CSR pattern (rp, ci): the reference keeps a K entry only when
// neither its row nor its column is fixed, plus one diagonal entry per DoF
// (dynamics.py:190-200).  src[e] = index of A entry e in K's value array (-1:
// a fixed DoF's diagonal); src == NULL means A shares K's pattern (no fixed
// DoFs).  fixed: per DoF, int8.
__global__ void system_matrix_kernel(int64_t n, const int64_t* __restrict__ rp, const int64_t* __restrict__ ci,
                                     const int64_t* __restrict__ src, const double* __restrict__ K,
                                     const double* __restrict__ m3, const int8_t* __restrict__ fixed,
                                     double k_scale, double m_scale, double* __restrict__ A) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const bool fr = fixed[r] != 0;
  for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
    const int64_t c = ci[e];
    double v;
    if (fr || fixed[c]) {
      v = (c == r) ? 1.0 : 0.0;
    } else {
      v = k_scale * K[src ? src[e] : e];
      if (c == r) v += m_scale * m3[r];
    }
    A[e] = v;
  }
}

// b = h (f_ext - f_el - alpha M v - beta Kv) - h^2 Kv, fixed -> 0; flags
// non-finite entries (NonFiniteForceError, dynamics.py:209-210).
__global__ void system_rhs_kernel(int64_t n, const double* __restrict__ fel, const double* __restrict__ Kv,
                                  const double* __restrict__ m3, const double* __restrict__ v,
                                  const double* __restrict__ fext, const int8_t* __restrict__ fixed, double h,
                                  double alpha, double beta, double* __restrict__ b, DevStatus* st) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const double f = fel[r] + alpha * (m3[r] * v[r]) + beta * Kv[r];
  double val = h * (fext[r] - f) - h * h * Kv[r];
  if (fixed[r]) val = 0.0;
  if (!isfinite(val)) raise_status(st, CNB_E_NONFINITE, (int)r, val);
  b[r] = val;
}

}  // namespace cnb

using namespace cnb;

extern "C" {

int cnb_fe_element(int64_t ntets, const int64_t* tets, const double* grads, const double* vol, const double* x,
                   const double* x0, double lam, double mu, int32_t corot, double* Kb, double* fe, double* R,
                   void* stream) {
  if (ntets <= 0) return CNB_OK;
  element_kernel<<<grid_for(ntets, 128), 128, 0, (cudaStream_t)stream>>>(ntets, tets, grads, vol, x, x0, lam, mu,
                                                                         corot, Kb, fe, R);
  CNB_LAUNCH_CHECK("element_kernel");
  return CNB_OK;
}

int cnb_fe_gather(int64_t nblocks, const int64_t* cptr, const int64_t* contrib, const double* Kb, const int64_t* dst,
                  double* vals, int64_t nnodes, const int64_t* fptr, const int64_t* fidx, const double* fe,
                  double* f, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (nblocks > 0 && vals) {
    gather_blocks_kernel<<<grid_for(nblocks, 128), 128, 0, st>>>(nblocks, cptr, contrib, Kb, dst, vals);
    CNB_LAUNCH_CHECK("gather_blocks_kernel");
  }
  if (nnodes > 0 && f) {
    gather_forces_kernel<<<grid_for(nnodes, 128), 128, 0, st>>>(nnodes, fptr, fidx, fe, f);
    CNB_LAUNCH_CHECK("gather_forces_kernel");
  }
  return CNB_OK;
}

int cnb_fe_system(int64_t n, const int64_t* rowptr, const int64_t* col, const int64_t* a_src, const double* Kvals,
                  const double* m3, const int8_t* fixed, double h, double alpha, double beta, const double* fel, const double* Kv,
                  const double* v, const double* fext, double* Avals, double* b, cnb_status_t* d_status,
                  void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n <= 0) return CNB_OK;
  if (Avals) {
    system_matrix_kernel<<<grid_for(n, 128), 128, 0, st>>>(n, rowptr, col, a_src, Kvals, m3, fixed, h * beta + h * h,
                                                           1.0 + h * alpha, Avals);
    CNB_LAUNCH_CHECK("system_matrix_kernel");
  }
  if (b) {
    system_rhs_kernel<<<grid_for(n, 128), 128, 0, st>>>(n, fel, Kv, m3, v, fext, fixed, h, alpha, beta, b,
                                                        (DevStatus*)d_status);
    CNB_LAUNCH_CHECK("system_rhs_kernel");
  }
  return CNB_OK;
}

}  // extern "C"
