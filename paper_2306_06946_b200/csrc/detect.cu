// Narrow-phase proximity detection: every surface vertex of mesh A against
// every triangle of mesh B (reference: _vertex_vs_mesh, collision.py:222-260,
// closest_points_on_triangles 138-184, triangle_normals 187-190).
//
// The per-vertex decision (closest triangle = LOWEST index whose distance is
// within _TIE_EPS of the minimum, then the signed distance gates the pair) is
// integer output that must match the reference bit for bit, so every
// quantity is computed in numpy's own operation order without FMA
// contraction:
//   einsum("ij,ij->i", x, y)      = (x0*y0 + x2*y2) + x1*y1
//   np.linalg.norm(x, axis=1)     = sqrt((x0*x0 + x1*x1) + x2*x2)
//   np.cross                      = a1*b2 - a2*b1, ...
//
// Layout / passes (thread per query vertex, triangles staged through shared
// memory in chunks, the triangle range split into slices so the grid covers
// every SM):
//   tri_prep   : a, b, c, unit normal and AABB per triangle (SoA, 18 doubles)
//   min pass   : exact minimum distance; a triangle whose AABB lower bound
//                exceeds the running minimum by more than a margin
//                (1e-9 relative + 1e-10 x coordinate scale, six orders above
//                fp64 rounding of the closest-point arithmetic) cannot be the
//                minimum and is skipped.
//                Slices combine with atomicMin on the distance bit pattern
//                (non-negative doubles order like int64): exact, deterministic.
//   first pass : lowest triangle index with dist <= min + eps (same pruning
//                against min + eps); slices combine with atomicMin on the index.
//   finalize   : closest point, barycentric weights, signed distance of the
//                selected triangle and the threshold gate.
#include "common.cuh"

namespace cnb {

constexpr int kDetThreads = 128;
constexpr int kDetChunk = 128;  // triangles staged per shared-memory chunk
constexpr double kTieEps = 1e-9;  // collision.py:25

struct TriSoA {
  const double* d;  // 18 x nt: a(3) b(3) c(3) n(3) lo(3) hi(3)
  int64_t nt;
  __device__ __forceinline__ double at(int k, int64_t t) const { return d[(int64_t)k * nt + t]; }
};

__device__ __forceinline__ double dot_einsum(double x0, double x1, double x2, double y0, double y1, double y2) {
  return add(add(mul(x0, y0), mul(x2, y2)), mul(x1, y1));
}

__device__ __forceinline__ double norm3(double x0, double x1, double x2) {
  return __dsqrt_rn(add(add(mul(x0, x0), mul(x1, x1)), mul(x2, x2)));
}

// closest point of p on triangle (a, b, c); numpy order of
// closest_points_on_triangles.  Returns the barycentric (u, v, w) and point.
__device__ __forceinline__ void closest_on_tri(const double p[3], const double a[3], const double b[3],
                                               const double c[3], double cp[3], double& u, double& v, double& w) {
  double ab[3], ac[3], ap[3], bp[3], cpv[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    ab[k] = sub(b[k], a[k]);
    ac[k] = sub(c[k], a[k]);
    ap[k] = sub(p[k], a[k]);
    bp[k] = sub(p[k], b[k]);
    cpv[k] = sub(p[k], c[k]);
  }
  const double d1 = dot_einsum(ab[0], ab[1], ab[2], ap[0], ap[1], ap[2]);
  const double d2 = dot_einsum(ac[0], ac[1], ac[2], ap[0], ap[1], ap[2]);
  const double d3 = dot_einsum(ab[0], ab[1], ab[2], bp[0], bp[1], bp[2]);
  const double d4 = dot_einsum(ac[0], ac[1], ac[2], bp[0], bp[1], bp[2]);
  const double d5 = dot_einsum(ab[0], ab[1], ab[2], cpv[0], cpv[1], cpv[2]);
  const double d6 = dot_einsum(ac[0], ac[1], ac[2], cpv[0], cpv[1], cpv[2]);
  const double va = sub(mul(d3, d6), mul(d5, d4));
  const double vb = sub(mul(d5, d2), mul(d1, d6));
  const double vc = sub(mul(d1, d4), mul(d3, d2));
  if (d1 <= 0.0 && d2 <= 0.0) {  // vertex a
    v = 0.0;
    w = 0.0;
  } else if (d3 >= 0.0 && d4 <= d3) {  // vertex b
    v = 1.0;
    w = 0.0;
  } else if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {  // edge ab
    v = d1 != d3 ? __ddiv_rn(d1, sub(d1, d3)) : 0.0;
    w = 0.0;
  } else if (d6 >= 0.0 && d5 <= d6) {  // vertex c
    v = 0.0;
    w = 1.0;
  } else if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {  // edge ac
    v = 0.0;
    w = d2 != d6 ? __ddiv_rn(d2, sub(d2, d6)) : 0.0;
  } else if (va <= 0.0 && sub(d4, d3) >= 0.0 && sub(d5, d6) >= 0.0) {  // edge bc
    const double den_bc = add(sub(d4, d3), sub(d5, d6));
    const double w_bc = den_bc != 0.0 ? __ddiv_rn(sub(d4, d3), den_bc) : 0.0;
    v = sub(1.0, w_bc);
    w = w_bc;
  } else {  // interior
    const double den = add(add(va, vb), vc);
    v = den != 0.0 ? __ddiv_rn(vb, den) : 1.0 / 3.0;
    w = den != 0.0 ? __ddiv_rn(vc, den) : 1.0 / 3.0;
  }
  u = sub(sub(1.0, v), w);
#pragma unroll
  for (int k = 0; k < 3; ++k) cp[k] = add(add(a[k], mul(v, ab[k])), mul(w, ac[k]));
}

__global__ void tri_prep_kernel(int64_t nt, const int64_t* __restrict__ tris, const double* __restrict__ pts,
                                double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  double v[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int64_t node = tris[3 * t + r];
#pragma unroll
    for (int k = 0; k < 3; ++k) v[r][k] = pts[3 * node + k];
  }
  double e1[3], e2[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    e1[k] = sub(v[1][k], v[0][k]);
    e2[k] = sub(v[2][k], v[0][k]);
  }
  const double n0 = sub(mul(e1[1], e2[2]), mul(e1[2], e2[1]));
  const double n1 = sub(mul(e1[2], e2[0]), mul(e1[0], e2[2]));
  const double n2 = sub(mul(e1[0], e2[1]), mul(e1[1], e2[0]));
  const double ln = norm3(n0, n1, n2);
  const double nn[3] = {ln > 0.0 ? __ddiv_rn(n0, ln) : 0.0, ln > 0.0 ? __ddiv_rn(n1, ln) : 0.0,
                        ln > 0.0 ? __ddiv_rn(n2, ln) : 0.0};
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k) out[(int64_t)(3 * r + k) * nt + t] = v[r][k];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    out[(int64_t)(9 + k) * nt + t] = nn[k];
    out[(int64_t)(12 + k) * nt + t] = fmin(v[0][k], fmin(v[1][k], v[2][k]));
    out[(int64_t)(15 + k) * nt + t] = fmax(v[0][k], fmax(v[1][k], v[2][k]));
  }
}

// squared distance lower bound from p to the box [lo, hi]
__device__ __forceinline__ double box_lb2(const double p[3], const double lo[3], const double hi[3]) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double g = fmax(fmax(lo[k] - p[k], p[k] - hi[k]), 0.0);
    s = fma(g, g, s);
  }
  return s;
}

// pass 0: exact min distance (mode 0) or first index within min + eps (mode 1)
template <int MODE>
__global__ void __launch_bounds__(kDetThreads) vm_scan_kernel(int64_t nv, const int64_t* __restrict__ vids,
                                                              const double* __restrict__ pa, TriSoA T,
                                                              int64_t slice, unsigned long long* __restrict__ dmin,
                                                              unsigned long long* __restrict__ first) {
  __shared__ double s[15][kDetChunk];  // a b c lo hi
  const int64_t q = (int64_t)blockIdx.x * kDetThreads + threadIdx.x;
  const bool live = q < nv;
  double p[3] = {0.0, 0.0, 0.0};
  if (live) {
    const int64_t vid = vids[q];
#pragma unroll
    for (int k = 0; k < 3; ++k) p[k] = pa[3 * vid + k];
  }
  const int64_t t0 = (int64_t)blockIdx.y * slice;
  const int64_t t1 = min(T.nt, t0 + slice);
  // absolute slack of the pruning test, see the header
  const double scale = 1e-10 * (1.0 + fmax(fabs(p[0]), fmax(fabs(p[1]), fabs(p[2]))));
  auto limit2 = [&](double d) {
    const double l = d + 1e-9 * d + scale;
    return l * l;
  };
  double best, lim2;
  if (MODE == 0) {
    best = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    lim2 = best;
  } else {
    best = live ? add(__longlong_as_double((long long)dmin[q]), kTieEps) : 0.0;
    lim2 = limit2(best);
  }
  long long found = 0x7fffffffffffffffLL;
  bool done = !live;
  for (int64_t c0 = t0; c0 < t1; c0 += kDetChunk) {
    const int cn = (int)min((int64_t)kDetChunk, t1 - c0);
    if (__syncthreads_and(done)) break;  // every vertex of the block resolved
    for (int e = threadIdx.x; e < 15 * kDetChunk; e += kDetThreads) {
      const int k = e / kDetChunk, j = e % kDetChunk;
      const int kk = k < 9 ? k : k + 3;  // skip the normal rows
      s[k][j] = j < cn ? T.at(kk, c0 + j) : 0.0;
    }
    __syncthreads();
    if (done) continue;
    for (int j = 0; j < cn; ++j) {
      const double lo[3] = {s[9][j], s[10][j], s[11][j]};
      const double hi[3] = {s[12][j], s[13][j], s[14][j]};
      if (box_lb2(p, lo, hi) > lim2) continue;
      const double a[3] = {s[0][j], s[1][j], s[2][j]};
      const double b[3] = {s[3][j], s[4][j], s[5][j]};
      const double c[3] = {s[6][j], s[7][j], s[8][j]};
      double cp[3], u, v, w;
      closest_on_tri(p, a, b, c, cp, u, v, w);
      const double dist = norm3(sub(p[0], cp[0]), sub(p[1], cp[1]), sub(p[2], cp[2]));
      if (MODE == 0) {
        if (dist < best) {
          best = dist;
          lim2 = limit2(best);
        }
      } else if (dist <= best) {
        found = c0 + j;
        done = true;
        break;
      }
    }
  }
  if (!live) return;
  if (MODE == 0) {
    atomicMin(dmin + q, (unsigned long long)__double_as_longlong(best));
  } else if (found != 0x7fffffffffffffffLL) {
    atomicMin(first + q, (unsigned long long)found);
  }
}

// out row (12 doubles): signed, dist, u, v, w, cp(3), normal(3), hit(0/1)
__global__ void vm_finalize_kernel(int64_t nv, const int64_t* __restrict__ vids, const double* __restrict__ pa,
                                   TriSoA T, const unsigned long long* __restrict__ first, double threshold,
                                   int64_t* __restrict__ best_out, double* __restrict__ out) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nv) return;
  const int64_t vid = vids[q];
  const double p[3] = {pa[3 * vid], pa[3 * vid + 1], pa[3 * vid + 2]};
  const int64_t t = (int64_t)first[q];
  double* o = out + 12 * q;
  if (t < 0 || t >= T.nt) {  // no triangles (cannot happen for nt > 0)
    best_out[q] = -1;
    o[11] = 0.0;
    return;
  }
  const double a[3] = {T.at(0, t), T.at(1, t), T.at(2, t)};
  const double b[3] = {T.at(3, t), T.at(4, t), T.at(5, t)};
  const double c[3] = {T.at(6, t), T.at(7, t), T.at(8, t)};
  const double n[3] = {T.at(9, t), T.at(10, t), T.at(11, t)};
  double cp[3], u, v, w;
  closest_on_tri(p, a, b, c, cp, u, v, w);
  const double d0 = sub(p[0], cp[0]), d1 = sub(p[1], cp[1]), d2 = sub(p[2], cp[2]);
  const double dist = norm3(d0, d1, d2);
  const double side = dot_einsum(d0, d1, d2, n[0], n[1], n[2]);
  const double sgn = side >= 0.0 ? dist : -dist;
  best_out[q] = t;
  o[0] = sgn;
  o[1] = dist;
  o[2] = u;
  o[3] = v;
  o[4] = w;
  o[5] = cp[0];
  o[6] = cp[1];
  o[7] = cp[2];
  o[8] = n[0];
  o[9] = n[1];
  o[10] = n[2];
  o[11] = sgn > threshold ? 0.0 : 1.0;
}

__global__ void fill_u64_kernel(int64_t n, unsigned long long* p, unsigned long long v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

}  // namespace cnb

using namespace cnb;

extern "C" {

// Workspace for cnb_detect_vertex_mesh: 18 nt doubles + 2 nv words.
int64_t cnb_detect_work_bytes(int64_t nv, int64_t nt) {
  return (int64_t)sizeof(double) * (18 * std::max<int64_t>(nt, 1) + 2 * std::max<int64_t>(nv, 1));
}

int cnb_detect_vertex_mesh(int64_t nv, const int64_t* vids, const double* pts_a, int64_t nt, const int64_t* tris,
                           const double* pts_b, double threshold, void* work, int64_t* best, double* out,
                           void* stream) {
  if (nv <= 0) return CNB_OK;
  if (nt <= 0) {
    set_error("detect_vertex_mesh: mesh B has no triangles");
    return CNB_E_VALIDATION;
  }
  cudaStream_t st = (cudaStream_t)stream;
  double* tri = (double*)work;
  unsigned long long* dmin = (unsigned long long*)(tri + 18 * nt);
  unsigned long long* first = dmin + nv;
  tri_prep_kernel<<<grid_for(nt, 256), 256, 0, st>>>(nt, tris, pts_b, tri);
  CNB_LAUNCH_CHECK("tri_prep_kernel");
  fill_u64_kernel<<<grid_for(2 * nv, 256), 256, 0, st>>>(2 * nv, dmin, 0x7fffffffffffffffULL);
  CNB_LAUNCH_CHECK("fill_u64_kernel");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t vblocks = (nv + kDetThreads - 1) / kDetThreads;
  int64_t slices = std::max<int64_t>(1, std::min<int64_t>((4 * sms + vblocks - 1) / vblocks,
                                                          (nt + kDetChunk - 1) / kDetChunk));
  const int64_t slice = (((nt + slices - 1) / slices + kDetChunk - 1) / kDetChunk) * kDetChunk;
  slices = (nt + slice - 1) / slice;
  TriSoA T{tri, nt};
  dim3 grid((unsigned)vblocks, (unsigned)slices);
  vm_scan_kernel<0><<<grid, kDetThreads, 0, st>>>(nv, vids, pts_a, T, slice, dmin, first);
  CNB_LAUNCH_CHECK("vm_scan_kernel<0>");
  vm_scan_kernel<1><<<grid, kDetThreads, 0, st>>>(nv, vids, pts_a, T, slice, dmin, first);
  CNB_LAUNCH_CHECK("vm_scan_kernel<1>");
  vm_finalize_kernel<<<grid_for(nv, 128), 128, 0, st>>>(nv, vids, pts_a, T, first, threshold, best, out);
  CNB_LAUNCH_CHECK("vm_finalize_kernel");
  return CNB_OK;
}

}  // extern "C"
