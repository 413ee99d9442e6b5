// Proximity refresh p = g(q) and signed gaps on the device.
//
// Reference: attachment_point / refresh_proximity collision.py:497-520,
// _element_normal / signed_gaps collision.py:523-548, the pen_before /
// pen_after reductions scene.py:658-662,713-718.
//
// Pair table layout (PairTable in collision.py): kind/obj (m,2), node (m,2,3)
// int64, w/local/world (m,2,3) f64; side 0 = A, side 1 = B.  Position views:
// views[oid] = node coordinates (n_o*3) of a deformable object, or null;
// poses[oid] = row-major R (9) + t (3) of a kinematic / rigid object.
#include "common.cuh"

namespace cnb {

enum { K_VERTEX = 0, K_BARY = 1, K_RIGID = 2, K_LOCAL = 3, K_WORLD = 4 };

__device__ __forceinline__ void attach_point(int i, int s, const int8_t* kind, const int* obj,
                                             const int64_t* node, const double* w, const double* local,
                                             const double* world, const double* const* views,
                                             const double* poses, double p[3]) {
  const int k = kind[2 * i + s];
  const int o = obj[2 * i + s];
  const int64_t* nd = node + 6 * i + 3 * s;
  const int base = 6 * i + 3 * s;
  if (k == K_VERTEX) {
    const double* q = views[o] + 3 * nd[0];
    p[0] = q[0];
    p[1] = q[1];
    p[2] = q[2];
  } else if (k == K_BARY) {
    const double* x0 = views[o] + 3 * nd[0];
    const double* x1 = views[o] + 3 * nd[1];
    const double* x2 = views[o] + 3 * nd[2];
    const double w0 = w[base], w1 = w[base + 1], w2 = w[base + 2];
#pragma unroll
    for (int d = 0; d < 3; ++d) p[d] = add(add(mul(w0, x0[d]), mul(w1, x1[d])), mul(w2, x2[d]));
  } else if (k == K_RIGID || k == K_LOCAL) {
    const double* P = poses + 12 * o;
    const double* l = local + base;
#pragma unroll
    for (int d = 0; d < 3; ++d)
      p[d] = add(add(add(mul(l[0], P[3 * d]), mul(l[1], P[3 * d + 1])), mul(l[2], P[3 * d + 2])), P[9 + d]);
  } else {
    p[0] = world[base];
    p[1] = world[base + 1];
    p[2] = world[base + 2];
  }
}

__global__ void refresh_kernel(int64_t m, const int8_t* kind, const int* obj, const int64_t* node,
                               const double* w, const double* local, const double* world,
                               const double* const* views, const double* poses, double* pa, double* pb) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double p[3];
  attach_point((int)i, 0, kind, obj, node, w, local, world, views, poses, p);
  pa[3 * i] = p[0];
  pa[3 * i + 1] = p[1];
  pa[3 * i + 2] = p[2];
  attach_point((int)i, 1, kind, obj, node, w, local, world, views, poses, p);
  pb[3 * i] = p[0];
  pb[3 * i + 1] = p[1];
  pb[3 * i + 2] = p[2];
}

__global__ void gaps_kernel(int64_t m, const int8_t* kind, const int* obj, const int64_t* node,
                            const double* w, const double* local, const double* world,
                            const double* lnormal, const int8_t* has_ln, const double* ref,
                            const double* const* views, const double* poses, double* gaps,
                            unsigned long long* pen_bits) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double pen = 0.0;
  if (i < m) {
    double a[3], b[3];
    attach_point((int)i, 0, kind, obj, node, w, local, world, views, poses, a);
    attach_point((int)i, 1, kind, obj, node, w, local, world, views, poses, b);
    double n[3] = {ref[3 * i], ref[3 * i + 1], ref[3 * i + 2]};
    const int kb = kind[2 * i + 1];
    const int ob = obj[2 * i + 1];
    if (kb == K_BARY) {
      const int64_t* nd = node + 6 * i + 3;
      const double* x0 = views[ob] + 3 * nd[0];
      const double* x1 = views[ob] + 3 * nd[1];
      const double* x2 = views[ob] + 3 * nd[2];
      double e1[3], e2[3], c[3];
      for (int d = 0; d < 3; ++d) {
        e1[d] = sub(x1[d], x0[d]);
        e2[d] = sub(x2[d], x0[d]);
      }
      c[0] = sub(mul(e1[1], e2[2]), mul(e1[2], e2[1]));
      c[1] = sub(mul(e1[2], e2[0]), mul(e1[0], e2[2]));
      c[2] = sub(mul(e1[0], e2[1]), mul(e1[1], e2[0]));
      const double nn = sqrt(add(add(mul(c[0], c[0]), mul(c[1], c[1])), mul(c[2], c[2])));
      if (nn > 0.0)
        for (int d = 0; d < 3; ++d) n[d] = __ddiv_rn(c[d], nn);
    } else if (kb == K_LOCAL && has_ln[i]) {
      const double* P = poses + 12 * ob;
      const double* l = lnormal + 3 * i;
      for (int d = 0; d < 3; ++d)
        n[d] = add(add(mul(P[3 * d], l[0]), mul(P[3 * d + 1], l[1])), mul(P[3 * d + 2], l[2]));
    }
    const double g = add(add(mul(n[0], sub(a[0], b[0])), mul(n[1], sub(a[1], b[1]))),
                         mul(n[2], sub(a[2], b[2])));
    gaps[i] = g;
    pen = -g > 0.0 ? -g : 0.0;
  }
  pen = warp_max(pen);
  if ((threadIdx.x & 31) == 0 && pen > 0.0) atomicMax(pen_bits, (unsigned long long)__double_as_longlong(pen));
}

}  // namespace cnb

using namespace cnb;

extern "C" {

int cnb_refresh_proximity(int64_t m, const int8_t* kind, const int32_t* obj, const int64_t* node,
                          const double* w, const double* local, const double* world,
                          const double* const* views, const double* poses, double* p_a, double* p_b,
                          void* stream) {
  if (m <= 0) return CNB_OK;
  refresh_kernel<<<grid_for(m, 128), 128, 0, (cudaStream_t)stream>>>(m, kind, obj, node, w, local, world,
                                                                       views, poses, p_a, p_b);
  CNB_LAUNCH_CHECK("refresh_kernel");
  return CNB_OK;
}

int cnb_signed_gaps(int64_t m, const int8_t* kind, const int32_t* obj, const int64_t* node, const double* w,
                    const double* local, const double* world, const double* lnormal, const int8_t* has_ln,
                    const double* ref_normal, const double* const* views, const double* poses, double* gaps,
                    double* pen, void* stream) {
  CNB_CUDA(cudaMemsetAsync(pen, 0, sizeof(double), (cudaStream_t)stream));
  if (m <= 0) return CNB_OK;
  gaps_kernel<<<grid_for(m, 128), 128, 0, (cudaStream_t)stream>>>(m, kind, obj, node, w, local, world, lnormal,
                                                                    has_ln, ref_normal, views, poses, gaps,
                                                                    (unsigned long long*)pen);
  CNB_LAUNCH_CHECK("gaps_kernel");
  return CNB_OK;
}

}  // extern "C"
