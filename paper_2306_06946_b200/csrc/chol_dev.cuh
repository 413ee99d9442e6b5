// Device-side structures of the supernodal Cholesky shared by the factor
// (chol.cu) and solve / compliance (solve.cu) translation units.
#pragma once

#include <algorithm>
#include <vector>

#include "chol.h"
#include "common.cuh"

namespace cnb {

struct CompliancePlan;  // solve.cu

struct DevSym {
  const int64_t* first;
  const int64_t* rows_ptr;
  const int64_t* rows;
  const int64_t* front_off;
  const int64_t* child_ptr;
  const int64_t* child;
  const int64_t* rel_ptr;
  const int32_t* rel;
  const int64_t* m_off;     // solve panels M_s = [L11^{-1}; P21] (f x nc, column-major, ld d_ldf)
  const int64_t* kk_off;    // first 32x32 diagonal-block inverse of each supernode (kkinv slots)
};

__device__ __forceinline__ int64_t d_nc(const DevSym& S, int64_t s) { return S.first[s + 1] - S.first[s]; }
__device__ __forceinline__ int64_t d_nr(const DevSym& S, int64_t s) { return S.rows_ptr[s + 1] - S.rows_ptr[s]; }
// column stride of front s (f rounded up to even: 16-byte aligned columns), Symbolic::ldf;
// also the stride of the solve panel M_s and of the right-hand-side blocks R_s
__device__ __forceinline__ int64_t d_ldf(const DevSym& S, int64_t s) {
  const int64_t f = d_nc(S, s) + d_nr(S, s);
  return f + (f & 1);
}

struct DevTasks {
  int32_t* ptr = nullptr;
  int64_t count = 0;
};


template <typename T>
inline int upload_vec(T** dptr, const std::vector<T>& v) {
  size_t bytes = std::max<size_t>(1, v.size()) * sizeof(T);
  CNB_CUDA(cudaMalloc((void**)dptr, bytes));
  if (!v.empty()) CNB_CUDA(cudaMemcpy(*dptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return CNB_OK;
}

// Dense-solve plan for right-hand-side chunks of a fixed width.
struct SolvePlan {
  int64_t width = -1;
  int32_t* d_tasks = nullptr;
  std::vector<DevTasks> asm_t, panel_t, bwd_t;  // per level
  int64_t *d_roff = nullptr, *d_lo = nullptr, *d_w = nullptr;
  double* d_rhs = nullptr;
  void* d_lv = nullptr;  // width 1: per-level task table of the cooperative solve (solve.cu SolveLevel)
  int32_t *d_cptr = nullptr, *d_csrc = nullptr;  // its assembly gathers (solve.cu gemv1_task)
  int32_t* d_g1 = nullptr;                         // its panel tasks (kG1Rows rows each)
  int coop_grid = 0;
  void release() {
    for (void* p : {(void*)d_tasks, (void*)d_roff, (void*)d_lo, (void*)d_w, (void*)d_rhs, d_lv, (void*)d_cptr,
                    (void*)d_csrc, (void*)d_g1})
      if (p) cudaFree(p);
    d_cptr = d_csrc = d_g1 = nullptr;
    d_tasks = nullptr;
    d_roff = d_lo = d_w = nullptr;
    d_rhs = nullptr;
    d_lv = nullptr;
    coop_grid = 0;
    width = -1;
  }
};

struct CholHandle {
  Symbolic S;
  bool uploaded = false;
  bool factored = false;
  int64_t *d_first = nullptr, *d_rows_ptr = nullptr, *d_rows = nullptr, *d_front_off = nullptr;
  int64_t *d_child_ptr = nullptr, *d_child = nullptr, *d_rel_ptr = nullptr, *d_perm = nullptr;
  int64_t* d_m_off = nullptr;
  int32_t* d_rel = nullptr;
  int32_t* d_ea_rng = nullptr;  // extend-add children's row ranges (Symbolic::ea_rng)
  int64_t *d_map_src = nullptr, *d_map_dst = nullptr;
  double* d_front = nullptr;
  double* d_m = nullptr;       // solve panels M_s = [L11^{-1}; P21 = L21 L11^{-1}], see DevSym::m_off
  double* d_kkinv = nullptr;  // inverse of every 32x32 panel diagonal block (slot kk_off[s] + panel)
  int64_t* d_kk_off = nullptr;
  std::vector<int64_t> kk_off;
  double* d_vals = nullptr;   // CSR values being factorised (fixed address for the graph)
  cudaGraphExec_t factor_exec = nullptr;
  cudaStream_t cap_stream = nullptr;
  // L11^{-1} / P21 of a level only feed the solves: they run on a side stream
  // beside the next levels' factorisation (fork per level, one join at the end)
  cudaStream_t side_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // the compliance's forward solve waits only for the levels of M_s it reads:
  // ev_level[l] is recorded (externally, from inside the factor graph) once level
  // l's M_s is formed; it runs on comp_stream after ev_pre (the caller's stream
  // just before the factor, or after the previous compliance's Gram)
  std::vector<cudaEvent_t> ev_level;
  cudaStream_t comp_stream = nullptr;
  cudaEvent_t ev_pre = nullptr, ev_comp = nullptr;
  bool level_events = false;
  void* factor_status = nullptr;
  long long factor_nodes = 0;
  std::vector<int64_t> m_off;
  int32_t* d_tasks = nullptr;
  std::vector<DevTasks> ea, trinv, p21;                  // per level
  std::vector<std::vector<DevTasks>> potrf, trsm, syrk, syrk_out;  // per level, per panel
  SolvePlan plan1, plan8;                                // single-RHS / multi-RHS dense solves
  GrowBuf bp, tbuf;                                      // permuted RHS, backward temp
  GrowBuf c_int, c_rhs, c_val, c_y;                      // compliance workspace
  PinnedBuf c_pin;                                       // pinned staging of the compliance plan
  double last_gram_flops = 0.0, last_fwd_flops = 0.0;
  CompliancePlan* cplan = nullptr;                       // multi-GPU split protocol state

  DevSym sym() const {
    return DevSym{d_first,   d_rows_ptr, d_rows, d_front_off, d_child_ptr,
                  d_child,   d_rel_ptr,  d_rel,  d_m_off,     d_kk_off};
  }
};

// solve.cu
int solve_profile(double* out);
int solve_dense(CholHandle* h, const double* B, int64_t ldb, double* X, int64_t ldx, int64_t k, cudaStream_t st);
int compliance(CholHandle* h, int64_t ncols, const int64_t* colptr, const int64_t* rowidx, const double* vals,
               double* U, int64_t ldu, double* flops_out, cudaStream_t st);
int compliance_split_plan(CholHandle* h, int64_t ncols, const int64_t* colptr, const int64_t* rowidx,
                          const double* vals, int rank, int world, int64_t* sizes, double* flops_out,
                          cudaStream_t st);
int compliance_split_forward(CholHandle* h, double* ysend, cudaStream_t st);
int compliance_split_gram(CholHandle* h, const double* yall, double* tiles, cudaStream_t st);
int compliance_split_finish(CholHandle* h, const double* tiles_all, double* U, int64_t ldu, cudaStream_t st);
void free_compliance_plan(CholHandle* h);
int trinv_level(CholHandle* h, int level, cudaStream_t st);

}  // namespace cnb
