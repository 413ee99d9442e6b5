// Supernodal multifrontal Cholesky: host-side structures shared by the
// symbolic analysis (symbolic.cpp) and the GPU numeric phases (chol.cu).
//
// Replaces the reference's SuperLU factorisation (linalg.py:68-87; scipy
// splu with MMD_AT_PLUS_A ordering, pivot-free, SymmetricMode) and its
// solves (linalg.py:89-106).  P A P^T = L L^T with P a nested-dissection
// permutation; every supernode s owns a dense column-major FRONT of order
// f_s = nc_s + nr_s (its nc_s pivot columns followed by its nr_s below-
// diagonal structure rows).  After factorisation the first nc_s columns of
// the front hold the L panel, the trailing nr_s x nr_s block the update
// matrix that the parent extend-adds.
#pragma once

#include <stdint.h>

#include <vector>

namespace cnb {

constexpr int kPanel = 32;   // pivot panel width of the dense front factorisation
constexpr int kBlkPanels = 16;  // panels per trailing-update block: the trailing matrix is
                               // updated once per kBlkPanels * kPanel = 512 columns (K <= 512,
                               // i.e. once per supernode piece: pieces are <= 512 wide)
constexpr int kTile = 64;    // SYRK / GEMM output tile
constexpr int kEaCols = 8;   // parent columns per extend-add task (small: more CTAs in flight)
constexpr int kInvCols = 8;  // columns of L11^{-1} per inversion task
constexpr int kMaxSnCols = 512;  // widest supernode (wider ones are split into chains)

struct LevelTasks {
  // extend-add: (parent supernode, parent col lo, parent col hi, offset into
  // Symbolic::ea_rng of the children's row ranges for that column range)
  std::vector<int32_t> ea;
  // per panel step p: potrf fronts, trsm (front, row chunk), syrk (front, ti, tj):
  // syrk[p] = in-block update of the block's remaining pivot columns by panel p,
  // syrk_out[p] = trailing update by the whole block (last panel of a block)
  std::vector<std::vector<int32_t>> potrf, trsm, syrk, syrk_out;
};

struct Symbolic {
  std::vector<int32_t> ea_rng;  // per extend-add task, per child: [k0, k1) of its rows mapping into [lo, hi)
  int64_t n = 0;   // DoFs
  int bs = 1;      // DoFs per graph node
  std::vector<int64_t> perm, iperm;        // DoF level: perm[new] = old
  int64_t ns = 0;                          // supernodes (postorder)
  std::vector<int64_t> first;              // ns+1: pivot DoF range [first[s], first[s+1])
  std::vector<int64_t> rows_ptr, rows;     // below-diagonal structure (new DoF ids, sorted)
  std::vector<int64_t> parent;             // -1 for roots
  std::vector<int32_t> level;              // 0 = leaf
  std::vector<int64_t> child_ptr, child;   // children lists (ascending)
  std::vector<int64_t> front_off;          // ns+1, doubles
  std::vector<int64_t> rel_ptr;            // ns+1
  std::vector<int32_t> rel;                // child row -> parent front position
  int32_t n_levels = 0;
  std::vector<int64_t> level_ptr, level_sn;  // supernodes grouped by level
  std::vector<LevelTasks> tasks;
  // value map of the CSR this handle was analysed with
  int64_t csr_nnz = 0;
  std::vector<int64_t> map_src, map_dst;
  int64_t nnz_L = 0;       // stored L entries (incl. structural zeros)
  double flops = 0.0;      // factorisation flops
  double solve_flops_per_rhs = 0.0;

  int64_t nc(int64_t s) const { return first[s + 1] - first[s]; }
  int64_t nr(int64_t s) const { return rows_ptr[s + 1] - rows_ptr[s]; }
  // column stride of front s: f rounded up to even, so every front column starts
  // 16-byte aligned (16-byte asynchronous copies in the dense kernels)
  int64_t ldf(int64_t s) const { const int64_t x = nc(s) + nr(s); return x + (x & 1); }
  int64_t f(int64_t s) const { return nc(s) + nr(s); }
};

// Analyse the pattern of a symmetric n x n CSR (both triangles present).
// bs > 1 groups consecutive DoFs into graph nodes (all bs DoFs of a node
// share their pattern, e.g. 3 for FE nodes); coords (n/bs x 3, may be
// null) enables geometric nested dissection.
int analyze(Symbolic& S, int64_t n, const int64_t* rowptr, const int64_t* col, int bs,
            const double* coords, int leaf_nodes);

}  // namespace cnb
