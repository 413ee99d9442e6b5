/*
 * cn_b200.h — C ABI of the B200-native recursive corrective-motion solver.
 *
 * Drop-in boundary for the hot path of the reference package `contactnewton`
 * (arXiv 2306.06946, fast scheme = paper Alg. 3).  The reference boundary is an
 * in-process Python API; every entry point below replaces one
 * reference function and is bound from Python with ctypes
 * (paper_2306_06946_b200/_lib.py).  INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - every pointer argument named d_* (and every double* / int* data array
 *     unless stated "host") is DEVICE memory owned by the caller; the library
 *     never frees caller memory;
 *   - `stream` is a cudaStream_t passed as void* (torch's current stream);
 *   - all floating point is IEEE fp64, matrices are row-major with a leading
 *     dimension `ld*` in elements;
 *   - every function returns a status code (CNB_OK on success); the message of
 *     the last failure on the calling thread is available from
 *     cnb_last_error();
 *   - kernels that detect data errors (non-positive pivots, singular contact
 *     blocks) record them in a device status word `d_status`
 *     (cnb_status_t, zero-initialised by the caller) that the host reads when
 *     it synchronises; status codes match the reference exceptions.
 */
#ifndef CN_B200_H
#define CN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (reference: contactnewton/errors.py:4-45) ------------- */
#define CNB_OK 0
#define CNB_E_DIMENSION 1          /* DimensionMismatchError  errors.py:8   */
#define CNB_E_NOT_SPD 2            /* NotSPDError             errors.py:12  */
#define CNB_E_SINGULAR_BLOCK 3     /* SingularBlockError      errors.py:36  */
#define CNB_E_DEGENERATE_FRAME 4   /* DegenerateFrameError    errors.py:32  */
#define CNB_E_NONFINITE 5          /* NonFiniteForceError     errors.py:24  */
#define CNB_E_VALIDATION 6         /* ValidationError         errors.py:44  */
#define CNB_E_INVALID_ATTACHMENT 7 /* InvalidAttachmentError  errors.py:28  */
#define CNB_E_DEGENERATE_TET 8     /* DegenerateTetError      errors.py:20  */
#define CNB_E_CUDA 100             /* CUDA runtime failure                  */
#define CNB_E_INTERNAL 200

typedef struct cnb_status {
  int32_t code;
  int32_t index;
  double value;
} cnb_status_t;

int cnb_abi_version(void);
const char* cnb_last_error(void);

/* ---- batched independent scenes (BASELINE configs[4]) ------------------- */
/* Copies of one soft body (shared mesh, linear material, one factorisation) on
 * their own planes.  Q: scene states (ns rows, pitch ldq); all other arrays are
 * device arrays over the concatenated pairs / packed per-scene matrices, with
 * exclusive prefix offsets poff (pairs), boff (3x3 blocks, m_s^2), woff
 * (doubles, ldw_s^2 with the even row stride ldw_s = 3 m_s + (m_s & 1)).  Replace, per copy: vertex-plane detection
 * (collision.py:264-287), W_g (constraints.py:155-179, as a gather from the
 * compliance C = E^T A^-1 E of the candidate surface DoFs), rebuild_W_fast
 * (constraints.py:182-191, bit-exact order), fast_update_proximity
 * (constraints.py:217-244), the backward-Euler right-hand side
 * (dynamics.py:183-211) and S^T acc (solver.py:250-257). */
/* d_i = float(n @ p_{vids[i]} - offset), bit-identical to the reference's plane
 * test (collision.py:264-270): numpy's 3-element dot is an FMA chain. */
int cnb_plane_distances(int64_t nv, const int64_t* vids, const double* pts, double n0, double n1, double n2,
                        double offset, double* out, void* stream);
int cnb_batch_detect_planes(int32_t ns, int64_t nsurf, const int64_t* vids, const double* Q, int64_t ldq,
                            const double* normals, const double* offsets, double threshold, int32_t* count,
                            int32_t* kept, void* stream);
int cnb_batch_pairs(int32_t ns, int64_t m, int64_t nsurf, const int64_t* poff, const int32_t* kept,
                    const int64_t* vids, const double* Q, int64_t ldq, const double* normals, const double* offsets,
                    int32_t* pscene, int32_t* pcand, double* pa, double* pb, double* ref, double* sdist,
                    void* stream);
int cnb_batch_gather_pa(int64_t m, const int32_t* pscene, const int32_t* pcand, const int64_t* vids, const double* Q,
                        int64_t ldq, double* pa, void* stream);
int cnb_batch_wg_gather(int32_t ns, int64_t nblocks, const int64_t* boff, const int64_t* poff, const int64_t* woff,
                        const int32_t* pcand, const int64_t* vids, const double* C, int64_t ldc, double* Wg,
                        void* stream);
/* C = A B (row-major fp64, DMMA tiles): the batched scenes' multi-RHS solves
 * against the shared inverse of A (formed once from the sparse factor). */
int cnb_gemm_dense(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B, int64_t ldb,
                   double* C, int64_t ldc, void* stream);
int cnb_batch_rebuild_w(int32_t ns, int64_t nblocks, const int64_t* boff, const int64_t* poff, const int64_t* woff,
                        const double* D, const double* Wg, double* W, void* stream);
int cnb_batch_prox(int32_t ns, int64_t m, const int64_t* poff, const int64_t* woff, const double* Wg, const double* t,
                   double h, double* pa, void* stream);
int cnb_batch_spmv(int32_t ns, int64_t n, const int64_t* rowptr, const int64_t* col, const double* val,
                   const double* x, int64_t ldx, double* y, int64_t ldy, void* stream);
int cnb_batch_rhs(int32_t ns, int64_t n, const double* fel, const double* Kv, const double* m3, const double* v,
                  const double* fext, const int8_t* fixed, double h, double alpha, double beta, double* b,
                  cnb_status_t* d_status, void* stream);
int cnb_batch_scatter_acc(int64_t m, const int32_t* pscene, const int32_t* pcand, const int64_t* vids,
                          const double* acc, double* rhs, int64_t ldr, void* stream);
/* PGS of independent scenes, one CTA each (solver.py:168-202 per scene);
 * g_off / w_off / mu are HOST arrays (nscenes + 1 / nscenes / nscenes); order
 * (HOST, optional) is the launch order, a permutation of the scenes (heaviest
 * expected solve first); results are per scene whatever the order.
 * delta_end may be NULL: the final pass over each scene's W is skipped. */
int cnb_pgs_batched(int32_t nscenes, const int64_t* g_off, const int64_t* w_off, const double* mu, const double* W,
                    const double* delta_base, double h, double tol, int32_t max_iter, double* lam, double* delta_end,
                    double* eps_hist, int32_t* iters_conv, const int32_t* order, cnb_status_t* d_status,
                    void* stream);

/* ---- constraint-space operators (contactnewton/constraints.py) ---------- */

/* W = D Wg D^T, D block-diagonal (groups x 3 x 3, rows n,t1,t2).
 * Replaces rebuild_W_fast  constraints.py:182-191 (+ gemm linalg.py:121-147);
 * bit-identical to the reference's naive-order double gemm. */
int cnb_rebuild_w(int64_t groups, const double* D, const double* Wg, int64_t ldwg,
                  double* W, int64_t ldw, void* stream);

/* U = S C S^T (m x m) for S (m x k) in ELL form, width 4 (ell_col int32, ell_val;
 * padding entries have value 0), C dense symmetric k x k.  The compact mapping
 * compliance U_o = S_o A^-1 S_o^T of constraints.py:175-178 is formed as
 * S_o (E^T A^-1 E) S_o^T, E = unit columns of the k DoFs S_o touches (k < m for
 * barycentric contacts that share triangle nodes).  k <= 29000. */
int cnb_sandwich(int64_t m, int64_t k, const int32_t* ell_col, const double* ell_val, const double* C,
                 int64_t ldc, double* U, int64_t ldu, void* stream);

/* total[3 idx[I] + a][3 idx[J] + b] += U[3I + a][3J + b] for one object's compact
 * compliance U (3 mo x 3 mo, idx ascending pair indices): the per-object sum of
 * W_g, constraints.py:175-179. */
int cnb_scatter_add_compliance(int64_t mo, const double* U, int64_t ldu, const int64_t* idx, double* total,
                               int64_t ldt, void* stream);

/* delta = D (p_a - p_b).  Replaces compute_violation constraints.py:208-214. */
int cnb_violation(int64_t groups, const double* D, const double* p_a, const double* p_b,
                  double* delta, void* stream);

/* t = D^T lam; if accumulated != NULL also accumulated += t.
 * Replaces DirectionMatrix.apply_transposed constraints.py:62-64 and the
 * impulse accumulation of newton_fast solver.py:346. */
int cnb_apply_dt(int64_t groups, const double* D, const double* lam, double* t,
                 double* accumulated, void* stream);

/* Fast proximity update for ONE dynamic object o:
 *   y = h^2 U_o t[idx],  p_a[idx[k]] += y_k (side +1)  or  p_b[idx[k]] -= y_k (side -1).
 * U_o is the compact (3*mo x 3*mo) restriction of the object's S A^-1 S^T to
 * the mo pairs it takes part in; idx (int64, mo) lists those pairs and
 * side (int8, mo) the side the object owns.  Replaces the per-object loop of
 * fast_update_proximity constraints.py:217-244.
 * U_o must be symmetric: from 8 row tiles of 128 up only its lower triangle is
 * read (CNB_PROX_SYM=0 forces the full-row GEMV).  The library's workspace for
 * this is shared: calls on different streams must not overlap. */
int cnb_prox_update(int64_t mo, const double* U, int64_t ldu, const int64_t* idx,
                    const int8_t* side, const double* t, double h, double* p_a, double* p_b,
                    void* stream);

/* ---- frames (contactnewton/collision.py) --------------------------------- */

/* Detection frames from p_a - p_b with the element normal as orientation
 * reference / fallback.  Replaces build_frames collision.py:359-375.
 * Degenerate pairs set d_status to CNB_E_DEGENERATE_FRAME. */
int cnb_build_frames(int64_t pairs, const double* p_a, const double* p_b,
                     const double* ref_normal, double* frames, cnb_status_t* d_status,
                     void* stream);

/* Re-linearised frames and the largest normal rotation (radians, written to
 * rotation[0]).  Replaces relinearize collision.py:381-405 and
 * max_frame_rotation collision.py:408-414. */
int cnb_relinearize(int64_t pairs, const double* p_a, const double* p_b,
                    const double* prev, double* frames, double* rotation, void* stream);

/* Proximity positions of both sides of every pair, p = g(q).  Replaces
 * refresh_proximity / attachment_point collision.py:497-520.
 * Pair table: kind, obj (m x 2), node (m x 2 x 3, int64), w, local, world
 * (m x 2 x 3); views: device array of per-object node-coordinate pointers
 * (deformable objects); poses: per-object R (9, row-major) + t (3). */
int cnb_refresh_proximity(int64_t m, const int8_t* kind, const int32_t* obj, const int64_t* node,
                          const double* w, const double* local, const double* world,
                          const double* const* views, const double* poses, double* p_a, double* p_b,
                          void* stream);

/* Signed gaps along the current supporting-element normal and
 * pen = max(0, -min gap) (pen[0]).  Replaces signed_gaps collision.py:523-548
 * and the pen_before/pen_after reductions scene.py:658-662,713-718. */
int cnb_signed_gaps(int64_t m, const int8_t* kind, const int32_t* obj, const int64_t* node, const double* w,
                    const double* local, const double* world, const double* lnormal, const int8_t* has_ln,
                    const double* ref_normal, const double* const* views, const double* poses, double* gaps,
                    double* pen, void* stream);

/* Narrow phase, vertex vs triangle mesh (replaces _vertex_vs_mesh
 * collision.py:222-260 with closest_points_on_triangles 138-184 and
 * triangle_normals 187-190).  For each query vertex vids[q] (row of pts_a,
 * n x 3) against every triangle of (tris (nt x 3, int64), pts_b): the
 * lowest triangle index within 1e-9 of the minimum distance -> best[q];
 * out[12 q + ...] = signed distance, distance, barycentric (u, v, w),
 * closest point (3), unit triangle normal (3), hit (1.0 when
 * signed <= threshold).  Same operation order as numpy (bit-exact
 * decisions).  work: cnb_detect_work_bytes(nv, nt) bytes of device memory. */
int64_t cnb_detect_work_bytes(int64_t nv, int64_t nt);
int cnb_detect_vertex_mesh(int64_t nv, const int64_t* vids, const double* pts_a, int64_t nt, const int64_t* tris,
                           const double* pts_b, double threshold, void* work, int64_t* best, double* out,
                           void* stream);

/* ---- projected Gauss-Seidel (contactnewton/solver.py) -------------------- */

/* PGS with Signorini + isotropic Coulomb disk in the reference's canonical
 * group order.  Replaces pgs solver.py:168-202, local_solve 124-165 and
 * regularize 99-121.
 *   lam (c): output; delta_end (c, may be NULL): delta_base + h^2 W_reg lam
 *   (solver.py:201; NULL skips that extra pass over W); eps_hist (max_iter):
 *   per-sweep epsilon; iters_conv (2 int32): sweeps performed, converged flag;
 *   shift_out (groups, may be NULL): the regularisation shift added to each
 *   group's diagonal block (0 where none).
 * Singular blocks set d_status to CNB_E_SINGULAR_BLOCK (index = group). */
int cnb_pgs(int64_t groups, const double* W, int64_t ldw, const double* delta_base,
            double h, double mu, double tol, int32_t max_iter, double* lam,
            double* delta_end, double* eps_hist, int32_t* iters_conv, double* shift_out,
            cnb_status_t* d_status, void* stream);

/* Graph-coloured PGS (north star option; NOT the reference's iterate): the
 * groups are visited colour by colour (colour_ptr[ncolours + 1] offsets into
 * colour_groups[groups], host arrays, built so that no two groups sharing a
 * DoF share a colour), all groups of a colour updated at once from the lambda
 * at the colour's start, one CTA per group streaming its rows of W.  Same
 * local solve, regularisation, stopping rule and outputs as cnb_pgs; W and lam
 * need 16-byte aligned rows (even ldw).  omega in (0, 1]: under-relaxation of
 * each group's change (a dense W makes plain Jacobi inside a colour diverge).
 * Validated on the converged lambda. */
int cnb_pgs_coloured(int64_t groups, const double* W, int64_t ldw, const double* delta_base, double h, double mu,
                     double tol, int32_t max_iter, const int64_t* colour_ptr, const int64_t* colour_groups,
                     int32_t ncolours, double omega, double* lam, double* delta_end, double* eps_hist,
                     int32_t* iters_conv, double* shift_out, cnb_status_t* d_status, void* stream);

/* One group's local solve (solver.py:124-165) as a device call, for API
 * parity with local_solve; out (3). */
int cnb_local_solve(int64_t alpha, int64_t groups, const double* W, int64_t ldw,
                    const double* delta_cur, const double* lam, double mu, double h2,
                    double* out, cnb_status_t* d_status, void* stream);

/* ---- sparse Cholesky (contactnewton/linalg.py:58-118) -------------------- */

typedef struct cnb_chol_opaque* cnb_chol_t;

/* Host-only symbolic analysis of a symmetric CSR pattern (host arrays, both
 * triangles): nested-dissection ordering (geometric when coords != NULL,
 * n/bs x 3 node coordinates), elimination tree, supernodes, fronts.
 * Replaces the ordering/symbolic part of Factorization.__init__
 * linalg.py:68-76 (SuperLU MMD_AT_PLUS_A). */
int cnb_chol_analyze(int64_t n, const int64_t* rowptr, const int64_t* col, int32_t bs,
                     const double* coords, int32_t leaf_nodes, cnb_chol_t* out);
int cnb_chol_destroy(cnb_chol_t h);
/* info[9] = {n, supernodes, nnz(L), front doubles, levels, csr nnz, bs, launches per factorisation, launches per solve};
 * flops[2] = {factorisation flops, solve flops per right-hand side}. */
int cnb_chol_info(cnb_chol_t h, int64_t* info, double* flops);
/* Copy a named host array of the symbolic structure (tests / tooling). */
int64_t cnb_chol_export_bytes(cnb_chol_t h, const char* name);
int cnb_chol_export(cnb_chol_t h, const char* name, void* dst);

/* Numeric factorisation on the device from CSR values (device, same pattern
 * as analysed).  A non-positive pivot sets d_status to CNB_E_NOT_SPD, as the
 * reference's pivot check (linalg.py:77-84).  Internally forks onto the
 * handle's side stream and joins back into `stream` before returning. */
int cnb_chol_factor(cnb_chol_t h, const double* vals, cnb_status_t* d_status, void* stream);

/* X = A^{-1} B for k right-hand sides stored as k contiguous length-n
 * vectors (leading dimensions ldb/ldx); X may alias B.  Replaces
 * Factorization.solve / solve_multi linalg.py:89-106.  k == 1 runs as one
 * cooperative (grid-barrier) kernel: do not overlap two such solves, or one
 * and cnb_pgs, on different streams (their grids could wait on each other's
 * co-residency); order them with events. */
int cnb_chol_solve(cnb_chol_t h, const double* B, int64_t ldb, double* X, int64_t ldx, int64_t k,
                   void* stream);

/* Mapping compliance of one object, U = S A^{-1} S^T (ncols x ncols, row-major
 * device output) for the ncols right-hand-side columns of S^T given in host
 * CSC form (colptr, rowidx = DoF ids, vals).  Y = L^{-1} P S^T is formed only
 * on the elimination paths of the columns and U = Y^T Y by fp64 MMA tiles.
 * Replaces solve_multi(S^T) + S @ X of assemble_Wg constraints.py:175-178.
 * flops_out (host, may be NULL) = {forward-solve flops, Gram flops}.
 * For small factors the forward solve overlaps the preceding cnb_chol_factor
 * (handle-internal stream, per-level events); U is written in `stream` order. */
int cnb_chol_compliance(cnb_chol_t h, int64_t ncols, const int64_t* colptr, const int64_t* rowidx,
                        const double* vals, double* U, int64_t ldu, double* flops_out, void* stream);

/* The same U over `world` GPUs, right-hand-side columns split per rank with the
 * factor replicated (constraints.py:155-179 -> linalg.py:98-106).
 * Protocol, every rank, in order (the caller owns the collectives):
 *   plan(rank, world) -> sizes[0] = doubles of every rank's compact Y (send
 *       count), sizes[1] = doubles of every rank's Gram tile buffer, sizes[2..3]
 *       = this rank's sorted column range; flops_out = this rank's share;
 *   forward(ysend): forward solve of the rank's columns into ysend;
 *   caller: all-gather ysend -> yall (world x sizes[0], rank-major);
 *   gram(yall, tiles): every rank's Y unpacked, this rank's 64x64 Gram tiles
 *       (tile t -> rank t mod world) into tiles (sizes[1]);
 *   caller: all-gather tiles -> tiles_all (world x sizes[1]);
 *   finish(tiles_all, U, ldu): every tile scattered into U (and its mirror).
 * Every column's forward solve and every tile's Gram sum are computed exactly
 * as by cnb_chol_compliance, so U is bit-identical for every world size.  The
 * plan lives in the handle until the next plan call. */
int cnb_chol_compliance_plan(cnb_chol_t h, int64_t ncols, const int64_t* colptr, const int64_t* rowidx,
                             const double* vals, int32_t rank, int32_t world, int64_t* sizes, double* flops_out,
                             void* stream);
int cnb_chol_compliance_forward(cnb_chol_t h, double* ysend, void* stream);
int cnb_chol_compliance_gram(cnb_chol_t h, const double* yall, double* tiles, void* stream);
int cnb_chol_compliance_finish(cnb_chol_t h, const double* tiles_all, double* U, int64_t ldu, void* stream);

/* ---- FE assembly (contactnewton/dynamics.py) ------------------------------ */

/* One thread per tet: the 16 (rotated) 3x3 stiffness blocks Kb (tets x 16 x 9)
 * and the 4 element elastic forces fe (tets x 4 x 3) at positions x.
 * corot = 0: linear material, K_e from rest gradients, fe = K_e (x - x0)
 * (dynamics.py:81-99,172-177); corot = 1: R_e = polar(F), R K_e R^T and
 * R K_e (R^T x - x0).  R (tets x 9, may be NULL) receives the rotations. */
int cnb_fe_element(int64_t ntets, const int64_t* tets, const double* grads, const double* vol, const double* x,
                   const double* x0, double lam, double mu, int32_t corot, double* Kb, double* fe, double* R,
                   void* stream);
/* Deterministic gathers: global 3x3 blocks into DoF-CSR values (dst = CSR
 * index of each block row's first entry) and nodal elastic forces. */
int cnb_fe_gather(int64_t nblocks, const int64_t* cptr, const int64_t* contrib, const double* Kb, const int64_t* dst,
                  double* vals, int64_t nnodes, const int64_t* fptr, const int64_t* fidx, const double* fe,
                  double* f, void* stream);
/* A = (1 + h alpha) M + (h beta + h^2) K with fixed rows/cols -> identity and
 * b = h (f_ext - f_el - alpha M v - beta K v) - h^2 K v, b[fixed] = 0
 * (SoftBody.assemble dynamics.py:183-211); non-finite b -> CNB_E_NONFINITE.
 * (rowptr, col) is A's pattern: K's entries whose row and column are both
 * free plus every diagonal (dynamics.py:192-200).  a_src[e] is A entry e's
 * index in Kvals (-1 for a fixed DoF's diagonal); a_src = NULL when A and K
 * share a pattern (no fixed DoFs).  Avals or b may be NULL. */
int cnb_fe_system(int64_t n, const int64_t* rowptr, const int64_t* col, const int64_t* a_src, const double* Kvals,
                  const double* m3, const int8_t* fixed, double h, double alpha, double beta, const double* fel, const double* Kv,
                  const double* v, const double* fext, double* Avals, double* b, cnb_status_t* d_status,
                  void* stream);

/* ---- sparse products ----------------------------------------------------- */

/* y = alpha A x, A in CSR (device), one row per thread in column order.
 * Used for S^T t of _mechanical_correction solver.py:250-257 and the
 * stiffness products of SoftBody.assemble dynamics.py:202-208. */
int cnb_csr_spmv(int64_t rows, const int64_t* rowptr, const int64_t* col, const double* val,
                 const double* x, double* y, double alpha, void* stream);

/* ---- dense products (contactnewton/linalg.py) ---------------------------- */

/* C (m x n) = op(A) op(B), accumulated over k in ascending order with
 * separately rounded products and sums: bit-identical to gemm
 * linalg.py:121-147. */
int cnb_gemm_naive(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
                   int32_t trans_a, const double* B, int64_t ldb, int32_t trans_b,
                   double* C, int64_t ldc, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CN_B200_H */
