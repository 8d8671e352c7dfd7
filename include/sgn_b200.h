/*
 * sgn_b200.h -- C ABI of the B200-native sparse Gauss-Newton (SGN) search-direction path.
 *
 * This is the drop-in boundary for the reference package `sgnopt` (arXiv 2107.03285).
 * The reference is pure Python; its solver plugin surface is a set of Python callables
 * (pkg/src/sgnopt/__init__.py:26-93).  The Python shim `paper_2107_03285_b200` re-exports
 * those callables with identical names/arguments/errors and binds the entry points below
 * through ctypes.  Each entry point names the reference interface it replaces.
 *
 * Conventions
 *   - every call returns a status code (SGN_OK ...); details via sgn_last_error();
 *   - "d_" pointers are device pointers owned by the caller; handles are owned by the
 *     library and freed by *_destroy;
 *   - every asynchronous call takes a cudaStream_t (passed as void*);  a handle is not
 *     thread-safe: one host thread per handle;
 *   - values are float64, matrix indices int64 on the host side (the reference's CscMatrix
 *     uses int64 indptr/indices, pkg/src/sgnopt/sparse.py:71-72);
 *   - KKT unknown order is the reference's (x[n_x], p[n_p], lambda[n_c]) with n_c == n_x
 *     (pkg/src/sgnopt/sparse.py:165-194).
 */
#ifndef SGN_B200_H
#define SGN_B200_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes -> errors.py types (mapped in paper_2107_03285_b200/_lib.py) */
#define SGN_OK             0
#define SGN_SINGULAR       1   /* SingularMatrix(pivot_index)           errors.py:26-35 */
#define SGN_NO_CONVERGENCE 2   /* NoConvergence(residual, iterations)   errors.py:46-54 */
#define SGN_DIMENSION      3   /* DimensionMismatch                     errors.py:9     */
#define SGN_CUDA_ERROR     4   /* CUDA runtime failure (message in sgn_last_error)      */
#define SGN_INVALID        5   /* bad argument / unsupported input                      */

/* solve flags */
#define SGN_SOLVE_LEADING  1   /* solve only with the leading (x, lambda) block of the
                                  factor; p unknowns are held at zero (adjoint solve)     */

typedef struct sgn_symbolic_s* sgn_symbolic;
typedef struct sgn_factor_s*   sgn_factor;

typedef struct {
    int64_t n;             /* dimension                                   */
    int64_t n_fronts;      /* fronts (dense supernodes) in the assembly tree */
    int64_t n_levels;      /* tree levels (height scheduling)             */
    int64_t nnz_l;         /* stored entries of L (incl. D)               */
    int64_t front_doubles; /* dense front storage per instance (doubles)  */
    int64_t max_front;     /* largest front order                         */
    int64_t max_piv;       /* largest pivot block of a front              */
    int64_t launches;      /* kernel launches of one numeric factorization */
    double  flops;         /* LDL^T flops of one numeric factorization    */
    int64_t pair_mode;     /* 1 = (x_i, lambda_pi(i)) 2x2 pivots; 2 = also p pairs in the dissection */
} sgn_symbolic_stats;

/* ---- library ------------------------------------------------------------------- */
const char* sgn_last_error(void);
int sgn_version(void);
/* total kernel launches issued by this library so far (launch-count evidence) */
int64_t sgn_launch_count(void);
int sgn_device_sync(void* stream);

/* ---- symbolic analysis (host, once per sparsity pattern) -----------------------
 * Replaces the ordering/symbolic half of SparseFactorization.__init__
 * (pkg/src/sgnopt/linear_solvers.py:70-91: structural checks + SuperLU COLAMD).
 * indptr/indices: full CSC pattern (sorted, unique rows) of a structurally symmetric
 * matrix.  n_x > 0 selects KKT mode (x, p, lambda blocks; 2x2 pivots on matched
 * (x_i, lambda_j) pairs, p unknowns eliminated last in one dense root front);
 * n_x == 0 selects generic mode (1x1 pivots).  leaf_size: max unknowns in a leaf front
 * (0 = default).  On structural singularity returns SGN_SINGULAR and *pivot_index.   */
int sgn_symbolic_create(int64_t n, const int64_t* indptr, const int64_t* indices,
                        int64_t n_x, int64_t n_p, int64_t n_c, int32_t leaf_size,
                        sgn_symbolic* out, int64_t* pivot_index);

/* Options of the symbolic analysis and of the task schedules it builds (all former
 * SGN_* environment knobs).  sgn_symbolic_options_default() fills the defaults; a zero
 * field of a default-filled struct is meaningful (e.g. noz_tiles = 0: off).            */
typedef struct {
    int32_t leaf_size;     /* max unknowns in a leaf front (default 64)                      */
    int32_t p_order;       /* KKT mode: 0 = p unknowns eliminated last in one dense root
                              front (needed when C = d2f/dp2 may be singular); 1 = p unknowns
                              join the nested dissection as consecutive 2x2 pairs (the caller
                              asserts C > 0: the stabilized KKT is then quasi-definite, and a
                              p pair's Schur block stays positive definite); an odd last p is
                              eliminated last on its own.  (default 0)                        */
    int32_t upd_group;     /* pivot steps per grouped Schur-update task (default 8)          */
    int32_t zinline;       /* fronts with >= zinline pivot tiles build Z inline (default 8)  */
    int32_t zquota;        /* queued Z blocks interleaved per pivot step (default 256)       */
    int32_t noz_tiles;     /* root p-front of >= noz_tiles tiles gets no Z (default 0: off)  */
    int32_t fat_tiles;     /* fronts of <= fat_tiles tiles factor as one task (default 0)    */
    int32_t fat_solve;     /* small fronts solve as one task (default 1)                     */
    int32_t generic_pairs; /* generic mode: 2x2 pivots on consecutive unknowns (default 1)   */
    int32_t upd_pair;      /* 64x64 task blocks: bit 0 grouped Schur updates, bit 1 struct-tile
                              solve-panel blocks, bit 2 front assembly, bit 3 single-column
                              updates as 64x32 row pairs, bit 4 the look-ahead and single-step
                              columns of a step as one 64x64 block per row pair below the
                              chain rows (default 31)                                         */
    int32_t pair_min_tiles;/* bits 0-1 of upd_pair apply to fronts of >= this many 32-row tiles;
                              0 (default) = auto: 4 when the factorization has >= 5e9 flops,
                              else none (small factorizations are pivot-chain bound)          */
    int32_t upd_group_cb;  /* pivot steps per grouped update of contribution-block columns
                              (tj >= P: off the pivot chain, only the parent's assembly reads
                              them; default 32)                                              */
    int32_t defer_groups;  /* 1: grouped updates of step k are listed after the panels and the diagonal
                            * update of step k + 1 (CTAs run them while that step's TRSMs are in flight) */
    int32_t zdist;         /* queued solve-panel blocks of fronts at levels <= lv - zdist are interleaved into
                            * the pivot steps of level lv (2: their fronts are finished by then; 1: the level
                            * below, whose fronts may still be finishing) */
    int32_t reserved[2];
} sgn_symbolic_options;
void sgn_symbolic_options_default(sgn_symbolic_options* o);
/* as sgn_symbolic_create, with options (NULL = defaults) */
int sgn_symbolic_create_ex(int64_t n, const int64_t* indptr, const int64_t* indices,
                           int64_t n_x, int64_t n_p, int64_t n_c, const sgn_symbolic_options* opts,
                           sgn_symbolic* out, int64_t* pivot_index);
int  sgn_symbolic_get_stats(sgn_symbolic s, sgn_symbolic_stats* out);
/* perm[k] = original unknown eliminated at position k */
int  sgn_symbolic_get_perm(sgn_symbolic s, int64_t* perm);
/* front tree export for host-side verification: per front (first position, npiv, nrow,
 * parent); rows_ptr (n_fronts+1) / rows (positions) */
int  sgn_symbolic_get_fronts(sgn_symbolic s, int64_t* first, int64_t* npiv, int64_t* nrow,
                             int64_t* parent, int64_t* rows_ptr, int64_t* rows);
void sgn_symbolic_destroy(sgn_symbolic s);

/* ---- numeric factorization (device) --------------------------------------------
 * Replaces spla.splu (linear_solvers.py:87) + the stabilization of stabilized_matrix
 * (linear_solvers.py:111-127): factors K + diag(+eps_x, 0, -eps_lambda) as
 * P^T K P = L D L^T (multifrontal, DMMA Schur updates).  `batch` independent instances
 * share the pattern; instance b's values start at d_values + b*values_stride.        */
int  sgn_factor_create(sgn_symbolic s, int32_t batch, sgn_factor* out);
int  sgn_factor_numeric(sgn_factor f, const double* d_values, int64_t values_stride,
                        double eps_x, double eps_lambda, void* stream);
/* as sgn_factor_numeric with per-instance shifts (device arrays of length batch; either may
 * be NULL = 0): the batched tau-regularized Newton of forward.py:171-186 needs one tau per
 * instance.                                                                           */
int  sgn_factor_numeric_v(sgn_factor f, const double* d_values, int64_t values_stride,
                          const double* d_eps_x, const double* d_eps_lambda, void* stream);
/* synchronizes; pivots[b] = first zero pivot of instance b (original index) or -1 */
int  sgn_factor_status(sgn_factor f, void* stream, int64_t* pivots);
/* synchronizes; returns SGN_SINGULAR with the first zero pivot (original index) */
int  sgn_factor_check(sgn_factor f, void* stream, int64_t* pivot_index);
/* x = (L D L^T)^{-1} b for every instance (b, x strided by n). Replaces
 * SparseFactorization.solve (linear_solvers.py:93-97); `transpose` is a no-op for the
 * symmetric factor.  flags: SGN_SOLVE_LEADING.  d_b may alias d_x.                 */
int  sgn_factor_solve(sgn_factor f, const double* d_b, double* d_x, int32_t flags, void* stream);
void sgn_factor_destroy(sgn_factor f);

/* Persistent grid (CTAs) of this factor's numeric factorization; ctas <= 0 restores the
 * default (every SM at the occupancy limit); *grid (may be NULL) = the grid in effect.
 * Two factorizations issued on concurrent streams -- the KKT factor and the adjoint's G_x
 * factor of one direction (sensitivity.py:194-198 next to linear_solvers.py:130-175) --
 * split the SMs' CTA slots instead of queueing.                                        */
int  sgn_factor_set_grid(sgn_factor f, int32_t ctas, int32_t* grid);
/* Late hand-over of CTA slots to a concurrent launch: the factorization starts on its full
 * grid, and once its task list reaches the first of the top levels that hold at most
 * max_level_fronts fronts each (the dependency-chain-bound end of the elimination tree), the
 * CTAs with index >= keep_ctas leave.  A launch queued on another stream (the adjoint's G_x
 * factorization, sensitivity.py:194-198) then becomes resident in their slots.  keep_ctas <=
 * 0 or max_level_fronts <= 0 turns it off; *retire_task (may be NULL) = the task index of
 * the hand-over, -1 when off or when no level qualifies. */
int  sgn_factor_set_retire(sgn_factor f, int32_t keep_ctas, int32_t max_level_fronts, int64_t* retire_task);

/* X[:, j] = (L D L^T)^{-1} B[:, j] for nrhs right-hand sides against ONE factor (batch 1),
 * column j at B + j*n.  Replaces the n_p back-substitutions of sensitivity_matrix
 * (reference sensitivity.py:167-178: factor.solve(dcdp dense)).                           */
int  sgn_factor_solve_multi(sgn_factor f, const double* d_B, double* d_X, int32_t nrhs, void* stream);

/* Smallest 1x1 pivot D_rr of a generic-mode factor (batch instance 0) and its unknown:
 * the positive-definiteness test of the dense Gauss-Newton factorization (reference
 * linear_solvers.py:214-240, cho_factor -> NotPositiveDefinite(pivot_index)).        */
int  sgn_factor_min_pivot(sgn_factor f, double* min_pivot, int64_t* position, void* stream);

/* ---- dense Gauss-Newton (DGN) building blocks, SURVEY 8(f) 2 -------------------------
 * Blocks of the stacked KKT [[A, B^T, G_x^T], [B, C, G_p^T], [G_x, G_p, 0]] are read from
 * its full CSC (int64 indptr / indices, symmetric so CSC == CSR).
 * sgn_csc_block_dense: out (column-major nr x nc) = K[r0:r0+nr, c0:c0+nc]  (dcdp.to_dense,
 *   blocks.C.to_dense; sensitivity.py:177, 240).
 * sgn_csc_spmm: Y[j][r] = sum_c K[r0+r, c0+c] X[j][c] (A @ sens, B @ sens; sensitivity.py:239-240).
 * sgn_gemm_tn: C (column-major n x n) = X Y^T for row-major X, Y (n x K): sens^T (A sens), DMMA.
 * sgn_gn_hessian: H = sym(STAS + BS + BS^T + C) (dense_gn_hessian, sensitivity.py:232-242). */
int  sgn_csc_block_dense(int64_t n_cols_total, const int64_t* d_ptr, const int64_t* d_idx, const double* d_val,
                         int64_t r0, int64_t nr, int64_t c0, int64_t nc, double* d_out, void* stream);
int  sgn_csc_spmm(const int64_t* d_ptr, const int64_t* d_idx, const double* d_val, int64_t r0, int64_t nr,
                  int64_t c0, int64_t ncol, const double* d_X, int64_t ldx, double* d_Y, int64_t ldy,
                  int64_t m, void* stream);
int  sgn_gemm_tn(const double* d_X, const double* d_Y, int64_t n, int64_t K, double* d_C, void* stream);
int  sgn_gn_hessian(const double* d_stas, const double* d_bs, const double* d_c, int64_t n, double* d_H,
                    void* stream);

/* Diagnostics (no reference counterpart): the persistent solve's task list and, when the
 * process ran with SGN_DAG_TRACE=1, the last solve's per-task trace -- 6 words per task
 * (start, (smid << 48) | signalled, prefetched, ready, combined, end; globaltimer ns,
 * 0 = phase not reached).  meta: 5 int32 per task
 * (kind, front, level, a, b); any output pointer may be NULL.                         */
int  sgn_debug_solve_trace(sgn_factor f, int64_t* out, int64_t cap, int64_t* n_tasks, int32_t* meta);
/* Same for the persistent factorization (SGN_FDAG_TRACE=1): 8 words per task (start,
 * ready, end ns; smid; 4 sub-phase ns or 0); meta: 6 int32 per task (kind, step, front,
 * level, a, b).                                                                        */
int  sgn_debug_factor_trace(sgn_factor f, int64_t* out, int64_t cap, int64_t* n_tasks, int32_t* meta);
/* Diagnostics: copy one internal buffer of a factor to the host (which: 0 fronts store,
 * 1 solve panels, 2 pivot-block scratch, 3 front table, 4 factor tasks, 5 solve tasks,
 * 6/7 gather map, 8 permutation, 9 tickets, 10 struct rows, 11 rel tile ranges).     */
int  sgn_debug_factor_buffer(sgn_factor f, int32_t which, void* out, int64_t cap_bytes, int64_t* size_bytes);
/* Diagnostics: fill the fronts, solve panels, pivot scratch and solve scratch with `value`
 * (tests use NaN to prove no kernel reads memory it has not written).                   */
int  sgn_debug_poison(sgn_factor f, double value);

/* y = K x on the full symmetric CSC pattern (which equals its CSR).  Replaces the
 * scipy SpMV of _relative_residual / _bicgstab_refine (linear_solvers.py:105-108,178-211).
 * flags: SGN_SOLVE_LEADING masks the p block (input and output).                   */
int  sgn_spmv(sgn_factor f, const double* d_values, int64_t values_stride,
              const double* d_x, double* d_y, int32_t flags, void* stream);

/* Post-factor half of solve_kkt_stabilized (linear_solvers.py:130-175) with
 * _bicgstab_refine (178-211) on the device: x0 = F^{-1} rhs; if the relative residual
 * against the UNSHIFTED K exceeds tol run restart-free left-preconditioned BiCGSTAB,
 * keeping the best iterate.  Per-instance results in rel_res[batch], iters[batch].
 * Returns SGN_NO_CONVERGENCE if any instance ends above tol (d_sol then holds the best
 * iterate, mirroring NoConvergence.best).                                          */
int  sgn_solve_refined(sgn_factor f, const double* d_values, int64_t values_stride,
                       const double* d_rhs, double* d_sol, double tol, int32_t max_iters,
                       int32_t flags, double* rel_res, int32_t* iters, void* stream);

/* Mixed-precision iterative refinement on the factor (the direction path's first solve,
 * ahead of the BiCGSTAB of linear_solvers.py:178-211): x = F^{-1} rhs, then `steps` times
 * x += F^{-1}(rhs - K x) with the residual evaluated in double-double (error-free products
 * and compensated row sums, then rounded).  rel_res[b] = |rhs - K x| / |rhs| of the final x
 * evaluated the same way (an exact residual, so it cannot be below the truth); corr[b] =
 * |last correction| / |x|.  x is carried as a double-double (hi in d_sol, lo copied to
 * d_sol_lo when non-NULL).  rel_res = corr = NULL: no final residual and no host sync
 * (graph-capturable).  The caller falls back to sgn_solve_refined when rel_res > tol.   */
int  sgn_solve_ir(sgn_factor f, const double* d_values, int64_t values_stride,
                  const double* d_rhs, double* d_sol, double* d_sol_lo, int32_t steps,
                  double* rel_res, double* corr, void* stream);
/* r = b - K (x + x_lo) with the same double-double evaluation (x_lo may be NULL).  The
 * adjoint gradient g = f_p + G_p^T lambda of the direction path is taken from it, with
 * lambda = (hi, lo) from sgn_solve_ir on the dc/dx factor (sensitivity.py:181-198). */
int  sgn_residual_dd(sgn_factor f, const double* d_values, int64_t values_stride,
                     const double* d_x, const double* d_x_lo, const double* d_b, double* d_r,
                     void* stream);

/* ---- element assembly (device) --------------------------------------------------
 * Replaces the NumPy element kernels + COO->CSC of constraint_jac_x / constraint_jac_p
 * (spring analog: forward.py:61-111, spring_bar.py:144-156).  Per element, writes the
 * element Hessian d2E/dx2 and mixed derivative d2E/dx dX (rest coordinates) in
 * row-major (nd x nd) blocks, nd = nodes_per_elem * dim.  d_mixed == NULL: Hessians
 * only (forward Newton).  d_mslot (neo-Hookean simplices, optional): compact mixed
 * slot per element (-1: not in the p-map support, skipped); NULL: one per element. */
#define SGN_ELEM_SPRING     1   /* 2-node spring, any dim (forward.py:61-111)        */
#define SGN_ELEM_NH_TRI     2   /* 3-node neo-Hookean triangle, plane strain         */
#define SGN_ELEM_NH_TET     3   /* 4-node neo-Hookean tetrahedron                    */
#define SGN_ELEM_SHELL_MEMBRANE 4 /* 3-node StVK membrane triangle in 3-D (config 4)  */
#define SGN_ELEM_HINGE      5   /* 4-node dihedral bending hinge (config 4)          */
int  sgn_element_derivs(int32_t elem_type, int64_t n_elems, int32_t batch,
                        const int32_t* d_conn, const double* d_pos, const double* d_rest,
                        int64_t vert_stride, const double* d_params, int64_t param_stride,
                        double* d_hess, double* d_mixed, const int32_t* d_mslot,
                        int64_t buf_stride, void* stream);
/* as sgn_element_derivs; rest_comp_mask (bit i = rest coordinate component i is moved by the
 * parameter map) lets the shell kinds skip the mixed columns of components the p-map never
 * reads (config 4: heights only, 4 of a hinge's 12 columns); those entries are not written. */
int  sgn_element_derivs_ex(int32_t elem_type, int64_t n_elems, int32_t batch,
                           const int32_t* d_conn, const double* d_pos, const double* d_rest,
                           int64_t vert_stride, const double* d_params, int64_t param_stride,
                           double* d_hess, double* d_mixed, const int32_t* d_mslot,
                           int64_t buf_stride, int32_t rest_comp_mask, void* stream);
/* element energies / gradients for the forward solve and line search
 * (spring_energy/spring_gradient analog, forward.py:34-48) */
int  sgn_element_energy_grad(int32_t elem_type, int64_t n_elems, int32_t batch,
                             const int32_t* d_conn, const double* d_pos, const double* d_rest,
                             int64_t vert_stride, const double* d_params, int64_t param_stride,
                             double* d_energy, double* d_grad, int64_t buf_stride, void* stream);

/* mixed blocks d2E/dx dX of the listed neo-Hookean simplices (the p-map support) into
 * compact slots: block t <- element d_elems[t] (constraint_jac_p's element terms).     */
int  sgn_element_mixed(int32_t elem_type, int64_t n_list, int32_t batch, const int32_t* d_elems,
                       const int32_t* d_conn, const double* d_pos, const double* d_rest,
                       int64_t vert_stride, const double* d_params, int64_t param_stride,
                       double* d_mixed, int64_t buf_stride, void* stream);
/* Fused vertex-centric assembly of the G_x entries of a single-group neo-Hookean mesh
 * (replaces constraint_jac_x's element triplets + COO->CSC for those entries,
 * spring analog forward.py:51-78, sensitivity.py:245-256 for the KKT placement): one
 * task per vertex, its incident elements' Hessian columns staged in shared memory, each
 * output the fixed-order sum of its element entries written to K (both symmetric copies)
 * and/or G_x.  Plan arrays from the host (engine.VertexPlan); group = lanes per vertex
 * (>= max incident elements: 6/8/16 for triangles, 16/32 for tetrahedra).              */
int  sgn_vertex_assemble(int32_t elem_type, int32_t n_task, int32_t group, int32_t batch,
                         const int32_t* d_inc_ptr, const int32_t* d_inc_ea, const int32_t* d_out_ptr,
                         const int32_t* d_out_dst, const int32_t* d_con_ptr, const int32_t* d_con_idx,
                         const int32_t* d_conn, const double* d_pos, const double* d_rest,
                         int64_t vert_stride, const double* d_params, int64_t param_stride,
                         double* d_kvals, int64_t kstride, double* d_gvals, int64_t gstride, void* stream);
/* out[dst[k]] = base[k] + sum coef * buf[idx]: the gather restricted to a list of outputs
 * (the KKT entries the vertex assembly does not produce: constants and G_p).          */
int  sgn_gather_to(int64_t n_out, int32_t batch, const int64_t* d_dst, const double* d_base,
                   const int64_t* d_ptr, const int64_t* d_idx, const double* d_coef, const double* d_buf,
                   int64_t buf_stride, double* d_out, int64_t out_stride, void* stream);
/* out[k] = base[k] + sum_{t in ptr[k]..ptr[k+1]} coef[t] * buf[idx[t]]  (atomic-free,
 * fixed-order segmented sum into a precomputed CSC pattern; per instance strided).  */
int  sgn_gather_values(int64_t n_out, int32_t batch, const double* d_base, int64_t base_stride,
                       const int64_t* d_ptr, const int64_t* d_idx, const double* d_coef,
                       const double* d_buf, int64_t buf_stride, double* d_out,
                       int64_t out_stride, void* stream);


/* ---- batched vector kernels of the direction / forward-solve pipeline -------------
 * sgn_reduce: op 0 = sum, 1 = dot(a, b), 2 = max|a|; one deterministic value per
 * instance (fixed reduction order).  Replaces the NumPy reductions of the objective,
 * energies and norms (sensitivity.py:83-85, forward.py:149,189-203).                */
int  sgn_reduce(int32_t op, int64_t n, int32_t batch, const double* d_a, const double* d_b,
                int64_t stride, double* d_out, void* stream);
/* out = y + alpha[b] * x  (per-instance step length; forward.py:197-199, optimize.py:472);
 * d_y = NULL: out = alpha[b] * x (out may alias x)                                    */
int  sgn_axpy(int64_t n, int32_t batch, const double* d_alpha, const double* d_x,
              const double* d_y, double* d_out, int64_t stride, void* stream);
/* dst[b] = src[b] for every instance b with mask[b] != 0 (per-instance acceptance in the
 * batched Newton / line search, forward.py:197-201, optimize.py:485-486)               */
/* 64-bit fingerprint of each instance's n-vector (XOR of mixed bit patterns; deterministic):
 * the forward Newton detects an iterate that repeats bitwise -- a deterministic iteration
 * is then periodic and can never meet its tolerance (forward.py:135-168 would fail after
 * max_iters; the device fails at once, with the same outcome).                         */
int  sgn_fingerprint(int64_t n, int32_t batch, const double* d_x, int64_t stride, uint64_t* d_out,
                     void* stream);
int  sgn_masked_copy(int64_t n, int32_t batch, const int32_t* d_mask, const double* d_src,
                     double* d_dst, int64_t stride, void* stream);
/* least-squares terms (sensitivity.py:83-93): d_vec (KKT order, dim = 2 n_x + n_p per
 * instance) receives (df/dx, df/dp, 0) for r = (sigma x[tdofs] - tvals - R p, p) with weights
 * (w_t, w_reg): f_x = sigma w_t r at the targets, f_p = -R^T w_t r + w_reg p; d_fobj[b] =
 * 0.5 sum w r^2.  Either output may be NULL.  sigma = x_scale (1 for a position state; the
 * shell's displacement state).  R (optional) is the CSR over targets
 * (rptr/ridx/rcoef) with its transpose over parameters (rtptr/...) and needs rscr
 * [batch x n_t].  part [batch x 128 doubles] and tickets [batch ints, zeroed once] are the
 * caller's scratch (one set per concurrently used engine; the tickets reset themselves).  */
typedef struct {
    int64_t n_x, n_p, n_t;
    const int64_t* tdofs; const double* tvals; int64_t tstride;
    double w_t, w_reg, x_scale;
    const int64_t* rptr; const int64_t* ridx; const double* rcoef;
    const int64_t* rtptr; const int64_t* rtidx; const double* rtcoef;
    double* rscr; double* part; int32_t* tickets;
} sgn_lsq_args;
int  sgn_lsq_eval(int32_t batch, const sgn_lsq_args* args, const double* d_x, const double* d_p,
                  double* d_vec, double* d_fobj, void* stream);
/* rest-length residual blocks of 2-D springs (reference spring bar regularizer,
 * spring_bar.py:159-184): per spring s (conn 2 x int32, rest positions d_rest, L0 rest
 * lengths at p0), 21 doubles at d_out + s*21: w j j^T (4x4), w r j (4), r^2 with
 * r = |X_a - X_b| - L0_s and j = dr/d(X_a, X_b).                                        */
int  sgn_restlen_blocks(int64_t ns, int32_t batch, const int32_t* d_conn, const double* d_rest,
                        int64_t rest_stride, const double* d_L0, double w, double* d_out,
                        int64_t out_stride, void* stream);
/* adjoint gradient from a leading-block KKT solve (sensitivity.py:181-198, 245-256):
 * mode 0: d_out = (0, 0, d_src[lambda]);  mode 1: g = d_fvec[p] - d_src[p] (d_src = K v),
 * d_out = (0, -g, 0), d_grad = g;  mode 2: d_out = (0, 0, w) for an n_x-vector w = d_src;
 * mode 3: d_out (n_x per instance) = x block of d_src;  mode 4: g = d_src[p] (d_src = f - K v
 * evaluated by sgn_residual_dd), d_out = (0, -g, 0), d_grad = g.                                           */
int  sgn_adjoint_step(int32_t mode, int32_t batch, int64_t n_x, int64_t n_p, const double* d_src,
                      const double* d_fvec, double* d_out, double* d_grad, void* stream);

/* FP64 peak microbenchmark (roofline denominator; MEASURED_PEAKS.json has no FP64 figure):
 * mode 0 = DMMA m8n8k4 tensor pipe, 1 = DFMA.  *tflops = achieved TFLOP/s (all SMs).   */
int  sgn_fp64_peak(int32_t mode, int32_t iters, double* tflops, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SGN_B200_H */
