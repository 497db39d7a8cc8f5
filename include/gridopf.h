/* gridopf.h -- C-ABI of the B200 condensed-space ACOPF solve path.
 *
 * One shared library (paper_2307_16830_b200/_lib/libgridopf.so) holds the
 * host symbolic analysis (C++) and the sm_100a CUDA kernels.  Every entry
 * point takes plain pointers and sizes; device pointers are caller-owned
 * (allocated by the Python layer through torch) and all device work is
 * stream-ordered on the `stream` argument (a cudaStream_t).
 *
 * The reference (gridnlp 0.1.0, /root/reference/pkg/src/gridnlp) has no
 * C FFI; its boundaries are Python duck types plus two numba kernels.  Each
 * declaration below names the reference interface it replaces.  See
 * INTEGRATION.md for the ctypes binding a gridnlp maintainer would add.
 *
 * Return codes: 0 = OK, negative = error; gn_last_error() has the text.
 * Plans are not thread-safe (one stream per plan), mirroring the
 * reference's exclusive-use solver instances.
 */
#ifndef GRIDOPF_H
#define GRIDOPF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gn_model gn_model;         /* compiled pattern-block model + AD plan */
typedef struct gn_condense gn_condense;   /* pattern of W + I + tril(A^T A) + maps   */
typedef struct gn_symbolic gn_symbolic;   /* ordering-dependent factor structure     */
typedef struct gn_kkt gn_kkt;             /* KKT vector-kernel plan (A, W gathers)   */

const char *gn_last_error(void);
int gn_version(void);
/* kernel launches and plan-upload bytes since the last reset */
void gn_stats(int64_t *launches, int64_t *h2d_bytes, int reset);
/* plan-upload host time, recorded only with GN_HOST_TIMING=1 (diagnostics) */
void gn_upload_stats(int64_t *n_alloc, double *malloc_ms, double *copy_ms, int reset);
/* Host threads the calling thread's structure analysis (condense, ordering
 * support, symbolic factor, front plan) may use; <= 0 restores the default.
 * Thread-local (an analysis worker leaves a core to the launching thread). */
int gn_set_host_threads(int k);

/* ------------------------------------------------------------------ */
/* Host structure (CPU; no device needed)                              */
/* ------------------------------------------------------------------ */

/* Deterministic record permutation: lexicographic on (targets,
 * var_idx[:,0..], params[:,0..]), stable.
 * Replaces model.py:128-140 (_canonical_order). */
int gn_canonical_order(int64_t n_records, int32_t n_var_slots, int32_t n_param_slots,
                       const int64_t *var_idx, const double *params,
                       const int64_t *targets /* nullable */, int64_t *order_out);

/* One pattern block = (instruction tape, data arrays).  kind: 0 objective
 * sum, 1 constraint define, 2 constraint increment (model.py:24-26).
 * Records must already be in canonical order. */
typedef struct gn_block_desc {
  int32_t kind;
  int32_t n_var_slots, n_param_slots;
  int64_t n_records;
  const int64_t *var_idx;  /* [n_records][n_var_slots]   */
  const double *params;    /* [n_records][n_param_slots] */
  const int64_t *targets;  /* [n_records] or NULL         */
  int32_t n_ops;           /* tape (expressions.py:126-145) */
  const int32_t *ops;      /* [n_ops][3] = (op, a, b)       */
  int32_t n_consts;
  const double *consts;
  int32_t out;
  int32_t n_first;         /* first-derivative slots (sorted)                   */
  const int32_t *first_slots;
  int32_t n_pairs;         /* second-derivative pairs (a >= b), sorted          */
  const int32_t *pairs;    /* [n_pairs][2] */
  const int32_t *grad_order; /* [n_first] slot order of the reverse sweep (dict order) */
} gn_block_desc;

/* Expand templates over records, dedup, build slot maps and the device
 * gather plans.  Replaces CompiledModel.__init__ (model.py:236-303). */
int gn_model_create(const gn_block_desc *blocks, int32_t n_blocks, int64_t n_var,
                    int64_t n_con, gn_model **out);
int gn_model_info(const gn_model *mdl, int64_t *nnz_jac, int64_t *nnz_hess,
                  int64_t *n_contrib);
/* jac_slots / hess_slots / hess_factor are concatenated block by block,
 * slot-major: block b contributes n_first*R (constraint blocks only) resp.
 * n_pairs*R entries. */
int gn_model_export(const gn_model *mdl, int64_t *jac_rows, int64_t *jac_cols,
                    int64_t *hess_rows, int64_t *hess_cols, int64_t *jac_slots,
                    int64_t *hess_slots, double *hess_factor);
void gn_model_destroy(gn_model *mdl);

/* Pattern of W + I + tril(A^T A), lower CSC, and its scatter maps.
 * Replaces kkt.py:243-283 (symbolic_condense) + csc.py:52-76. */
int gn_condense_create(int64_t n, int64_t nnz_h, const int64_t *hess_rows,
                       const int64_t *hess_cols, int64_t nnz_j, const int64_t *jac_rows,
                       const int64_t *jac_cols, gn_condense **out);
int gn_condense_info(const gn_condense *cs, int64_t *nnz_k, int64_t *n_products);
int gn_condense_export(const gn_condense *cs, int64_t *indptr, int64_t *indices,
                       int64_t *w_map, int64_t *diag_map, int64_t *ata_map,
                       int64_t *ata_row, int64_t *ata_s1, int64_t *ata_s2);
void gn_condense_destroy(gn_condense *cs);

/* Generic lower-CSC -> (CSC, slot map) conversion (csc.py:52-76).
 * Two-phase: call with indptr_out == NULL to get *nnz_out. */
int gn_coo_to_csc(int64_t n, int64_t nnz, const int64_t *rows, const int64_t *cols,
                  int64_t *nnz_out, int64_t *indptr_out, int64_t *indices_out,
                  int64_t *slot_map_out);

/* Exact greedy minimum degree, key (degree, initial degree, index).
 * Replaces amd.py:18-54 (amd_order); bit-identical permutation. */
int gn_min_degree(int64_t n, const int64_t *indptr, const int64_t *indices,
                  int64_t *perm_out);

/* Symbolic Cholesky of the permuted pattern + the supernodal front plan.
 * Replaces cholesky.py:56-144 (elimination_tree, _row_patterns,
 * symbolic_cholesky). */
int gn_symbolic_create(int64_t n, const int64_t *indptr, const int64_t *indices,
                       const int64_t *perm, gn_symbolic **out);
typedef struct gn_symbolic_info_t {
  int64_t n, nnz_a, nnz_l, n_fronts, front_doubles, vec_doubles, max_front, max_cols;
  int64_t n_levels, flops;
} gn_symbolic_info_t;
/* condense + (minimum degree when perm is NULL) + symbolic + front plan in
 * one call; perm_out[n] receives the ordering used.  Same results as the
 * separate calls. */
int gn_analyze(int64_t n, int64_t nh, const int64_t *hr, const int64_t *hc, int64_t nj,
               const int64_t *jr, const int64_t *jc, const int64_t *perm, int64_t *perm_out,
               gn_condense **cs_out, gn_symbolic **sym_out);
int gn_symbolic_info(const gn_symbolic *sym, gn_symbolic_info_t *info);
int gn_symbolic_export(const gn_symbolic *sym, int64_t *parent, int64_t *a_rowptr,
                       int64_t *a_rowcol, int64_t *a_srcslot, int64_t *row_ptr,
                       int64_t *row_cols, int64_t *l_colptr, int64_t *l_rowidx);
/* Supernodal front plan (n_fronts entries each): first column, width,
 * rows, parent front (-1 = root), task order; *nf_small = number of
 * warp-task fronts (a prefix of order). */
int gn_symbolic_fronts(const gn_symbolic *sym, int32_t *first, int32_t *ncols, int32_t *nrows,
                       int32_t *parent, int32_t *order, int64_t *nf_small);
void gn_symbolic_destroy(gn_symbolic *sym);

/* ------------------------------------------------------------------ */
/* Device (sm_100a)                                                    */
/* ------------------------------------------------------------------ */

/* what-mask for gn_ad_eval */
#define GN_AD_F 1u
#define GN_AD_C 2u
#define GN_AD_GRAD 4u
#define GN_AD_JAC 8u
#define GN_AD_HESS 16u
#define GN_AD_RESET_FLAGS 256u   /* zero *flags before evaluating (stream-ordered) */

/* Uploads the plan and compiles one straight-line device function per
 * distinct pattern tape (NVRTC, sm_100a, cached per process); without NVRTC
 * (or with GN_AD_INTERPRETER=1) a generic tape-interpreter kernel is used. */
int gn_model_upload(gn_model *mdl);
/* the generated CUDA source of the pattern kernels (host only; two-phase:
 * *needed = bytes incl. the terminator) */
int gn_model_pattern_source(const gn_model *mdl, char *buf, size_t len, size_t *needed);
/* compulsory HBM bytes of one gn_ad_eval with this what-mask: inputs once,
 * index maps once, outputs once (the roofline numerator) */
int gn_model_traffic(const gn_model *mdl, uint32_t what, int64_t *bytes);
/* "patterns" or "interpreter: <reason>" */
int gn_model_ad_backend(const gn_model *mdl, char *buf, size_t len);
/* free the device copy of the plan (the host structure stays valid) */
int gn_model_release(gn_model *mdl);
/* Objective, constraints, gradient, Jacobian and Lagrangian Hessian values.
 * Replaces autodiff.py:45-142 (eval_*), with the _Problem scaling
 * (ipm.py:208-249) folded in: f *= obj_scale, c[i] *= con_scale[i],
 * grad *= obj_scale, jac[k] *= con_scale[row k], Hessian weights
 * obj_weight and y[i]*con_scale[i].  con_scale may be NULL (= 1).
 * Non-finite results set bits of *flags (GN_AD_* of the offending
 * output) instead of raising.  f points to ONE device double. */
int gn_ad_eval(gn_model *mdl, const double *x, const double *y, double obj_weight,
               const double *con_scale, double obj_scale, double *f, double *c,
               double *grad, double *jac, double *hess, uint32_t what,
               double *contrib_ws, int32_t *flags, void *stream);

int gn_symbolic_upload(gn_symbolic *sym);
/* Numeric refactorisation on the fixed pivot order.  kvals are the matrix
 * values in the CSC layout given to gn_symbolic_create.  *fail_col
 * (device int64) receives the smallest failing pivot position or n.
 * Replaces _chol_kernel/factorize (cholesky.py:147-205). */
int gn_chol_factor(gn_symbolic *sym, const double *kvals, double *fronts,
                   int64_t *fail_pos, void *stream);
/* x = P^T L^-T L^-1 P b; b and x may alias.  ws: vec_doubles scratch.
 * Replaces _solve_kernel/solve (cholesky.py:175-217). */
int gn_chol_solve(gn_symbolic *sym, const double *fronts, const double *b, double *x,
                  double *ws, void *stream);
/* The calling thread will run k solves concurrently on k streams: its
 * persistent kernels (which need every CTA co-resident) are sized to 1/k of
 * the device from now on (thread-local; default 1). */
int gn_set_concurrency(int k);
/* Return every cached device block of the plan allocator to the driver
 * (freed plan memory is otherwise kept for reuse, invisible to torch's
 * allocator).  cached_bytes_before (may be NULL) receives the cache size. */
int gn_alloc_trim(int64_t *cached_bytes_before);
/* Diagnostics: when trace (device int64[3][n_fronts][4]) is non-NULL the
 * factor / forward / backward kernels stamp %globaltimer per front (task
 * start, dependencies met, assembled, done).  NULL turns it off. */
int gn_chol_set_trace(gn_symbolic *sym, int64_t *trace);
/* Diagnostics: measured FP64 tensor-core (DMMA) throughput of this device
 * in TFLOP/s (the refactorisation's FLOP-roofline denominator). */
int gn_measure_dmma_peak(double *tflops, void *stream);
/* Factor values in the reference CSC layout (l_colptr/l_rowidx). */
int gn_chol_export_l(gn_symbolic *sym, const double *fronts, double *l_vals, void *stream);

/* ------------------------------------------------------------------ */
/* Condensed KKT system (device)                                       */
/* ------------------------------------------------------------------ */

/* Values of the seven-block Newton system at the current iterate
 * (KKTWorkspace, kkt.py:96-129).  Widths are +inf for absent bounds. */
typedef struct gn_kkt_state {
  const double *w, *a;                   /* W lower-COO values, Jacobian values */
  const double *dxl, *dxu, *dsl, *dsu;   /* bound widths                       */
  const double *zxl, *zxu, *zsl, *zsu;   /* bound duals                        */
  const double *sx, *ss;                 /* Sigma_x, Sigma_s                   */
  double dw, dc;                         /* delta_w, delta_c                   */
} gn_kkt_state;

/* seven-block vector (PVec / Steps, kkt.py:60-85) */
typedef struct gn_vec7 {
  double *x, *s, *y, *zxl, *zxu, *zsl, *zsu;
} gn_vec7;

/* Gather plans for W v, A v, A^T u and the K assembly (cs may be NULL when
 * no assembly is needed). */
int gn_kkt_create(int64_t n, int64_t m, int64_t nnz_h, const int64_t *hess_rows,
                  const int64_t *hess_cols, int64_t nnz_j, const int64_t *jac_rows,
                  const int64_t *jac_cols, const gn_condense *cs, gn_kkt **out);
void gn_kkt_destroy(gn_kkt *k);
/* sigma = zl/dl + zu/du over finite widths (kkt.py:121-129) */
int gn_kkt_sigma(int64_t len, const double *dl, const double *du, const double *zl,
                 const double *zu, double *sigma, void *stream);
/* kind 0: W v (symmetric, from the lower triangle), 1: A v, 2: A^T u
 * (kkt.py:132-150); accumulation order = the reference's np.add.at order */
int gn_kkt_matvec(gn_kkt *k, int kind, const double *vals, const double *v, double *out,
                  void *stream);
/* K = W + (Sigma_x + dw) I + A^T D A in the condensed CSC layout
 * (CondensedBackend.assemble, kkt.py:300-312) */
int gn_kkt_assemble(gn_kkt *k, const gn_kkt_state *st, double *kvals, void *stream);
/* compulsory HBM bytes of one gn_kkt_assemble (roofline numerator) */
int gn_kkt_assembly_traffic(const gn_kkt *k, int64_t *bytes);
/* (qx, qs, qy) = condense_pvec(pv); rhs = qx + A^T (C qs + D qy)
 * (kkt.py:159-167) */
int gn_kkt_condense_rhs(gn_kkt *k, const gn_kkt_state *st, const gn_vec7 *pv, double *qx,
                        double *qs, double *qy, double *rhs, void *stream);
/* ds = C (A dx + dc qs - qy), dy = (Sigma_s + dw) ds - qs (kkt.py:169-173) */
int gn_kkt_recover_slack_dual(gn_kkt *k, const gn_kkt_state *st, const double *dx,
                              const double *qs, const double *qy, double *ds, double *dy,
                              void *stream);
/* bound-dual steps (kkt.py:175-187); sets bit 1 of *flags when a finite
 * width is not positive (DegenerateInterior) */
int gn_kkt_recover_bound_duals(gn_kkt *k, const gn_kkt_state *st, const double *dx,
                               const double *ds, const gn_vec7 *pv, double *dzxl, double *dzxu,
                               double *dzsl, double *dzsu, int32_t *flags, void *stream);
/* res = pv - M_full * steps accumulated in double-double, rounded to
 * double; *norm = residual_norm(res) (kkt.py:190-209, 224-229) */
int gn_kkt_residual(gn_kkt *k, const gn_kkt_state *st, const gn_vec7 *steps,
                    const gn_vec7 *pv, gn_vec7 *res, double *norm, void *stream);
/* matrix_scale (kkt.py:211-221) into *out (device) */
int gn_kkt_matrix_scale(gn_kkt *k, const gn_kkt_state *st, double *out, void *stream);
/* y += alpha x over all seven blocks (Steps.axpy, kkt.py:83-85) */
int gn_vec7_axpy(gn_kkt *k, gn_vec7 *y, const gn_vec7 *x, double alpha, void *stream);

/* ------------------------------------------------------------------ */
/* Interior-point vector algebra (device)                              */
/* ------------------------------------------------------------------ */

/* Device vectors of one interior-point solve (ipm.py:326-548). */
typedef struct gn_ipm_vecs {
  double *x, *s, *y, *zxl, *zxu, *zsl, *zsu;   /* iterate                       */
  const double *xl, *xu, *sl, *su;             /* bounds (+-inf when absent)     */
  double *dxl, *dxu, *dsl, *dsu;               /* widths (+inf when absent)      */
  double *sx, *ss;                             /* Sigma_x, Sigma_s               */
  double *grad, *c, *jac;                      /* scaled AD outputs              */
  double *dual_x, *dual_s, *primal;            /* KKT residual blocks            */
} gn_ipm_vecs;

/* ------------------------------------------------------------------ */
/* Instance batches: B problems of ONE sparsity pattern share
 * every plan (model, KKT, symbolic factor); their vectors are stored
 * instance-major ([B][n], [B][m], [B][nnzH], [B][nnzJ], [B][nnzK], fronts
 * [B][front_doubles], solve workspace [B][vec_doubles]) and each *_batched
 * entry point is one launch per kernel for all B instances.  Per-instance
 * scalar operands are read from a device array bp[B][GN_BP_STRIDE]; scalar
 * outputs go to per-instance blocks scal + b * GN_BATCH_SCAL. */
#define GN_BP_MU 0         /* barrier parameter                                */
#define GN_BP_TAU 1        /* fraction-to-boundary factor                      */
#define GN_BP_ALPHA 2      /* primal step (trial point, accept, axpy)          */
#define GN_BP_ALPHA_Z 3    /* dual step (accept)                               */
#define GN_BP_DW 4         /* delta_w                                          */
#define GN_BP_DC 5         /* delta_c                                          */
#define GN_BP_ACTIVE 6     /* 0: state-changing kernels leave the instance alone */
#define GN_BP_OBJW 7       /* objective weight / scale (AD)                    */
#define GN_BP_STRIDE 8
#define GN_BATCH_SCAL 64   /* doubles per instance in batched scalar blocks    */

/* layout of the scalar block written by gn_ipm_prep (device doubles) */
#define GN_IPM_MAX_MU 16
#define GN_PREP_X_DUAL 0     /* max |dual_x|                         */
#define GN_PREP_X_ZL1 1      /* sum |zxl| + |zxu|                    */
#define GN_PREP_X_LOGL 2     /* sum log dxl (finite)                 */
#define GN_PREP_X_LOGU 3     /* sum log dxu (finite)                 */
#define GN_PREP_X_COMP 4     /* [n_mu] max |z w - mu_k| (finite w)   */
#define GN_PREP_S 24         /* start of the s-side block            */
#define GN_PREP_S_DUAL 0     /* max |dual_s|                         */
#define GN_PREP_S_PRIMAL 1   /* max |primal|                         */
#define GN_PREP_S_ZL1 2      /* sum |zsl| + |zsu|                    */
#define GN_PREP_S_YL1 3      /* sum |y|                              */
#define GN_PREP_S_THETA 4    /* sum |g - s|                          */
#define GN_PREP_S_LOGL 5
#define GN_PREP_S_LOGU 6
#define GN_PREP_S_COMP 7     /* [n_mu]                               */
#define GN_PREP_DOUBLES 48

/* widths, Sigma, dual_x = grad + A^T y - zxl + zxu, dual_s, primal and the
 * reductions of kkt_residual / barrier_phi (ipm.py:150-157, 393-429) for
 * the barrier candidates mus[0..n_mu) */
int gn_ipm_prep(gn_kkt *k, const gn_ipm_vecs *v, int32_t n_mu, const double *mus_host,
                double *scal, void *stream);
/* seven-block right-hand side (ipm.py:434-442) */
int gn_ipm_pvec(gn_kkt *k, const gn_ipm_vecs *v, double mu, gn_vec7 *pv, void *stream);
/* scal[0..4) = (alpha_x, alpha_s, alpha_z, dphi): fraction-to-boundary and
 * the barrier directional derivative (ipm.py:455-476) */
int gn_ipm_direction(gn_kkt *k, const gn_ipm_vecs *v, const gn_vec7 *steps, double mu, double tau,
                     double *scal, void *stream);
/* xt = x + alpha dx, st = s + alpha ds (ipm.py:482-483) */
int gn_ipm_trial_point(gn_kkt *k, const gn_ipm_vecs *v, const gn_vec7 *steps, double alpha,
                       double *xt, double *st, void *stream);
/* same at alpha = min(alpha_pair[0], alpha_pair[1]) read from the device
 * (the gn_ipm_direction output), so the first line-search trial needs no
 * host round trip */
int gn_ipm_trial_point_at(gn_kkt *k, const gn_ipm_vecs *v, const gn_vec7 *steps,
                          const double *alpha_pair, double *xt, double *st, void *stream);
/* scal[0..5) = (theta_t, log-sums of the four trial widths) (ipm.py:490-492);
 * a non-positive finite width yields a NaN log-sum */
int gn_ipm_trial_merit(gn_kkt *k, const gn_ipm_vecs *v, const double *ct, const double *xt,
                       const double *st, double *scal, void *stream);
/* accept the step, apply the kappa_sigma dual safeguard, flag (bit 2) lost
 * interiority (ipm.py:521-548) */
int gn_ipm_accept(gn_kkt *k, const gn_ipm_vecs *v, const gn_vec7 *steps, double alpha,
                  double alpha_z, double mu, double kappa_sigma, int32_t *flags, void *stream);

/* problem setup of one solve (replaces the _Problem constructor's scaling,
 * relax_equalities and the start/dual initialisation, ipm.py:112-123,
 * 179-193, 360-369): from g0 = grad f(x0) and j0 = J(x0) (row-major COO rows
 * jac_rows on the device) obj_scale / con_scale (when `scaling`), the relaxed
 * slack bounds sl/su of the scaled ranges [rlo, rhi], x = x0, s = y = 0 and
 * the unit bound duals of the finite bounds.  scratch: m + 1 uint64. */
int gn_ipm_setup(int64_t n, int64_t m, int64_t nj, const double *g0, const double *j0,
                 const int64_t *jac_rows, const double *x0, const double *xl, const double *xu,
                 const double *rlo, const double *rhi, int32_t scaling, double tol_r, uint64_t *scratch,
                 double *x, double *s, double *y, double *zxl, double *zxu, double *zsl, double *zsu,
                 double *con_scale, double *sl, double *su, double *obj_scale, void *stream);
/* initial slacks (ipm.py:371-380): s = clip(g, sl + push_tol, su - push_tol)
 * (midpoint of [sl, su] where that interval is empty) and theta = sum |g - s|.
 * red_partials: GN_RED_PARTIALS doubles; red_counter: one zeroed uint32 (left
 * zeroed). */
#define GN_RED_PARTIALS (1184 * 40)
int gn_ipm_init_slacks(int64_t m, const double *g, const double *sl, const double *su, double push_tol,
                       double *s, double *theta, double *red_partials, uint32_t *red_counter, void *stream);

/* ---- batched entry points (K12; layout and bp/scal conventions above).
 * Each replaces B back-to-back calls of its single-instance counterpart on
 * B problems sharing one plan -- the reference's multi-instance path is
 * run_suite(parallel=P) over independent solves (src/bench.py:166-186). */
/* gn_ad_eval for B instances: x [B][n], y/con_scale [B][m], c [B][m], grad
 * [B][n], jac [B][nnzJ], hess [B][nnzH]; objw_b / objs_b [B] objective
 * weight (Hessian) and scale (f, gradient), NULL = 1; params_b [B][P] per-
 * instance parameter values in the plan's layout (gn_model_param_count),
 * NULL = the model's own; f at f + b f_stride; flags [B]; contrib_ws [B][..] */
int gn_ad_eval_batched(gn_model *mdl, int32_t B, const double *x, const double *y, const double *objw_b,
                       const double *con_scale, const double *objs_b, const double *params_b, double *f,
                       int64_t f_stride, double *c, double *grad, double *jac, double *hess, uint32_t what,
                       double *contrib_ws, int32_t *flags, void *stream);
/* size P of the device parameter layout (per pattern block: param slot-major) */
int gn_model_param_count(const gn_model *mdl, int64_t *count);
/* kvals [B][nnzK]; delta_w / delta_c from bp */
int gn_kkt_assemble_batched(gn_kkt *k, int32_t B, const gn_kkt_state *st, const double *bp, double *kvals,
                            void *stream);
int gn_kkt_condense_rhs_batched(gn_kkt *k, int32_t B, const gn_kkt_state *st, const double *bp, const gn_vec7 *pv,
                                double *qx, double *qs, double *qy, double *rhs, void *stream);
int gn_kkt_recover_slack_dual_batched(gn_kkt *k, int32_t B, const gn_kkt_state *st, const double *bp,
                                      const double *dx, const double *qs, const double *qy, double *ds, double *dy,
                                      void *stream);
/* flags [B] */
int gn_kkt_recover_bound_duals_batched(gn_kkt *k, int32_t B, const gn_kkt_state *st, const double *dx,
                                       const double *ds, const gn_vec7 *pv, double *dzxl, double *dzxu,
                                       double *dzsl, double *dzsu, int32_t *flags, void *stream);
/* norm: instance b's residual max at norm[b * GN_BATCH_SCAL] (+1 scratch) */
int gn_kkt_residual_batched(gn_kkt *k, int32_t B, const gn_kkt_state *st, const double *bp, const gn_vec7 *steps,
                            const gn_vec7 *pv, gn_vec7 *res, double *norm, void *stream);
int gn_kkt_matrix_scale_batched(gn_kkt *k, int32_t B, const gn_kkt_state *st, const double *bp, double *out,
                                void *stream);
/* y += bp[b].alpha * x per instance (alpha 0: instance untouched) */
int gn_vec7_axpy_batched(gn_kkt *k, int32_t B, gn_vec7 *y, const gn_vec7 *x, const double *bp, void *stream);
/* fronts [B][front_doubles], fail_pos [B] (instance-local positions) */
int gn_chol_factor_batched(gn_symbolic *sym, int32_t B, const double *kvals, double *fronts, int64_t *fail_pos,
                           void *stream);
/* b, x [B][n], ws [B][vec_doubles] */
int gn_chol_solve_batched(gn_symbolic *sym, int32_t B, const double *fronts, const double *b, double *x,
                          double *ws, void *stream);
/* mus_dev [B][GN_IPM_MAX_MU] barrier candidates; scal [B][GN_BATCH_SCAL] */
int gn_ipm_prep_batched(gn_kkt *k, int32_t B, const gn_ipm_vecs *v, int32_t n_mu, const double *mus_dev,
                        double *scal, void *stream);
int gn_ipm_pvec_batched(gn_kkt *k, int32_t B, const gn_ipm_vecs *v, const double *bp, gn_vec7 *pv, void *stream);
int gn_ipm_direction_batched(gn_kkt *k, int32_t B, const gn_ipm_vecs *v, const gn_vec7 *steps, const double *bp,
                             double *scal, void *stream);
int gn_ipm_trial_point_batched(gn_kkt *k, int32_t B, const gn_ipm_vecs *v, const gn_vec7 *steps, const double *bp,
                               double *xt, double *st, void *stream);
/* alpha = min of the pair at alpha_pairs + b * GN_BATCH_SCAL */
int gn_ipm_trial_point_at_batched(gn_kkt *k, int32_t B, const gn_ipm_vecs *v, const gn_vec7 *steps,
                                  const double *alpha_pairs, double *xt, double *st, void *stream);
int gn_ipm_trial_merit_batched(gn_kkt *k, int32_t B, const gn_ipm_vecs *v, const double *ct, const double *xt,
                               const double *st, double *scal, void *stream);
/* instances with bp[b].active == 0 are left untouched; flags [B] */
int gn_ipm_accept_batched(gn_kkt *k, int32_t B, const gn_ipm_vecs *v, const gn_vec7 *steps, const double *bp,
                          double kappa_sigma, int32_t *flags, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GRIDOPF_H */
