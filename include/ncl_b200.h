/*
 * ncl_b200.h -- C ABI of the B200 (sm_100a) Newton-step hot path.
 *
 * Drop-in boundary for the reference's KKT plugin interface
 * (/root/reference/proj/include/ncl/kkt.hpp:58-125, proj/src/kkt.cpp) and
 * for the sparse layer it sits on (proj/include/ncl/sparse.hpp:26-99).  Plain
 * pointers and sizes only; every entry point returns 0 on success, a negative
 * code on invalid arguments / CUDA errors (message via ncl_last_error()).
 * Numerical failure is never an error code: it is reported in the stats
 * (ok = 0), exactly as the reference reports it in KktStep::ok / LdlFactors::ok.
 *
 * Index conventions are the reference's: int32 indices, FP64 values,
 * Hessian pattern lower CSC over the nt decision variables
 * (HessianPattern, model.hpp:44-48), Jacobian pattern CSR with sorted columns,
 * equality rows first (JacobianPattern, model.hpp:38-42), slack column -1 of
 * inequality row m_eq+k implicit (model.hpp:115-122).
 *
 * Threading: one context per solver thread (the reference's bench runs
 * independent solves in parallel, proj/tools/main.cpp:186-201); every context
 * owns its CUDA stream and device workspace, no global mutable state.
 */
#ifndef NCL_B200_H
#define NCL_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define NCL_OK 0
#define NCL_EINVAL (-1)  /* std::invalid_argument in the reference */
#define NCL_ELOGIC (-2)  /* std::logic_error ("kkt: missing slot") */
#define NCL_ECUDA (-3)
#define NCL_ENOMEM (-4)

enum { NCL_K2 = 0, NCL_K2R = 1, NCL_K1S = 2 }; /* KktForm, kkt.hpp:22 */

/* KktOptions (kkt.hpp:27-33) */
typedef struct {
  double pivot_eps;  /* 1e-10 */
  int max_refine;    /* 10 */
  double refine_tol; /* 1e-12 */
  double delta_max;  /* 1e40 */
  double accept_tol; /* 1e-8 */
} ncl_kkt_opts;

/* KktStep scalars (kkt.hpp:48-56) */
typedef struct {
  double delta;
  int factor_attempts;
  int refine_steps;
  int perturbed_pivots;
  double rel_residual;
  int ok;
  int accepted;  /* an attempt passed the acceptance test: delta, refine_steps,
                    perturbed_pivots, rel_residual and dx/dr/dy are filled
                    (KktStep keeps them even when ok = 0 for a non-finite step,
                    kkt.cpp:291-298) */
} ncl_kkt_stats;

/* symbolic / structural facts of a context (for parity checks and roofline
 * accounting: SURVEY.md section 8(d)) */
typedef struct {
  int n;              /* KKT dimension N */
  int nnz;            /* lower nnz of K incl. diagonal */
  long long l_nnz;    /* strictly lower nnz of L (SymbolicLdl::l_nnz) */
  long long flops;    /* sum_j c_j (c_j + 2) */
  int n_supernodes;
  int sn_height;      /* supernodal elimination-tree height */
  int n_paths;        /* warp-tier heavy paths */
  int n_wide;         /* wide-tier fronts */
  int n_levels;       /* wide-tier levels */
  int max_front;
  long long npairs;   /* K1s J^T J pair contributions */
} ncl_kkt_info;

typedef struct ncl_kkt ncl_kkt;

const char* ncl_last_error(void);
int ncl_device_count(void);

/* KktContext::KktContext (kkt.hpp:60-61, kkt.cpp:41-138).  opt may be NULL
 * (defaults).  Symbolic analysis (AMD, etree, column counts, supernodes, all
 * gather maps) happens here, once. */
int ncl_kkt_create(int nt, const int* hp_ptr, const int* hp_idx, int m,
                   const int* jp_ptr, const int* jp_idx, int ns, int m_eq,
                   int form, const ncl_kkt_opts* opt, ncl_kkt** out);
void ncl_kkt_destroy(ncl_kkt* ctx);

/* KktContext::solve (kkt.hpp:65, kkt.cpp:266-314) with HOST buffers:
 * hval (nnz_H), jval (nnz_J), sigma (n), rbar1 (n), rbar2 (m), rbar3 (m) in;
 * dx (n), dr (m), dy (m) out.  n = nt + ns. */
int ncl_kkt_solve(ncl_kkt* ctx, const double* hval, const double* jval,
                  const double* sigma, const double* rbar1,
                  const double* rbar2, const double* rbar3, double rho,
                  double warm_delta, double* dx, double* dr, double* dy,
                  ncl_kkt_stats* stats);
/* Same with DEVICE pointers (inputs resident in HBM, outputs left there). */
int ncl_kkt_solve_device(ncl_kkt* ctx, const double* hval, const double* jval,
                         const double* sigma, const double* rbar1,
                         const double* rbar2, const double* rbar3, double rho,
                         double warm_delta, double* dx, double* dr, double* dy,
                         ncl_kkt_stats* stats);

int ncl_kkt_info_get(const ncl_kkt* ctx, ncl_kkt_info* info);
/* inertia_target() (kkt.cpp:140-147) */
int ncl_kkt_inertia_target(const ncl_kkt* ctx, int* tgt3);
/* symbolic analysis of the KKT pattern: perm, parent (N), lcol_ptr (N+1);
 * any pointer may be NULL.  Bit-exact with analyze() (sparse.cpp:178-180). */
int ncl_kkt_symbolic(const ncl_kkt* ctx, int* perm, int* parent,
                     int* lcol_ptr);
/* matrix(): pattern (N+1, nnz) and values of the last refill (kkt.hpp:70) */
int ncl_kkt_matrix(const ncl_kkt* ctx, int* col_ptr, int* row_ind,
                   double* val);
/* refill only (KktContext::refill, kkt.cpp:149-186), host inputs; the values
 * land in the context's K (read back with ncl_kkt_matrix). */
int ncl_kkt_refill(ncl_kkt* ctx, const double* hval, const double* jval,
                   const double* sigma, double rho, double delta);
/* last factorization in the reference layout (LdlFactors, sparse.hpp:59-68):
 * lcol_ptr (N+1), lrow_ind/lval (l_nnz), d (N), info4 = ok,n_pos,n_neg,
 * perturbed.  Test/diagnostic path (device -> host conversion). */
int ncl_kkt_factors(const ncl_kkt* ctx, int* lcol_ptr, int* lrow_ind,
                    double* lval, double* d, int* info4);
/* per-phase device time of the last solve in milliseconds:
 * [0] assembly [1] factorization [2] rhs+refined solve [3] recover, summed
 * over attempts; [4] total; [5] number of accepted solves so far */
int ncl_kkt_last_timing(const ncl_kkt* ctx, double* ms6);
int ncl_kkt_set_timing(ncl_kkt* ctx, int enable);
/* the context's CUDA stream (cudaStream_t) for event timing by callers */
int ncl_kkt_get_stream(const ncl_kkt* ctx, void** stream);
/* number of kernels this context has launched so far */
int ncl_kkt_launch_count(const ncl_kkt* ctx, long long* count);

/* ---- host-only symbolic plan (no GPU needed) ------------------------------
 * The symbolic-once half of KktContext construction (pattern, slot maps,
 * AMD, etree, column counts, supernodes, schedules), exposed for parity
 * checks on machines without a GPU. */
typedef struct ncl_plan ncl_plan;
int ncl_plan_create(int nt, const int* hp_ptr, const int* hp_idx, int m,
                    const int* jp_ptr, const int* jp_idx, int ns, int m_eq,
                    int form, ncl_plan** out);
void ncl_plan_destroy(ncl_plan* plan);
int ncl_plan_info(const ncl_plan* plan, ncl_kkt_info* info);
int ncl_plan_symbolic(const ncl_plan* plan, int* perm, int* parent,
                      int* lcol_ptr);
int ncl_plan_pattern(const ncl_plan* plan, int* col_ptr, int* row_ind);
/* Checks the invariants of the warp-tier schedule built from the plan (paths,
 * hand-out orders of the persistent kernels, light-child extend-add chunks,
 * path-position records); internal = 1: the re-postordered structure the
 * device factorization uses.  NCL_ELOGIC + ncl_last_error() on a violation.
 * Test hook, no reference counterpart. */
int ncl_plan_check_schedule(const ncl_plan* plan, int internal);
/* Builds the tile-dataflow schedules of the wide tier (one per segment of
 * wide levels, for `workers` resident workers) exactly as a context would and
 * replays them: every task runs once, in panel order per tile, without
 * deadlock.  stats4 (may be NULL): segments, tasks, simulated makespan and
 * critical path (us, summed over segments).  NCL_ELOGIC on a violation.
 * Test hook, no reference counterpart. */
int ncl_plan_check_dag(const ncl_plan* plan, int workers, double* stats4);
/* Eigen AMDOrdering<int> restated (the ordering the reference calls at
 * sparse.cpp:81-100) on a full symmetric CSC pattern with sorted rows:
 * perm[k] = node eliminated k-th.  Lets a reference build without Eigen use
 * the same ordering as this library. */
int ncl_amd_full_pattern(int n, const int* Ap, const int* Ai, int* perm);
/* analyze / analyze_with_permutation of a triplet pattern (perm_in may be
 * NULL = AMD); outputs perm, parent (n), lcol_ptr (n+1) */
int ncl_analyze_host(int n, int ntrip, const int* rows, const int* cols,
                     const int* perm_in, int* perm, int* parent,
                     int* lcol_ptr);

/* ---- sparse layer (sparse.hpp) on the same device LDL^T ---------------- */
typedef struct ncl_sparse ncl_sparse;
/* sym_from_triplets + analyze / analyze_with_permutation (perm may be NULL) */
int ncl_sparse_create(int n, int ntrip, const int* rows, const int* cols,
                      const double* vals, const int* perm, ncl_sparse** out);
void ncl_sparse_destroy(ncl_sparse* sp);
int ncl_sparse_nnz(const ncl_sparse* sp, int* nnz, long long* l_nnz);
int ncl_sparse_symbolic(const ncl_sparse* sp, int* perm, int* parent,
                        int* lcol_ptr);
/* factorize (sparse.cpp:182-256); info4 = ok, n_pos, n_neg, perturbed */
int ncl_sparse_factorize(ncl_sparse* sp, double pivot_eps, int* info4);
int ncl_sparse_factors(const ncl_sparse* sp, int* lcol_ptr, int* lrow_ind,
                       double* lval, double* d);
/* ldl_solve (sparse.cpp:258-276), host vectors */
int ncl_sparse_ldl_solve(ncl_sparse* sp, const double* b, double* x);
/* solve_refined (sparse.cpp:278-322); out: steps, rel_residual, converged */
int ncl_sparse_solve_refined(ncl_sparse* sp, const double* b, int max_ref,
                             double tol, double* x, int* steps,
                             double* rel_residual, int* converged);
/* y += A x (sparse.cpp:70-79), host vectors */
int ncl_sparse_matvec(ncl_sparse* sp, const double* x, double* y);

/* ---- fused NCL vector kernels ------------------
 * Device pointers throughout; per-element arithmetic bitwise the reference's.
 * An ncl_nlp holds the Jacobian pattern (+ its transpose) and the NLP-form
 * bounds (x = (t, s), n = nt + ns; +-inf for absent bounds). */
typedef struct ncl_nlp ncl_nlp;
int ncl_nlp_create(int nt, int ns, int m_eq, int m, const int* jp_ptr,
                   const int* jp_idx, const double* lb, const double* ub,
                   ncl_nlp** out);
void ncl_nlp_destroy(ncl_nlp* h);
int ncl_nlp_sync(ncl_nlp* h);
/* InnerSolver::solve_prepared's KktInput (ipm.cpp:184-208) */
int ncl_nlp_kkt_input(ncl_nlp* h, const double* jval, const double* grad,
                      const double* c, const double* x, const double* zl,
                      const double* zu, const double* r, const double* y,
                      const double* yk, double mu, double rho, double* sigma,
                      double* rbar1, double* rbar2, double* rbar3);
/* barrier_kkt_residual (kkt.cpp:341-366); block vectors may be NULL;
 * norm5 (host) = stat, mult, primal, compl_l, compl_u inf-norms */
int ncl_nlp_residual(ncl_nlp* h, const double* jval, const double* grad,
                     const double* c, const double* r, const double* y,
                     const double* yk, double rho, const double* x,
                     const double* zl, const double* zu, double mu,
                     double* stat, double* mult, double* primal,
                     double* compl_l, double* compl_u, double* norm5);
/* recover_bound_duals (kkt.cpp:316-328) and the fraction-to-boundary
 * minima (ipm.cpp:124-141): alpha3 (host) = primal, dual zl, dual zu */
int ncl_nlp_step(ncl_nlp* h, const double* x, const double* zl,
                 const double* zu, double mu, const double* dx, double tau,
                 double* dzl, double* dzu, double* alpha3);
/* out = v + a d (trial point / commit, ipm.cpp:267-271) */
int ncl_nlp_axpy(ncl_nlp* h, int n, const double* v, double a, const double* d,
                 double* out);
/* clip_duals (ipm.cpp:232-249), in place */
int ncl_nlp_clip_duals(ncl_nlp* h, const double* x, double mu, double* zl,
                       double* zu);
/* ||r||_inf (host out) and, if update, y_k += rho_used r (solver.cpp:213-217) */
int ncl_nlp_outer(ncl_nlp* h, const double* r, double* yk, double rho_used,
                  int update, double* rnorm);
/* outer schedule (solver.cpp:21-41) on {mu, eta, omega, rho, rho_max} */
void ncl_initial_outer_state(double mu0, double rho0, double rho_max,
                             double* state5);
int ncl_outer_update(double* state5, double rnorm);


/* ---- Schur mode: one rank's share of a block-arrowhead problem ----------
 * (SCOPF with contingency blocks; no reference counterpart --
 * the reference factors the whole KKT on one core).  The sub-problem's first
 * n0 variables couple the blocks; they are ordered last and not eliminated:
 * the factorization leaves the rank's Schur contribution
 * S_g = A00_g - sum_k A0k Akk^-1 Ak0, which the caller sums over ranks
 * (NCCL allreduce) and factors densely on every rank.  K1s form only.  All
 * vectors are DEVICE pointers; every call returns after its work finished.
 * stats4 = n_pos, n_neg, perturbed, fail. */
typedef struct ncl_schur ncl_schur;
int ncl_schur_create(int nt, const int* hp_ptr, const int* hp_idx, int m,
                     const int* jp_ptr, const int* jp_idx, int ns, int m_eq,
                     int n0, const ncl_kkt_opts* opt, ncl_schur** out);
void ncl_schur_destroy(ncl_schur* h);
int ncl_schur_info(const ncl_schur* h, ncl_kkt_info* info);
int ncl_schur_n0(const ncl_schur* h);
/* refill (kkt.cpp:149-186) + factorization of the blocks; S: n0 x n0
 * column-major, lower part = S_g, upper zero */
int ncl_schur_factor(ncl_schur* h, const double* hval, const double* jval,
                     const double* sigma, double rho, double delta,
                     int* stats4, double* S);
/* dense static-pivot LDL^T of S (+ diag_shift on its diagonal) */
int ncl_schur_factor_dense(ncl_schur* h, const double* S, double diag_shift,
                           int* stats4);
/* K1s right-hand side (kkt.cpp:188-222) of the sub-problem */
int ncl_schur_rhs(ncl_schur* h, const double* jval, const double* sigma,
                  const double* rbar1, const double* rbar2, const double* rbar3,
                  double rho, double delta, double* b);
/* forward solve through the blocks: b0 = this rank's reduced coupling rhs */
int ncl_schur_forward(ncl_schur* h, const double* b, double* b0);
/* x0 = S^-1 b0 with the dense factors */
int ncl_schur_solve0(ncl_schur* h, const double* b0, double* x0);
/* backward solve through the blocks given the coupling solution x0 */
int ncl_schur_backward(ncl_schur* h, const double* x0, double* x);
/* r = b - K_g x with the sub-problem's matrix of the last refill */
int ncl_schur_residual(ncl_schur* h, const double* x, const double* b,
                       double* r);
/* recover (kkt.cpp:224-264) of the sub-problem's rows */
int ncl_schur_recover(ncl_schur* h, const double* jval, const double* sol,
                      const double* rbar2, double rho, double delta, double* dx,
                      double* dr, double* dy);
int ncl_schur_launch_count(const ncl_schur* h, long long* count);


/* ---- init_multipliers (proj/src/solver.cpp:43-91) ------------------------
 * least-squares multiplier estimate (JJ^T + 1e-8 I [+1 on slack rows]) y =
 * J grad, clipped to +-1e3, HOST buffers.  Same triplets as the reference's
 * all-pairs loop (nonzero dots only, bit-identical values), found from the
 * rows sharing a column instead of all m^2 pairs; factored on the device with
 * eps = 1e-14, unrefined solve.  seconds4 (optional): candidate pairs, device
 * dots, symbolic analysis, numeric factor+solve. */
int ncl_init_multipliers(int m, int m_eq, int nt, const int* jp_ptr,
                         const int* jp_idx, const double* jval,
                         const double* grad, double* y, double* seconds4);
/* host-only: the candidate pairs (i, j <= i sharing a column, ascending);
 * count always set, pairs written when cap >= count */
int ncl_jjt_candidates(int m, int nt, const int* jp_ptr, const int* jp_idx,
                       long long cap, long long* count, int* pi, int* pj);

#ifdef __cplusplus
}
#endif
#endif
