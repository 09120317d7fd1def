/*
 * ncl_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C11) of the reference's Newton-step hot path, used as
 * the parity checker for the sm_100a implementation.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library.  The product (paper_2510_05885_b200/) never links it.
 *
 * Every function cites the reference file:line it restates
 * (/root/reference/proj/...).  Third-party arithmetic restated here:
 *   Eigen 3 AMDOrdering<int> (Eigen/src/OrderingMethods/Amd.h, a port of
 *   CSparse cs_amd with the structural-diagonal rule), version unpinned by the
 *   reference (proj/CMakeLists.txt:14); called at proj/src/sparse.cpp:81-100.
 *
 * Parity pinning: tests/test_oracle_kat.py checks this restatement against
 * every known-answer test of proj/tests/test_sparse.cpp, test_kkt.cpp,
 * test_ipm.cpp and test_solver.cpp, and (when oracle/_ref was built from the
 * reference sources in this container) against the reference itself on
 * seeded inputs -- see tests/golden/make_golden.py.
 */
#ifndef NCL_ORACLE_H
#define NCL_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

/* ---- sparse layer: proj/src/sparse.cpp ---------------------------------- */

/* Lower-CSC symmetric matrix (sparse.hpp:15-22). */
typedef struct {
  int n;
  int nnz;
  int* col_ptr; /* n+1 */
  int* row_ind; /* nnz */
  double* val;  /* nnz */
} orc_csc;

typedef struct {
  int n;
  int* perm;      /* perm[k] = original index eliminated k-th */
  int* iperm;
  int* parent;    /* etree of permuted pattern */
  int* lcol_ptr;  /* n+1 */
  int* a_col_ptr; /* n+1: permuted upper pattern by column */
  int* a_row_ind; /* nnz */
  int* a_map;     /* nnz: orig slot -> permuted slot */
  int nnz;
} orc_symbolic;

typedef struct {
  int n;
  int ok;
  int* lcol_ptr;
  int* lrow_ind;
  double* lval;
  double* d;
  int n_pos, n_neg, n_zero, perturbed;
  double pivot_eps;
} orc_factors;

/* returns 0, or -1 on invalid input (reference throws invalid_argument) */
int orc_sym_from_triplets(int n, int nt, const int* rows, const int* cols,
                          const double* vals, orc_csc* out);
void orc_csc_free(orc_csc* A);
void orc_sym_matvec(const orc_csc* A, const double* x, double* y);
int orc_amd_order(const orc_csc* A, int* perm);
/* Eigen-style entry used by the Eigen shim: full symmetric CSC pattern. */
int orc_amd_full_pattern(int n, const int* Ap, const int* Ai, int* perm);
int orc_analyze_with_permutation(const orc_csc* A, const int* perm,
                                 orc_symbolic* S);
int orc_analyze(const orc_csc* A, orc_symbolic* S);
void orc_symbolic_free(orc_symbolic* S);
int orc_factorize(const orc_symbolic* S, const orc_csc* A, double pivot_eps,
                  orc_factors* F);
void orc_factors_free(orc_factors* F);
void orc_ldl_solve(const orc_symbolic* S, const orc_factors* F,
                   const double* b, double* x);
/* x (n) out; returns steps; rel_residual/converged via pointers */
int orc_solve_refined(const orc_symbolic* S, const orc_factors* F,
                      const orc_csc* A, const double* b, int max_ref,
                      double tol, double* x, double* rel_residual,
                      int* converged);

/* ---- KKT layer: proj/src/kkt.cpp ----------------------------------------- */

enum { ORC_K2 = 0, ORC_K2R = 1, ORC_K1S = 2 };

typedef struct {
  double pivot_eps;  /* 1e-10 */
  int max_refine;    /* 10 */
  double refine_tol; /* 1e-12 */
  double delta_max;  /* 1e40 */
  double accept_tol; /* 1e-8 */
} orc_kkt_opts;

typedef struct {
  double delta;
  int factor_attempts;
  int refine_steps;
  int perturbed_pivots;
  double rel_residual;
  int ok;
} orc_kkt_stats;

typedef struct orc_kkt orc_kkt;

/* hp: lower CSC (n=nt); jp: CSR rows x nt.  Returns NULL on invalid shape. */
orc_kkt* orc_kkt_create(int nt, const int* hp_ptr, const int* hp_idx,
                        int m, const int* jp_ptr, const int* jp_idx,
                        int ns, int m_eq, int form, const orc_kkt_opts* opt);
void orc_kkt_destroy(orc_kkt* K);
int orc_kkt_system_size(const orc_kkt* K);
int orc_kkt_nnz(const orc_kkt* K);
void orc_kkt_inertia_target(const orc_kkt* K, int* tgt3);
/* copies of the pattern / last refilled values / symbolic analysis */
void orc_kkt_matrix(const orc_kkt* K, int* col_ptr, int* row_ind, double* val);
const orc_symbolic* orc_kkt_symbolic(const orc_kkt* K);
void orc_kkt_slots(const orc_kkt* K, int* h_slot, int* diag_slot,
                   int* pair_or_j_slot, int* slack_slot, int* ydiag_slot);
int orc_kkt_num_pairs(const orc_kkt* K);
/* refill only (for bit-exact assembly checks) */
void orc_kkt_refill(orc_kkt* K, const double* hval, const double* jval,
                    const double* sigma, double rho, double delta);
void orc_kkt_build_rhs(const orc_kkt* K, const double* jval,
                       const double* sigma, const double* rbar1,
                       const double* rbar2, const double* rbar3, double rho,
                       double delta, double* rhs);
int orc_kkt_solve(orc_kkt* K, const double* hval, const double* jval,
                  const double* sigma, const double* rbar1,
                  const double* rbar2, const double* rbar3, double rho,
                  double warm_delta, double* dx, double* dr, double* dy,
                  orc_kkt_stats* st);
/* last factorization (valid after a solve/factor attempt) */
const orc_factors* orc_kkt_last_factors(const orc_kkt* K);

/* ---- NCL vector kernels: kkt.cpp:316-366, ipm.cpp:124-141,180-212,232-249,
 *      solver.cpp:21-41 ------------------------------------------------------ */

void orc_recover_bound_duals(int n, const double* x, const double* lb,
                             const double* ub, const double* zl,
                             const double* zu, double mu, const double* dx,
                             double* dzl, double* dzu);
/* out5 = {stat, mult, primal, compl_l, compl_u} inf-norms; block vectors
 * optional (may be NULL). */
void orc_barrier_kkt_residual(int nt, int ns, int m, const int* jp_ptr,
                              const int* jp_idx, const double* jval,
                              const double* grad_phi, const double* c,
                              const double* r, const double* y,
                              const double* yk, double rho, const double* x,
                              const double* lb, const double* ub,
                              const double* zl, const double* zu, double mu,
                              double* stat, double* mult, double* primal,
                              double* compl_l, double* compl_u, double* out5);
double orc_fraction_to_boundary(int n, const double* x, const double* lb,
                                const double* ub, const double* dx,
                                double tau);
double orc_dual_fraction_to_boundary(int n, const double* z, const double* dz,
                                     double tau);
void orc_clip_duals(int n, const double* x, const double* lb,
                    const double* ub, double mu, double* zl, double* zu);
/* KktInput formation of solve_prepared (ipm.cpp:180-212) */
void orc_kkt_input(int nt, int ns, int m, const int* jp_ptr,
                   const int* jp_idx, const double* jval, const double* grad,
                   const double* c, const double* x, const double* lb,
                   const double* ub, const double* zl, const double* zu,
                   const double* r, const double* y, const double* yk,
                   double mu, double rho, double* sigma, double* rbar1,
                   double* rbar2, double* rbar3);
/* outer schedule (solver.cpp:21-41); state = {mu, eta, omega, rho, rho_max} */
void orc_initial_outer_state(double mu0, double rho0, double rho_max,
                             double* state5);
int orc_outer_update(double* state5, double rnorm);
/* (J J^T + 1e-8 I [+1 slack rows]) y = J g (solver.cpp:43-91) */
void orc_init_multipliers(int m, int m_eq, const int* jp_ptr,
                          const int* jp_idx, const double* jval,
                          const double* g, double* y);

#ifdef __cplusplus
}
#endif
#endif
