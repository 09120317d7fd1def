// harness_impl.hpp -- extern "C" surface over a build of the reference's
// driver (proj/src): instance construction (instances.hpp), the KktContext,
// the sparse layer and full NCL solves with their iteration logs.
//
// Included twice, with different NCL_HARNESS_PREFIX:
//   oracle/ref_harness.cpp  (ref_)  -> oracle/_ref/libncl_ref.so, the
//       reference compiled unmodified: the CPU oracle / baseline;
//   integration/harness.cpp (drop_) -> integration/_build/libncl_drop.so, the
//       same driver with the B200 KktContext dropped in.
#ifndef NCL_HARNESS_PREFIX
#error "define NCL_HARNESS_PREFIX"
#endif
#define NCL_CAT2(a, b) a##b
#define NCL_CAT(a, b) NCL_CAT2(a, b)
#define NCL_H(name) NCL_CAT(NCL_HARNESS_PREFIX, name)

#include <chrono>
#include <cstring>
#include <exception>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include <ncl/ipm.hpp>
#include <ncl/kkt.hpp>
#include <ncl/model.hpp>
#include <ncl/problems.hpp>
#include <ncl/solver.hpp>
#include <ncl/sparse.hpp>

#include "instances.hpp"

using namespace ncl;

namespace {

struct ModelH {
  std::unique_ptr<Model> m;
  NlpForm f;
};

struct KktH {
  std::unique_ptr<KktContext> ctx;
  HessianPattern hp;
  JacobianPattern jp;
  std::vector<double> hv, jv;
};

struct SparseH {
  SparseSymMatrix A;
  SymbolicLdl S;
  LdlFactors F;
};

struct ReportH {
  SolveReport rep;
  double init_mult_seconds = 0.0;
};

KktOptions opts_from(const double* o) {
  KktOptions k;
  if (o) {
    k.pivot_eps = o[0];
    k.max_refine = static_cast<int>(o[1]);
    k.refine_tol = o[2];
    k.delta_max = o[3];
    k.accept_tol = o[4];
  }
  return k;
}

KktForm form_of(int f) {
  return f == 0 ? KktForm::K2 : (f == 1 ? KktForm::K2r : KktForm::K1s);
}

}  // namespace

extern "C" {

void* NCL_H(model_new)(const char* spec) {
  try {
    auto* h = new ModelH;
    h->m = std::make_unique<Model>(ncl_inst::build(spec));
    h->f = to_nlp_form(*h->m);
    return h;
  } catch (const std::exception&) {
    return nullptr;
  }
}

void NCL_H(model_free)(void* p) { delete static_cast<ModelH*>(p); }

// out: nt, ns, m_eq, m, hnnz, jnnz
void NCL_H(model_dims)(void* p, int* out) {
  auto* h = static_cast<ModelH*>(p);
  out[0] = h->f.nt;
  out[1] = h->f.ns;
  out[2] = h->f.m_eq;
  out[3] = h->f.m;
  out[4] = h->m->hessian_pattern().nnz();
  out[5] = h->m->jacobian_pattern().nnz();
}

void NCL_H(model_patterns)(void* p, int* hp_ptr, int* hp_idx, int* jp_ptr,
                        int* jp_idx) {
  auto* h = static_cast<ModelH*>(p);
  const auto& hp = h->m->hessian_pattern();
  const auto& jp = h->m->jacobian_pattern();
  std::memcpy(hp_ptr, hp.ptr.data(), sizeof(int) * hp.ptr.size());
  std::memcpy(hp_idx, hp.idx.data(), sizeof(int) * hp.idx.size());
  std::memcpy(jp_ptr, jp.ptr.data(), sizeof(int) * jp.ptr.size());
  std::memcpy(jp_idx, jp.idx.data(), sizeof(int) * jp.idx.size());
}

// NLP-form bounds (n) and model start (nt)
void NCL_H(model_bounds)(void* p, double* lb, double* ub, double* start) {
  auto* h = static_cast<ModelH*>(p);
  for (int i = 0; i < h->f.n; ++i) {
    lb[i] = h->f.lb[i];
    ub[i] = h->f.ub[i];
  }
  for (int i = 0; i < h->f.nt; ++i) start[i] = h->m->start()[i];
}

// Derivative values at t (nt) with multipliers y (m): hval (obj_scale 1),
// jval, gradient (nt), constraints (m).
void NCL_H(model_eval)(void* p, const double* t, const double* y, double* hval,
                    double* jval, double* grad, double* c) {
  auto* h = static_cast<ModelH*>(p);
  auto ws = h->m->make_workspace();
  dvec tv(h->f.nt), yv(h->f.m);
  for (int i = 0; i < h->f.nt; ++i) tv[i] = t[i];
  for (int i = 0; i < h->f.m; ++i) yv[i] = y[i];
  std::vector<double> hv, jv;
  h->m->eval_lag_hessian(tv, 1.0, yv, ws, hv);
  h->m->eval_jacobian(tv, ws, jv);
  dvec g, cv;
  h->m->eval_gradient(tv, ws, g);
  h->m->eval_constraints(tv, ws, cv);
  std::memcpy(hval, hv.data(), sizeof(double) * hv.size());
  std::memcpy(jval, jv.data(), sizeof(double) * jv.size());
  for (int i = 0; i < h->f.nt; ++i) grad[i] = g[i];
  for (int i = 0; i < h->f.m; ++i) c[i] = cv[i];
}

// proj/tests/test_kkt.cpp:40-68 ("from_model") recipe
void NCL_H(kkt_case)(void* p, unsigned seed, double* hval, double* jval,
                  double* sigma, double* r1, double* r2, double* r3) {
  auto* h = static_cast<ModelH*>(p);
  const NlpForm& f = h->f;
  auto ws = h->m->make_workspace();
  std::mt19937_64 gen(seed);
  auto uni = [&](double lo, double hi) {
    const double u = static_cast<double>(gen() >> 11) * 0x1.0p-53;
    return lo + (hi - lo) * u;
  };
  dvec t = h->m->start();
  for (int i = 0; i < t.size(); ++i) t[i] += uni(-0.05, 0.05);
  dvec y(f.m);
  for (int i = 0; i < f.m; ++i) y[i] = uni(-0.01, 0.01);
  std::vector<double> hv, jv;
  h->m->eval_lag_hessian(t, 1.0, y, ws, hv);
  h->m->eval_jacobian(t, ws, jv);
  std::memcpy(hval, hv.data(), sizeof(double) * hv.size());
  std::memcpy(jval, jv.data(), sizeof(double) * jv.size());
  for (int i = 0; i < f.n; ++i) sigma[i] = uni(0.5, 2.0);
  for (int i = 0; i < f.n; ++i) r1[i] = uni(-1.0, 1.0);
  for (int i = 0; i < f.m; ++i) r2[i] = uni(-1.0, 1.0);
  for (int i = 0; i < f.m; ++i) r3[i] = uni(-1.0, 1.0);
}

// KktContext of the reference (kkt.cpp) on raw patterns
void* NCL_H(kkt_new)(int nt, const int* hp_ptr, const int* hp_idx, int m,
                  const int* jp_ptr, const int* jp_idx, int ns, int m_eq,
                  int form, const double* opts5) {
  try {
    auto* h = new KktH;
    h->hp.n = nt;
    h->hp.ptr.assign(hp_ptr, hp_ptr + nt + 1);
    h->hp.idx.assign(hp_idx, hp_idx + hp_ptr[nt]);
    h->jp.rows = m;
    h->jp.cols = nt;
    h->jp.ptr.assign(jp_ptr, jp_ptr + m + 1);
    h->jp.idx.assign(jp_idx, jp_idx + jp_ptr[m]);
    h->ctx = std::make_unique<KktContext>(h->hp, h->jp, nt, ns, m_eq,
                                          form_of(form), opts_from(opts5));
    return h;
  } catch (const std::exception&) {
    return nullptr;
  }
}

void NCL_H(kkt_free)(void* p) { delete static_cast<KktH*>(p); }
int NCL_H(kkt_size)(void* p) { return static_cast<KktH*>(p)->ctx->system_size(); }
int NCL_H(kkt_nnz)(void* p) { return static_cast<KktH*>(p)->ctx->matrix().nnz(); }

void NCL_H(kkt_matrix)(void* p, int* col_ptr, int* row_ind, double* val) {
  const auto& A = static_cast<KktH*>(p)->ctx->matrix();
  if (col_ptr) std::memcpy(col_ptr, A.col_ptr.data(), sizeof(int) * A.col_ptr.size());
  if (row_ind) std::memcpy(row_ind, A.row_ind.data(), sizeof(int) * A.row_ind.size());
  if (val) std::memcpy(val, A.val.data(), sizeof(double) * A.val.size());
}

// stats6: delta, attempts, refine_steps, perturbed, rel_residual, ok
int NCL_H(kkt_solve_n)(void* p, int n, const double* hval, const double* jval,
                    const double* sigma, const double* r1, const double* r2,
                    const double* r3, double rho, double warm, double* dx,
                    double* dr, double* dy, double* stats6) {
  auto* h = static_cast<KktH*>(p);
  const int nt = h->hp.n, m = h->jp.rows;
  h->hv.assign(hval, hval + h->hp.ptr[nt]);
  h->jv.assign(jval, jval + h->jp.ptr[m]);
  KktInput in;
  in.hval = &h->hv;
  in.jval = &h->jv;
  in.rho = rho;
  in.sigma.resize(n);
  in.rbar1.resize(n);
  in.rbar2.resize(m);
  in.rbar3.resize(m);
  for (int i = 0; i < n; ++i) {
    in.sigma[i] = sigma[i];
    in.rbar1[i] = r1[i];
  }
  for (int i = 0; i < m; ++i) {
    in.rbar2[i] = r2[i];
    in.rbar3[i] = r3[i];
  }
  const KktStep st = h->ctx->solve(in, warm);
  for (int i = 0; i < st.dx.size(); ++i) dx[i] = st.dx[i];
  for (int i = 0; i < st.dr.size(); ++i) dr[i] = st.dr[i];
  for (int i = 0; i < st.dy.size(); ++i) dy[i] = st.dy[i];
  stats6[0] = st.delta;
  stats6[1] = st.factor_attempts;
  stats6[2] = st.refine_steps;
  stats6[3] = st.perturbed_pivots;
  stats6[4] = st.rel_residual;
  stats6[5] = st.ok ? 1.0 : 0.0;
  return 0;
}

// ---- sparse layer (sparse.cpp) ---------------------------------------------
void* NCL_H(sparse_new)(int n, int nt, const int* rows, const int* cols,
                     const double* vals, const int* perm_or_null) {
  try {
    auto* h = new SparseH;
    h->A = sym_from_triplets(n, std::vector<int>(rows, rows + nt),
                             std::vector<int>(cols, cols + nt),
                             std::vector<double>(vals, vals + nt));
    if (perm_or_null)
      h->S = analyze_with_permutation(h->A,
                                      std::vector<int>(perm_or_null, perm_or_null + n));
    else
      h->S = analyze(h->A);
    return h;
  } catch (const std::exception&) {
    return nullptr;
  }
}
void NCL_H(sparse_free)(void* p) { delete static_cast<SparseH*>(p); }
int NCL_H(sparse_nnz)(void* p) { return static_cast<SparseH*>(p)->A.nnz(); }
int NCL_H(sparse_lnz)(void* p) { return static_cast<SparseH*>(p)->S.l_nnz(); }
void NCL_H(sparse_matrix)(void* p, int* col_ptr, int* row_ind, double* val) {
  const auto& A = static_cast<SparseH*>(p)->A;
  std::memcpy(col_ptr, A.col_ptr.data(), sizeof(int) * A.col_ptr.size());
  std::memcpy(row_ind, A.row_ind.data(), sizeof(int) * A.row_ind.size());
  std::memcpy(val, A.val.data(), sizeof(double) * A.val.size());
}
void NCL_H(sparse_symbolic)(void* p, int* perm, int* parent, int* lcol_ptr,
                         int* a_map) {
  const auto& S = static_cast<SparseH*>(p)->S;
  std::memcpy(perm, S.perm.data(), sizeof(int) * S.perm.size());
  std::memcpy(parent, S.parent.data(), sizeof(int) * S.parent.size());
  std::memcpy(lcol_ptr, S.lcol_ptr.data(), sizeof(int) * S.lcol_ptr.size());
  std::memcpy(a_map, S.a_map.data(), sizeof(int) * S.a_map.size());
}
// info4: ok, n_pos, n_neg, perturbed
void NCL_H(sparse_factorize)(void* p, double eps, int* info4, int* lrow_ind,
                          double* lval, double* d) {
  auto* h = static_cast<SparseH*>(p);
  h->F = factorize(h->S, h->A, eps);
  info4[0] = h->F.ok;
  info4[1] = h->F.n_pos;
  info4[2] = h->F.n_neg;
  info4[3] = h->F.perturbed;
  if (lrow_ind)
    std::memcpy(lrow_ind, h->F.lrow_ind.data(), sizeof(int) * h->F.lrow_ind.size());
  if (lval) std::memcpy(lval, h->F.lval.data(), sizeof(double) * h->F.lval.size());
  if (d) std::memcpy(d, h->F.d.data(), sizeof(double) * h->F.d.size());
}
// returns steps; out2: rel_residual, converged
int NCL_H(sparse_solve_refined)(void* p, const double* b, int max_ref,
                             double tol, double* x, double* out2) {
  auto* h = static_cast<SparseH*>(p);
  const int n = h->A.n;
  const RefineResult r = solve_refined(h->S, h->F, h->A,
                                       std::vector<double>(b, b + n), max_ref, tol);
  std::memcpy(x, r.x.data(), sizeof(double) * n);
  out2[0] = r.rel_residual;
  out2[1] = r.converged ? 1.0 : 0.0;
  return r.steps;
}
void NCL_H(sparse_ldl_solve)(void* p, const double* b, double* x) {
  auto* h = static_cast<SparseH*>(p);
  ldl_solve(h->S, h->F, b, x);
}

// ---- full NCL solve (solver.cpp) ------------------------------------------
void* NCL_H(solve)(void* model, int form, double tol, int max_outer,
                int max_inner, double pivot_eps, int scaling) {
  auto* mh = static_cast<ModelH*>(model);
  SolverOptions o;
  o.kkt_form = form_of(form);
  o.tol = tol;
  o.max_outer = max_outer;
  o.max_inner = max_inner;
  o.pivot_eps = pivot_eps;
  o.scaling = scaling != 0;
  auto* r = new ReportH;
  r->rep = ncl::solve(*mh->m, o);
  return r;
}
void NCL_H(report_free)(void* p) { delete static_cast<ReportH*>(p); }
// out12: status, outer, inner, extrap_accepts, objective, kkt_residual,
// primal_feas, mu_final, rho_final, solve_seconds, nlog, n_extrap
void NCL_H(report_scalars)(void* p, double* out) {
  const auto& r = static_cast<ReportH*>(p)->rep;
  out[0] = static_cast<double>(static_cast<int>(r.status));
  out[1] = r.outer_iters;
  out[2] = r.inner_iters;
  out[3] = r.extrapolation_accepts;
  out[4] = r.objective;
  out[5] = r.kkt_residual;
  out[6] = r.primal_feas;
  out[7] = r.mu_final;
  out[8] = r.rho_final;
  out[9] = r.solve_seconds;
  out[10] = static_cast<double>(r.log.size());
  out[11] = static_cast<double>(r.extrap_alpha.size());
}
// 13 columns per row: k_outer k_inner f_stat f_mult f_primal f_compl_l
// f_compl_u mu rho delta alpha refine_steps perturbed_pivots
void NCL_H(report_log)(void* p, double* rows, double* extrap_alpha) {
  const auto& r = static_cast<ReportH*>(p)->rep;
  for (size_t k = 0; k < r.log.size(); ++k) {
    const LogRow& l = r.log[k];
    double* o = rows + 13 * k;
    o[0] = l.k_outer;
    o[1] = l.k_inner;
    o[2] = l.f_stat;
    o[3] = l.f_mult;
    o[4] = l.f_primal;
    o[5] = l.f_compl_l;
    o[6] = l.f_compl_u;
    o[7] = l.mu;
    o[8] = l.rho;
    o[9] = l.delta;
    o[10] = l.alpha;
    o[11] = l.refine_steps;
    o[12] = l.perturbed_pivots;
  }
  for (size_t k = 0; k < r.extrap_alpha.size(); ++k)
    extrap_alpha[k] = r.extrap_alpha[k];
}
// final iterate, unscaled: x (n), y (m)
void NCL_H(report_xy)(void* p, double* x, double* y) {
  const auto& r = static_cast<ReportH*>(p)->rep;
  for (int i = 0; i < r.x.size(); ++i) x[i] = r.x[i];
  for (int i = 0; i < r.y.size(); ++i) y[i] = r.y[i];
}

// init_multipliers timing split (solver.cpp:43-91), seconds
double NCL_H(time_init_multipliers)(void* model) {
  auto* mh = static_cast<ModelH*>(model);
  ScaledProblem sp(*mh->m, true);
  const auto t0 = std::chrono::steady_clock::now();
  IterState s = initial_state(sp, 0.1);
  (void)s;
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0)
      .count();
}

}  // extern "C"
