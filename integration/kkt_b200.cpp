// Drop-in KktContext over the B200 C ABI (include/ncl_b200.h).  Replaces
// proj/src/kkt.cpp in a reference build; see INTEGRATION.md.
//
// recover_bound_duals / barrier_kkt_residual keep the reference's host
// expressions (kkt.cpp:316-366) so a host-resident driver sees bitwise the
// reference's residuals; their device counterparts (ncl_nlp_*) serve a
// device-resident driver.
#include <ncl/kkt.hpp>

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>

#include "../include/ncl_b200.h"

namespace ncl {

KktForm parse_kkt_form(const std::string& name) {
  if (name == "k2") return KktForm::K2;
  if (name == "k2r") return KktForm::K2r;
  if (name == "k1s") return KktForm::K1s;
  throw std::invalid_argument("unknown kkt form: " + name);
}

const char* kkt_form_name(KktForm f) {
  switch (f) {
    case KktForm::K2: return "k2";
    case KktForm::K2r: return "k2r";
    case KktForm::K1s: return "k1s";
  }
  return "?";
}

namespace {

[[noreturn]] void rethrow(int rc, const char* what) {
  const std::string msg = std::string(what) + ": " + ncl_last_error();
  if (rc == NCL_EINVAL) throw std::invalid_argument(msg);
  if (rc == NCL_ELOGIC) throw std::logic_error(msg);
  throw std::runtime_error(msg);
}

int form_code(KktForm f) {
  return f == KktForm::K2 ? NCL_K2 : (f == KktForm::K2r ? NCL_K2R : NCL_K1S);
}

double inf_norm_or_zero(const dvec& v) {
  return v.size() ? v.lpNorm<Eigen::Infinity>() : 0.0;
}

}  // namespace

KktContext::KktContext(const HessianPattern& hp, const JacobianPattern& jp, int nt, int ns,
                       int m_eq, KktForm form, KktOptions opt)
    : form_(form), nt_(nt), ns_(ns), n_(nt + ns), m_(jp.rows) {
  if (hp.n != nt || jp.cols != nt || jp.rows - m_eq != ns)
    throw std::invalid_argument("kkt: inconsistent problem shape");
  ncl_kkt_opts o{opt.pivot_eps, opt.max_refine, opt.refine_tol, opt.delta_max, opt.accept_tol};
  const int rc = ncl_kkt_create(nt, hp.ptr.data(), hp.idx.data(), jp.rows, jp.ptr.data(),
                                jp.idx.data(), ns, m_eq, form_code(form), &o, &h_);
  if (rc) rethrow(rc, "KktContext");
  ncl_kkt_info info;
  ncl_kkt_info_get(h_, &info);
  n_sys_ = info.n;
}

KktContext::~KktContext() { ncl_kkt_destroy(h_); }

std::array<int, 3> KktContext::inertia_target() const {
  int t[3];
  ncl_kkt_inertia_target(h_, t);
  return {t[0], t[1], t[2]};
}

const SparseSymMatrix& KktContext::matrix() const {
  if (mat_stale_) {
    ncl_kkt_info info;
    ncl_kkt_info_get(h_, &info);
    mat_.n = info.n;
    mat_.col_ptr.assign(static_cast<size_t>(info.n) + 1, 0);
    mat_.row_ind.assign(static_cast<size_t>(info.nnz), 0);
    mat_.val.assign(static_cast<size_t>(info.nnz), 0.0);
    const int rc = ncl_kkt_matrix(h_, mat_.col_ptr.data(), mat_.row_ind.data(), mat_.val.data());
    if (rc) rethrow(rc, "KktContext::matrix");
    mat_stale_ = false;
  }
  return mat_;
}

KktStep KktContext::solve(const KktInput& in, double warm_delta) {
  KktStep st;
  dvec dx(n_), dr(m_), dy(m_);
  ncl_kkt_stats s{};
  const int rc = ncl_kkt_solve(h_, in.hval->data(), in.jval->data(), in.sigma.data(),
                               in.rbar1.data(), in.rbar2.data(), in.rbar3.data(), in.rho,
                               warm_delta, dx.data(), dr.data(), dy.data(), &s);
  if (rc) rethrow(rc, "KktContext::solve");
  mat_stale_ = true;
  st.factor_attempts = s.factor_attempts;
  st.ok = s.ok != 0;
  if (s.accepted) {  // kkt.cpp:291-298: every field of an accepted attempt, finite or not
    st.delta = s.delta;
    st.refine_steps = s.refine_steps;
    st.perturbed_pivots = s.perturbed_pivots;
    st.rel_residual = s.rel_residual;
    st.dx = std::move(dx);
    st.dr = std::move(dr);
    st.dy = std::move(dy);
  }
  return st;
}

void recover_bound_duals(const dvec& x, const dvec& lb, const dvec& ub, const dvec& zl,
                         const dvec& zu, double mu, const dvec& dx, dvec& dzl, dvec& dzu) {
  const int n = static_cast<int>(x.size());
  dzl = dvec::Zero(n);
  dzu = dvec::Zero(n);
  for (int i = 0; i < n; ++i) {
    if (std::isfinite(lb[i])) dzl[i] = -(zl[i] * dx[i] - mu) / (x[i] - lb[i]) - zl[i];
    if (std::isfinite(ub[i])) dzu[i] = (zu[i] * dx[i] + mu) / (ub[i] - x[i]) - zu[i];
  }
}

double ResidualParts::stat_norm() const { return inf_norm_or_zero(stat); }
double ResidualParts::mult_norm() const { return inf_norm_or_zero(mult); }
double ResidualParts::primal_norm() const { return inf_norm_or_zero(primal); }
double ResidualParts::compl_l_norm() const { return inf_norm_or_zero(compl_l); }
double ResidualParts::compl_u_norm() const { return inf_norm_or_zero(compl_u); }

double ResidualParts::inf_norm() const {
  return std::max({stat_norm(), mult_norm(), primal_norm(), compl_l_norm(), compl_u_norm()});
}

ResidualParts barrier_kkt_residual(const dvec& grad_phi, const std::vector<double>& jval,
                                   const JacobianPattern& jp, int ns, const dvec& c,
                                   const dvec& r, const dvec& y, const dvec& yk, double rho,
                                   const dvec& x, const dvec& lb, const dvec& ub, const dvec& zl,
                                   const dvec& zu, double mu) {
  const int nt = jp.cols, m = jp.rows;
  const int m_eq = m - ns;
  ResidualParts res;
  res.stat = grad_phi - zl + zu;
  for (int i = 0; i < m; ++i)
    for (int p = jp.ptr[i]; p < jp.ptr[i + 1]; ++p) res.stat[jp.idx[p]] -= jval[p] * y[i];
  for (int k = 0; k < ns; ++k) res.stat[nt + k] += y[m_eq + k];
  res.mult = yk + rho * r - y;
  res.primal = c + r;
  const int n = static_cast<int>(x.size());
  res.compl_l = dvec::Zero(n);
  res.compl_u = dvec::Zero(n);
  for (int i = 0; i < n; ++i) {
    if (std::isfinite(lb[i])) res.compl_l[i] = zl[i] * (x[i] - lb[i]) - mu;
    if (std::isfinite(ub[i])) res.compl_u[i] = zu[i] * (ub[i] - x[i]) - mu;
  }
  return res;
}

}  // namespace ncl
