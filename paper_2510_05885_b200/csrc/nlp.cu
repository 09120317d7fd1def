// C ABI of the fused NCL vector kernels (ncl_vec.cu): the per-iteration work
// of the IPM / NCL loop around the KKT solve, on device-resident vectors.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <memory>
#include <vector>

#include "../../include/ncl_b200.h"
#include "cuda_util.hpp"

namespace nclb {

struct NlpDev {
  int nt, ns, n, m_eq, m;
  const int* jp_ptr;
  const int* jp_idx;
  const int* jt_ptr;
  const int* jt_row;
  const int* jt_slot;
  const double* lb;
  const double* ub;
};

void launch_kkt_input(const NlpDev& P, const double* jval, const double* grad, const double* c,
                      const double* x, const double* zl, const double* zu, const double* r,
                      const double* y, const double* yk, double mu, double rho, double* sigma,
                      double* rbar1, double* rbar2, double* rbar3, cudaStream_t st);
void launch_nlp_residual(const NlpDev& P, const double* jval, const double* grad, const double* c,
                         const double* r, const double* y, const double* yk, double rho,
                         const double* x, const double* zl, const double* zu, double mu,
                         double* stat, double* mult, double* primal, double* cl, double* cu,
                         double* norm5, cudaStream_t st);
void launch_nlp_step(const NlpDev& P, const double* x, const double* zl, const double* zu,
                     double mu, const double* dx, double tau, double* dzl, double* dzu,
                     double* alpha3, cudaStream_t st);
void launch_axpy(int n, const double* v, double a, const double* d, double* out, cudaStream_t st);
void launch_clip(const NlpDev& P, const double* x, double mu, double* zl, double* zu,
                 cudaStream_t st);
void launch_outer(int m, const double* r, double* yk, double rho_used, int update, double* norm,
                  cudaStream_t st);

class NlpSystem {
 public:
  NlpSystem(int nt, int ns, int m_eq, int m, const int* jp_ptr, const int* jp_idx,
            const double* lb, const double* ub) {
    if (nt < 0 || ns < 0 || m_eq < 0 || m - m_eq != ns)
      throw std::invalid_argument("nlp: inconsistent problem shape");
    const int n = nt + ns;
    std::vector<int> jpp(jp_ptr, jp_ptr + m + 1), jpi(jp_idx, jp_idx + jp_ptr[m]);
    for (int i = 0; i < m; ++i)
      for (int p = jpp[i]; p < jpp[i + 1]; ++p)
        if (jpi[p] < 0 || jpi[p] >= nt) throw std::invalid_argument("nlp: jacobian column out of range");
    std::vector<int> jtp(static_cast<size_t>(nt) + 1, 0), jtr(jpi.size()), jts(jpi.size());
    for (int p = 0; p < jpp[m]; ++p) jtp[jpi[p] + 1]++;
    for (int c = 0; c < nt; ++c) jtp[c + 1] += jtp[c];
    std::vector<int> nx(jtp.begin(), jtp.end() - 1);
    for (int i = 0; i < m; ++i)
      for (int p = jpp[i]; p < jpp[i + 1]; ++p) {
        const int q = nx[jpi[p]]++;
        jtr[q] = i;
        jts[q] = p;
      }
    CK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    jp_ptr_.upload(jpp);
    jp_idx_.upload(jpi);
    jt_ptr_.upload(jtp);
    jt_row_.upload(jtr);
    jt_slot_.upload(jts);
    lb_.upload(std::vector<double>(lb, lb + n));
    ub_.upload(std::vector<double>(ub, ub + n));
    red_.alloc(8);
    CK(cudaMallocHost(&hred_, 8 * sizeof(double)));
    P_ = {nt, ns, n, m_eq, m, jp_ptr_.p, jp_idx_.p, jt_ptr_.p, jt_row_.p, jt_slot_.p, lb_.p, ub_.p};
    CK(cudaStreamSynchronize(st_));
  }
  ~NlpSystem() {
    if (hred_) cudaFreeHost(hred_);
    if (st_) cudaStreamDestroy(st_);
  }
  const NlpDev& P() const { return P_; }
  cudaStream_t st() const { return st_; }
  double* red() { return red_.p; }
  double* hred() { return hred_; }
  void fetch(int k) {
    CK(cudaMemcpyAsync(hred_, red_.p, k * sizeof(double), cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
  }

 private:
  NlpDev P_{};
  cudaStream_t st_ = nullptr;
  DBuf<int> jp_ptr_, jp_idx_, jt_ptr_, jt_row_, jt_slot_;
  DBuf<double> lb_, ub_, red_;
  double* hred_ = nullptr;
};

}  // namespace nclb

struct ncl_nlp {
  std::unique_ptr<nclb::NlpSystem> sys;
};

using nclb::guard;

extern "C" {

int ncl_nlp_create(int nt, int ns, int m_eq, int m, const int* jp_ptr, const int* jp_idx,
                   const double* lb, const double* ub, ncl_nlp** out) {
  if (!out || !jp_ptr || !lb || !ub) return NCL_EINVAL;
  *out = nullptr;
  return guard([&] {
    auto* h = new ncl_nlp;
    try {
      h->sys = std::make_unique<nclb::NlpSystem>(nt, ns, m_eq, m, jp_ptr, jp_idx, lb, ub);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void ncl_nlp_destroy(ncl_nlp* h) { delete h; }

int ncl_nlp_sync(ncl_nlp* h) {
  if (!h) return NCL_EINVAL;
  return guard([&] { CK(cudaStreamSynchronize(h->sys->st())); });
}

int ncl_nlp_kkt_input(ncl_nlp* h, const double* jval, const double* grad, const double* c,
                      const double* x, const double* zl, const double* zu, const double* r,
                      const double* y, const double* yk, double mu, double rho, double* sigma,
                      double* rbar1, double* rbar2, double* rbar3) {
  if (!h) return NCL_EINVAL;
  return guard([&] {
    nclb::launch_kkt_input(h->sys->P(), jval, grad, c, x, zl, zu, r, y, yk, mu, rho, sigma, rbar1,
                           rbar2, rbar3, h->sys->st());
    CK(cudaGetLastError());
  });
}

int ncl_nlp_residual(ncl_nlp* h, const double* jval, const double* grad, const double* c,
                     const double* r, const double* y, const double* yk, double rho,
                     const double* x, const double* zl, const double* zu, double mu,
                     double* stat, double* mult, double* primal, double* compl_l,
                     double* compl_u, double* norm5) {
  if (!h || !norm5) return NCL_EINVAL;
  return guard([&] {
    auto& S = *h->sys;
    CK(cudaMemsetAsync(S.red(), 0, 5 * sizeof(double), S.st()));
    nclb::launch_nlp_residual(S.P(), jval, grad, c, r, y, yk, rho, x, zl, zu, mu, stat, mult,
                              primal, compl_l, compl_u, S.red(), S.st());
    CK(cudaGetLastError());
    S.fetch(5);
    std::copy(S.hred(), S.hred() + 5, norm5);
  });
}

int ncl_nlp_step(ncl_nlp* h, const double* x, const double* zl, const double* zu, double mu,
                 const double* dx, double tau, double* dzl, double* dzu, double* alpha3) {
  if (!h || !alpha3) return NCL_EINVAL;
  return guard([&] {
    auto& S = *h->sys;
    const double one[3] = {1.0, 1.0, 1.0};
    CK(cudaMemcpyAsync(S.red(), one, 3 * sizeof(double), cudaMemcpyHostToDevice, S.st()));
    nclb::launch_nlp_step(S.P(), x, zl, zu, mu, dx, tau, dzl, dzu, S.red(), S.st());
    CK(cudaGetLastError());
    S.fetch(3);
    std::copy(S.hred(), S.hred() + 3, alpha3);
  });
}

int ncl_nlp_axpy(ncl_nlp* h, int n, const double* v, double a, const double* d, double* out) {
  if (!h) return NCL_EINVAL;
  return guard([&] {
    nclb::launch_axpy(n, v, a, d, out, h->sys->st());
    CK(cudaGetLastError());
  });
}

int ncl_nlp_clip_duals(ncl_nlp* h, const double* x, double mu, double* zl, double* zu) {
  if (!h) return NCL_EINVAL;
  return guard([&] {
    nclb::launch_clip(h->sys->P(), x, mu, zl, zu, h->sys->st());
    CK(cudaGetLastError());
  });
}

int ncl_nlp_outer(ncl_nlp* h, const double* r, double* yk, double rho_used, int update,
                  double* rnorm) {
  if (!h || !rnorm) return NCL_EINVAL;
  return guard([&] {
    auto& S = *h->sys;
    CK(cudaMemsetAsync(S.red(), 0, sizeof(double), S.st()));
    nclb::launch_outer(S.P().m, r, yk, rho_used, update, S.red(), S.st());
    CK(cudaGetLastError());
    S.fetch(1);
    *rnorm = S.hred()[0];
  });
}

// outer_update (solver.cpp:31-41) on the five schedule scalars
// {mu, eta, omega, rho, rho_max}; returns 1 on the multiplier branch
int ncl_outer_update(double* s, double rnorm) {
  if (rnorm <= s[1]) {
    const double mu_old = s[0];
    s[0] = std::max(std::min(std::pow(mu_old, 1.99), 0.2 * mu_old), 1e-14);
    s[1] = std::max(std::min(std::pow(s[0], 1.1), 0.1 * mu_old), 1e-12);
    s[2] = std::max(100.0 * std::pow(s[0], 1.05), 1e-12);
    return 1;
  }
  s[3] = std::min(s[4], 10.0 * s[3]);
  return 0;
}

void ncl_initial_outer_state(double mu0, double rho0, double rho_max, double* s) {
  s[0] = mu0;
  s[1] = std::pow(mu0, 1.1);
  s[2] = 100.0 * std::pow(mu0, 1.05);
  s[3] = rho0;
  s[4] = rho_max;
}

}  // extern "C"
