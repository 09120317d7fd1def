// Fused NCL vector kernels for sm_100a.
//
//   k_kkt_input       solve_prepared's KktInput formation   ipm.cpp:180-208
//   k_residual_*      barrier_kkt_residual + 5 inf-norms    kkt.cpp:341-366
//   k_step            recover_bound_duals + the three
//                     fraction-to-boundary minima           kkt.cpp:316-328,
//                                                           ipm.cpp:124-141
//   k_trial / k_clip  w+ = w + a d, dual clipping           ipm.cpp:232-249,
//                                                           267-272
//   k_outer           ||r||_inf and y_k += rho r            solver.cpp:213-217
// Per element the arithmetic is the reference's expression with explicit
// round-to-nearest intrinsics (no FMA contraction), and the J^T y
// accumulations gather each column's entries in increasing row order -- the
// reference's scatter order -- so every vector is bitwise the reference's;
// max / min reductions are order-independent.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "device.cuh"

namespace nclb {

struct NlpDev {
  int nt, ns, n, m_eq, m;
  const int* jp_ptr;
  const int* jp_idx;
  const int* jt_ptr;   // J^T: column -> entries in increasing row order
  const int* jt_row;
  const int* jt_slot;
  const double* lb;
  const double* ub;
};

__device__ __forceinline__ double dsub(double a, double b) { return __dadd_rn(a, -b); }

// sigma, rbar1..3 (ipm.cpp:184-208)
__global__ void k_kkt_input(NlpDev P, const double* __restrict__ jval,
                            const double* __restrict__ grad, const double* __restrict__ c,
                            const double* __restrict__ x, const double* __restrict__ zl,
                            const double* __restrict__ zu, const double* __restrict__ r,
                            const double* __restrict__ y, const double* __restrict__ yk, double mu,
                            double rho, double* sigma, double* rbar1, double* rbar2,
                            double* rbar3) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < P.n) {
    double sg = 0.0, r1 = grad[i];
    if (isfinite(P.lb[i])) {
      const double gl = dsub(x[i], P.lb[i]);
      sg = __dadd_rn(sg, __ddiv_rn(zl[i], gl));
      r1 = dsub(r1, __ddiv_rn(mu, gl));
    }
    if (isfinite(P.ub[i])) {
      const double gu = dsub(P.ub[i], x[i]);
      sg = __dadd_rn(sg, __ddiv_rn(zu[i], gu));
      r1 = __dadd_rn(r1, __ddiv_rn(mu, gu));
    }
    if (i < P.nt) {
      for (int q = P.jt_ptr[i]; q < P.jt_ptr[i + 1]; ++q)
        r1 = dsub(r1, __dmul_rn(jval[P.jt_slot[q]], y[P.jt_row[q]]));
    } else {
      r1 = __dadd_rn(r1, y[P.m_eq + (i - P.nt)]);
    }
    sigma[i] = sg;
    rbar1[i] = r1;
  }
  if (i < P.m) {
    rbar2[i] = dsub(__dadd_rn(yk[i], __dmul_rn(rho, r[i])), y[i]);
    rbar3[i] = __dadd_rn(c[i], r[i]);
  }
}

__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, v, o);
    v = v < t ? t : v;
  }
  return v;
}

__device__ __forceinline__ double warp_min(double v) {
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, v, o);
    v = t < v ? t : v;
  }
  return v;
}

__device__ __forceinline__ void atomic_min_pos(double* addr, double v) {
  // v in [0, 1]: non-negative doubles order like their bit patterns
  atomicMin(reinterpret_cast<unsigned long long*>(addr),
            static_cast<unsigned long long>(__double_as_longlong(v)));
}

// barrier_kkt_residual (kkt.cpp:341-366): stat, mult, primal, compl_l,
// compl_u and their inf-norms (norm5 must be zeroed); block vectors optional
__global__ void k_residual(NlpDev P, const double* __restrict__ jval,
                           const double* __restrict__ grad, const double* __restrict__ c,
                           const double* __restrict__ r, const double* __restrict__ y,
                           const double* __restrict__ yk, double rho,
                           const double* __restrict__ x, const double* __restrict__ zl,
                           const double* __restrict__ zu, double mu, double* stat, double* mult,
                           double* primal, double* compl_l, double* compl_u, double* norm5) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0;
  if (i < P.n) {
    double st = __dadd_rn(dsub(grad[i], zl[i]), zu[i]);
    if (i < P.nt) {
      for (int q = P.jt_ptr[i]; q < P.jt_ptr[i + 1]; ++q)
        st = dsub(st, __dmul_rn(jval[P.jt_slot[q]], y[P.jt_row[q]]));
    } else {
      st = __dadd_rn(st, y[P.m_eq + (i - P.nt)]);
    }
    double cl = 0.0, cu = 0.0;
    if (isfinite(P.lb[i])) cl = dsub(__dmul_rn(zl[i], dsub(x[i], P.lb[i])), mu);
    if (isfinite(P.ub[i])) cu = dsub(__dmul_rn(zu[i], dsub(P.ub[i], x[i])), mu);
    if (stat) stat[i] = st;
    if (compl_l) compl_l[i] = cl;
    if (compl_u) compl_u[i] = cu;
    a0 = fabs(st);
    a3 = fabs(cl);
    a4 = fabs(cu);
  }
  if (i < P.m) {
    const double mv = dsub(__dadd_rn(yk[i], __dmul_rn(rho, r[i])), y[i]);
    const double pv = __dadd_rn(c[i], r[i]);
    if (mult) mult[i] = mv;
    if (primal) primal[i] = pv;
    a1 = fabs(mv);
    a2 = fabs(pv);
  }
  // Eigen's lpNorm<Infinity> (a plain max); NaN entries are skipped by the
  // atomic (atomic_max_nonneg ignores them)
  a0 = warp_max(a0);
  a1 = warp_max(a1);
  a2 = warp_max(a2);
  a3 = warp_max(a3);
  a4 = warp_max(a4);
  if ((threadIdx.x & 31) == 0) {
    atomic_max_nonneg(norm5 + 0, a0);
    atomic_max_nonneg(norm5 + 1, a1);
    atomic_max_nonneg(norm5 + 2, a2);
    atomic_max_nonneg(norm5 + 3, a3);
    atomic_max_nonneg(norm5 + 4, a4);
  }
}

// recover_bound_duals + the three FTB minima (alpha3 must be set to 1.0):
// [0] primal (ipm.cpp:124-135), [1] dual zl, [2] dual zu (ipm.cpp:137-141)
__global__ void k_step(NlpDev P, const double* __restrict__ x, const double* __restrict__ zl,
                       const double* __restrict__ zu, double mu, const double* __restrict__ dx,
                       double tau, double* dzl, double* dzu, double* alpha3) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double ap = 1.0, al = 1.0, au = 1.0;
  if (i < P.n) {
    const double l = P.lb[i], u = P.ub[i], xi = x[i], d = dx[i];
    double gl = 0.0, gu = 0.0;
    if (isfinite(l)) {
      gl = dsub(-__ddiv_rn(dsub(__dmul_rn(zl[i], d), mu), dsub(xi, l)), zl[i]);
    }
    if (isfinite(u)) {
      gu = dsub(__ddiv_rn(__dadd_rn(__dmul_rn(zu[i], d), mu), dsub(u, xi)), zu[i]);
    }
    dzl[i] = gl;
    dzu[i] = gu;
    if (d < 0.0 && isfinite(l))
      ap = __ddiv_rn(__dmul_rn(tau, dsub(xi, l)), -d);
    else if (d > 0.0 && isfinite(u))
      ap = __ddiv_rn(__dmul_rn(tau, dsub(u, xi)), d);
    if (zl[i] > 0.0 && gl < 0.0) al = __ddiv_rn(__dmul_rn(tau, zl[i]), -gl);
    if (zu[i] > 0.0 && gu < 0.0) au = __ddiv_rn(__dmul_rn(tau, zu[i]), -gu);
    ap = ap < 1.0 ? ap : 1.0;
    al = al < 1.0 ? al : 1.0;
    au = au < 1.0 ? au : 1.0;
  }
  ap = warp_min(ap);
  al = warp_min(al);
  au = warp_min(au);
  if ((threadIdx.x & 31) == 0) {
    // std::max(a, 0.0) at the end of the reference: clamp negatives to 0
    atomic_min_pos(alpha3 + 0, ap > 0.0 ? ap : 0.0);
    atomic_min_pos(alpha3 + 1, al > 0.0 ? al : 0.0);
    atomic_min_pos(alpha3 + 2, au > 0.0 ? au : 0.0);
  }
}

// out = v + a * d (the trial point / commit, ipm.cpp:267-271, 366-369)
__global__ void k_axpy(int n, const double* __restrict__ v, double a, const double* __restrict__ d,
                       double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __dadd_rn(v[i], __dmul_rn(a, d[i]));
}

// clip_duals (ipm.cpp:232-249)
__global__ void k_clip(NlpDev P, const double* __restrict__ x, double mu, double* zl, double* zu) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  const double kap = 1e10;
  if (isfinite(P.lb[i])) {
    const double gap = fmax(dsub(x[i], P.lb[i]), 1e-300);
    const double lo = __ddiv_rn(mu, __dmul_rn(kap, gap)), hi = __ddiv_rn(__dmul_rn(kap, mu), gap);
    const double z = zl[i];
    zl[i] = z < lo ? lo : (hi < z ? hi : z);
  } else {
    zl[i] = 0.0;
  }
  if (isfinite(P.ub[i])) {
    const double gap = fmax(dsub(P.ub[i], x[i]), 1e-300);
    const double lo = __ddiv_rn(mu, __dmul_rn(kap, gap)), hi = __ddiv_rn(__dmul_rn(kap, mu), gap);
    const double z = zu[i];
    zu[i] = z < lo ? lo : (hi < z ? hi : z);
  } else {
    zu[i] = 0.0;
  }
}

// ||r||_inf (norm must be zeroed) and, when `update`, yk += rho_used * r
__global__ void k_outer(int m, const double* __restrict__ r, double* yk, double rho_used,
                        int update, double* norm) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double a = 0.0;
  if (i < m) {
    a = fabs(r[i]);
    if (update) yk[i] = __dadd_rn(yk[i], __dmul_rn(rho_used, r[i]));
  }
  a = warp_max(a);
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(norm, a);
}

// ---------------------------------------------------------------------------
static inline int nblk(int n) { return n > 0 ? (n + 255) / 256 : 1; }

void launch_kkt_input(const NlpDev& P, const double* jval, const double* grad, const double* c,
                      const double* x, const double* zl, const double* zu, const double* r,
                      const double* y, const double* yk, double mu, double rho, double* sigma,
                      double* rbar1, double* rbar2, double* rbar3, cudaStream_t st) {
  const int n = P.n > P.m ? P.n : P.m;
  if (n) k_kkt_input<<<nblk(n), 256, 0, st>>>(P, jval, grad, c, x, zl, zu, r, y, yk, mu, rho, sigma,
                                             rbar1, rbar2, rbar3);
}

void launch_nlp_residual(const NlpDev& P, const double* jval, const double* grad, const double* c,
                         const double* r, const double* y, const double* yk, double rho,
                         const double* x, const double* zl, const double* zu, double mu,
                         double* stat, double* mult, double* primal, double* cl, double* cu,
                         double* norm5, cudaStream_t st) {
  const int n = P.n > P.m ? P.n : P.m;
  if (n) k_residual<<<nblk(n), 256, 0, st>>>(P, jval, grad, c, r, y, yk, rho, x, zl, zu, mu, stat,
                                            mult, primal, cl, cu, norm5);
}

void launch_nlp_step(const NlpDev& P, const double* x, const double* zl, const double* zu,
                     double mu, const double* dx, double tau, double* dzl, double* dzu,
                     double* alpha3, cudaStream_t st) {
  if (P.n) k_step<<<nblk(P.n), 256, 0, st>>>(P, x, zl, zu, mu, dx, tau, dzl, dzu, alpha3);
}

void launch_axpy(int n, const double* v, double a, const double* d, double* out, cudaStream_t st) {
  if (n) k_axpy<<<nblk(n), 256, 0, st>>>(n, v, a, d, out);
}

void launch_clip(const NlpDev& P, const double* x, double mu, double* zl, double* zu,
                 cudaStream_t st) {
  if (P.n) k_clip<<<nblk(P.n), 256, 0, st>>>(P, x, mu, zl, zu);
}

void launch_outer(int m, const double* r, double* yk, double rho_used, int update, double* norm,
                  cudaStream_t st) {
  if (m) k_outer<<<nblk(m), 256, 0, st>>>(m, r, yk, rho_used, update, norm);
}

}  // namespace nclb
