// KKT-layer kernels for sm_100a: bit-exact refill (proj/src/kkt.cpp:149-186),
// right-hand sides (kkt.cpp:188-222), recovery (kkt.cpp:224-264), the
// symmetric residual matvec of the refinement loop (sparse.cpp:70-79,
// 292-300) and the small reductions the delta loop needs.
//
// Everything that the reference computes with a defined operation order is
// written with explicit round-to-nearest intrinsics (__dadd_rn, __dmul_rn,
// __ddiv_rn) so no FMA contraction can change a bit: the assembled K, the
// right-hand side and the recovery formulas are bitwise the reference's for
// identical inputs.
#include <cuda_runtime.h>
#include <stdint.h>

#include "device.cuh"
#include "kkt_plan.hpp"
#include "launch.hpp"

namespace nclb {

// w_i = rho_hat * omega_i, omega_i = 1 (eq) or ss/(ss + rho_hat) with
// ss = sigma_s + delta (kkt.cpp:160-166)
__global__ void k_row_weight(int m, int m_eq, int nt, const double* __restrict__ sigma,
                             double rho_hat, double delta, double* wrow) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double omega = 1.0;
  if (i >= m_eq) {
    const double ss = __dadd_rn(sigma[nt + (i - m_eq)], delta);
    omega = __ddiv_rn(ss, __dadd_rn(ss, rho_hat));
  }
  wrow[i] = __dmul_rn(rho_hat, omega);
}

// one refill contribution (kkt.cpp:149-186 term types)
__device__ __forceinline__ double refill_term(const AsmDev& a, int q, const double* __restrict__ hval,
                                              const double* __restrict__ jval,
                                              const double* __restrict__ sigma,
                                              const double* __restrict__ wrow, double rho_hat,
                                              double delta) {
  const uint32_t code = a.c_code[q];
  const uint32_t idx = code & kIdxMask;
  switch (code >> kTypeShift) {
    case kCH: return hval[idx];
    case kCDiag: return __dadd_rn(sigma[idx], delta);
    case kCPair:
      return __dmul_rn(__dmul_rn(wrow[a.pair_row[idx]], jval[a.pair_pa[idx]]), jval[a.pair_pb[idx]]);
    case kCJ: return jval[idx];
    case kCMinus1: return -1.0;
    case kCYdiag: return __ddiv_rn(-1.0, rho_hat);
    case kCRho: return rho_hat;
    default: return 1.0;
  }
}

// acc + v_0 + v_1 + ... + v_{n-1} left to right (v_i held by lane i), every
// lane returning the same bitwise result of the sequential sum
__device__ __forceinline__ double ordered_warp_sum(double acc, double v, int n) {
  for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, v, i));
  return acc;
}

// one thread per K slot: acc = 0; acc += contribution, in refill order
__global__ void k_assemble(AsmDev a, const double* __restrict__ hval,
                           const double* __restrict__ jval,
                           const double* __restrict__ sigma,
                           const double* __restrict__ wrow, double rho_hat,
                           double delta, double* kval) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.nnz) return;
  const int b = a.c_ptr[s], e = a.c_ptr[s + 1];
  if (e - b > kLongSum) return;  // k_assemble_long
  double acc = 0.0;
  for (int q = b; q < e; ++q)
    acc = __dadd_rn(acc, refill_term(a, q, hval, jval, sigma, wrow, rho_hat, delta));
  kval[s] = acc;
}

// slots with more than kLongSum contributions (SCOPF: the coupling rows sum
// over every contingency block): one warp per slot, 32 terms evaluated at a
// time (their loads in flight together), then added in the refill order by
// every lane (shuffle broadcast) -- bitwise the sequential sum
__global__ void k_assemble_long(AsmDev a, const double* __restrict__ hval,
                                const double* __restrict__ jval,
                                const double* __restrict__ sigma,
                                const double* __restrict__ wrow, double rho_hat,
                                double delta, double* kval) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= a.nlong) return;
  const int s = a.long_slots[w];
  const int b = a.c_ptr[s], e = a.c_ptr[s + 1];
  double acc = 0.0;
  for (int q0 = b; q0 < e; q0 += 32) {
    const int q = q0 + lane;
    const double v = q < e ? refill_term(a, q, hval, jval, sigma, wrow, rho_hat, delta) : 0.0;
    acc = ordered_warp_sum(acc, v, min(32, e - q0));
  }
  if (lane == 0) kval[s] = acc;
}

// hmax = max(|hval|, |sigma[0:n]|) (kkt.cpp:269-271); out must be zeroed
__global__ void k_absmax2(int n1, const double* __restrict__ a, int n2,
                          const double* __restrict__ b, double* out) {
  double m = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n1 + n2;
       i += gridDim.x * blockDim.x) {
    const double v = fabs(i < n1 ? a[i] : b[i - n1]);
    m = (m < v) ? v : m;  // std::max(m, v): NaN skipped
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, m, o);
    m = (m < t) ? t : m;
  }
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, m);
}

// ---- right-hand sides -------------------------------------------------------
__global__ void k_rhs_k2(int n, int m, const double* __restrict__ r1,
                         const double* __restrict__ r2, const double* __restrict__ r3,
                         double* rhs) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) rhs[i] = -r1[i];
  if (i < m) {
    rhs[n + i] = -r2[i];
    rhs[n + m + i] = -r3[i];
  }
}

__global__ void k_rhs_k2r(int n, int m, const double* __restrict__ r1,
                          const double* __restrict__ r2, const double* __restrict__ r3,
                          double rho_hat, double* rhs) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) rhs[i] = -r1[i];
  if (i < m) rhs[n + i] = __dadd_rn(-r3[i], __ddiv_rn(r2[i], rho_hat));
}

// K1s helpers: v_i = rbar2_i - rho_hat rbar3_i ; for inequality rows also
// rs_k = -rbar1[nt+k] - v[row], pk = (sigma_s + delta) + rho_hat and the
// scaled weight rho_hat*rs/pk (kkt.cpp:205-218)
__global__ void k_k1s_rowvec(int m, int m_eq, int nt, const double* __restrict__ sigma,
                             const double* __restrict__ r1, const double* __restrict__ r2,
                             const double* __restrict__ r3, double rho_hat, double delta,
                             double* v, double* wk, double* rs, double* pk) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double vi = __dadd_rn(r2[i], -__dmul_rn(rho_hat, r3[i]));
  v[i] = vi;
  if (i >= m_eq) {
    const int k = i - m_eq;
    const double rsk = __dadd_rn(-r1[nt + k], -vi);
    const double pkk = __dadd_rn(__dadd_rn(sigma[nt + k], delta), rho_hat);
    rs[k] = rsk;
    pk[k] = pkk;
    wk[k] = __ddiv_rn(__dmul_rn(rho_hat, rsk), pkk);
  }
}

// rhs[c] = -rbar1[c] + sum_{rows i asc} jv*v_i, then + sum_{ineq rows asc} jv*w_k
__global__ void k_rhs_k1s(int nt, int m_eq, const int* __restrict__ jt_ptr,
                          const int* __restrict__ jt_row, const int* __restrict__ jt_slot,
                          const double* __restrict__ jval, const double* __restrict__ r1,
                          const double* __restrict__ v, const double* __restrict__ wk,
                          double* rhs) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nt) return;
  const int b = jt_ptr[c], e = jt_ptr[c + 1];
  if (e - b > kLongSum) return;  // k_rhs_k1s_long
  double acc = -r1[c];
  for (int q = b; q < e; ++q)
    acc = __dadd_rn(acc, __dmul_rn(jval[jt_slot[q]], v[jt_row[q]]));
  for (int q = b; q < e; ++q) {
    const int i = jt_row[q];
    if (i >= m_eq) acc = __dadd_rn(acc, __dmul_rn(jval[jt_slot[q]], wk[i - m_eq]));
  }
  rhs[c] = acc;
}

// columns with more than kLongSum Jacobian entries: one warp each, the two
// passes of k_rhs_k1s as chunked in-order sums (bitwise the same)
__global__ void k_rhs_k1s_long(int m_eq, const int* __restrict__ long_cols, int nlong,
                               const int* __restrict__ jt_ptr, const int* __restrict__ jt_row,
                               const int* __restrict__ jt_slot, const double* __restrict__ jval,
                               const double* __restrict__ r1, const double* __restrict__ v,
                               const double* __restrict__ wk, double* rhs) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= nlong) return;
  const int c = long_cols[w];
  const int b = jt_ptr[c], e = jt_ptr[c + 1];
  double acc = -r1[c];
  for (int q0 = b; q0 < e; q0 += 32) {
    const int q = q0 + lane;
    const double t = q < e ? __dmul_rn(jval[jt_slot[q]], v[jt_row[q]]) : 0.0;
    acc = ordered_warp_sum(acc, t, min(32, e - q0));
  }
  for (int q0 = b; q0 < e; q0 += 32) {
    const int q = q0 + lane;
    const int i = q < e ? jt_row[q] : -1;
    const bool ineq = i >= m_eq;
    const double t = ineq ? __dmul_rn(jval[jt_slot[q]], wk[i - m_eq]) : 0.0;
    // only the inequality rows are added (in order)
    unsigned msk = __ballot_sync(0xffffffffu, ineq);
    while (msk) {
      const int src = __ffs(msk) - 1;
      acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, t, src));
      msk &= msk - 1;
    }
  }
  if (lane == 0) rhs[c] = acc;
}

// ---- recovery ---------------------------------------------------------------
__global__ void k_recover_k2(int n, int m, const double* __restrict__ sol, double* dx,
                             double* dr, double* dy) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dx[i] = sol[i];
  if (i < m) {
    dr[i] = sol[n + i];
    dy[i] = -sol[n + m + i];
  }
}

__global__ void k_recover_k2r(int n, int m, const double* __restrict__ sol,
                              const double* __restrict__ r2, double rho_hat, double* dx,
                              double* dr, double* dy) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dx[i] = sol[i];
  if (i < m) {
    const double yi = -sol[n + i];
    dy[i] = yi;
    dr[i] = __ddiv_rn(__dadd_rn(yi, -r2[i]), rho_hat);
  }
}

// K1s: jdt = J dt (row order), slack steps, dy, dr (kkt.cpp:238-262)
__global__ void k_recover_k1s(int nt, int m, int m_eq, const int* __restrict__ jp_ptr,
                              const int* __restrict__ jp_idx, const double* __restrict__ jval,
                              const double* __restrict__ sol, const double* __restrict__ v,
                              const double* __restrict__ rs, const double* __restrict__ pk,
                              const double* __restrict__ r2, double rho_hat, double* dx,
                              double* dr, double* dy) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nt) dx[i] = sol[i];
  if (i >= m) return;
  double jdt = 0.0;
  for (int p = jp_ptr[i]; p < jp_ptr[i + 1]; ++p)
    jdt = __dadd_rn(jdt, __dmul_rn(jval[p], sol[jp_idx[p]]));
  double jxdx = jdt;
  if (i >= m_eq) {
    const int k = i - m_eq;
    const double dxs = __ddiv_rn(__dadd_rn(__dmul_rn(rho_hat, jdt), rs[k]), pk[k]);
    dx[nt + k] = dxs;
    jxdx = __dadd_rn(jxdx, -dxs);
  }
  const double yi = __dadd_rn(v[i], -__dmul_rn(rho_hat, jxdx));
  dy[i] = yi;
  dr[i] = __ddiv_rn(__dadd_rn(yi, -r2[i]), rho_hat);
}

// all-finite check of the step (kkt.cpp:298)
__global__ void k_nonfinite(int n, const double* __restrict__ a, int* flag) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (!isfinite(a[i])) {
      atomicOr(flag, 1);
      return;
    }
}
// the step's three outputs (dx[n], dr[m], dy[m]) in one pass
__global__ void k_nonfinite3(int n, const double* __restrict__ a, int m, const double* __restrict__ b,
                             const double* __restrict__ c, int* flag) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n + 2 * m; i += gridDim.x * blockDim.x) {
    const double v = i < n ? a[i] : (i < n + m ? b[i - n] : c[i - n - m]);
    if (!isfinite(v)) {
      atomicOr(flag, 1);
      return;
    }
  }
}

// ---- refinement pieces --------------------------------------------------------
// r = b - A x over the full symmetric row pattern; norm = max |r_i| (NaN
// entries skipped exactly as std::max(nrm, nan) skips them, sparse.cpp:296)
constexpr int kRowLanes = 8;
constexpr int kLongRow = 256;  // longer residual rows: k_residual_long
__global__ void k_residual(int N, const int* __restrict__ fr_ptr, const int* __restrict__ fr_col,
                           const int* __restrict__ fr_slot, const double* __restrict__ kval,
                           const double* __restrict__ x, const double* __restrict__ b,
                           double* r, double* norm) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  int row = gt / kRowLanes;
  const int sub = gt % kRowLanes;
  if (row < N && fr_ptr[row + 1] - fr_ptr[row] > kLongRow) row = N;  // k_residual_long
  double acc = 0.0;
  if (row < N)
    for (int q = fr_ptr[row] + sub; q < fr_ptr[row + 1]; q += kRowLanes)
      acc += kval[fr_slot[q]] * x[fr_col[q]];
#pragma unroll
  for (int o = kRowLanes / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  double mag = 0.0;
  if (row < N && sub == 0) {
    const double ri = b[row] - acc;
    r[row] = ri;
    mag = fabs(ri);
    if (mag != mag) mag = 0.0;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, mag, o);
    mag = mag < t ? t : mag;
  }
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(norm, mag);
}

// rows longer than kLongRow: one CTA each, fixed-order tree reduction
__global__ void __launch_bounds__(256)
k_residual_long(const int* __restrict__ long_rows, const int* __restrict__ fr_ptr,
                const int* __restrict__ fr_col, const int* __restrict__ fr_slot,
                const double* __restrict__ kval, const double* __restrict__ x,
                const double* __restrict__ b, double* r, double* norm) {
  __shared__ double red[8];
  const int row = long_rows[blockIdx.x];
  double acc = 0.0;
  for (int q = fr_ptr[row] + threadIdx.x; q < fr_ptr[row + 1]; q += 256) acc += kval[fr_slot[q]] * x[fr_col[q]];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 8; ++i) t += red[i];
    const double ri = b[row] - t;
    r[row] = ri;
    double mag = fabs(ri);
    if (mag != mag) mag = 0.0;
    atomic_max_nonneg(norm, mag);
  }
}

__global__ void k_axpy_to(int n, const double* __restrict__ x, const double* __restrict__ dx,
                          double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = x[i] + dx[i];
}

// ---------------------------------------------------------------------------
static inline int nb(int n, int t = 256) { return n > 0 ? (n + t - 1) / t : 1; }

void launch_assemble(const AsmDev& a, int form, int m, int m_eq, int nt,
                     const double* hval, const double* jval, const double* sigma,
                     double* wrow, double rho, double delta, double* kval,
                     cudaStream_t st) {
  const double rho_hat = rho + delta;
  if (form == kK1s && m > 0)
    k_row_weight<<<nb(m), 256, 0, st>>>(m, m_eq, nt, sigma, rho_hat, delta, wrow);
  if (a.nnz > 0)
    k_assemble<<<nb(a.nnz), 256, 0, st>>>(a, hval, jval, sigma, wrow, rho_hat, delta, kval);
  if (a.nlong > 0)
    k_assemble_long<<<nb(a.nlong * 32), 256, 0, st>>>(a, hval, jval, sigma, wrow, rho_hat, delta, kval);
}

void launch_absmax2(int n1, const double* a, int n2, const double* b, double* out,
                    cudaStream_t st) {
  const int n = n1 + n2;
  if (n == 0) return;
  int g = nb(n);
  if (g > 1184) g = 1184;
  k_absmax2<<<g, 256, 0, st>>>(n1, a, n2, b, out);
}

void launch_rhs(const KktPlan& P, const int* jt_ptr, const int* jt_row, const int* jt_slot,
                const double* jval, const double* sigma, const double* r1,
                const double* r2, const double* r3, double rho, double delta, double* v,
                double* wk, double* rs, double* pk, double* rhs, const int* long_cols, int nlong_cols,
                cudaStream_t st) {
  const double rho_hat = rho + delta;
  const int n = P.n, m = P.m;
  const int big = n > m ? n : m;
  if (P.form == kK2) {
    if (big) k_rhs_k2<<<nb(big), 256, 0, st>>>(n, m, r1, r2, r3, rhs);
  } else if (P.form == kK2r) {
    if (big) k_rhs_k2r<<<nb(big), 256, 0, st>>>(n, m, r1, r2, r3, rho_hat, rhs);
  } else {
    if (m) k_k1s_rowvec<<<nb(m), 256, 0, st>>>(m, P.m_eq, P.nt, sigma, r1, r2, r3, rho_hat,
                                             delta, v, wk, rs, pk);
    if (P.nt) k_rhs_k1s<<<nb(P.nt), 256, 0, st>>>(P.nt, P.m_eq, jt_ptr, jt_row, jt_slot, jval,
                                                r1, v, wk, rhs);
    if (nlong_cols)
      k_rhs_k1s_long<<<nb(nlong_cols * 32), 256, 0, st>>>(P.m_eq, long_cols, nlong_cols, jt_ptr, jt_row,
                                                        jt_slot, jval, r1, v, wk, rhs);
  }
}

void launch_recover(const KktPlan& P, const int* jp_ptr, const int* jp_idx,
                    const double* jval, const double* sol, const double* v,
                    const double* rs, const double* pk, const double* r2, double rho,
                    double delta, double* dx, double* dr, double* dy, cudaStream_t st) {
  const double rho_hat = rho + delta;
  const int n = P.n, m = P.m;
  const int big = n > m ? n : m;
  if (!big) return;
  if (P.form == kK2)
    k_recover_k2<<<nb(big), 256, 0, st>>>(n, m, sol, dx, dr, dy);
  else if (P.form == kK2r)
    k_recover_k2r<<<nb(big), 256, 0, st>>>(n, m, sol, r2, rho_hat, dx, dr, dy);
  else {
    const int b2 = P.nt > m ? P.nt : m;
    if (b2)
      k_recover_k1s<<<nb(b2), 256, 0, st>>>(P.nt, m, P.m_eq, jp_ptr, jp_idx, jval, sol, v, rs,
                                            pk, r2, rho_hat, dx, dr, dy);
  }
}

void launch_nonfinite(int n, const double* a, int* flag, cudaStream_t st) {
  if (n <= 0) return;
  int g = nb(n);
  if (g > 1184) g = 1184;
  k_nonfinite<<<g, 256, 0, st>>>(n, a, flag);
}

void launch_nonfinite3(int n, const double* a, int m, const double* b, const double* c, int* flag,
                       cudaStream_t st) {
  if (n + 2 * m <= 0) return;
  int g = nb(n + 2 * m);
  if (g > 1184) g = 1184;
  k_nonfinite3<<<g, 256, 0, st>>>(n, a, m, b, c, flag);
}

void launch_residual(int N, const int* fr_ptr, const int* fr_col, const int* fr_slot,
                     const double* kval, const double* x, const double* b, double* r,
                     double* norm, const int* long_rows, int nlong_rows, cudaStream_t st) {
  if (N == 0) return;
  const long long threads = static_cast<long long>(N) * kRowLanes;
  k_residual<<<static_cast<int>((threads + 255) / 256), 256, 0, st>>>(N, fr_ptr, fr_col, fr_slot,
                                                                     kval, x, b, r, norm);
  if (nlong_rows)
    k_residual_long<<<nlong_rows, 256, 0, st>>>(long_rows, fr_ptr, fr_col, fr_slot, kval, x, b, r, norm);
}

void launch_axpy_to(int n, const double* x, const double* dx, double* out, cudaStream_t st) {
  if (n) k_axpy_to<<<nb(n), 256, 0, st>>>(n, x, dx, out);
}

}  // namespace nclb
