// Small-front tier: wide-tier levels whose fronts all have at most 64 rows
// (the bottom of the wide tree -- on the 78k-bus mesh, levels of 200-1600
// fronts of 33-64 rows).  One WARP per front, the whole front in shared
// memory (64 x 65 doubles), four fronts per CTA, so a level runs ~600 fronts
// at a time instead of one 512-thread cluster CTA per front.  Same storage as
// the wide tier (f x f column-major, leading dimension wide_ld(f), L in the
// first k columns, the update matrix in the trailing corner), same pivot rule
// (sparse.cpp:235-247) and the warp tier's l = u / d.
#include <cuda_runtime.h>
#include <stdint.h>

#include "device.cuh"
#include "launch.hpp"
#include "layout.hpp"
#include "symbolic.hpp"

namespace nclb {

constexpr int kSmallF = 64;
constexpr int kSmallLd = kSmallF + 1;  // conflict-free column-major shared front
constexpr int kSmallWarps = 4;
constexpr unsigned kSFull = 0xffffffffu;

// assembly of one column into the shared front (warp): zero, A entries, the
// children's columns in child order (same lists and order as the wide tier)
__device__ __forceinline__ void small_assemble_col(const SnDev& sd, const FactorDev& fd,
                                                   const double* __restrict__ kval, int s, int c0,
                                                   int k, int f, int J, double* a) {
  const int lane = threadIdx.x & 31;
  const int cb = sd.cc_off[s] + J;
  const int e0 = sd.cc_ptr[cb], e1 = sd.cc_ptr[cb + 1];
  const int a0 = J < k ? sd.asm_cp[c0 + J] : 0, a1 = J < k ? sd.asm_cp[c0 + J + 1] : 0;
  for (int r = J + lane; r < f; r += 32) a[r] = 0.0;
  __syncwarp();
  for (int q = a0 + lane; q < a1; q += 32) a[sd.asm_pos[q] & 0xffff] += __ldg(kval + sd.asm_slot[q]);
  __syncwarp();
  for (int e = e0; e < e1; ++e) {
    const long long ub = sd.cc_ubase[e];
    const int rb = sd.cc_rbase[e], cw = sd.cc_cnt[e];
    const int cnt = cw & ((1 << 30) - 1);
    const double* U = ((cw >> 30) ? fd.lval : fd.upd) + ub;
    const int* rel = sd.rel + rb;
    for (int i = lane; i < cnt; i += 32) a[rel[i]] += __ldcg(U + i);
    __syncwarp();
  }
}

__global__ void __launch_bounds__(kSmallWarps * 32)
k_small_front(SnDev sd, FactorDev fd, const double* __restrict__ kval,
              const int* __restrict__ nodes, int count, double eps) {
  extern __shared__ double small_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fi = blockIdx.x * kSmallWarps + warp;
  if (fi >= count) return;  // warp-level work only below: no CTA barriers
  double* S = small_smem + static_cast<size_t>(warp) * kSmallF * kSmallLd;
  const int s = nodes[fi];
  const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
  const int kp = s == sd.schur ? 0 : k;
  const size_t ld = wide_ld(f);
  double* F = fd.lval + sd.l_off[s];
  for (int J = 0; J < f; ++J) small_assemble_col(sd, fd, kval, s, c0, k, f, J, S + J * kSmallLd);
  __syncwarp();
  int npos = 0, nneg = 0, pert = 0;
  bool bad = false;
  const int i0 = lane, i1 = lane + 32;  // the two rows of this lane
  for (int p = 0; p < kp; ++p) {
    const double* colp = S + p * kSmallLd;
    double dp = colp[p];
    int pflag = 0;
    if (fabs(dp) < eps) {
      dp = (dp >= 0.0) ? eps : -eps;
      pflag = 1;
    }
    const double l0 = (i0 > p && i0 < f) ? colp[i0] / dp : 0.0;
    const double l1 = (i1 > p && i1 < f) ? colp[i1] / dp : 0.0;
    bad |= !isfinite(l0) || !isfinite(l1);
    if (lane == 0) {
      fd.d[c0 + p] = dp;
      pert += pflag;
      if (!isfinite(dp) || dp == 0.0) bad = true;
      if (dp > 0.0)
        npos++;
      else
        nneg++;
    }
    // trailing update with the unscaled column p (untouched until below)
    for (int j = p + 1; j < f; ++j) {
      const double uj = colp[j];
      double* cj = S + j * kSmallLd;
      if (i0 >= j && i0 < f) cj[i0] -= l0 * uj;
      if (i1 >= j && i1 < f) cj[i1] -= l1 * uj;
    }
    __syncwarp();
    if (i0 > p && i0 < f) S[p * kSmallLd + i0] = l0;
    if (i1 > p && i1 < f) S[p * kSmallLd + i1] = l1;
    __syncwarp();
  }
  for (int j = 0; j < f; ++j)
    for (int i = j + lane; i < f; i += 32) F[i + j * ld] = S[j * kSmallLd + i];
  const bool fail = __any_sync(kSFull, bad);
  if (lane == 0) {
    if (npos) atomicAdd(fd.stats + 0, npos);
    if (nneg) atomicAdd(fd.stats + 1, nneg);
    if (pert) atomicAdd(fd.stats + 2, pert);
    if (fail) atomicOr(fd.stats + 3, 1);
  }
}

// forward solve of a small front (warp): gather, k-step substitution with
// the L column loaded per step (coalesced), update vector for the parent
__global__ void __launch_bounds__(kSmallWarps * 32)
k_fwd_small(SnDev sd, const double* __restrict__ lval, double* w, double* uvec,
            const int* __restrict__ nodes, int count) {
  __shared__ double Ts[kSmallWarps][kSmallF];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fi = blockIdx.x * kSmallWarps + warp;
  if (fi >= count) return;
  double* T = Ts[warp];
  const int s = nodes[fi];
  const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
  const int kp = s == sd.schur ? 0 : k;
  const size_t ld = wide_ld(f);
  const double* L = lval + sd.l_off[s];
  for (int r = lane; r < f; r += 32) T[r] = r < k ? __ldcg(w + c0 + r) : 0.0;
  __syncwarp();
  for (int cc = sd.ch_ptr[s]; cc < sd.ch_ptr[s + 1]; ++cc) {
    const int c = sd.ch[cc];
    const int fu = f_minus_k(sd, c), rp = sd.rel_ptr[c];
    for (int i = lane; i < fu; i += 32) T[sd.rel[rp + i]] += __ldcg(uvec + rp + i);
    __syncwarp();
  }
  const int i0 = lane, i1 = lane + 32;
  double t0 = i0 < f ? T[i0] : 0.0, t1 = i1 < f ? T[i1] : 0.0;
  for (int p = 0; p < kp; ++p) {
    const double* Lp = L + p * ld;
    const double a0 = (i0 > p && i0 < f) ? __ldg(Lp + i0) : 0.0;
    const double a1 = (i1 > p && i1 < f) ? __ldg(Lp + i1) : 0.0;
    const double xp = __shfl_sync(kSFull, p < 32 ? t0 : t1, p & 31);
    t0 -= a0 * xp;
    t1 -= a1 * xp;
  }
  double* u = uvec + sd.rel_ptr[s];
  if (i0 < f) (i0 < k ? w[c0 + i0] : u[i0 - k]) = t0;
  if (i1 < f) (i1 < k ? w[c0 + i1] : u[i1 - k]) = t1;
}

// backward solve of a small front (warp): L^T x = D^-1 w with the parent's
// rows already solved; warp reductions per pivot, last pivot first
__global__ void __launch_bounds__(kSmallWarps * 32)
k_bwd_small(SnDev sd, const double* __restrict__ lval, const double* __restrict__ d,
            const double* __restrict__ w, double* x, const int* __restrict__ nodes, int count) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fi = blockIdx.x * kSmallWarps + warp;
  if (fi >= count) return;
  const int s = nodes[fi];
  if (s == sd.schur) return;
  const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
  const size_t ld = wide_ld(f);
  const double* L = lval + sd.l_off[s];
  const int* rows = sd.rows + sd.rows_ptr[s];
  const int i0 = lane, i1 = lane + 32;
  double x0 = 0.0, x1 = 0.0;  // solved values of this lane's rows
  if (i0 >= k && i0 < f) x0 = __ldcg(x + rows[i0]);
  if (i1 >= k && i1 < f) x1 = __ldcg(x + rows[i1]);
  for (int p = k - 1; p >= 0; --p) {
    const double* Lp = L + p * ld;
    double part = 0.0;
    if (i0 > p && i0 < f) part += __ldg(Lp + i0) * x0;
    if (i1 > p && i1 < f) part += __ldg(Lp + i1) * x1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(kSFull, part, o);
    const double xp = __ldcg(w + c0 + p) / __ldcg(d + c0 + p) - part;
    if (i0 == p) x0 = xp;
    if (i1 == p) x1 = xp;
  }
  if (i0 < k) x[c0 + i0] = x0;
  if (i1 < k) x[c0 + i1] = x1;
}

// ---------------------------------------------------------------------------
static size_t small_front_smem() { return sizeof(double) * kSmallWarps * kSmallF * kSmallLd; }

int small_front_limit() { return kSmallF; }

void launch_small_front(const SnDev& sd, const FactorDev& fd, const double* kval, const int* nodes,
                        int count, double eps, cudaStream_t st) {
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_small_front, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(small_front_smem()));
    init = true;
  }
  if (count)
    k_small_front<<<(count + kSmallWarps - 1) / kSmallWarps, kSmallWarps * 32, small_front_smem(), st>>>(
        sd, fd, kval, nodes, count, eps);
}

void launch_fwd_small(const SnDev& sd, const double* lval, double* w, double* uvec,
                      const int* nodes, int count, cudaStream_t st) {
  if (count)
    k_fwd_small<<<(count + kSmallWarps - 1) / kSmallWarps, kSmallWarps * 32, 0, st>>>(sd, lval, w, uvec,
                                                                                      nodes, count);
}

void launch_bwd_small(const SnDev& sd, const double* lval, const double* d, const double* w,
                      double* x, const int* nodes, int count, cudaStream_t st) {
  if (count)
    k_bwd_small<<<(count + kSmallWarps - 1) / kSmallWarps, kSmallWarps * 32, 0, st>>>(sd, lval, d, w, x,
                                                                                      nodes, count);
}

}  // namespace nclb
