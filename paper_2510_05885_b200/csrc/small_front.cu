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

#include "cuda_util.hpp"
#include "device.cuh"
#include "launch.hpp"
#include "layout.hpp"
#include "symbolic.hpp"

namespace nclb {

// instances: R rows per lane (fronts <= 32 R rows), W warps (fronts) per CTA.
// Factorization: levels of fronts <= 64 rows (R = 2, W = 4; a one-warp
// 128-row front was measured slower than the cluster kernel).  Solves: levels
// of fronts <= 128 rows (R = 4, no shared front needed).
constexpr int kSmallFactorF = 64;
constexpr int kSmallSolveF = 128;
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
  const int ng = sd.split_ng[s];
  if (ng) {  // group sums of the contributions (split.cu), in group order
    const double* P = fd.ccpart + sd.split_off[s] + static_cast<size_t>(J) * ng * f;
    for (int r = J + lane; r < f; r += 32) {
      double v = a[r];
#pragma unroll 8
      for (int g = 0; g < ng; ++g) v += __ldcg(P + static_cast<size_t>(g) * f + r);
      a[r] = v;
    }
    __syncwarp();
    return;
  }
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

template <int R, int W>
__global__ void __launch_bounds__(W * 32)
k_small_front(SnDev sd, FactorDev fd, const double* __restrict__ kval,
              const int* __restrict__ nodes, int count, double eps, int fm) {
  // column-major shared front sized for the level's largest front (fm <= 32 R
  // rows): leading dimension fm + 1 (odd: conflict-free); a level of 48-row
  // fronts then fits three CTAs per SM instead of one
  const int LDS = fm + 1;
  extern __shared__ double small_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fi = blockIdx.x * W + warp;
  if (fi >= count) return;  // warp-level work only below: no CTA barriers
  double* S = small_smem + static_cast<size_t>(warp) * fm * LDS;
  const int s = nodes[fi];
  const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
  const int kp = s == sd.schur ? 0 : k;
  const size_t ld = wide_ld(f);
  double* F = fd.lval + sd.l_off[s];
  if (sd.split_ng[s]) {
    for (int J = 0; J < f; ++J) small_assemble_col(sd, fd, kval, s, c0, k, f, J, S + J * LDS);
  } else {
    // whole-front assembly: zero, every A entry of the front at once, then the
    // children one by one with all of a child's loads in flight (a column-
    // by-column pass waits one L2 round trip per child column); per position
    // the same order as the column pass: A, then the children in order
    for (int J = 0; J < f; ++J)
      for (int r = lane; r < f; r += 32) S[J * LDS + r] = 0.0;
    __syncwarp();
    for (int q = sd.asm_ptr[s] + lane; q < sd.asm_ptr[s + 1]; q += 32) {
      const int pos = sd.asm_pos[q];
      S[(pos >> 16) * LDS + (pos & 0xffff)] += __ldg(kval + sd.asm_slot[q]);
    }
    __syncwarp();
    for (int cc = sd.ch_ptr[s]; cc < sd.ch_ptr[s + 1]; ++cc) {
      const int c = sd.ch[cc];
      const int fu = f_minus_k(sd, c);
      const size_t uld = sd.u_ld[c];
      const double* U = (sd.wide[c] ? fd.lval : fd.upd) + sd.u_off[c];
      const int* rel = sd.rel + sd.rel_ptr[c];
      int ri[R];  // this lane's rows of the child, as front positions
#pragma unroll
      for (int r = 0; r < R; ++r) ri[r] = lane + 32 * r < fu ? rel[lane + 32 * r] : 0;
#pragma unroll 4
      for (int j = 0; j < fu; ++j) {
        const int cj = rel[j];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int i = lane + 32 * r;
          if (i >= j && i < fu) S[cj * LDS + ri[r]] += __ldcg(U + i + j * uld);
        }
      }
      __syncwarp();
    }
  }
  __syncwarp();
  int npos = 0, nneg = 0, pert = 0;
  bool bad = false;
  for (int p = 0; p < kp; ++p) {
    const double* colp = S + p * LDS;
    double dp = colp[p];
    int pflag = 0;
    if (fabs(dp) < eps) {
      dp = (dp >= 0.0) ? eps : -eps;
      pflag = 1;
    }
    double l[R];  // rows lane + 32 r
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = lane + 32 * r;
      l[r] = (i > p && i < f) ? colp[i] / dp : 0.0;
      bad |= !isfinite(l[r]);
    }
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
      double* cj = S + j * LDS;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = lane + 32 * r;
        if (i >= j && i < f) cj[i] -= l[r] * uj;
      }
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = lane + 32 * r;
      if (i > p && i < f) S[p * LDS + i] = l[r];
    }
    __syncwarp();
  }
  for (int j = 0; j < f; ++j)
    for (int i = j + lane; i < f; i += 32) F[i + j * ld] = S[j * LDS + i];
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
template <int R, int W>
__global__ void __launch_bounds__(W * 32)
k_fwd_small(SnDev sd, const double* __restrict__ lval, double* w, double* uvec,
            const int* __restrict__ nodes, int count) {
  __shared__ double Ts[W][32 * R];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fi = blockIdx.x * W + warp;
  if (fi >= count) return;
  double* T = Ts[warp];
  const int s = nodes[fi];
  const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
  const int kp = s == sd.schur ? 0 : k;
  const size_t ld = wide_ld(f);
  const double* L = lval + sd.l_off[s];
  for (int r = lane; r < f; r += 32) T[r] = r < k ? __ldcg(w + c0 + r) : 0.0;
  __syncwarp();
  if (const int ng = sd.usplit_ng[s]) {  // group sums (split.cu), in group order
    const double* P = sd.uvpart + sd.usplit_off[s];
    for (int r = lane; r < f; r += 32) {
      double v = T[r];
#pragma unroll 8
      for (int g = 0; g < ng; ++g) v += __ldcg(P + static_cast<size_t>(g) * f + r);
      T[r] = v;
    }
    __syncwarp();
  } else {
    for (int cc = sd.ch_ptr[s]; cc < sd.ch_ptr[s + 1]; ++cc) {
      const int c = sd.ch[cc];
      const int fu = f_minus_k(sd, c), rp = sd.rel_ptr[c];
      for (int i = lane; i < fu; i += 32) T[sd.rel[rp + i]] += __ldcg(uvec + rp + i);
      __syncwarp();
    }
  }
  double t[R];
#pragma unroll
  for (int r = 0; r < R; ++r) t[r] = lane + 32 * r < f ? T[lane + 32 * r] : 0.0;
  for (int p = 0; p < kp; ++p) {
    const double* Lp = L + p * ld;
    double a[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = lane + 32 * r;
      a[r] = (i > p && i < f) ? __ldg(Lp + i) : 0.0;
    }
    double src = t[0];
#pragma unroll
    for (int r = 1; r < R; ++r) src = (p >> 5) == r ? t[r] : src;
    const double xp = __shfl_sync(kSFull, src, p & 31);
#pragma unroll
    for (int r = 0; r < R; ++r) t[r] -= a[r] * xp;
  }
  double* u = uvec + sd.rel_ptr[s];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = lane + 32 * r;
    if (i < f) (i < k ? w[c0 + i] : u[i - k]) = t[r];
  }
}

// backward solve of a small front (warp): L^T x = D^-1 w with the parent's
// rows already solved; warp reductions per pivot, last pivot first
template <int R, int W>
__global__ void __launch_bounds__(W * 32)
k_bwd_small(SnDev sd, const double* __restrict__ lval, const double* __restrict__ d,
            const double* __restrict__ w, double* x, const int* __restrict__ nodes, int count) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fi = blockIdx.x * W + warp;
  if (fi >= count) return;
  const int s = nodes[fi];
  if (s == sd.schur) return;
  const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
  const size_t ld = wide_ld(f);
  const double* L = lval + sd.l_off[s];
  const int* rows = sd.rows + sd.rows_ptr[s];
  double xv[R];  // solved values of this lane's rows
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = lane + 32 * r;
    xv[r] = (i >= k && i < f) ? __ldcg(x + rows[i]) : 0.0;
  }
  for (int p = k - 1; p >= 0; --p) {
    const double* Lp = L + p * ld;
    double part = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = lane + 32 * r;
      if (i > p && i < f) part += __ldg(Lp + i) * xv[r];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(kSFull, part, o);
    const double xp = __ldcg(w + c0 + p) / __ldcg(d + c0 + p) - part;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (lane + 32 * r == p) xv[r] = xp;
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = lane + 32 * r;
    if (i < k) x[c0 + i] = xv[r];
  }
}

// ---------------------------------------------------------------------------
template <int R, int W>
static size_t small_front_smem(int fm) { return sizeof(double) * W * fm * (fm + 1); }

int small_factor_limit() { return kSmallFactorF; }
int small_solve_limit() { return kSmallSolveF; }

template <int R, int W>
static void small_launch(const SnDev& sd, const FactorDev& fd, const double* kval, const int* nodes,
                         int count, int fmax, double eps, cudaStream_t st) {
  static PerDeviceOnce init;
  init([] {
    cudaFuncSetAttribute(k_small_front<R, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(small_front_smem<R, W>(32 * R)));
  });
  const int fm = fmax < 1 ? 1 : fmax;
  k_small_front<R, W><<<(count + W - 1) / W, W * 32, small_front_smem<R, W>(fm), st>>>(sd, fd, kval, nodes,
                                                                                       count, eps, fm);
}

void launch_small_front(const SnDev& sd, const FactorDev& fd, const double* kval, const int* nodes,
                        int count, int fmax, double eps, cudaStream_t st) {
  if (count && fmax <= kSmallFactorF) small_launch<2, 4>(sd, fd, kval, nodes, count, fmax, eps, st);
}

void launch_fwd_small(const SnDev& sd, const double* lval, double* w, double* uvec,
                      const int* nodes, int count, int fmax, cudaStream_t st) {
  if (!count) return;
  if (fmax <= 64)
    k_fwd_small<2, 4><<<(count + 3) / 4, 128, 0, st>>>(sd, lval, w, uvec, nodes, count);
  else
    k_fwd_small<4, 4><<<(count + 3) / 4, 128, 0, st>>>(sd, lval, w, uvec, nodes, count);
}

void launch_bwd_small(const SnDev& sd, const double* lval, const double* d, const double* w,
                      double* x, const int* nodes, int count, int fmax, cudaStream_t st) {
  if (!count) return;
  if (fmax <= 64)
    k_bwd_small<2, 4><<<(count + 3) / 4, 128, 0, st>>>(sd, lval, d, w, x, nodes, count);
  else
    k_bwd_small<4, 4><<<(count + 3) / 4, 128, 0, st>>>(sd, lval, d, w, x, nodes, count);
}

}  // namespace nclb
