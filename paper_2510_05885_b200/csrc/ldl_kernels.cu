// Static-pivot supernodal multifrontal LDL^T and its triangular solves for
// sm_100a.  Numeric semantics follow proj/src/sparse.cpp:182-276: pivots in
// the fixed (AMD) order, |d| < eps replaced by sign(d)*eps (exact zero -> +eps)
// and counted, inertia from the signs of D, ok = false on a non-finite or
// zero pivot or a non-finite L entry.
//
// Two tiers (see symbolic.hpp):
//  * warp tier  -- fronts of <= 32 rows.  One persistent kernel; each warp
//    pulls a heavy path of the supernodal elimination tree from a global
//    counter and walks it bottom-up (factor, forward solve) or top-down
//    (backward solve) with the front in shared memory, one front row per
//    lane.  Light children are other warps' paths that precede it in the
//    path order, so a warp only ever spins on work that an already-running
//    warp owns: no deadlock, no per-level launches, and long chains
//    (ring-shaped power grids) run at on-chip latency.
//  * wide tier  -- fronts above 32 rows and all their ancestors:
//    wide_kernels.cu (factorization) and wide_solve.cu (solves).
#include <cuda_runtime.h>
#include <stdint.h>

#include "device.cuh"
#include "launch.hpp"

namespace nclb {

constexpr int kWF = 32;       // warp-tier front limit (rows)
constexpr int kFLD = 33;      // padded leading dimension of a warp front
constexpr int kWarpsPerCta = 4;
constexpr int kWideThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int next_path(int* counter, int lane) {
  int pi = 0;
  if (lane == 0) pi = atomicAdd(counter, 1);
  return __shfl_sync(0xffffffffu, pi, 0);
}

__device__ __forceinline__ void publish(int* flag, int epoch, int lane) {
  __threadfence();
  __syncwarp();
  if (lane == 0) st_release(flag, epoch);
}

// ---------------------------------------------------------------------------
// warp-tier numeric factorization
__global__ void __launch_bounds__(kWarpsPerCta * 32)
k_factor_warp(SnDev sd, FactorDev fd, const double* __restrict__ kval,
              int* flags, int epoch, int* counter, int npaths, double eps) {
  __shared__ double smem[kWarpsPerCta][kWF * kFLD];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* F = smem[wid];
  int npos = 0, nneg = 0, pert = 0, fail = 0;
  for (;;) {
    const int pi = next_path(counter, lane);
    if (pi >= npaths) break;
    const int pb = sd.path_ptr[pi], pe = sd.path_ptr[pi + 1];
    for (int q = pb; q < pe; ++q) {
      const int s = sd.path_nodes[q];
      const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
      const int chb = sd.ch_ptr[s], che = sd.ch_ptr[s + 1];
      for (int c = chb + lane; c < che; c += 32)
        while (ld_acquire(flags + sd.ch[c]) != epoch) {
        }
      __syncwarp();
      for (int c = 0; c < f; ++c) F[c * kFLD + lane] = 0.0;
      __syncwarp();
      for (int a = sd.asm_ptr[s] + lane; a < sd.asm_ptr[s + 1]; a += 32) {
        const int pos = sd.asm_pos[a];
        F[(pos >> 16) * kFLD + (pos & 0xffff)] += __ldg(kval + sd.asm_slot[a]);
      }
      __syncwarp();
      for (int cc = chb; cc < che; ++cc) {
        const int c = sd.ch[cc];
        const int fu = sd.u_ld[c];
        const int* rel = sd.rel + sd.rel_ptr[c];
        const double* U = fd.upd + sd.u_off[c];
        if (lane < fu) {
          const int ri = rel[lane];
          for (int j = 0; j <= lane; ++j)
            F[rel[j] * kFLD + ri] += __ldcg(U + lane + static_cast<size_t>(j) * fu);
        }
        __syncwarp();
      }
      double* Lb = fd.lval + sd.l_off[s];
      for (int p = 0; p < k; ++p) {
        const double u = (lane < f) ? F[p * kFLD + lane] : 0.0;
        double dp = __shfl_sync(0xffffffffu, u, p);
        int pflag = 0;
        if (fabs(dp) < eps) {
          dp = (dp >= 0.0) ? eps : -eps;
          pflag = 1;
        }
        const bool bad = !isfinite(dp) || dp == 0.0;
        const bool mine = lane > p && lane < f;
        const double l = mine ? u / dp : 0.0;
#pragma unroll 4
        for (int j = p + 1; j < f; ++j) {
          const double uj = F[p * kFLD + j];
          if (lane >= j && lane < f) F[j * kFLD + lane] -= l * uj;
        }
        if (mine) {
          Lb[lane + static_cast<size_t>(p) * f] = l;
          if (!isfinite(l)) fail = 1;
        }
        if (lane == 0) {
          fd.d[c0 + p] = dp;
          pert += pflag;
          if (bad) fail = 1;
          if (dp > 0.0)
            npos++;
          else
            nneg++;
        }
        __syncwarp();
      }
      const int fu = f - k;
      double* Us = fd.upd + sd.u_off[s];
      if (lane >= k && lane < f) {
        const int i = lane - k;
        for (int j = 0; j <= i; ++j)
          Us[i + static_cast<size_t>(j) * fu] = F[(k + j) * kFLD + lane];
      }
      publish(flags + s, epoch, lane);
    }
  }
  fail = __any_sync(0xffffffffu, fail);
  if (lane == 0) {
    if (npos) atomicAdd(fd.stats + 0, npos);
    if (nneg) atomicAdd(fd.stats + 1, nneg);
    if (pert) atomicAdd(fd.stats + 2, pert);
    if (fail) atomicOr(fd.stats + 3, 1);
  }
}

// ---------------------------------------------------------------------------
// forward solve L w = b (in place on the permuted vector w); update vectors of
// the multifrontal solve live at uvec + rel_ptr[s] (f - k entries).  The L
// block's column entries of a lane's row are all loaded before the
// substitution chain, and the heavy child's update vector is kept in shared
// memory along the path (path tops still write theirs for other readers).
__global__ void __launch_bounds__(kWarpsPerCta * 32)
k_fwd_warp(SnDev sd, const double* __restrict__ lval, double* w, double* uvec,
           int* flags, int epoch, int* counter, int npaths) {
  __shared__ double Ts[kWarpsPerCta][kWF];
  __shared__ double Hs[kWarpsPerCta][kWF];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* T = Ts[wid];
  double* Hv = Hs[wid];
  for (;;) {
    const int pi = next_path(counter, lane);
    if (pi >= npaths) break;
    const int pb = sd.path_ptr[pi], pe = sd.path_ptr[pi + 1];
    int heavy = -1;
    for (int q = pb; q < pe; ++q) {
      const int s = sd.path_nodes[q];
      const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
      const int chb = sd.ch_ptr[s], che = sd.ch_ptr[s + 1];
      const double* Lb = lval + sd.l_off[s];
      double lv[kWF];  // L(lane, p), p < lane
#pragma unroll
      for (int p = 0; p < kWF; ++p)
        lv[p] = (p < k && lane > p && lane < f) ? __ldg(Lb + lane + static_cast<size_t>(p) * f) : 0.0;
      const double wv = (lane < k) ? __ldcg(w + c0 + lane) : 0.0;
      for (int c = chb + lane; c < che; c += 32) {
        const int ch = sd.ch[c];
        if (ch != heavy)
          while (ld_acquire(flags + ch) != epoch) {
          }
      }
      __syncwarp();
      T[lane] = wv;
      __syncwarp();
      for (int cc = chb; cc < che; ++cc) {
        const int c = sd.ch[cc];
        const int fu = f_minus_k(sd, c);
        if (lane < fu)
          T[sd.rel[sd.rel_ptr[c] + lane]] += (c == heavy) ? Hv[lane] : __ldcg(uvec + sd.rel_ptr[c] + lane);
        __syncwarp();
      }
      double t = (lane < f) ? T[lane] : 0.0;
#pragma unroll
      for (int p = 0; p < kWF; ++p) {
        if (p < k) {
          const double wp = __shfl_sync(0xffffffffu, t, p);
          t -= lv[p] * wp;
        }
      }
      __syncwarp();
      if (lane >= k && lane < f) Hv[lane - k] = t;
      if (lane < k)
        w[c0 + lane] = t;
      else if (lane < f && q == pe - 1)
        uvec[sd.rel_ptr[s] + lane - k] = t;
      if (q == pe - 1) publish(flags + s, epoch, lane);
      heavy = s;
      __syncwarp();
    }
  }
}

// backward solve L^T x = D^-1 w, paths taken in reverse order, top-down.
// Lane q owns pivot q and its L column (loaded up front); the rows below the
// block enter through one shuffle-broadcast dot product per lane, then the
// pivots resolve last-first with one shuffle + FMA each.
__global__ void __launch_bounds__(kWarpsPerCta * 32)
k_bwd_warp(SnDev sd, const double* __restrict__ lval, const double* __restrict__ d,
           const double* __restrict__ w, double* x, int* flags, int epoch,
           const int8_t* __restrict__ wide, int* counter, int npaths) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    const int pj = next_path(counter, lane);
    if (pj >= npaths) break;
    const int pi = npaths - 1 - pj;
    const int pb = sd.path_ptr[pi], pe = sd.path_ptr[pi + 1];
    {
      const int top = sd.path_nodes[pe - 1];
      const int par = sd.sparent[top];
      if (par >= 0 && !wide[par] && lane == 0)
        while (ld_acquire(flags + par) != epoch) {
        }
      __syncwarp();
    }
    for (int q = pe - 1; q >= pb; --q) {
      const int s = sd.path_nodes[q];
      const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
      const double* Lb = lval + sd.l_off[s];
      double lc[kWF];  // L(r, lane), r > lane
#pragma unroll
      for (int r = 0; r < kWF; ++r)
        lc[r] = (lane < k && r > lane && r < f) ? __ldg(Lb + r + static_cast<size_t>(lane) * f) : 0.0;
      const double xr = (lane >= k && lane < f) ? __ldcg(x + sd.rows[sd.rows_ptr[s] + lane]) : 0.0;
      double z = (lane < k) ? w[c0 + lane] / d[c0 + lane] : 0.0;
#pragma unroll
      for (int r = 0; r < kWF; ++r) {
        if (r >= k && r < f) {
          const double xv = __shfl_sync(0xffffffffu, xr, r);
          z -= lc[r] * xv;
        }
      }
#pragma unroll
      for (int p = kWF - 1; p >= 0; --p) {
        if (p < k) {
          const double xp = __shfl_sync(0xffffffffu, z, p);
          if (lane < p) z -= lc[p] * xp;
        }
      }
      if (lane < k) x[c0 + lane] = z;
      publish(flags + s, epoch, lane);
    }
  }
}

__global__ void k_permute_in(int n, const int* __restrict__ perm,
                             const double* __restrict__ b, double* w) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) w[i] = b[perm[i]];
}

__global__ void k_permute_out(int n, const int* __restrict__ perm,
                              const double* __restrict__ xp, double* x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[perm[i]] = xp[i];
}

// ---------------------------------------------------------------------------
// launch helpers (host)
void launch_factor_warp(const SnDev& sd, const FactorDev& fd, const double* kval,
                        int* flags, int epoch, int* counter, int npaths,
                        double eps, int grid, cudaStream_t st) {
  if (npaths == 0) return;
  k_factor_warp<<<grid, kWarpsPerCta * 32, 0, st>>>(sd, fd, kval, flags, epoch,
                                                   counter, npaths, eps);
}

void launch_fwd_warp(const SnDev& sd, const double* lval, double* w, double* uvec,
                     int* flags, int epoch, int* counter, int npaths, int grid,
                     cudaStream_t st) {
  if (npaths == 0) return;
  k_fwd_warp<<<grid, kWarpsPerCta * 32, 0, st>>>(sd, lval, w, uvec, flags, epoch,
                                                counter, npaths);
}

void launch_bwd_warp(const SnDev& sd, const double* lval, const double* d,
                     const double* w, double* x, int* flags, int epoch,
                     const int8_t* wide, int* counter, int npaths, int grid,
                     cudaStream_t st) {
  if (npaths == 0) return;
  k_bwd_warp<<<grid, kWarpsPerCta * 32, 0, st>>>(sd, lval, d, w, x, flags, epoch,
                                                wide, counter, npaths);
}

void launch_permute_in(int n, const int* perm, const double* b, double* w,
                       cudaStream_t st) {
  if (n == 0) return;
  k_permute_in<<<(n + 255) / 256, 256, 0, st>>>(n, perm, b, w);
}

void launch_permute_out(int n, const int* perm, const double* xp, double* x,
                        cudaStream_t st) {
  if (n == 0) return;
  k_permute_out<<<(n + 255) / 256, 256, 0, st>>>(n, perm, xp, x);
}

int warp_tier_grid() {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_factor_warp,
                                                kWarpsPerCta * 32, 0);
  int a = 0, b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_fwd_warp, kWarpsPerCta * 32, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_bwd_warp, kWarpsPerCta * 32, 0);
  per_sm = per_sm < a ? per_sm : a;
  per_sm = per_sm < b ? per_sm : b;
  if (per_sm < 1) per_sm = 1;
  return sms * per_sm;
}

}  // namespace nclb
