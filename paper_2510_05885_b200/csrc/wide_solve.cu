// Wide-tier triangular solves (ldl_solve, sparse.cpp:258-276, restated for
// the supernodal fronts): one launch per tree level, one thread-block cluster
// per front.
//
// Forward  (L w = b on the permuted vector):
//   rank 0   -- gathers the pivot values and the children's update vectors,
//               then solves the k x k unit-lower L11 block by block: warp 0
//               runs the 32-step substitution chain with its L11 rows already
//               in registers (static indices, one shuffle + FMA per step)
//               while the other warps prefetch the L entries of the rows
//               below the block, then fold the solved block in (GEMV);
//   all CTAs -- after one cluster barrier, the (f-k) x k GEMV that forms the
//               update vector the parent adds (thread per row, coalesced
//               column-major reads, rows split across the cluster).
// Backward (L^T x = D^-1 w):
//   all CTAs -- the k x (f-k) transposed GEMV against the parent's solved
//               rows (warp per pivot column, lanes along the column);
//   rank 0   -- after one cluster barrier, the blocked L11^T solve from the
//               last block up: GEMV against the later pivots, then warp 0's
//               32-step chain with its L11 column in registers.
// No atomics on values; every sum has a fixed order (bitwise reproducible).
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "device.cuh"
#include "launch.hpp"
#include "symbolic.hpp"
#include "layout.hpp"

namespace cg = cooperative_groups;

namespace nclb {

constexpr int kSolveThreads = 512;
constexpr int kSolveWarps = kSolveThreads / 32;
constexpr int kBlk = 32;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kSolveThreads, 1)
k_fwd_front(SnDev sd, const double* __restrict__ lval, double* w, double* uvec,
            const int* __restrict__ nodes) {
  extern __shared__ double T[];
  cg::cluster_group cl = cg::this_cluster();
  const int C = static_cast<int>(cl.num_blocks());
  const int rank = static_cast<int>(cl.block_rank());
  const int s = nodes[blockIdx.x / C];
  const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
  const size_t ld = wide_ld(f);
  const double* L = lval + sd.l_off[s];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* u = uvec + sd.rel_ptr[s];
  if (rank == 0) {
    for (int r = tid; r < f; r += kSolveThreads) T[r] = r < k ? __ldcg(w + c0 + r) : 0.0;
    __syncthreads();
    for (int cc = sd.ch_ptr[s]; cc < sd.ch_ptr[s + 1]; ++cc) {
      const int c = sd.ch[cc];
      const int fu = f_minus_k(sd, c), rp = sd.rel_ptr[c];
      for (int i = tid; i < fu; i += kSolveThreads) T[sd.rel[rp + i]] += __ldcg(uvec + rp + i);
      __syncthreads();
    }
    for (int p0 = 0; p0 < k; p0 += kBlk) {
      const int p1 = min(p0 + kBlk, k), nb = p1 - p0;
      double lv[kBlk];
      int r = -1;
      if (warp == 0) {
        // lane owns row p0+lane of L11: L(p0+lane, p0+q), q < lane
#pragma unroll
        for (int q = 0; q < kBlk; ++q)
          lv[q] = (q < lane && lane < nb) ? __ldcg(L + (p0 + lane) + (p0 + q) * ld) : 0.0;
        double t = lane < nb ? T[p0 + lane] : 0.0;
#pragma unroll
        for (int q = 0; q < kBlk; ++q) {
          if (q < nb) {
            const double wq = __shfl_sync(0xffffffffu, t, q);
            if (lane > q) t -= lv[q] * wq;
          }
        }
        if (lane < nb) T[p0 + lane] = t;
      } else {
        // prefetch this thread's row below the block while the chain runs
        r = p1 + tid - 32;
        if (r < k) {
#pragma unroll
          for (int q = 0; q < kBlk; ++q) lv[q] = q < nb ? __ldcg(L + r + (p0 + q) * ld) : 0.0;
        }
      }
      __syncthreads();
      if (warp != 0) {
        for (; r < k; r += kSolveThreads - 32) {
          if (r >= p1 + kSolveThreads - 32) {  // rows beyond the prefetched one
#pragma unroll
            for (int q = 0; q < kBlk; ++q) lv[q] = q < nb ? __ldcg(L + r + (p0 + q) * ld) : 0.0;
          }
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
          for (int q = 0; q < kBlk; q += 4) {
            a0 += lv[q] * T[p0 + q];
            a1 += lv[q + 1] * T[p0 + q + 1];
            a2 += lv[q + 2] * T[p0 + q + 2];
            a3 += lv[q + 3] * T[p0 + q + 3];
          }
          T[r] -= (a0 + a1) + (a2 + a3);
        }
      }
      __syncthreads();
    }
    for (int q = tid; q < f; q += kSolveThreads) {
      if (q < k)
        w[c0 + q] = T[q];
      else
        u[q - k] = T[q];
    }
  }
  cl.sync();
  // update vector rows [k, f): u_r -= sum_{q<k} L(r, q) w_q, rows split over the cluster
  const int rows = f - k;
  if (rows == 0) return;
  if (rank != 0) {
    for (int q = tid; q < k; q += kSolveThreads) T[q] = __ldcg(w + c0 + q);
    __syncthreads();
  }
  const int chunk = (rows + C - 1) / C;
  const int lo = k + rank * chunk, hi = min(f, lo + chunk);
  for (int r = lo + tid; r < hi; r += kSolveThreads) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const double* Lr = L + r;
    int q = 0;
    for (; q + 4 <= k; q += 4) {
      a0 += __ldcg(Lr + q * ld) * T[q];
      a1 += __ldcg(Lr + (q + 1) * ld) * T[q + 1];
      a2 += __ldcg(Lr + (q + 2) * ld) * T[q + 2];
      a3 += __ldcg(Lr + (q + 3) * ld) * T[q + 3];
    }
    for (; q < k; ++q) a0 += __ldcg(Lr + q * ld) * T[q];
    u[r - k] = __ldcg(u + (r - k)) - ((a0 + a1) + (a2 + a3));
  }
}

__global__ void __launch_bounds__(kSolveThreads, 1)
k_bwd_front(SnDev sd, const double* __restrict__ lval, const double* __restrict__ d,
            const double* __restrict__ w, double* x, const int* __restrict__ nodes) {
  extern __shared__ double X[];
  cg::cluster_group cl = cg::this_cluster();
  const int C = static_cast<int>(cl.num_blocks());
  const int rank = static_cast<int>(cl.block_rank());
  const int s = nodes[blockIdx.x / C];
  const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
  const size_t ld = wide_ld(f);
  const double* L = lval + sd.l_off[s];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int* rows = sd.rows + sd.rows_ptr[s];
  for (int r = k + tid; r < f; r += kSolveThreads) X[r] = __ldcg(x + rows[r]);
  __syncthreads();
  // z_p = w_p / d_p - sum_{r >= k} L(r, p) x_r, warp per pivot column
  for (int p = rank * kSolveWarps + warp; p < k; p += C * kSolveWarps) {
    const double* Lp = L + p * ld;
    double part = 0.0;
    for (int r = k + lane; r < f; r += 32) part += __ldcg(Lp + r) * X[r];
    part = wsum(part);
    if (lane == 0) x[c0 + p] = __ldcg(w + c0 + p) / __ldcg(d + c0 + p) - part;
  }
  cl.sync();
  if (rank != 0) return;
  for (int p = tid; p < k; p += kSolveThreads) X[p] = __ldcg(x + c0 + p);
  __syncthreads();
  const int nblk = (k + kBlk - 1) / kBlk;
  for (int b = nblk - 1; b >= 0; --b) {
    const int p0 = b * kBlk, p1 = min(p0 + kBlk, k), nb = p1 - p0;
    double lc[kBlk];
    if (warp == 0) {
      // lane owns column p0+lane of L11: L(p0+j, p0+lane), j > lane
#pragma unroll
      for (int j = 0; j < kBlk; ++j)
        lc[j] = (j > lane && j < nb) ? __ldcg(L + (p0 + j) + (p0 + lane) * ld) : 0.0;
    } else {
      // later pivots of this front: x_p -= sum_{r in [p1, k)} L(r, p) x_r
      for (int p = p0 + warp - 1; p < p1; p += kSolveWarps - 1) {
        const double* Lp = L + p * ld;
        double part = 0.0;
        for (int r = p1 + lane; r < k; r += 32) part += __ldcg(Lp + r) * X[r];
        part = wsum(part);
        if (lane == 0) X[p] -= part;
      }
    }
    __syncthreads();
    if (warp == 0) {
      double xv = lane < nb ? X[p0 + lane] : 0.0;
#pragma unroll
      for (int p = kBlk - 1; p >= 0; --p) {
        if (p < nb) {
          const double xp = __shfl_sync(0xffffffffu, xv, p);
          if (lane < p) xv -= lc[p] * xp;
        }
      }
      if (lane < nb) X[p0 + lane] = xv;
    }
    __syncthreads();
  }
  for (int p = tid; p < k; p += kSolveThreads) x[c0 + p] = X[p];
}

// ---------------------------------------------------------------------------
template <typename Kern, typename... Args>
static int launch_clustered(Kern kern, int count, int cluster, size_t smem, cudaStream_t st,
                            Args... args) {
  for (; cluster >= 1; cluster >>= 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(count * cluster));
    cfg.blockDim = dim3(kSolveThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(cluster);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess || ncl < 1) {
      cudaGetLastError();
      continue;
    }
    if (cudaLaunchKernelEx(&cfg, kern, args...) == cudaSuccess) return cluster;
    cudaGetLastError();
  }
  return 0;
}

static void solve_init() {
  static bool done = false;
  if (done) return;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncSetAttribute(k_fwd_front, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_bwd_front, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_fwd_front, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
  cudaFuncSetAttribute(k_bwd_front, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
  done = true;
}

int launch_fwd_front(const SnDev& sd, const double* lval, double* w, double* uvec,
                     const int* nodes, int count, int cluster, int max_f, cudaStream_t st) {
  if (count == 0) return cluster;
  solve_init();
  return launch_clustered(k_fwd_front, count, cluster, sizeof(double) * max_f, st, sd, lval, w,
                          uvec, nodes);
}

int launch_bwd_front(const SnDev& sd, const double* lval, const double* d, const double* w,
                     double* x, const int* nodes, int count, int cluster, int max_f,
                     cudaStream_t st) {
  if (count == 0) return cluster;
  solve_init();
  return launch_clustered(k_bwd_front, count, cluster, sizeof(double) * max_f, st, sd, lval, d,
                          w, x, nodes);
}

}  // namespace nclb
