// Wide-tier numeric factorization (fronts above 32 rows and their ancestors).
//
// A wide front is f x f column-major, resident in HBM/L2 inside the L buffer
// (its first k columns are the L block, the trailing (f-k)^2 corner the
// update matrix the parent extend-adds from).  Building blocks:
//   assemble_tile    -- (CTA) zero a 64x64 tile, scatter A, extend-add the
//                       children's update sub-blocks that land in it, child
//                       by child (deterministic order);
//   panel_step       -- (CTA) static-pivot LDL^T of 32 pivots: warp 0 factors
//                       the 32x32 diagonal block in registers
//                       (sparse.cpp:235-247 pivot rule, inertia, perturbed
//                       counts), every other thread solves one row below it
//                       (TRSM) in registers; L stored scaled in place;
//   warp_update_tile -- (WARP) F22 -= L21 D L21^T on a 32x32 tile with FP64
//                       tensor cores (mma.sync.m8n8k4.f64 = DMMA), operand
//                       fragments loaded straight from L2, no CTA barrier.
// k_wide_front runs a whole tree level in ONE launch: one thread-block
// cluster (1..16 CTAs) per front walks assembly -> [panel -> trailing
// update]* with cluster barriers between phases.  Levels holding huge fronts
// use the three-kernel path (k_wide_assemble / k_wide_panel /
// k_wide_update) so one front can spread over every SM.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "device.cuh"
#include "launch.hpp"
#include "symbolic.hpp"

namespace cg = cooperative_groups;

namespace nclb {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

struct WideSmem {
  double Ud[kWidePanel][kWidePanel + 1];  // unscaled diagonal-block columns u_jp
  double dsh[kWidePanel];
  double rinv[kWidePanel];
  int rg[4];
};

__device__ __forceinline__ const double* child_update(const SnDev& sd, const FactorDev& fd,
                                                      int c) {
  return (sd.wide[c] ? fd.lval : fd.upd) + sd.u_off[c];
}

__device__ __forceinline__ int lower_bound_dev(const int* a, int n, int v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// lower-triangular tile index -> (row block, col block), row >= col
__device__ __forceinline__ void tri_decode(int t, int& i, int& j) {
  int r = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while (r * (r + 1) / 2 > t) --r;
  while ((r + 1) * (r + 2) / 2 <= t) ++r;
  i = r;
  j = t - r * (r + 1) / 2;
}

__device__ __noinline__ void assemble_tile(const SnDev& sd, const FactorDev& fd, const double* kval, int s,
                              int f, int k, double* F, int r_lo, int c_lo, WideSmem& sm) {
  const int tid = threadIdx.x, nth = blockDim.x;
  const int r_hi = min(f, r_lo + kWideTile), c_hi = min(f, c_lo + kWideTile);
  const int tr = r_hi - r_lo, tc = c_hi - c_lo;
  for (int idx = tid; idx < tr * tc; idx += nth) {
    const int r = r_lo + idx % tr, c = c_lo + idx / tr;
    if (r >= c) F[r + static_cast<size_t>(c) * f] = 0.0;
  }
  __syncthreads();
  if (c_lo < k) {
    for (int a = sd.asm_ptr[s] + tid; a < sd.asm_ptr[s + 1]; a += nth) {
      const int pos = sd.asm_pos[a];
      const int c = pos >> 16, r = pos & 0xffff;
      if (c >= c_lo && c < c_hi && r >= r_lo && r < r_hi)
        F[r + static_cast<size_t>(c) * f] += kval[sd.asm_slot[a]];
    }
  }
  __syncthreads();
  for (int cc = sd.ch_ptr[s]; cc < sd.ch_ptr[s + 1]; ++cc) {
    const int c = sd.ch[cc];
    const int fu = f_minus_k(sd, c);
    const int ld = sd.u_ld[c];
    const int* rel = sd.rel + sd.rel_ptr[c];
    const double* U = child_update(sd, fd, c);
    if (tid < 4)
      sm.rg[tid] = lower_bound_dev(rel, fu, tid == 0 ? r_lo : tid == 1 ? r_hi : tid == 2 ? c_lo : c_hi);
    __syncthreads();
    const int i0 = sm.rg[0], i1 = sm.rg[1], j0 = sm.rg[2], j1 = sm.rg[3];
    const int ni = i1 - i0, nj = j1 - j0;
    for (int idx = tid; idx < ni * nj; idx += nth) {
      const int i = i0 + idx % ni, j = j0 + idx / ni;
      if (i >= j) F[rel[i] + static_cast<size_t>(rel[j]) * f] += __ldcg(U + i + static_cast<size_t>(j) * ld);
    }
    __syncthreads();
  }
}

// pivots [p0, p1) of front s; this CTA solves rows [row_lo, row_hi) below
// the diagonal block; `publish`: write L11, D and the counts (one CTA only)
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __noinline__ void panel_step(const FactorDev& fd, int c0, int f, double* F, int p0, int p1,
                           int row_lo, int row_hi, bool publish, double eps, WideSmem& sm,
                           unsigned long long* tr = nullptr) {
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nb = p1 - p0;
  if (tr && tid == 0) tr[0] = globaltimer();
  if (warp == 0) {
    double a[kWidePanel];  // lane owns row `lane` of the diagonal block
#pragma unroll
    for (int j = 0; j < kWidePanel; ++j)
      a[j] = (j <= lane && lane < nb) ? __ldcg(F + (p0 + lane) + static_cast<size_t>(p0 + j) * f) : 0.0;
    int npos = 0, nneg = 0, pert = 0, fail = 0;
#pragma unroll
    for (int p = 0; p < kWidePanel; ++p) {
      if (p < nb) {
        double dp = __shfl_sync(0xffffffffu, a[p], p);
        int pflag = 0;
        if (fabs(dp) < eps) {
          dp = (dp >= 0.0) ? eps : -eps;
          pflag = 1;
        }
        const double rp = __drcp_rn(dp);
        const bool below = lane > p && lane < nb;
        const double u = below ? a[p] : 0.0;
        const double l = u * rp;
        sm.Ud[lane][p] = u;
        if (below) {
          a[p] = l;
          if (!isfinite(l)) fail = 1;
        }
        __syncwarp();
        // batch the column loads before the FMAs: one LDS latency per pivot
        // instead of one per (pivot, row)
        double uv[kWidePanel];
#pragma unroll
        for (int j = p + 1; j < kWidePanel; ++j) uv[j] = sm.Ud[j][p];
#pragma unroll
        for (int j = p + 1; j < kWidePanel; ++j)
          if (j <= lane) a[j] -= l * uv[j];
        if (lane == 0) {
          sm.dsh[p] = dp;
          sm.rinv[p] = rp;
          pert += pflag;
          if (!isfinite(dp) || dp == 0.0) fail = 1;
          if (dp > 0.0)
            npos++;
          else
            nneg++;
        }
      }
    }
    fail = __any_sync(0xffffffffu, fail);
    if (publish) {
#pragma unroll
      for (int p = 0; p < kWidePanel; ++p)
        if (lane > p && lane < nb) F[(p0 + lane) + static_cast<size_t>(p0 + p) * f] = a[p];
      __syncwarp();
      for (int p = lane; p < nb; p += 32) fd.d[c0 + p0 + p] = sm.dsh[p];
      if (lane == 0) {
        if (npos) atomicAdd(fd.stats + 0, npos);
        if (nneg) atomicAdd(fd.stats + 1, nneg);
        if (pert) atomicAdd(fd.stats + 2, pert);
        if (fail) atomicOr(fd.stats + 3, 1);
      }
    }
    if (tr && tid == 0) tr[1] = globaltimer();
  }
  __syncthreads();
  if (tr && tid == 0) tr[2] = globaltimer();
  bool bad = false;
  for (int r = row_lo + tid; r < row_hi; r += nth) {
    double x[kWidePanel];
#pragma unroll
    for (int q = 0; q < kWidePanel; ++q)
      x[q] = q < nb ? __ldcg(F + r + static_cast<size_t>(p0 + q) * f) : 0.0;
#pragma unroll
    for (int p = 0; p < kWidePanel; ++p) {
      double uv[kWidePanel];
#pragma unroll
      for (int j = p + 1; j < kWidePanel; ++j) uv[j] = sm.Ud[j][p];
      const double l = x[p] * sm.rinv[p];
      x[p] = l;
#pragma unroll
      for (int j = p + 1; j < kWidePanel; ++j) x[j] -= l * uv[j];
    }
#pragma unroll
    for (int q = 0; q < kWidePanel; ++q)
      if (q < nb) {
        F[r + static_cast<size_t>(p0 + q) * f] = x[q];
        bad |= !isfinite(x[q]);
      }
  }
  if (bad) atomicOr(fd.stats + 3, 1);
  if (tr && tid == 0) tr[3] = globaltimer();
}

__device__ __forceinline__ void dmma_m8n8k4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// One warp: F[r][c] -= sum_{q in [p0,p1)} L[r][q] d_q L[c][q] on the 32x32
// tile at (r0, q0).  A fragments (row g, k tq) and B fragments (k tq, col g)
// of mma.m8n8k4.f64 are read directly from the column-major front.
__device__ __noinline__ void warp_update_tile(const double* __restrict__ dv, int f, double* F,
                                                 int r0, int q0, int p0, int nb) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 2
  for (int kk = 0; kk < kWidePanel; kk += 4) {
    if (kk >= nb) break;
    const int q = kk + tq;
    const bool qv = q < nb;
    const double* col = F + static_cast<size_t>(p0 + q) * f;
    const double dq = qv ? __ldcg(dv + q) : 0.0;
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = r0 + i * 8 + g;
      a[i] = (qv && r < f) ? __ldcg(col + r) : 0.0;
      const int c = q0 + i * 8 + g;
      b[i] = (qv && c < f) ? __ldcg(col + c) * dq : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_m8n8k4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
  double cur[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = r0 + i * 8 + g, c = q0 + j * 8 + tq * 2 + e;
        cur[i][j][e] = (r < f && c < f && r >= c) ? __ldcg(F + r + static_cast<size_t>(c) * f) : 0.0;
      }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = r0 + i * 8 + g, c = q0 + j * 8 + tq * 2 + e;
        if (r < f && c < f && r >= c) F[r + static_cast<size_t>(c) * f] = cur[i][j][e] - acc[i][j][e];
      }
}

// ---------------------------------------------------------------------------
// one launch per level, one cluster per front
// trace (optional, diagnostic): per front, timestamps (ns) after assembly
// and after every panel / update phase, recorded by cluster rank 0
__global__ void __launch_bounds__(kThreads)
k_wide_front(SnDev sd, FactorDev fd, const double* __restrict__ kval,
             const int* __restrict__ nodes, double eps, unsigned long long* trace) {
  __shared__ WideSmem sm;
  cg::cluster_group cl = cg::this_cluster();
  const int C = static_cast<int>(cl.num_blocks());
  const int rank = static_cast<int>(cl.block_rank());
  const int fi = blockIdx.x / C;
  const int s = nodes[fi];
  const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
  double* F = fd.lval + sd.l_off[s];
  const bool tr = trace && rank == 0 && threadIdx.x == 0;
  int ti = 0;
  if (tr) trace[fi * 128 + ti++] = globaltimer();
  {
    const int T = (f + kWideTile - 1) / kWideTile;
    for (int t = rank; t < T * (T + 1) / 2; t += C) {
      int i, j;
      tri_decode(t, i, j);
      assemble_tile(sd, fd, kval, s, f, k, F, i * kWideTile, j * kWideTile, sm);
    }
  }
  cl.sync();
  if (tr) trace[fi * 128 + ti++] = globaltimer();
  const int warp = threadIdx.x >> 5;
  for (int p0 = 0; p0 < k; p0 += kWidePanel) {
    const int p1 = min(p0 + kWidePanel, k);
    const int rows = f - p1;
    const int chunk = (rows + C - 1) / C;
    const int lo = p1 + rank * chunk, hi = min(f, lo + chunk);
    panel_step(fd, c0, f, F, p0, p1, lo, max(lo, hi), rank == 0, eps, sm,
               (trace && rank == 0 && p0 == 0) ? trace + fi * 128 + 120 : nullptr);
    cl.sync();
    if (tr && ti < 119) trace[fi * 128 + ti++] = globaltimer();
    const int T = (rows + kUpdTile - 1) / kUpdTile;
    for (int t = rank * kWarps + warp; t < T * (T + 1) / 2; t += C * kWarps) {
      int i, j;
      tri_decode(t, i, j);
      warp_update_tile(fd.d + c0 + p0, f, F, p1 + i * kUpdTile, p1 + j * kUpdTile, p0, p1 - p0);
    }
    cl.sync();
    if (tr && ti < 119) trace[fi * 128 + ti++] = globaltimer();
  }
}

// ---------------------------------------------------------------------------
// three-kernel path for levels with huge fronts
__global__ void __launch_bounds__(kThreads)
k_wide_assemble(SnDev sd, FactorDev fd, const double* __restrict__ kval,
                const int4* __restrict__ tasks) {
  __shared__ WideSmem sm;
  const int4 t = tasks[blockIdx.x];
  const int s = t.x;
  const int f = sd.f[s], k = sd.first[s + 1] - sd.first[s];
  assemble_tile(sd, fd, kval, s, f, k, fd.lval + sd.l_off[s], t.y, t.z, sm);
}

__global__ void __launch_bounds__(kThreads)
k_wide_panel(SnDev sd, FactorDev fd, const int2* __restrict__ tasks, int panel, double eps) {
  __shared__ WideSmem sm;
  const int2 task = tasks[blockIdx.x];
  const int s = task.x, rb = task.y;
  const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
  const int p0 = panel * kWidePanel, p1 = min(p0 + kWidePanel, k);
  const int lo = p1 + rb * kPanelRows, hi = min(f, lo + kPanelRows);
  panel_step(fd, c0, f, fd.lval + sd.l_off[s], p0, p1, lo, max(lo, hi), rb == 0, eps, sm);
}

// 8 warps per CTA, one 32x32 tile per warp
__global__ void __launch_bounds__(kThreads)
k_wide_update(SnDev sd, FactorDev fd, const int4* __restrict__ tiles, int count) {
  const int w = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (w >= count) return;
  const int4 t = tiles[w];
  const int s = t.x;
  const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
  const int p0 = t.w * kWidePanel, p1 = min(p0 + kWidePanel, k);
  warp_update_tile(fd.d + c0 + p0, f, fd.lval + sd.l_off[s], t.y, t.z, p0, p1 - p0);
}

// ---------------------------------------------------------------------------
static void wide_init() {
  static bool done = false;
  if (done) return;
  cudaFuncSetAttribute(k_wide_front, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  done = true;
}

int launch_wide_front(const SnDev& sd, const FactorDev& fd, const double* kval, const int* nodes,
                      int count, int cluster, double eps, cudaStream_t st,
                      unsigned long long* trace) {
  if (!count) return cluster;
  wide_init();
  for (; cluster >= 1; cluster >>= 1) {  // largest cluster the device can place
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(count * cluster));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(cluster);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, k_wide_front, &cfg) != cudaSuccess ||
        nclusters < 1) {
      cudaGetLastError();
      continue;
    }
    if (cudaLaunchKernelEx(&cfg, k_wide_front, sd, fd, kval, nodes, eps, trace) == cudaSuccess)
      return cluster;
    cudaGetLastError();
  }
  return 0;
}

void launch_wide_assemble(const SnDev& sd, const FactorDev& fd, const double* kval,
                          const int4* tasks, int count, cudaStream_t st) {
  if (count) k_wide_assemble<<<count, kThreads, 0, st>>>(sd, fd, kval, tasks);
}

void launch_wide_panel(const SnDev& sd, const FactorDev& fd, const int2* tasks, int count,
                       int panel, double eps, cudaStream_t st) {
  if (count) k_wide_panel<<<count, kThreads, 0, st>>>(sd, fd, tasks, panel, eps);
}

void launch_wide_update(const SnDev& sd, const FactorDev& fd, const int4* tiles, int count,
                        cudaStream_t st) {
  if (count)
    k_wide_update<<<(count + kWarps - 1) / kWarps, kThreads, 0, st>>>(sd, fd, tiles, count);
}

}  // namespace nclb
