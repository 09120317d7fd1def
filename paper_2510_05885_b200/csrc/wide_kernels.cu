// Wide-tier numeric factorization (fronts above 32 rows and their ancestors).
//
// A wide front is f x f column-major, resident in HBM/L2 inside the L buffer
// (its first k columns are the L block, the trailing (f-k)^2 corner the
// update matrix the parent extend-adds from).  Building blocks, all written
// as compact loops so the code stays resident in the instruction cache (a
// fully unrolled 32-pivot body is tens of KB of straight-line SASS that is
// fetched from L2 on every panel -- that, not arithmetic, was the cost):
//   assemble_col  -- (WARP) one front column: zero, scatter A, extend-add the
//                    children's columns that land in it, child by child
//                    (deterministic order), accumulated in shared memory and
//                    written once;
//   diag_block    -- (WARP) static-pivot LDL^T of a <=32-pivot diagonal block
//                    (sparse.cpp:235-247 pivot rule, inertia, perturbed
//                    counts); a lane owns one row in registers and the row is
//                    rotated one column per pivot, so every register index is
//                    static while the pivot loop stays a loop;
//   trsm_rows     -- (THREAD per row) the rows below the block against the
//                    unscaled diagonal columns, same rotation scheme;
//   warp_update_tile -- (WARP) F22 -= L21 D L21^T on a 32x32 tile with FP64
//                    tensor cores (mma.sync.m8n8k4.f64 = DMMA).
// k_wide_front runs a whole tree level in ONE launch: one thread-block
// cluster (1..16 CTAs) per front walks assembly -> [panel -> trailing
// update]* with cluster barriers between phases.  Levels holding huge fronts
// use the multi-kernel path (k_wide_assemble / k_wide_diag / k_wide_panel /
// k_wide_update) so one front spreads over every SM.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "device.cuh"
#include "launch.hpp"
#include "symbolic.hpp"

namespace cg = cooperative_groups;

namespace nclb {

constexpr int kThreads = 384;
constexpr int kWarps = kThreads / 32;
constexpr int kHugeThreads = 256;
constexpr unsigned kFull = 0xffffffffu;

// Us[p][j] = unscaled u = F(p0+p+1+j, p0+p) after the first p pivots (zero
// past the block); row p is what every row below subtracts at pivot p.
struct PanelSmem {
  double Us[kWidePanel][kWidePanel];
  double rinv[kWidePanel];
  double Lsh[kWidePanel][kWidePanel + 1];  // scaled L11 (published late)
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// lower-triangular tile index -> (row block, col block), row >= col
__device__ __forceinline__ void tri_decode(int t, int& i, int& j) {
  int r = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while (r * (r + 1) / 2 > t) --r;
  while ((r + 1) * (r + 2) / 2 <= t) ++r;
  i = r;
  j = t - r * (r + 1) / 2;
}

// ---------------------------------------------------------------------------
// assembly of front column J (one warp).  acc: f doubles of shared memory
// private to this warp, or nullptr to accumulate in place (huge fronts).
__device__ __noinline__ void assemble_col(const SnDev& sd, const FactorDev& fd,
                                          const double* __restrict__ kval, int s, int c0, int k,
                                          int f, double* F, int J, double* acc) {
  const int lane = threadIdx.x & 31;
  double* col = F + static_cast<size_t>(J) * f;
  double* a = acc ? acc : col;
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
  if (acc)
    for (int r = J + lane; r < f; r += 32) col[r] = a[r];
}

// ---------------------------------------------------------------------------
// static-pivot LDL^T of the nb-pivot diagonal block at p0 (one warp).  Fills
// sm.Us / sm.rinv (and sm.Lsh with the scaled L11).  With `dout` (publisher
// only) writes D and adds the inertia / perturbed / failure counts.
__device__ __noinline__ void diag_block(const double* F, int f, int p0, int nb, double eps,
                                        PanelSmem& sm, double* dout, int* stats) {
  const int lane = threadIdx.x & 31;
  double* us = &sm.Us[0][0];
  for (int i = lane; i < kWidePanel * kWidePanel; i += 32) us[i] = 0.0;
  double a[kWidePanel];  // a[j] = current F(p0+lane, p0+p+j)
#pragma unroll
  for (int j = 0; j < kWidePanel; ++j)
    a[j] = (lane < nb && j <= lane) ? __ldcg(F + (p0 + lane) + static_cast<size_t>(p0 + j) * f) : 0.0;
  __syncwarp();
  int npos = 0, nneg = 0, pert = 0, fail = 0;
#pragma unroll 1
  for (int p = 0; p < nb; ++p) {
    double dp = __shfl_sync(kFull, a[0], p);
    int pflag = 0;
    if (fabs(dp) < eps) {
      dp = (dp >= 0.0) ? eps : -eps;
      pflag = 1;
    }
    const double rp = __drcp_rn(dp);
    const bool below = lane > p && lane < nb;
    const double u = below ? a[0] : 0.0;
    const double l = u * rp;
    if (below) {
      sm.Us[p][lane - p - 1] = u;
      sm.Lsh[lane][p] = l;
      if (!isfinite(l)) fail = 1;
    }
    if (lane == 0) {
      sm.rinv[p] = rp;
      if (dout) dout[p] = dp;
      pert += pflag;
      if (!isfinite(dp) || dp == 0.0) fail = 1;
      if (dp > 0.0)
        npos++;
      else
        nneg++;
    }
    __syncwarp();
    const double2* up = reinterpret_cast<const double2*>(sm.Us[p]);
#pragma unroll
    for (int j = 0; j < kWidePanel; j += 2) {
      const double2 v = up[j >> 1];
      a[j] = a[j + 1] - l * v.x;
      a[j + 1] = (j + 2 < kWidePanel ? a[j + 2] : 0.0) - l * v.y;
    }
  }
  __syncwarp();
  if (stats) {
    fail = __any_sync(kFull, fail);
    if (lane == 0) {
      if (npos) atomicAdd(stats + 0, npos);
      if (nneg) atomicAdd(stats + 1, nneg);
      if (pert) atomicAdd(stats + 2, pert);
      if (fail) atomicOr(stats + 3, 1);
    }
  }
}

// rows [row_lo, row_hi) of panel columns [p0, p0+nb): L(r, :) from the
// unscaled diagonal columns us (32x32) and 1/d (thread per row)
__device__ __noinline__ void trsm_rows(double* F, int f, int p0, int nb, int row_lo, int row_hi,
                                       const double* us, const double* rinv, int* stats) {
  bool bad = false;
  for (int r = row_lo + static_cast<int>(threadIdx.x); r < row_hi; r += blockDim.x) {
    double x[kWidePanel];
    double* row = F + r + static_cast<size_t>(p0) * f;
#pragma unroll
    for (int q = 0; q < kWidePanel; ++q) x[q] = q < nb ? __ldcg(row + static_cast<size_t>(q) * f) : 0.0;
#pragma unroll 1
    for (int p = 0; p < nb; ++p) {
      const double l = x[0] * rinv[p];
      row[static_cast<size_t>(p) * f] = l;
      bad |= !isfinite(l);
      const double2* up = reinterpret_cast<const double2*>(us + p * kWidePanel);
#pragma unroll
      for (int j = 0; j < kWidePanel; j += 2) {
        const double2 v = up[j >> 1];
        x[j] = x[j + 1] - l * v.x;
        x[j + 1] = (j + 2 < kWidePanel ? x[j + 2] : 0.0) - l * v.y;
      }
    }
  }
  if (bad) atomicOr(stats + 3, 1);
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
  // all 32 loads in flight before the first store
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
// one launch per level, one cluster per front.
// trace (optional, diagnostic): per front, timestamps (ns) after assembly
// and after every panel / update phase, recorded by cluster rank 0
__global__ void __launch_bounds__(kThreads, 1)
k_wide_front(SnDev sd, FactorDev fd, const double* __restrict__ kval,
             const int* __restrict__ nodes, double eps, int acc_f, unsigned long long* trace) {
  __shared__ PanelSmem sm;
  extern __shared__ double acc_smem[];
  cg::cluster_group cl = cg::this_cluster();
  const int C = static_cast<int>(cl.num_blocks());
  const int rank = static_cast<int>(cl.block_rank());
  const int fi = blockIdx.x / C;
  const int s = nodes[fi];
  const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
  double* F = fd.lval + sd.l_off[s];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool tr = trace && rank == 0 && threadIdx.x == 0;
  int ti = 0;
  if (tr) trace[fi * 128 + ti++] = globaltimer();
  {
    double* acc = acc_smem + static_cast<size_t>(warp) * acc_f;
    for (int J = rank * kWarps + warp; J < f; J += C * kWarps)
      assemble_col(sd, fd, kval, s, c0, k, f, F, J, acc);
  }
  cl.sync();
  if (tr) trace[fi * 128 + ti++] = globaltimer();
  for (int p0 = 0; p0 < k; p0 += kWidePanel) {
    const int p1 = min(p0 + kWidePanel, k), nb = p1 - p0;
    const int rows = f - p1;
    const int chunk = (rows + C - 1) / C;
    const int lo = p1 + rank * chunk, hi = min(f, lo + chunk);
    // detailed stamps of the second panel (the first when k <= 32)
    unsigned long long* dt = (tr && p0 == (k > kWidePanel ? kWidePanel : 0)) ? trace + fi * 128 + 120
                                                                             : nullptr;
    if (dt) dt[0] = globaltimer();
    // every CTA factors the diagonal block itself (no extra cluster barrier);
    // rank 0 publishes D and the counts now, L11 after the barrier below
    // (other CTAs may still be reading the unfactored block until then)
    if (warp == 0)
      diag_block(F, f, p0, nb, eps, sm, rank == 0 ? fd.d + c0 + p0 : nullptr,
                 rank == 0 ? fd.stats : nullptr);
    if (dt) dt[1] = globaltimer();
    __syncthreads();
    if (dt) dt[2] = globaltimer();
    trsm_rows(F, f, p0, nb, lo, max(lo, hi), &sm.Us[0][0], sm.rinv, fd.stats);
    if (dt) dt[3] = globaltimer();
    cl.sync();
    if (dt) dt[4] = globaltimer();
    if (tr && ti < 119) trace[fi * 128 + ti++] = globaltimer();
    if (rank == 0 && warp == 0)
      for (int p = 0; p < nb; ++p)
        if (lane > p && lane < nb) F[(p0 + lane) + static_cast<size_t>(p0 + p) * f] = sm.Lsh[lane][p];
    if (dt) dt[5] = globaltimer();
    const int T = (rows + kUpdTile - 1) / kUpdTile;
    for (int t = rank * kWarps + warp; t < T * (T + 1) / 2; t += C * kWarps) {
      int i, j;
      tri_decode(t, i, j);
      warp_update_tile(fd.d + c0 + p0, f, F, p1 + i * kUpdTile, p1 + j * kUpdTile, p0, nb);
    }
    if (dt) dt[6] = globaltimer();
    cl.sync();
    if (dt) dt[7] = globaltimer();
    if (tr && ti < 119) trace[fi * 128 + ti++] = globaltimer();
  }
}

// ---------------------------------------------------------------------------
// multi-kernel path for levels with huge fronts
__global__ void __launch_bounds__(kHugeThreads)
k_wide_assemble(SnDev sd, FactorDev fd, const double* __restrict__ kval,
                const int4* __restrict__ tasks) {
  const int4 t = tasks[blockIdx.x];
  const int s = t.x, J = t.y + (threadIdx.x >> 5);
  const int c0 = sd.first[s], f = sd.f[s], k = sd.first[s + 1] - c0;
  if (J < min(f, t.y + kAsmCols)) assemble_col(sd, fd, kval, s, c0, k, f, fd.lval + sd.l_off[s], J, nullptr);
}

// one warp per front: diagonal block of panel `panel`, publishes L11, D and
// the counts, and leaves {Us, rinv} in the scratch slot of the task
__global__ void __launch_bounds__(32)
k_wide_diag(SnDev sd, FactorDev fd, const int* __restrict__ fronts, int panel, double eps) {
  __shared__ PanelSmem sm;
  const int s = fronts[blockIdx.x];
  const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
  const int p0 = panel * kWidePanel, nb = min(p0 + kWidePanel, k) - p0;
  double* F = fd.lval + sd.l_off[s];
  diag_block(F, f, p0, nb, eps, sm, fd.d + c0 + p0, fd.stats);
  const int lane = threadIdx.x;
  for (int p = 0; p < nb; ++p)
    if (lane > p && lane < nb) F[(p0 + lane) + static_cast<size_t>(p0 + p) * f] = sm.Lsh[lane][p];
  double* scr = fd.dscr + static_cast<size_t>(blockIdx.x) * (kWidePanel * kWidePanel + kWidePanel);
  for (int i = lane; i < kWidePanel * kWidePanel; i += 32) scr[i] = (&sm.Us[0][0])[i];
  scr[kWidePanel * kWidePanel + lane] = sm.rinv[lane];
}

__global__ void __launch_bounds__(kHugeThreads)
k_wide_panel(SnDev sd, FactorDev fd, const int4* __restrict__ tasks, int panel) {
  __shared__ __align__(16) double us[kWidePanel * kWidePanel + kWidePanel];
  const int4 task = tasks[blockIdx.x];
  const int s = task.x, rb = task.y;
  const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
  const int p0 = panel * kWidePanel, p1 = min(p0 + kWidePanel, k);
  const double* scr = fd.dscr + static_cast<size_t>(task.z) * (kWidePanel * kWidePanel + kWidePanel);
  for (int i = threadIdx.x; i < kWidePanel * kWidePanel + kWidePanel; i += blockDim.x) us[i] = scr[i];
  __syncthreads();
  const int lo = p1 + rb * kPanelRows, hi = min(f, lo + kPanelRows);
  trsm_rows(fd.lval + sd.l_off[s], f, p0, p1 - p0, lo, max(lo, hi), us,
            us + kWidePanel * kWidePanel, fd.stats);
}

// 8 warps per CTA, one 32x32 tile per warp
__global__ void __launch_bounds__(kHugeThreads)
k_wide_update(SnDev sd, FactorDev fd, const int4* __restrict__ tiles, int count) {
  const int w = blockIdx.x * (kHugeThreads / 32) + (threadIdx.x >> 5);
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
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncSetAttribute(k_wide_front, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       optin - static_cast<int>(sizeof(PanelSmem)));
  done = true;
}

int wide_front_smem(int max_f) {
  return static_cast<int>(sizeof(double)) * kWarps * (max_f > 0 ? max_f : 1);
}

int launch_wide_front(const SnDev& sd, const FactorDev& fd, const double* kval, const int* nodes,
                      int count, int cluster, int max_f, double eps, cudaStream_t st,
                      unsigned long long* trace) {
  if (!count) return cluster;
  wide_init();
  for (; cluster >= 1; cluster >>= 1) {  // largest cluster the device can place
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(count * cluster));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = static_cast<size_t>(wide_front_smem(max_f));
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
    if (cudaLaunchKernelEx(&cfg, k_wide_front, sd, fd, kval, nodes, eps, max_f, trace) ==
        cudaSuccess)
      return cluster;
    cudaGetLastError();
  }
  return 0;
}

void launch_wide_assemble(const SnDev& sd, const FactorDev& fd, const double* kval,
                          const int4* tasks, int count, cudaStream_t st) {
  if (count) k_wide_assemble<<<count, kHugeThreads, 0, st>>>(sd, fd, kval, tasks);
}

void launch_wide_diag(const SnDev& sd, const FactorDev& fd, const int* fronts, int count,
                      int panel, double eps, cudaStream_t st) {
  if (count) k_wide_diag<<<count, 32, 0, st>>>(sd, fd, fronts, panel, eps);
}

void launch_wide_panel(const SnDev& sd, const FactorDev& fd, const int4* tasks, int count,
                       int panel, cudaStream_t st) {
  if (count) k_wide_panel<<<count, kHugeThreads, 0, st>>>(sd, fd, tasks, panel);
}

void launch_wide_update(const SnDev& sd, const FactorDev& fd, const int4* tiles, int count,
                        cudaStream_t st) {
  if (count)
    k_wide_update<<<(count + kHugeThreads / 32 - 1) / (kHugeThreads / 32), kHugeThreads, 0, st>>>(
        sd, fd, tiles, count);
}

}  // namespace nclb
