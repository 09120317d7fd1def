// Split extend-add for fronts with very many children -- in Schur mode the
// coupling front receives one contribution per contingency block in every
// column (symbolic.hpp split_ng / usplit_ng).  A wide grid pre-sums groups
// of contributions; the front's own kernel then adds the group sums in group
// order.  Each group is 8 warps, each warp a contiguous slice of the
// contributions (children order) accumulated privately in shared memory, the
// 8 slices combined in warp order: every sum has a fixed order
// (deterministic), only not the child-by-child one of an unsplit front.
#include <cuda_runtime.h>
#include <stdint.h>

#include "cuda_util.hpp"
#include "device.cuh"
#include "launch.hpp"

namespace nclb {

constexpr int kSplitWarps = 8;

// grid (f, ng): column J = blockIdx.x, group g = blockIdx.y.
// Output part[(J * ng + g) * f + r], rows r >= J.
__global__ void __launch_bounds__(kSplitWarps * 32)
k_cc_partial(SnDev sd, FactorDev fd, int s, int ng) {
  extern __shared__ double acc[];  // kSplitWarps x f
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int J = blockIdx.x, g = blockIdx.y;
  const int f = sd.f[s];
  double* a = acc + static_cast<size_t>(warp) * f;
  for (int r = J + lane; r < f; r += 32) a[r] = 0.0;
  __syncwarp();
  const int cb = sd.cc_off[s] + J;
  const int e0 = sd.cc_ptr[cb], n = sd.cc_ptr[cb + 1] - e0;
  const long long W = static_cast<long long>(ng) * kSplitWarps, w = static_cast<long long>(g) * kSplitWarps + warp;
  const int eb = e0 + static_cast<int>(n * w / W), ee = e0 + static_cast<int>(n * (w + 1) / W);
  for (int e = eb; e < ee; ++e) {
    const long long ub = sd.cc_ubase[e];
    const int rb = sd.cc_rbase[e], cw = sd.cc_cnt[e];
    const int cnt = cw & ((1 << 30) - 1);
    const double* U = ((cw >> 30) ? fd.lval : fd.upd) + ub;
    const int* rel = sd.rel + rb;
    for (int i = lane; i < cnt; i += 32) a[rel[i]] += __ldcg(U + i);
    __syncwarp();
  }
  __syncthreads();
  double* out = fd.ccpart + sd.split_off[s] + (static_cast<size_t>(J) * ng + g) * f;
  for (int r = J + threadIdx.x; r < f; r += kSplitWarps * 32) {
    double v = acc[r];
#pragma unroll
    for (int q = 1; q < kSplitWarps; ++q) v += acc[static_cast<size_t>(q) * f + r];
    out[r] = v;
  }
}

// grid ng: group g of the children of s, their forward-solve update vectors
// summed into part[g * f + r]
__global__ void __launch_bounds__(kSplitWarps * 32)
k_uv_partial(SnDev sd, const double* __restrict__ uvec, int s, int ng) {
  extern __shared__ double acc[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x;
  const int f = sd.f[s];
  double* a = acc + static_cast<size_t>(warp) * f;
  for (int r = lane; r < f; r += 32) a[r] = 0.0;
  __syncwarp();
  const int cb = sd.ch_ptr[s], n = sd.ch_ptr[s + 1] - cb;
  const long long W = static_cast<long long>(ng) * kSplitWarps, w = static_cast<long long>(g) * kSplitWarps + warp;
  const int qb = cb + static_cast<int>(n * w / W), qe = cb + static_cast<int>(n * (w + 1) / W);
  for (int q = qb; q < qe; ++q) {
    const int c = sd.ch[q];
    const int fu = f_minus_k(sd, c), rp = sd.rel_ptr[c];
    for (int i = lane; i < fu; i += 32) a[sd.rel[rp + i]] += __ldcg(uvec + rp + i);
    __syncwarp();
  }
  __syncthreads();
  double* out = sd.uvpart + sd.usplit_off[s] + static_cast<size_t>(g) * f;
  for (int r = threadIdx.x; r < f; r += kSplitWarps * 32) {
    double v = acc[r];
#pragma unroll
    for (int q = 1; q < kSplitWarps; ++q) v += acc[static_cast<size_t>(q) * f + r];
    out[r] = v;
  }
}

void launch_cc_partial(const SnDev& sd, const FactorDev& fd, int s, int f, int ng, cudaStream_t st) {
  const size_t smem = sizeof(double) * kSplitWarps * f;
  static PerDeviceOnce init;
  init([] {
    cudaFuncSetAttribute(k_cc_partial, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(double) * kSplitWarps * 512));
  });
  k_cc_partial<<<dim3(f, ng), kSplitWarps * 32, smem, st>>>(sd, fd, s, ng);
}

void launch_uv_partial(const SnDev& sd, const double* uvec, int s, int f, int ng, cudaStream_t st) {
  const size_t smem = sizeof(double) * kSplitWarps * f;
  static PerDeviceOnce init;
  init([] {
    cudaFuncSetAttribute(k_uv_partial, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(double) * kSplitWarps * 512));
  });
  k_uv_partial<<<ng, kSplitWarps * 32, smem, st>>>(sd, uvec, s, ng);
}

}  // namespace nclb
