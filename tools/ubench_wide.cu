// Micro-benchmark of the wide-tier building blocks in isolation (measurement
// only): cycles of diag_block and group_tile on a synthetic front, alone and
// with several groups running concurrently; plus dependent-latency floors.
#include "../paper_2510_05885_b200/csrc/wide_kernels.cu"
#include <cstdio>
#include <vector>
using namespace nclb;

__global__ void fill(double* F, int f, size_t ld) {
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < (size_t)f * ld; idx += (size_t)gridDim.x * blockDim.x) {
    const int i = idx % ld, j = idx / ld;
    F[idx] = (i == j) ? 50.0 : 0.01 * ((i * 7 + j * 3) % 11 - 5);
  }
}

__global__ void __launch_bounds__(512, 1) k_diag(double* F, size_t ld, double* d, long long* out) {
  __shared__ PanelSmem sm;
  __shared__ __align__(16) double D[32 * kSL];
  for (int rep = 0; rep < 40; ++rep) {
    __syncthreads();
    long long t0 = clock64();
    if (threadIdx.x < 32) diag_block(F, ld, 32 * (rep % 8), 32, 1e-10, sm, D, d, nullptr, nullptr);
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0 && rep < 3) out[rep] = t1 - t0;
  }
}

__global__ void __launch_bounds__(512, 1) k_group(double* F, size_t ld, int f, double* d, long long* out, int ngroups, int ntiles) {
  extern __shared__ __align__(16) double dyn[];
  GroupSmem* G = reinterpret_cast<GroupSmem*>(dyn);
  const int grp = threadIdx.x >> 7, gt = threadIdx.x & 127;
  __syncthreads();
  long long t0 = clock64();
  if (grp < ngroups)
    for (int t = 0; t < ntiles; ++t)
      group_tile(F, ld, f, d, 0, 32, 32 + 32 * (grp * ntiles + t) % 3000, 64, G[grp], gt, 1 + grp);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) *out = t1 - t0;
}

int main() {
  const int f = 3200;
  const size_t ld = wide_ld(f);
  double *F, *d; long long* out;
  cudaMalloc(&F, (size_t)f * ld * 8); cudaMalloc(&d, f * 8); cudaMalloc(&out, 64 * 8);
  fill<<<1024, 256>>>(F, f, ld);
  cudaMemcpy(d, F, 8 * 32, cudaMemcpyDeviceToDevice);
  long long ho[8];
  k_diag<<<1, 512>>>(F, ld, d, out);
  cudaMemcpy(ho, out, 24, cudaMemcpyDeviceToHost);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  printf("diag_block: %lld %lld %lld cycles\n", ho[0], ho[1], ho[2]);
  cudaFuncSetAttribute(k_group, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * (int)sizeof(GroupSmem));
  for (int ng : {1, 2, 4})
    for (int nt : {1, 4}) {
      k_group<<<1, 512, 4 * sizeof(GroupSmem)>>>(F, ld, f, d, out, ng, nt);
      cudaMemcpy(ho, out, 8, cudaMemcpyDeviceToHost);
      printf("group_tile: %d groups x %d tiles: %lld cycles (%lld per tile per group)  %s\n", ng, nt, ho[0], ho[0] / nt,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
