// Micro-benchmarks of the latencies the wide-tier factorization is built on
// (measurement only): cluster barrier cost by cluster size, dependent L2 load
// latency, __syncthreads cost.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_csync(long long* out, int iters) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = (t1 - t0) / iters;
}
__global__ void k_bsync(long long* out, int iters) {
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = (t1 - t0) / iters;
}
__global__ void k_chase(const int* next, int iters, long long* out, int* sink) {
  int p = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = __ldcg(next + p);
  long long t1 = clock64();
  *out = (t1 - t0) / iters;
  *sink = p;
}
int main() {
  long long* d; cudaMalloc(&d, 8); long long h;
  for (int C : {1, 2, 4, 8, 16}) {
    for (int th : {256, 384, 512}) {
      cudaFuncSetAttribute(k_csync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(C); cfg.blockDim = dim3(th);
      cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = C; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
      cfg.attrs = a; cfg.numAttrs = 1;
      cudaError_t e = cudaLaunchKernelEx(&cfg, k_csync, d, 1000);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("cluster.sync C=%2d threads=%d: %lld cycles (%s)\n", C, th, h, cudaGetErrorString(e));
    }
  }
  k_bsync<<<1, 384>>>(d, 1000); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("__syncthreads 384: %lld cycles\n", h);
  for (int kb : {64, 1024, 16384, 65536}) {
    int n = kb * 256;  // ints
    int* hn = new int[n];
    int stride = 4099;  // pseudo-random walk in units of 32 ints
    int lines = n / 32;
    for (int i = 0; i < lines; ++i) hn[i * 32] = ((i + stride) % lines) * 32;
    int* dn; cudaMalloc(&dn, n * 4); cudaMemcpy(dn, hn, n * 4, cudaMemcpyHostToDevice);
    int* sink; cudaMalloc(&sink, 4);
    k_chase<<<1, 1>>>(dn, 20000, d, sink); cudaDeviceSynchronize();
    k_chase<<<1, 1>>>(dn, 20000, d, sink); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("dependent ldcg chase over %d KB: %lld cycles/load\n", kb, h);
    cudaFree(dn); delete[] hn;
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock %d kHz\n", clk);
  return 0;
}
