// Load-path micro-benchmark (measurement only): how fast one warp pulls
// 32x32 FP64 blocks of a column-major front (ld = f) out of L2.
//   slice-ldcg / slice-plain : the DMMA-fragment pattern (8 rows x 4 columns
//                              per instruction), 48 loads
//   col-ldcg / col-plain     : lane = row, 32 loads each a coalesced column
//   cpasync16                : cp.async.cg 16 B per lane into shared memory
// Every repetition reads columns no earlier repetition touched (cold L1,
// warm L2: the buffer was written by a previous kernel).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__device__ __forceinline__ double ld(const double* p) {
  if (MODE == 0) return __ldcg(p);
  return *p;
}
__global__ void fill(double* F, size_t n) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) F[i] = 1.0 + i % 7;
}
template <int MODE>
__global__ void k_slice(const double* F, int f, double* out, long long* t) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  double s = 0;
  for (int rep = 0; rep < 4; ++rep) {
    const double* B = F + (size_t)(32 * rep) * f;
    __syncwarp();
    long long t0 = clock64();
    double a[8], b[8][4];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const double* col = B + (size_t)(kk * 4 + tq) * f;
      a[kk] = ld<MODE>(col + 64 + g);
#pragma unroll
      for (int j = 0; j < 4; ++j) b[kk][j] = ld<MODE>(col + 128 + j * 8 + g);
    }
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) { s += a[kk]; for (int j = 0; j < 4; ++j) s += b[kk][j]; }
    __syncwarp();
    long long t1 = clock64();
    if (threadIdx.x == 0) t[rep] = t1 - t0;
  }
  out[threadIdx.x] = s;
}
template <int MODE>
__global__ void k_col(const double* F, int f, double* out, long long* t) {
  const int lane = threadIdx.x & 31;
  double s = 0;
  for (int rep = 0; rep < 4; ++rep) {
    const double* B = F + (size_t)(32 * rep) * f;
    __syncwarp();
    long long t0 = clock64();
    double a[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) a[q] = ld<MODE>(B + (size_t)q * f + 64 + lane);
#pragma unroll
    for (int q = 0; q < 32; ++q) s += a[q];
    __syncwarp();
    long long t1 = clock64();
    if (threadIdx.x == 0) t[rep] = t1 - t0;
  }
  out[threadIdx.x] = s;
}
__global__ void k_cpasync(const double* F, int f, double* out, long long* t) {
  __shared__ __align__(16) double sm[32 * 32];
  const int lane = threadIdx.x & 31;
  double s = 0;
  for (int rep = 0; rep < 4; ++rep) {
    const double* B = F + (size_t)(32 * rep) * f;
    __syncwarp();
    long long t0 = clock64();
    // 32 columns x 256 B = 512 chunks of 16 B, 16 per lane
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const int chunk = c * 32 + lane, col = chunk >> 4, off = (chunk & 15) * 2;
      const double* src = B + (size_t)col * f + 64 + off;
      unsigned dst = (unsigned)__cvta_generic_to_shared(sm + col * 32 + off);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    long long t1 = clock64();
    s += sm[lane * 32 + 3];
    if (threadIdx.x == 0) t[rep] = t1 - t0;
  }
  out[threadIdx.x] = s;
}
int main() {
  const int f = 4000;  // even: 16-byte aligned column starts for cp.async
  size_t n = (size_t)f * f;
  double* F; cudaMalloc(&F, n * 8);
  fill<<<1024, 256>>>(F, n);
  double* out; cudaMalloc(&out, 1024); long long* t; cudaMalloc(&t, 64); long long h[4];
  auto pr = [&](const char* nm) {
    cudaDeviceSynchronize(); cudaMemcpy(h, t, 32, cudaMemcpyDeviceToHost);
    printf("%-12s: %lld %lld %lld %lld cycles\n", nm, h[0], h[1], h[2], h[3]);
  };
  k_slice<0><<<1, 32>>>(F, f, out, t); pr("slice-ldcg");
  k_slice<1><<<1, 32>>>(F + 200 * f, f, out, t); pr("slice-plain");
  k_col<0><<<1, 32>>>(F + 400 * f, f, out, t); pr("col-ldcg");
  k_col<1><<<1, 32>>>(F + 600 * f, f, out, t); pr("col-plain");
  k_cpasync<<<1, 32>>>(F + 800 * f, f, out, t); pr("cpasync16");
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
