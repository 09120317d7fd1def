// Micro-benchmark of the wide-tier building blocks in isolation (measurement
// only): per-call cycles of diag_block / trsm_rows / warp_update_tile on a
// synthetic SPD front, first (cold i-cache) and repeated calls; plus DFMA /
// SHFL dependent-chain latencies.
#include "../paper_2510_05885_b200/csrc/wide_kernels.cu"
#include <cstdio>
#include <vector>
using namespace nclb;

__global__ void k_parts(double* F, int f, double* d, int* stats, long long* out) {
  __shared__ PanelSmem sm;
  const int warp = threadIdx.x >> 5;
  for (int rep = 0; rep < 3; ++rep) {
    __syncthreads();
    long long t0 = clock64();
    if (warp == 0) diag_block(F, f, 0, 32, 1e-10, sm, d, nullptr);
    __syncwarp();
    long long t1 = clock64();
    __syncthreads();
    long long t2 = clock64();
    trsm_rows(F + 0, f, 0, 32, 32, 32 + blockDim.x, &sm.Us[0][0], sm.rinv, stats);
    long long t3 = clock64();
    __syncthreads();
    long long t4 = clock64();
    if (warp == 0) warp_update_tile(d, f, F, 32, 32, 0, 32);
    __syncwarp();
    long long t5 = clock64();
    if (threadIdx.x == 0) {
      out[rep * 4 + 0] = t1 - t0;
      out[rep * 4 + 1] = t3 - t2;
      out[rep * 4 + 2] = t5 - t4;
    }
  }
}

__global__ void k_lat(double* io, long long* out) {
  double x = io[threadIdx.x], y = io[threadIdx.x + 32];
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = fma(x, y, 0.5);
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = __drcp_rn(x);
  long long t3 = clock64();
  io[threadIdx.x] = x;
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / 1000; out[1] = (t2 - t1) / 1000; out[2] = (t3 - t2) / 1000; }
}

int main() {
  const int f = 400;
  std::vector<double> h((size_t)f * f, 0.0);
  for (int j = 0; j < f; ++j)
    for (int i = j; i < f; ++i) h[i + (size_t)j * f] = (i == j) ? 50.0 : 0.01 * ((i * 7 + j * 3) % 11 - 5);
  double *F, *d; int* st; long long* out;
  cudaMalloc(&F, h.size() * 8); cudaMalloc(&d, f * 8); cudaMalloc(&st, 16); cudaMalloc(&out, 64 * 8);
  cudaMemcpy(F, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  k_parts<<<1, 384>>>(F, f, d, st, out);
  long long ho[64];
  cudaMemcpy(ho, out, sizeof(ho), cudaMemcpyDeviceToHost);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  for (int r = 0; r < 3; ++r) printf("rep %d: diag %lld  trsm(384 rows) %lld  update_tile %lld cycles\n", r, ho[r*4], ho[r*4+1], ho[r*4+2]);
  double* io; cudaMalloc(&io, 64 * 8); cudaMemcpy(io, h.data(), 64 * 8, cudaMemcpyHostToDevice);
  k_lat<<<1, 32>>>(io, out); cudaMemcpy(ho, out, 24, cudaMemcpyDeviceToHost);
  printf("dependent latency: DFMA %lld  SHFL %lld  DRCP_RN %lld cycles\n", ho[0], ho[1], ho[2]);
  return 0;
}
