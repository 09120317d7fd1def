// Micro-benchmark: the wide tier's 32-pivot diagonal block (diag_block), one
// warp, staged block in shared memory, repeated; cycles per block for
// variants: V0 plain, V1 with the lock-step progress flag, V2 + the stats
// atomics.  Built against a copy of wide_kernels.cu (WK=path), so the same
// source can be compared before and after a change:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I paper_2510_05885_b200/csrc -DWK='"<path>/wide_kernels.cu"' tools/ubench_diag.cu -o tools/ubench_diag
#include WK
#include <cstdio>
#include <string>
#include <vector>

namespace nclb {
std::string& last_error() {
  static thread_local std::string s;
  return s;
}
template <int V>
__global__ void k_ub_diag(const double* A, double* dout, int* stats, long long* cyc, int iters, double eps) {
  __shared__ PanelSmem sm;
  __shared__ __align__(16) double D[kWidePanel * kSL];
  const int lane = threadIdx.x;
  for (int j = 0; j < 32; ++j) D[j * kSL + lane] = A[j * 32 + lane];
  if (lane == 0) sm.prog = 0;
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    diag_block(nullptr, 0, 0, 32, eps, sm, D, V >= 2 ? dout : nullptr, V >= 2 ? stats : nullptr,
               V >= 1 ? &sm.prog : nullptr, true);
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) cyc[0] = (t1 - t0) / iters;
  if (V < 2) dout[lane] = sm.rinv[lane];
}
#ifdef HAVE_DIAG2
// two-warp variant (diag_block2): 64 threads
__global__ void k_ub_diag2(const double* A, double* dout, long long* cyc, int iters, double eps) {
  __shared__ PanelSmem sm;
  __shared__ __align__(16) double D[kWidePanel * kSL];
  const int t = threadIdx.x;
  for (int j = t >> 5; j < 32; j += 2) D[j * kSL + (t & 31)] = A[j * 32 + (t & 31)];
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (t == 0) {
      sm.prog = 0;
      sm.hw = 0;
    }
    __syncthreads();
    diag_block2(t >> 5, 32, eps, sm, D, nullptr, nullptr, &sm.prog);
    __syncthreads();
  }
  long long t1 = clock64();
  if (t == 0) cyc[0] = (t1 - t0) / iters;
  if (t < 32) {
    dout[t] = sm.rinv[t];
    for (int p = 0; p < 32; ++p) dout[64 + p * 32 + t] = sm.Lsh[t][p];
  }
}
#endif
template <int V>
__global__ void k_ub_lsh(const double* A, double* dout, double eps) {
  __shared__ PanelSmem sm;
  __shared__ __align__(16) double D[kWidePanel * kSL];
  const int lane = threadIdx.x;
  for (int j = 0; j < 32; ++j) D[j * kSL + lane] = A[j * 32 + lane];
  if (lane == 0) sm.prog = 0;
  __syncwarp();
  diag_block(nullptr, 0, 0, 32, eps, sm, D, nullptr, nullptr, nullptr, true);
  __syncwarp();
  dout[lane] = sm.rinv[lane];
  for (int p = 0; p < 32; ++p) dout[64 + p * 32 + lane] = sm.Lsh[lane][p];
}
}  // namespace nclb

int main(int argc, char** argv) {
  using namespace nclb;
  std::vector<double> h(32 * 32);
  unsigned s = 12345;
  for (int j = 0; j < 32; ++j)
    for (int i = 0; i < 32; ++i) {
      s = s * 1664525u + 1013904223u;
      const double r = (s >> 8) * (1.0 / 16777216.0) - 0.5;
      h[j * 32 + i] = (i == j) ? 40.0 + r : r;
    }
  for (int j = 0; j < 32; ++j)
    for (int i = 0; i < j; ++i) h[j * 32 + i] = h[i * 32 + j];
  double *A, *dout;
  int* stats;
  long long* cyc;
  cudaMalloc(&A, 8 * 1024);
  cudaMalloc(&dout, 8 * 64);
  cudaMalloc(&stats, 16);
  cudaMalloc(&cyc, 8);
  cudaMemcpy(A, h.data(), 8 * 1024, cudaMemcpyHostToDevice);
  long long c[3];
  for (int v = 0; v < 3; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      if (v == 0) k_ub_diag<0><<<1, 32>>>(A, dout, stats, cyc, 200, 1e-10);
      if (v == 1) k_ub_diag<1><<<1, 32>>>(A, dout, stats, cyc, 200, 1e-10);
      if (v == 2) k_ub_diag<2><<<1, 32>>>(A, dout, stats, cyc, 200, 1e-10);
    }
    cudaMemcpy(&c[v], cyc, 8, cudaMemcpyDeviceToHost);
  }
  std::printf("diag_block 32 pivots, cycles per block: plain %lld  +progress flag %lld  +stats %lld  (%.1f / pivot)\n",
              c[0], c[1], c[2], c[0] / 32.0);
  if (argc > 1) {  // dump 1/d and L of the block (bitwise comparison of two builds)
    double* o;
    cudaMalloc(&o, 8 * (64 + 1024));
    std::vector<double> r(64 + 1024);
    for (int m = 0; m < 2; ++m) {  // m = 1: a block with a tiny pivot (static perturbation)
      if (m == 1) {
        std::vector<double> h2 = h;
        h2[5 * 32 + 5] = 1e-14;
        cudaMemcpy(A, h2.data(), 8 * 1024, cudaMemcpyHostToDevice);
      }
      k_ub_lsh<0><<<1, 32>>>(A, o, 1e-10);
      cudaMemcpy(r.data(), o, r.size() * 8, cudaMemcpyDeviceToHost);
      FILE* f = std::fopen((std::string(argv[1]) + (m ? ".tiny" : "")).c_str(), "wb");
      std::fwrite(r.data(), 8, r.size(), f);
      std::fclose(f);
    }
  }
#ifdef HAVE_DIAG2
  double* o2;
  cudaMalloc(&o2, 8 * (64 + 1024));
  std::vector<double> r1(64 + 1024), r2(64 + 1024);
  k_ub_lsh<0><<<1, 32>>>(A, o2, 1e-10);
  cudaMemcpy(r1.data(), o2, r1.size() * 8, cudaMemcpyDeviceToHost);
  long long c2 = 0;
  for (int rep = 0; rep < 2; ++rep) k_ub_diag2<<<1, 64>>>(A, o2, cyc, 200, 1e-10);
  cudaMemcpy(&c2, cyc, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(r2.data(), o2, r2.size() * 8, cudaMemcpyDeviceToHost);
  int diff = 0;
  for (int i = 0; i < 32; ++i) diff += r1[i] != r2[i];
  for (int p = 0; p < 32; ++p)
    for (int i = p + 1; i < 32; ++i) diff += r1[64 + p * 32 + i] != r2[64 + p * 32 + i];
  std::printf("diag_block2 (two warps): %lld cycles per block (%.1f / pivot), entries differing from diag_block: %d\n",
              c2, c2 / 32.0, diff);
#ifdef DIAG2_PROBE
  long long pr[4];
  cudaMemcpyFromSymbol(pr, g_probe, sizeof(pr));
  std::printf("  per block: chain waits for hand-over %lld cycles, bulk waits for pivots %lld cycles\n",
              pr[0] / 400, pr[1] / 400);
#endif
#endif
  return cudaGetLastError() != cudaSuccess;
}
