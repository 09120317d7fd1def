// Micro-benchmark: one warp, the warp-tier register pivot loop (k pivots of a
// f-row front), repeated; reports cycles per front for variants.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kWF = 32, kFLD = 33;
template <int V>
__global__ void kpiv(const double* __restrict__ A, double* Lout, double* dout, int k, int f, int iters,
                     long long* cyc, double eps) {
  __shared__ double F[kWF * kFLD];
  const int lane = threadIdx.x;
  for (int j = 0; j < f; ++j) F[j * kFLD + lane] = A[j * 32 + lane];
  __syncwarp();
  int fail = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    double fr[kWF];
#pragma unroll
    for (int j = 0; j < kWF; ++j) fr[j] = (j < f && lane < f) ? F[j * kFLD + lane] : 0.0;
    double* Lb = Lout + (it & 63) * 1024;
    for (int p = 0; p < k; ++p) {
      double dp = __shfl_sync(0xffffffffu, fr[0], p);
      if (fabs(dp) < eps) dp = (dp >= 0.0) ? eps : -eps;
      const bool mine = lane > p && lane < f;
      const double u = fr[0];
      double l;
      if (V == 2)
        l = mine ? u * dp : 0.0;
      else
        l = mine ? u / dp : 0.0;
      const int fmp = f - p;
#pragma unroll
      for (int b8 = 0; b8 < kWF; b8 += 8) {
        if (b8 < fmp) {
#pragma unroll
          for (int j = b8; j < b8 + 8; ++j) {
            if (j > 0) {
              const double uj = __shfl_sync(0xffffffffu, u, (p + j) & 31);
              fr[j - 1] = fr[j] - l * uj;
            }
          }
        }
      }
      fr[kWF - 1] = 0.0;
      if (V != 1) {
        if (mine) {
          Lb[lane + p * f] = l;
          if (!isfinite(l)) fail = 1;
        }
        if (lane == 0) dout[(it & 63) * 32 + p] = dp;
      }
    }
    if (V == 1) Lb[lane] = fr[0] + fr[1];
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) cyc[V] = (t1 - t0) / iters;
  if (fail) Lout[0] = 1;
}

__device__ __forceinline__ double rcp_nr(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}
// register rows + shared-memory column broadcast + reciprocal + lookahead
template <int V>
__global__ void kv3(const double* __restrict__ A, double* Lout, double* dout, int k, int f, int iters,
                    long long* cyc, double eps) {
  __shared__ double F[kWF * kFLD];
  __shared__ __align__(16) double cb[2][kWF + 2];
  const int lane = threadIdx.x;
  for (int j = 0; j < f; ++j) F[j * kFLD + lane] = A[j * 32 + lane];
  __syncwarp();
  int fail = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    double fr[kWF + 1];
#pragma unroll
    for (int j = 0; j < kWF; ++j) fr[j] = (j < f && lane < f) ? F[j * kFLD + lane] : 0.0;
    fr[kWF] = 0.0;
    double* Lb = Lout + (it & 63) * 1024;
    double dnext = __shfl_sync(0xffffffffu, fr[0], 0);
    for (int p = 0; p < k; ++p) {
      double dp = dnext;
      if (fabs(dp) < eps) dp = (dp >= 0.0) ? eps : -eps;
      const bool mine = lane > p && lane < f;
      const double u = fr[0];
      double* cbp = cb[p & 1];
      if (lane >= p) cbp[lane - p] = u;
      const double rp = rcp_nr(dp);
      const double l = mine ? u * rp : 0.0;
      __syncwarp();
      fr[0] = fr[1] - l * cbp[1];
      dnext = __shfl_sync(0xffffffffu, fr[0], (p + 1) & 31);
      const int fmp = f - p;
#pragma unroll
      for (int b8 = 0; b8 < kWF; b8 += 8) {
        if (b8 < fmp) {
#pragma unroll
          for (int j = (b8 == 0 ? 2 : b8); j < b8 + 8; j += 2) {
            const double2 v = *reinterpret_cast<const double2*>(cbp + j);
            fr[j - 1] = fr[j] - l * v.x;
            fr[j] = fr[j + 1] - l * v.y;
          }
        }
      }
      if (V != 1) {
        if (mine) {
          Lb[lane + p * f] = l;
          if (!isfinite(l)) fail = 1;
        }
        if (lane == 0) dout[(it & 63) * 32 + p] = dp;
      }
    }
    if (V == 1) Lb[lane] = fr[0] + fr[1];
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) cyc[4 + V] = (t1 - t0) / iters;
  if (fail) Lout[0] = 1;
}
// smem variant (the pre-register kernel)
__global__ void ksm(const double* __restrict__ A, double* Lout, double* dout, int k, int f, int iters,
                    long long* cyc, double eps) {
  __shared__ double F0[kWF * kFLD];
  __shared__ double F[kWF * kFLD];
  const int lane = threadIdx.x;
  for (int j = 0; j < f; ++j) F0[j * kFLD + lane] = A[j * 32 + lane];
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int j = 0; j < f; ++j) F[j * kFLD + lane] = F0[j * kFLD + lane];
    __syncwarp();
    double* Lb = Lout + (it & 63) * 1024;
    for (int p = 0; p < k; ++p) {
      const double u = (lane < f) ? F[p * kFLD + lane] : 0.0;
      double dp = __shfl_sync(0xffffffffu, u, p);
      if (fabs(dp) < eps) dp = (dp >= 0.0) ? eps : -eps;
      const bool mine = lane > p && lane < f;
      const double l = mine ? u / dp : 0.0;
#pragma unroll 4
      for (int j = p + 1; j < f; ++j) {
        const double uj = F[p * kFLD + j];
        if (lane >= j && lane < f) F[j * kFLD + lane] -= l * uj;
      }
      if (mine) Lb[lane + p * f] = l;
      if (lane == 0) dout[(it & 63) * 32 + p] = dp;
      __syncwarp();
    }
  }
  long long t1 = clock64();
  if (lane == 0) cyc[3] = (t1 - t0) / iters;
}
int main() {
  double *A, *L, *d;
  long long* cyc;
  cudaMalloc(&A, 32 * 32 * 8);
  cudaMalloc(&L, 64 * 1024 * 8);
  cudaMalloc(&d, 64 * 32 * 8);
  cudaMallocManaged(&cyc, 8 * 8);
  double h[1024];
  for (int j = 0; j < 32; ++j)
    for (int i = 0; i < 32; ++i) h[j * 32 + i] = (i == j) ? 40.0 + i : 1.0 / (1 + i + j);
  cudaMemcpy(A, h, sizeof(h), cudaMemcpyHostToDevice);
  int cases[][2] = {{12, 16}, {12, 28}, {24, 32}, {4, 8}};
  for (auto& c : cases) {
    const int k = c[0], f = c[1];
    kpiv<0><<<1, 32>>>(A, L, d, k, f, 2000, cyc, 1e-10);
    kpiv<1><<<1, 32>>>(A, L, d, k, f, 2000, cyc, 1e-10);
    kpiv<2><<<1, 32>>>(A, L, d, k, f, 2000, cyc, 1e-10);
    ksm<<<1, 32>>>(A, L, d, k, f, 2000, cyc, 1e-10);
    kv3<0><<<1, 32>>>(A, L, d, k, f, 2000, cyc, 1e-10);
    kv3<1><<<1, 32>>>(A, L, d, k, f, 2000, cyc, 1e-10);
    cudaDeviceSynchronize();
    printf("k %2d f %2d: reg %lld  reg-nostore %lld  reg-nodiv %lld  smem %lld  v3 %lld  v3-nostore %lld cycles/front\n",
           k, f, cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5]);
  }
  return 0;
}
