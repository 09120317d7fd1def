// Micro-benchmark: dependent-chain latencies (cycles) of FP64 ops, shuffles
// and shared-memory round trips for one warp on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void klat(double* out, long long* cyc, double a, double b, int n) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  double x = a + lane;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, b, a);
  long long t1 = clock64();
  double y = x;
  for (int i = 0; i < n; ++i) y = __shfl_sync(0xffffffffu, y, (lane + 1) & 31);
  long long t2 = clock64();
  double z = y;
  for (int i = 0; i < n; ++i) z = a / (z + b);
  long long t3 = clock64();
  sm[lane] = z;
  double w = z;
  for (int i = 0; i < n; ++i) {
    sm[(lane + i) & 31] = w;
    __syncwarp();
    w = sm[(lane + 1 + i) & 31] + 1.0;
    __syncwarp();
  }
  long long t4 = clock64();
  float fx = (float)w;
  for (int i = 0; i < n; ++i) fx = fmaf(fx, (float)b, (float)a);
  long long t5 = clock64();
  double r = fx;
  for (int i = 0; i < n; ++i) {
    double q;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(q) : "d"(r));
    r = q + b;
  }
  long long t6 = clock64();
  out[lane] = r;
  if (lane == 0) {
    cyc[0] = (t1 - t0) / n;
    cyc[1] = (t2 - t1) / n;
    cyc[2] = (t3 - t2) / n;
    cyc[3] = (t4 - t3) / n;
    cyc[4] = (t5 - t4) / n;
    cyc[5] = (t6 - t5) / n;
  }
}
int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 256);
  cudaMallocManaged(&c, 64);
  klat<<<1, 32>>>(o, c, 0.5, 0.25, 4096);
  klat<<<1, 32>>>(o, c, 0.5, 0.25, 4096);
  cudaDeviceSynchronize();
  printf("dfma %lld  shfl(f64) %lld  ddiv(+dadd) %lld  smem st/ld round %lld  ffma %lld  rcp64+dadd %lld cycles\n",
         c[0], c[1], c[2], c[3], c[4], c[5]);
  return 0;
}
