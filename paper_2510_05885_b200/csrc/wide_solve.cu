// Wide-tier triangular solves (ldl_solve, sparse.cpp:258-276, restated for
// the supernodal fronts): one launch per tree level, one thread-block cluster
// per front.
//
// Forward  (L w = b on the permuted vector):
//   rank 0   -- gathers the pivot values and the children's update vectors,
//               then solves the k x k unit-lower L11 block by block: warp 0
//               runs the 32-step substitution chain with its L11 rows already
//               in registers (static indices, one shuffle + FMA per step)
//               while the other warps prefetch the L entries of the rows
//               below the block, then fold the solved block in (GEMV);
//   all CTAs -- after one cluster barrier, the (f-k) x k GEMV that forms the
//               update vector the parent adds (thread per row, coalesced
//               column-major reads, rows split across the cluster).
// Backward (L^T x = D^-1 w):
//   all CTAs -- the k x (f-k) transposed GEMV against the parent's solved
//               rows (warp per pivot column, lanes along the column);
//   rank 0   -- after one cluster barrier, the blocked L11^T solve from the
//               last block up: GEMV against the later pivots, then warp 0's
//               32-step chain with its L11 column in registers.
// No atomics on values; every sum has a fixed order (bitwise reproducible).
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdlib>
#include <stdint.h>

#include "cuda_util.hpp"
#include "device.cuh"
#include "launch.hpp"
#include "symbolic.hpp"
#include "layout.hpp"

namespace cg = cooperative_groups;

namespace nclb {

constexpr int kSolveThreads = 512;
constexpr int kSolveWarps = kSolveThreads / 32;
constexpr int kBlk = 32;
constexpr int kRows = 240;        // rows per staged panel chunk
constexpr int kSLP = kRows + 2;   // its column stride in shared memory
constexpr unsigned kFull = 0xffffffffu;
constexpr int kParK = 1024;       // pivot blocks from which the L11 solve is cluster-parallel

// dynamic shared memory: the front vector (f doubles) after two panel buffers
struct SolveSmem {
  double P[2][kBlk * kSLP];
  double Z[kBlk];
};

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ void cp16(void* dst, const void* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// rows [r0, r0+nr) x columns [c0, c0+nc) of L (ld even) -> S, element
// (r0+i, c0+j) at S[j*kSLP + i + sh], sh = r0 & 1; warp per column, lanes
// along it in 16-byte chunks (cp.async: many copies in flight per warp --
// register loads from L2 stall on too few outstanding requests).
__device__ __forceinline__ int stage_cols(double* S, const double* L, size_t ld, int r0, int nr,
                                          int c0, int nc, int warp, int lane, int nwarps = kSolveWarps) {
  const int a = r0 & ~1, sh = r0 - a, n2 = (nr + sh + 1) >> 1;
  for (int j = warp; j < nc; j += nwarps) {
    const double* src = L + a + (c0 + j) * ld;
    double* dst = S + j * kSLP;
    for (int ch = lane; ch < n2; ch += 32) cp16(dst + 2 * ch, src + 2 * ch);
  }
  return r0 - a;
}

template <bool PAR>
__global__ void __launch_bounds__(kSolveThreads, 1)
k_fwd_front(SnDev sd, const double* __restrict__ lval, double* w, double* uvec,
            const int* __restrict__ nodes) {
  extern __shared__ __align__(16) double dyn[];
  SolveSmem& sm = *reinterpret_cast<SolveSmem*>(dyn);
  double* T = dyn + sizeof(SolveSmem) / sizeof(double);
  cg::cluster_group cl = cg::this_cluster();
  const int C = static_cast<int>(cl.num_blocks());
  const int rank = static_cast<int>(cl.block_rank());
  const int s = nodes[blockIdx.x / C];
  const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
  const size_t ld = wide_ld(f);
  const double* L = lval + sd.l_off[s];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* u = uvec + sd.rel_ptr[s];
  const int kp = s == sd.schur ? 0 : k;  // Schur mode: assemble the coupling rhs only
  pdl_launch_dependents();
  // the children's update vectors (previous level) are read by rank 0 only,
  // after its first L11 stage is in flight; the other CTAs read nothing of
  // the previous level before the cluster barrier that follows rank 0's work
  if (rank == 0 && !(k > 0)) pdl_wait();
  // big pivot blocks: the L11 solve itself is spread over the cluster
  // (per 32-block: rank 0's chain, then every CTA's share of the rows below)
  const bool par = PAR && kp >= kParK && C > 1;
  if (rank == 0 && k > 0) {
    // stages: block b (columns [32b, 32b+nb)), rows [32b, k) in chunks of kRows
    int sb = 0, sr = 0, buf = 0;
    int shv[2];
    auto issue = [&](int b, int r0, int bf) {
      const int p0 = b * kBlk, nb = min(kBlk, k - p0);
      shv[bf] = stage_cols(sm.P[bf], L, ld, r0, min(kRows, k - r0), p0, nb, warp, lane);
      cp_commit();
    };
    if (kp > 0 && !par) issue(0, 0, 0);
    pdl_wait();
    for (int r = tid; r < f; r += kSolveThreads) T[r] = r < k ? __ldcg(w + c0 + r) : 0.0;
    __syncthreads();
    if (const int ng = sd.usplit_ng[s]) {  // group sums (split.cu), in group order
      const double* P = sd.uvpart + sd.usplit_off[s];
      for (int r = tid; r < f; r += kSolveThreads) {
        double v = T[r];
#pragma unroll 8
        for (int g = 0; g < ng; ++g) v += __ldcg(P + static_cast<size_t>(g) * f + r);
        T[r] = v;
      }
      __syncthreads();
    } else {
      for (int cc = sd.ch_ptr[s]; cc < sd.ch_ptr[s + 1]; ++cc) {
        const int c = sd.ch[cc];
        const int fu = f_minus_k(sd, c), rp = sd.rel_ptr[c];
        for (int i = tid; i < fu; i += kSolveThreads) T[sd.rel[rp + i]] += __ldcg(uvec + rp + i);
        __syncthreads();
      }
    }
    for (; kp > 0 && !par;) {
      const int p0 = sb * kBlk, p1 = min(p0 + kBlk, k), nb = p1 - p0;
      const int nr = min(kRows, k - sr);
      // next stage into the other buffer
      int nbk = sb, nr0 = sr + kRows;
      if (nr0 >= k) {
        ++nbk;
        nr0 = nbk * kBlk;
      }
      const bool more = nbk * kBlk < k;
      if (more) {
        issue(nbk, nr0, buf ^ 1);
        cp_wait<1>();
      } else {
        cp_wait<0>();
      }
      __syncthreads();
      const double* P = sm.P[buf];
      const int sh = shv[buf];
      if (sr == p0) {  // chunk holding L11: the substitution chain first
        if (warp == 0) {
          double lv[kBlk];
#pragma unroll
          for (int q = 0; q < kBlk; ++q) lv[q] = (q < lane && lane < nb) ? P[q * kSLP + lane + sh] : 0.0;
          double t = lane < nb ? T[p0 + lane] : 0.0;
#pragma unroll
          for (int q = 0; q < kBlk; ++q) {
            if (q < nb) {
              const double wq = __shfl_sync(kFull, t, q);
              if (lane > q) t -= lv[q] * wq;
            }
          }
          if (lane < nb) T[p0 + lane] = t;
        }
        __syncthreads();
      }
      // rows of this chunk below the block: T[r] -= L(r, block) w_block
      for (int r = max(sr, p1) + tid; r < sr + nr; r += kSolveThreads) {
        const int i = r - sr + sh;
        double a0 = 0.0, a1 = 0.0;
        int q = 0;
        for (; q + 2 <= nb; q += 2) {
          a0 += P[q * kSLP + i] * T[p0 + q];
          a1 += P[(q + 1) * kSLP + i] * T[p0 + q + 1];
        }
        if (q < nb) a0 += P[q * kSLP + i] * T[p0 + q];
        T[r] -= a0 + a1;
      }
      __syncthreads();
      if (!more) break;
      sb = nbk;
      sr = nr0;
      buf ^= 1;
    }
    for (int q = tid; q < f; q += kSolveThreads) {
      if (q < k)
        w[c0 + q] = T[q];
      else
        u[q - k] = T[q];
    }
  }
  cl.sync();
  if (par) {
    const int ch = (k + C - 1) / C;
    const int mlo = rank * ch, mhi = min(k, mlo + ch);  // this CTA's rows of the L11 part
    for (int p0 = 0; p0 < k; p0 += kBlk) {
      const int p1 = min(p0 + kBlk, k), nb = p1 - p0;
      const int r0 = max(p1, mlo), nr = mhi - r0;
      int sh = 0;
      if (nr > 0) sh = stage_cols(sm.P[1], L, ld, r0, nr, p0, nb, warp, lane);  // rows below, prefetched
      cp_commit();
      if (rank == 0 && warp == 0) {
        const int sd0 = stage_cols(sm.P[0], L, ld, p0, nb, p0, nb, 0, lane, 1);
        cp_commit();
        cp_wait<0>();
        __syncwarp();
        double lv[kBlk];
#pragma unroll
        for (int q = 0; q < kBlk; ++q) lv[q] = (q < lane && lane < nb) ? sm.P[0][q * kSLP + lane + sd0] : 0.0;
        double t = lane < nb ? __ldcg(w + c0 + p0 + lane) : 0.0;
#pragma unroll
        for (int q = 0; q < kBlk; ++q) {
          if (q < nb) {
            const double wq = __shfl_sync(kFull, t, q);
            if (lane > q) t -= lv[q] * wq;
          }
        }
        if (lane < nb) w[c0 + p0 + lane] = t;
      }
      cl.sync();
      cp_wait<0>();
      __syncthreads();
      if (tid < kBlk) sm.Z[tid] = tid < nb ? __ldcg(w + c0 + p0 + tid) : 0.0;
      __syncthreads();
      for (int r = tid; r < nr; r += kSolveThreads) {
        double a0 = 0.0, a1 = 0.0;
        int q = 0;
        for (; q + 2 <= nb; q += 2) {
          a0 += sm.P[1][q * kSLP + r + sh] * sm.Z[q];
          a1 += sm.P[1][(q + 1) * kSLP + r + sh] * sm.Z[q + 1];
        }
        if (q < nb) a0 += sm.P[1][q * kSLP + r + sh] * sm.Z[q];
        w[c0 + r0 + r] = __ldcg(w + c0 + r0 + r) - (a0 + a1);
      }
      cl.sync();
    }
  }
  // update vector rows [k, f): u_r -= sum_{q<k} L(r, q) w_q, rows split over
  // the cluster; column chunks of 32 streamed through the two buffers
  const int rows = f - k;
  if (rows == 0 || k == 0) return;
  if (rank != 0 || par) {
    for (int q = tid; q < k; q += kSolveThreads) T[q] = __ldcg(w + c0 + q);
  }
  const int chunk = (rows + C - 1) / C;
  const int lo = k + rank * chunk, hi = min(f, lo + chunk);
  const int ncc = (k + kBlk - 1) / kBlk;
  for (int base = lo; base < hi; base += kRows) {
    const int nr = min(kRows, hi - base);
    int shv[2];
    shv[0] = stage_cols(sm.P[0], L, ld, base, nr, 0, min(kBlk, k), warp, lane);
    cp_commit();
    double acc = 0.0;
    for (int cb = 0; cb < ncc; ++cb) {
      const int bf = cb & 1;
      if (cb + 1 < ncc) {
        shv[bf ^ 1] = stage_cols(sm.P[bf ^ 1], L, ld, base, nr, (cb + 1) * kBlk,
                                 min(kBlk, k - (cb + 1) * kBlk), warp, lane);
        cp_commit();
        cp_wait<1>();
      } else {
        cp_wait<0>();
      }
      __syncthreads();
      if (tid < nr) {
        const double* P = sm.P[bf];
        const int i = tid + shv[bf], q0 = cb * kBlk, nq = min(kBlk, k - q0);
        double a1 = 0.0;
        int q = 0;
        for (; q + 2 <= nq; q += 2) {
          acc += P[q * kSLP + i] * T[q0 + q];
          a1 += P[(q + 1) * kSLP + i] * T[q0 + q + 1];
        }
        if (q < nq) acc += P[q * kSLP + i] * T[q0 + q];
        acc += a1;
      }
      __syncthreads();
    }
    if (tid < nr) u[base + tid - k] = __ldcg(u + (base + tid - k)) - acc;
  }
}

template <bool PAR>
__global__ void __launch_bounds__(kSolveThreads, 1)
k_bwd_front(SnDev sd, const double* __restrict__ lval, const double* __restrict__ d,
            const double* __restrict__ w, double* x, const int* __restrict__ nodes, double* scr) {
  extern __shared__ __align__(16) double dyn[];
  SolveSmem& sm = *reinterpret_cast<SolveSmem*>(dyn);
  double* X = dyn + sizeof(SolveSmem) / sizeof(double);
  cg::cluster_group cl = cg::this_cluster();
  const int C = static_cast<int>(cl.num_blocks());
  const int rank = static_cast<int>(cl.block_rank());
  const int s = nodes[blockIdx.x / C];
  const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
  const size_t ld = wide_ld(f);
  const double* L = lval + sd.l_off[s];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int* rows = sd.rows + sd.rows_ptr[s];
  pdl_launch_dependents();
  if (k == 0 || s == sd.schur) {  // Schur mode: coupling solution set by the host
    pdl_wait();
    return;
  }
  // z_p = w_p / d_p - sum_{r >= k} L(r, p) x_r for this CTA's pivot columns,
  // 32 columns x kRows rows per staged chunk, two columns per warp.  The
  // first chunk of L is staged before waiting for the parent's solution rows
  // (the previous level's output)
  {
    const int pc = (k + C - 1) / C;
    const int pa = rank * pc, pb = min(k, pa + pc);
    const int nch = (f - k + kRows - 1) / kRows;
    int shv0 = 0;
    if (pa < pb && nch > 0) {
      shv0 = stage_cols(sm.P[0], L, ld, k, min(kRows, f - k), pa, min(kBlk, pb - pa), warp, lane);
      cp_commit();
    }
    pdl_wait();
    for (int r = k + tid; r < f; r += kSolveThreads) X[r] = __ldcg(x + rows[r]);
    __syncthreads();
    for (int q0 = pa; q0 < pb; q0 += kBlk) {
      const int nq = min(kBlk, pb - q0);
      double part0 = 0.0, part1 = 0.0;
      int shv[2];
      if (nch > 0) {
        if (q0 == pa) {
          shv[0] = shv0;
        } else {
          shv[0] = stage_cols(sm.P[0], L, ld, k, min(kRows, f - k), q0, nq, warp, lane);
          cp_commit();
        }
      }
      for (int ci = 0; ci < nch; ++ci) {
        const int bf = ci & 1, r0 = k + ci * kRows, nr = min(kRows, f - r0);
        if (ci + 1 < nch) {
          shv[bf ^ 1] = stage_cols(sm.P[bf ^ 1], L, ld, r0 + kRows, min(kRows, f - r0 - kRows), q0,
                                   nq, warp, lane);
          cp_commit();
          cp_wait<1>();
        } else {
          cp_wait<0>();
        }
        __syncthreads();
        const double* P = sm.P[bf];
        for (int i = lane; i < nr; i += 32) {
          const double xv = X[r0 + i];
          if (warp < nq) part0 += P[warp * kSLP + i + shv[bf]] * xv;
          if (warp + kSolveWarps < nq) part1 += P[(warp + kSolveWarps) * kSLP + i + shv[bf]] * xv;
        }
        __syncthreads();
      }
      part0 = wsum(part0);
      part1 = wsum(part1);
      if (lane == 0) {
        int p = q0 + warp;
        if (warp < nq) x[c0 + p] = __ldcg(w + c0 + p) / __ldcg(d + c0 + p) - part0;
        p += kSolveWarps;
        if (warp + kSolveWarps < nq) x[c0 + p] = __ldcg(w + c0 + p) / __ldcg(d + c0 + p) - part1;
      }
    }
  }
  cl.sync();
  if (PAR && k >= kParK && C > 1) {  // big pivot blocks: the L11^T solve spread over the cluster
    const int ch = (k + C - 1) / C;
    const int mlo = rank * ch, mhi = min(k, mlo + ch);
    double* part = scr + static_cast<size_t>(blockIdx.x / C) * (16 * kBlk);  // [rank][32]
    for (int p1 = k; p1 > 0;) {
      const int p0 = ((p1 - 1) / kBlk) * kBlk, nb = p1 - p0;
      const int r0 = max(p1, mlo), nr = mhi - r0;
      int sh = 0;
      if (nr > 0) sh = stage_cols(sm.P[1], L, ld, r0, nr, p0, nb, warp, lane);
      cp_commit();
      for (int r = tid; r < nr; r += kSolveThreads) X[r] = __ldcg(x + c0 + r0 + r);
      cp_wait<0>();
      __syncthreads();
      for (int j = warp; j < kBlk; j += kSolveWarps) {
        double a = 0.0;
        if (j < nb)
          for (int r = lane; r < nr; r += 32) a += sm.P[1][j * kSLP + r + sh] * X[r];
        a = wsum(a);
        if (lane == 0) part[rank * kBlk + j] = a;
      }
      cl.sync();
      if (rank == 0 && warp == 0) {
        const int sd0 = stage_cols(sm.P[0], L, ld, p0, nb, p0, nb, 0, lane, 1);
        cp_commit();
        double z = 0.0;
        for (int c = 0; c < C; ++c) z += __ldcg(part + c * kBlk + lane);  // fixed order
        double xv = lane < nb ? __ldcg(x + c0 + p0 + lane) - z : 0.0;
        cp_wait<0>();
        __syncwarp();
        double lc[kBlk];
#pragma unroll
        for (int j = 0; j < kBlk; ++j) lc[j] = (j > lane && j < nb) ? sm.P[0][lane * kSLP + j + sd0] : 0.0;
#pragma unroll
        for (int p = kBlk - 1; p >= 0; --p) {
          if (p < nb) {
            const double xp = __shfl_sync(kFull, xv, p);
            if (lane < p) xv -= lc[p] * xp;
          }
        }
        if (lane < nb) x[c0 + p0 + lane] = xv;
      }
      cl.sync();
      p1 = p0;
    }
    return;
  }
  if (rank != 0) return;
  for (int p = tid; p < k; p += kSolveThreads) X[p] = __ldcg(x + c0 + p);
  __syncthreads();
  // blocked L11^T solve from the last block up; block b's chunks (rows
  // [32b, k) in kRows pieces) are visited last-first so the chunk holding
  // L11 is still resident for the chain
  const int nblk = (k + kBlk - 1) / kBlk;
  auto nchunks = [&](int b) { return (k - b * kBlk + kRows - 1) / kRows; };
  int b = nblk - 1, ci = nchunks(b) - 1, buf = 0;
  int shv[2];
  auto issue = [&](int bb, int cc, int bf) {
    const int p0 = bb * kBlk, r0 = p0 + cc * kRows;
    shv[bf] = stage_cols(sm.P[bf], L, ld, r0, min(kRows, k - r0), p0, min(kBlk, k - p0), warp, lane);
    cp_commit();
  };
  issue(b, ci, 0);
  if (tid < kBlk) sm.Z[tid] = 0.0;
  for (;;) {
    const int p0 = b * kBlk, p1 = min(p0 + kBlk, k), nb = p1 - p0;
    const int r0 = p0 + ci * kRows, nr = min(kRows, k - r0);
    int nb2 = b, nc2 = ci - 1;
    if (nc2 < 0) {
      --nb2;
      nc2 = nb2 >= 0 ? nchunks(nb2) - 1 : 0;
    }
    const bool more = nb2 >= 0;
    if (more) {
      issue(nb2, nc2, buf ^ 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const double* P = sm.P[buf];
    const int sh = shv[buf];
    // later pivots of this front: z_p -= sum_{r in chunk, r >= p1} L(r, p) x_r
    for (int j = warp; j < nb; j += kSolveWarps) {
      double part = 0.0;
      for (int r = max(r0, p1) + lane; r < r0 + nr; r += 32) part += P[j * kSLP + r - r0 + sh] * X[r];
      part = wsum(part);
      if (lane == 0) sm.Z[j] += part;
    }
    __syncthreads();
    if (ci == 0) {  // all chunks of block b done; P holds L11
      if (warp == 0) {
        double lc[kBlk];  // lane owns column p0+lane of L11: L(p0+j, p0+lane), j > lane
#pragma unroll
        for (int j = 0; j < kBlk; ++j) lc[j] = (j > lane && j < nb) ? P[lane * kSLP + j + sh] : 0.0;
        double xv = lane < nb ? X[p0 + lane] - sm.Z[lane] : 0.0;
#pragma unroll
        for (int p = kBlk - 1; p >= 0; --p) {
          if (p < nb) {
            const double xp = __shfl_sync(kFull, xv, p);
            if (lane < p) xv -= lc[p] * xp;
          }
        }
        if (lane < nb) X[p0 + lane] = xv;
        sm.Z[lane] = 0.0;
      }
      __syncthreads();
    }
    if (!more) break;
    b = nb2;
    ci = nc2;
    buf ^= 1;
  }
  for (int p = tid; p < k; p += kSolveThreads) x[c0 + p] = X[p];
}

// ---------------------------------------------------------------------------
// programmatic dependent launch of the level kernels (NCL_NO_PDL=1: off)
static bool pdl_enabled() {
  static const bool on = std::getenv("NCL_NO_PDL") == nullptr;
  return on;
}

template <typename Kern, typename... Args>
static int launch_clustered(Kern kern, int count, int cluster, size_t smem, cudaStream_t st,
                            Args... args) {
  for (; cluster >= 1; cluster >>= 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(count * cluster));
    cfg.blockDim = dim3(kSolveThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(cluster);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // device: pdl_wait()
    attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess || ncl < 1) {
      cudaGetLastError();
      continue;
    }
    if (cudaLaunchKernelEx(&cfg, kern, args...) == cudaSuccess) return cluster;
    cudaGetLastError();
  }
  return 0;
}

template <bool PAR>
static void solve_init_one(int optin) {
  cudaFuncSetAttribute(k_fwd_front<PAR>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_bwd_front<PAR>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_fwd_front<PAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
  cudaFuncSetAttribute(k_bwd_front<PAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
}

static void solve_init() {
  static PerDeviceOnce once;
  once([] {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    solve_init_one<false>(optin);
    solve_init_one<true>(optin);
  });
}

// par: the level holds a front with >= kParK pivots (cluster-parallel L11)
int launch_fwd_front(const SnDev& sd, const double* lval, double* w, double* uvec,
                     const int* nodes, int count, int cluster, int max_f, bool par,
                     cudaStream_t st) {
  if (count == 0) return cluster;
  solve_init();
  const size_t smem = sizeof(SolveSmem) + sizeof(double) * max_f;
  return par ? launch_clustered(k_fwd_front<true>, count, cluster, smem, st, sd, lval, w, uvec, nodes)
             : launch_clustered(k_fwd_front<false>, count, cluster, smem, st, sd, lval, w, uvec, nodes);
}

int launch_bwd_front(const SnDev& sd, const double* lval, const double* d, const double* w,
                     double* x, const int* nodes, int count, int cluster, int max_f, double* scr,
                     bool par, cudaStream_t st) {
  if (count == 0) return cluster;
  solve_init();
  const size_t smem = sizeof(SolveSmem) + sizeof(double) * max_f;
  return par ? launch_clustered(k_bwd_front<true>, count, cluster, smem, st, sd, lval, d, w, x, nodes, scr)
             : launch_clustered(k_bwd_front<false>, count, cluster, smem, st, sd, lval, d, w, x, nodes, scr);
}

int solve_par_k() { return kParK; }

}  // namespace nclb
