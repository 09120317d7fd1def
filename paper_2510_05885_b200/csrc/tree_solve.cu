// Wide-tier triangular solves (ldl_solve, sparse.cpp:258-276, restated for
// the supernodal fronts) as ONE persistent dataflow launch per direction.
//
// The level kernels (wide_solve.cu) pay a launch and a whole-level barrier
// per tree level, and each front's 32-step substitution chains wait behind
// L2 round trips for the L panels.  Here a grid of resident CTAs walks the
// wide fronts of a run of levels in topological order -- CTA i takes list
// positions i, i+G, i+2G, ... (forward: children before parents; backward:
// the reversed list) -- and a front waits only for the fronts it reads:
// its children's update vectors (forward) or its parent's solution rows
// (backward), through one flag per front (st.release.gpu / relaxed polls +
// fence.acq_rel.gpu).  Every CTA runs its positions in list order, so a
// front is only ever waited on by CTAs holding later positions: no deadlock
// while all CTAs are resident (grid <= resident CTAs).
//
// Inside a front (one CTA, 9 warps):
//   warp 0 ("chain")  -- the 32-pivot substitution chains, block by block; its
//                        L data (the 32x32 diagonal block and the 32x32 block
//                        next to it) is staged in shared memory by cp.async
//                        two blocks ahead, so the chain never waits on L2;
//   warps 1-8 ("bulk") -- apply every solved block to the rest of the front
//                        (forward: the rows below; backward: the pivot
//                        columns above) from register-prefetched L, one
//                        32x32 block per step, overlapped with the chain.
// Only the chain and the one block beside it are on the critical path.
// Chain and bulk warps hand over through shared-memory counters
// (st.release / ld.acquire at CTA scope).
//
// Arithmetic per front (row r of the front, panel = 32 pivot columns):
//   forward   T_r = w_r + sum_children u  (child order), then per panel c in
//             order T_r -= sum_q L(r, q) x_q (two interleaved partial sums),
//             x_c = L_cc^-1 T_c by the shuffle chain;
//   backward  z_q = w_q / d_q - [sum over update rows, pivot blocks from the
//             top] L(r, q) x_r, then x_c = L_cc^-T z_c by the shuffle chain.
// Every sum has a fixed order, independent of the CTA that runs the front
// (bitwise reproducible solves).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "cuda_util.hpp"
#include "device.cuh"
#include "launch.hpp"
#include "layout.hpp"

namespace nclb {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kBulk = 8;                   // bulk warps
constexpr int kThr = 32 * (1 + kBulk);     // threads per CTA
constexpr int kStages = 3;                 // chain head stages in flight
constexpr int kHeadSL = 66;                // forward head: column stride (64 rows + pad; 16-byte multiple)
constexpr int kMaxRB = 80;                 // row blocks per front (f <= kTreeMaxF)
constexpr int kTsSL = 33;                  // backward transpose buffer stride

__device__ __forceinline__ unsigned sptr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sptr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void st_rel_cta(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(sptr(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acq_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(sptr(p)) : "memory");
  return v;
}
// trace stamps: SM clock (durations within a CTA; %globaltimer reads slowed
// this kernel 4x when they were used for the stamps)
__device__ __forceinline__ unsigned long long gtime() { return static_cast<unsigned long long>(clock64()); }
__device__ __forceinline__ void wait_ge(const int* p, int v) {
  while (ld_acq_cta(p) < v) __nanosleep(16);
}
// a flag of another CTA (gpu scope): relaxed polls, then one acquire fence
__device__ __forceinline__ void gwait_ge(const int* p, int v) {
  if (ld_relaxed(p) < v) {
    unsigned ns = 32;
    while (ld_relaxed(p) < v) {
      __nanosleep(ns);
      if (ns < 256) ns <<= 1;
    }
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// row blocks of a front: pivot blocks [32R, min(32R+32, k)), then update
// blocks [k + 32(R-P), ...)
__device__ __forceinline__ int rb_start(int k, int P, int R) { return R < P ? 32 * R : k + 32 * (R - P); }
__device__ __forceinline__ int rb_size(int k, int f, int P, int R) {
  const int s = rb_start(k, P, R);
  return (R < P ? min(s + 32, k) : min(s + 32, f)) - s;
}

struct FrontGeo {
  int s, c0, k, f, P, NR;
  size_t ld;
  const double* L;
};

__device__ __forceinline__ FrontGeo front_geo(const SnDev& sd, const double* lval, int s) {
  FrontGeo g;
  g.s = s;
  g.c0 = __ldg(sd.first + s);
  g.k = __ldg(sd.first + s + 1) - g.c0;
  g.f = __ldg(sd.f + s);
  g.P = (g.k + 31) >> 5;
  g.NR = g.P + ((g.f - g.k + 31) >> 5);
  g.ld = wide_ld(g.f);
  g.L = lval + __ldg(sd.l_off + s);
  return g;
}

// ---------------------------------------------------------------------------
// forward
struct FwdSmem {
  double head[kStages][32 * kHeadSL];  // rows [32b, 32b+64) x the 32 columns of block b
  int xdone;                           // pivot blocks solved
  int cnt[kMaxRB];                     // per row block: panels applied by the bulk warps
};

// chain head of block b: rows [32b, 32b+64) of block b's columns, column j at
// S[j * kHeadSL], lane = 16-byte chunk (coalesced 512-byte columns)
__device__ __forceinline__ void fwd_stage(double* S, const FrontGeo& g, int b, int lane) {
  if (b < g.P) {
    const int p0 = 32 * b, nb = min(32, g.k - p0);
    const double* src = g.L + p0 + 2 * lane + static_cast<size_t>(p0) * g.ld;
    for (int j = 0; j < nb; ++j) cp16(S + j * kHeadSL + 2 * lane, src + j * g.ld);
  }
  cp_commit();
}

__device__ __forceinline__ void fwd_chain(const FrontGeo& g, double* T, FwdSmem& sm) {
  const int lane = threadIdx.x & 31;
  __syncwarp();  // the warp enters converged (the CTA's tid-0 branches)
  double psum = 0.0;  // panel b-1 applied to block b's rows (this warp's share)
  for (int b = 0; b < g.P; ++b) {
    const int p0 = 32 * b, nb = min(32, g.k - p0);
    cp_wait<kStages - 1>();
    __syncwarp();
    const double* S = sm.head[b % kStages];
    double lv[32];
    const bool nxt = b + 1 < g.P;
    const int nbn = nxt ? min(32, g.k - p0 - 32) : 0;
#pragma unroll
    for (int q = 0; q < 32; ++q) lv[q] = (q < lane && lane < nb) ? S[q * kHeadSL + lane] : 0.0;
    if (b >= 2) wait_ge(&sm.cnt[b], b - 1);
    double t = lane < nb ? T[p0 + lane] - psum : 0.0;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const double wq = __shfl_sync(kFull, t, q);
      if (lane > q) t = fma(-lv[q], wq, t);
    }
    if (lane < nb) T[p0 + lane] = t;
    __syncwarp();
    if (lane == 0) st_rel_cta(&sm.xdone, b + 1);
    if (nxt) {  // panel b on block b+1's rows: L(32b+32+lane, 32b+q) from the head
      const bool ok = lane < nbn;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int q = 0; q < 32; q += 2) {
        const double l0 = (ok && q < nb) ? S[q * kHeadSL + 32 + lane] : 0.0;
        const double l1 = (ok && q + 1 < nb) ? S[(q + 1) * kHeadSL + 32 + lane] : 0.0;
        a0 = fma(l0, __shfl_sync(kFull, t, q), a0);
        a1 = fma(l1, __shfl_sync(kFull, t, q + 1), a1);
      }
      psum = a0 + a1;
    }
    __syncwarp();
    fwd_stage(sm.head[b % kStages], g, b + kStages, lane);
  }
  cp_wait<0>();
}

// bulk items (c, R): panel c applied to row block R, R owned by this warp
// (R % kBulk == wb), in (c, R) order; pivot blocks take panels c <= R-2
// (panel R-1 is the chain warp's), update blocks every panel
__device__ __forceinline__ bool fwd_valid(const FrontGeo& g, int c, int R) {
  return R < g.P ? R >= c + 2 : true;
}
__device__ __forceinline__ bool fwd_next(const FrontGeo& g, int wb, int& c, int& R) {
  for (;;) {
    R += kBulk;
    if (R >= g.NR) {
      if (++c >= g.P) return false;
      R = wb;
    }
    if (fwd_valid(g, c, R)) return true;
  }
}
__device__ __forceinline__ void fwd_load(double (&v)[32], const FrontGeo& g, int c, int R, int lane) {
  const int r0 = rb_start(g.k, g.P, R), nr = rb_size(g.k, g.f, g.P, R);
  const int q0 = 32 * c, nq = min(32, g.k - q0);
  const double* src = g.L + r0 + lane + static_cast<size_t>(q0) * g.ld;
  const bool ok = lane < nr;
#pragma unroll
  for (int q = 0; q < 32; ++q) v[q] = (ok && q < nq) ? __ldg(src + q * g.ld) : 0.0;
}
__device__ __forceinline__ void fwd_apply(const double (&v)[32], const FrontGeo& g, int c, int R,
                                          double* T, FwdSmem& sm, int lane) {
  wait_ge(&sm.xdone, c + 1);
  const int q0 = 32 * c, nq = min(32, g.k - q0);
  double a0 = 0.0, a1 = 0.0;
#pragma unroll
  for (int q = 0; q < 32; q += 2) {
    a0 = fma(v[q], q < nq ? T[q0 + q] : 0.0, a0);
    a1 = fma(v[q + 1], q + 1 < nq ? T[q0 + q + 1] : 0.0, a1);
  }
  const int r0 = rb_start(g.k, g.P, R), nr = rb_size(g.k, g.f, g.P, R);
  if (lane < nr) T[r0 + lane] -= a0 + a1;
  __syncwarp();
  if (lane == 0 && R < g.P) st_rel_cta(&sm.cnt[R], c + 1);
}

__device__ __forceinline__ void fwd_bulk(const FrontGeo& g, int wb, double* T, FwdSmem& sm) {
  const int lane = threadIdx.x & 31;
  __syncwarp();  // the warp enters converged (the CTA's tid-0 branches)
  int c = 0, R = wb;
  if (R >= g.NR || g.P == 0) return;
  if (!fwd_valid(g, c, R) && !fwd_next(g, wb, c, R)) return;
  double A[32], B[32];
  fwd_load(A, g, c, R, lane);
  for (;;) {
    int cb = c, Rb = R;
    const bool hb = fwd_next(g, wb, cb, Rb);
    if (hb) fwd_load(B, g, cb, Rb, lane);
    fwd_apply(A, g, c, R, T, sm, lane);
    if (!hb) break;
    c = cb;
    R = Rb;
    const bool ha = fwd_next(g, wb, cb, Rb);
    if (ha) fwd_load(A, g, cb, Rb, lane);
    fwd_apply(B, g, c, R, T, sm, lane);
    if (!ha) break;
    c = cb;
    R = Rb;
  }
}

__global__ void __launch_bounds__(kThr, 1)
k_fwd_tree(SnDev sd, TreeDev td, const double* __restrict__ lval, double* w, double* uvec) {
  extern __shared__ __align__(16) double dyn[];
  FwdSmem& sm = *reinterpret_cast<FwdSmem*>(dyn);
  double* T = dyn + (sizeof(FwdSmem) + 7) / 8;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int li = blockIdx.x; li < td.n; li += gridDim.x) {
    const FrontGeo g = front_geo(sd, lval, __ldg(td.list + li));
    unsigned long long* tr = td.trace ? td.trace + 4 * static_cast<size_t>(li) : nullptr;
    if (tr && tid == 0) tr[0] = gtime();
    if (warp == 0)  // the chain's first L blocks do not depend on anything
      for (int b = 0; b < kStages; ++b) fwd_stage(sm.head[b], g, b, lane);
    for (int i = tid; i < kMaxRB; i += kThr) sm.cnt[i] = 0;
    if (tid == 0) sm.xdone = 0;
    // children's update vectors: wide children in the list publish flags
    if (warp == 1) {
      const int e0 = __ldg(td.wait_ptr + li), e1 = __ldg(td.wait_ptr + li + 1);
      for (int e = e0 + lane; e < e1; e += 32) gwait_ge(td.flags + __ldg(td.wait + e), 1);
    }
    __syncthreads();
    if (tr && tid == 0) tr[1] = gtime();
    // gather: T_r = w_r (pivot rows) + the children's entries, child order
    {
      const int* gp = td.g_row + __ldg(td.g_base + li);
      for (int r = tid; r < g.f; r += kThr) {
        double v = r < g.k ? __ldcg(w + g.c0 + r) : 0.0;
        const int e0 = __ldg(gp + r), e1 = __ldg(gp + r + 1);
        for (int e = e0; e < e1; ++e) v += __ldcg(uvec + __ldg(td.g_src + e));
        T[r] = v;
      }
    }
    __syncthreads();
    if (tr && tid == 0) tr[2] = gtime();
    if (warp == 0)
      fwd_chain(g, T, sm);
    else
      fwd_bulk(g, warp - 1, T, sm);
    __syncthreads();
    double* u = uvec + __ldg(sd.rel_ptr + g.s);
    for (int r = tid; r < g.f; r += kThr) {
      if (r < g.k)
        w[g.c0 + r] = T[r];
      else
        u[r - g.k] = T[r];
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release(td.flags + g.s, 1);
      if (tr) tr[3] = gtime();
    }
  }
}

// ---------------------------------------------------------------------------
// backward
struct BwdSmem {
  // chain head of block b: rows [32b, 32b+64) x block b's columns; column q,
  // 16-byte chunk c at chunk index q*32 + (c ^ (q & 7)) (lane = column reads)
  double head[kStages][32 * 64];
  double Ts[kBulk][32 * kTsSL];  // per bulk warp: one 32x32 block, row-major
  int xdone;                     // pivot blocks solved, counted from the last
  int cnt[kMaxRB];               // per column block: bulk items applied
};

__device__ __forceinline__ void bwd_stage(double* S, const FrontGeo& g, int b, int lane) {
  if (b >= 0) {
    const int p0 = 32 * b, nb = min(32, g.k - p0);
    const double* src = g.L + p0 + 2 * lane + static_cast<size_t>(p0) * g.ld;
    for (int j = 0; j < nb; ++j) cp16(S + 2 * (j * 32 + (lane ^ (j & 7))), src + j * g.ld);
  }
  cp_commit();
}
__device__ __forceinline__ double head_at(const double* S, int i, int q) {  // L(32b+i, 32b+q)
  return S[2 * (q * 32 + ((i >> 1) ^ (q & 7))) + (i & 1)];
}

__device__ __forceinline__ int bwd_nexp(const FrontGeo& g, int b) {
  return (g.NR - g.P) + max(0, g.P - 2 - b);
}

__device__ __forceinline__ void bwd_chain(const FrontGeo& g, double* X, const double* acc, int pstride,
                                          double* x, BwdSmem& sm) {
  const int lane = threadIdx.x & 31;
  __syncwarp();  // the warp enters converged (the CTA's tid-0 branches)
  for (int o = 0; o < g.P; ++o) {
    const int b = g.P - 1 - o, p0 = 32 * b, nb = min(32, g.k - p0);
    cp_wait<kStages - 1>();
    __syncwarp();
    const double* S = sm.head[o % kStages];
    double lc[32];
    double psum = 0.0;  // block b+1's solved rows applied to column p0+lane
    if (b + 1 < g.P) {
      const int nbn = min(32, g.k - p0 - 32);
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        if (i < nbn) a0 = fma(head_at(S, 32 + i, lane), X[p0 + 32 + i], a0);
        if (i + 1 < nbn) a1 = fma(head_at(S, 33 + i, lane), X[p0 + 33 + i], a1);
      }
      psum = a0 + a1;
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) lc[i] = (i > lane && i < nb) ? head_at(S, i, lane) : 0.0;
    __syncwarp();
    bwd_stage(sm.head[o % kStages], g, b - kStages, lane);
    wait_ge(&sm.cnt[b], bwd_nexp(g, b));
    double sb = 0.0;
#pragma unroll
    for (int w = 0; w < kBulk; ++w) sb += acc[(w * pstride + b) * 32 + lane];
    double xv = lane < nb ? X[p0 + lane] - sb - psum : 0.0;
#pragma unroll
    for (int p = 31; p >= 0; --p) {
      const double xp = __shfl_sync(kFull, xv, p);
      if (lane < p) xv = fma(-lc[p], xp, xv);
    }
    if (lane < nb) {
      X[p0 + lane] = xv;
      x[g.c0 + p0 + lane] = xv;
    }
    __syncwarp();
    if (lane == 0) st_rel_cta(&sm.xdone, o + 1);
  }
  cp_wait<0>();
}

// bulk items (R, b): row block R applied to column block b.  Phase 1 -- the
// update rows, known from the start: items t = (P-1-b) * U + (R-P) (column
// blocks from the last, where the chain starts) dealt round-robin over the
// bulk warps; phase 2 -- pivot blocks R = P-1 .. 2 as the chain solves them,
// items b <= R-2 with b % kBulk == wb, from b = R-2 down (the one the chain
// needs next first).  Each warp sums into its own partials accW[wb][b]; the
// chain adds the warps' partials in warp order.
struct BwdIt {
  int t, R, b;
};
__device__ __forceinline__ bool bwd_phase2_from(const FrontGeo& g, int wb, BwdIt& it, int R) {
  it.t = 0x7fffffff;
  for (; R >= 2; --R) {
    const int m = R - 2;
    if (m >= wb) {
      it.R = R;
      it.b = wb + ((m - wb) / kBulk) * kBulk;
      return true;
    }
  }
  return false;
}
__device__ __forceinline__ bool bwd_set1(const FrontGeo& g, BwdIt& it) {
  const int U = g.NR - g.P;
  if (it.t >= g.P * U) return false;
  it.b = g.P - 1 - it.t / U;
  it.R = g.P + it.t % U;
  return true;
}
__device__ __forceinline__ bool bwd_first(const FrontGeo& g, int wb, BwdIt& it) {
  it.t = wb;
  if (bwd_set1(g, it)) return true;
  return bwd_phase2_from(g, wb, it, g.P - 1);
}
__device__ __forceinline__ bool bwd_next(const FrontGeo& g, int wb, BwdIt& it) {
  if (it.t != 0x7fffffff) {
    it.t += kBulk;
    if (bwd_set1(g, it)) return true;
    return bwd_phase2_from(g, wb, it, g.P - 1);
  }
  it.b -= kBulk;
  if (it.b >= 0) return true;
  return bwd_phase2_from(g, wb, it, it.R - 1);
}
__device__ __forceinline__ void bwd_load(double (&v)[32], const FrontGeo& g, int R, int b, int lane) {
  const int r0 = rb_start(g.k, g.P, R), nr = rb_size(g.k, g.f, g.P, R);
  const int q0 = 32 * b, nq = min(32, g.k - q0);
  const double* src = g.L + r0 + lane + static_cast<size_t>(q0) * g.ld;
  const bool ok = lane < nr;
#pragma unroll
  for (int q = 0; q < 32; ++q) v[q] = (ok && q < nq) ? __ldg(src + q * g.ld) : 0.0;
}
__device__ __forceinline__ void red_rel_cta(int* p, int v) {
  asm volatile("red.release.cta.shared::cta.add.s32 [%0], %1;" ::"r"(sptr(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void bwd_apply(const double (&v)[32], const FrontGeo& g, int R, int b,
                                          const double* X, double* accw, double* Ts, BwdSmem& sm,
                                          int lane) {
  if (R < g.P) wait_ge(&sm.xdone, g.P - R);
  const int r0 = rb_start(g.k, g.P, R), nr = rb_size(g.k, g.f, g.P, R);
#pragma unroll
  for (int q = 0; q < 32; ++q) Ts[lane * kTsSL + q] = v[q];
  __syncwarp();
  double a = accw[32 * b + lane];
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i < nr) a = fma(Ts[i * kTsSL + lane], X[r0 + i], a);
  accw[32 * b + lane] = a;
  __syncwarp();
  if (lane == 0) red_rel_cta(&sm.cnt[b], 1);
}

__device__ __forceinline__ void bwd_bulk(const FrontGeo& g, int wb, const double* X, double* accw,
                                         BwdSmem& sm) {
  const int lane = threadIdx.x & 31;
  __syncwarp();  // the warp enters converged (the CTA's tid-0 branches)
  BwdIt it;
  if (!bwd_first(g, wb, it)) return;
  double* Ts = sm.Ts[wb];
  double A[32], B[32];
  bwd_load(A, g, it.R, it.b, lane);
  for (;;) {
    BwdIt nx = it;
    const bool hb = bwd_next(g, wb, nx);
    if (hb) bwd_load(B, g, nx.R, nx.b, lane);
    bwd_apply(A, g, it.R, it.b, X, accw, Ts, sm, lane);
    if (!hb) break;
    it = nx;
    const bool ha = bwd_next(g, wb, nx);
    if (ha) bwd_load(A, g, nx.R, nx.b, lane);
    bwd_apply(B, g, it.R, it.b, X, accw, Ts, sm, lane);
    if (!ha) break;
    it = nx;
  }
}

__global__ void __launch_bounds__(kThr, 1)
k_bwd_tree(SnDev sd, TreeDev td, const double* __restrict__ lval, const double* __restrict__ d,
           const double* __restrict__ w, double* x, int pmax) {
  extern __shared__ __align__(16) double dyn[];
  BwdSmem& sm = *reinterpret_cast<BwdSmem*>(dyn);
  double* acc = dyn + (sizeof(BwdSmem) + 7) / 8;  // kBulk x pmax x 32: the bulk warps' partials
  double* X = acc + kBulk * 32 * pmax;             // front rows
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int li0 = blockIdx.x; li0 < td.n; li0 += gridDim.x) {
    const int li = td.n - 1 - li0;
    const FrontGeo g = front_geo(sd, lval, __ldg(td.list + li));
    unsigned long long* tr = td.trace ? td.trace + 4 * static_cast<size_t>(td.n + li) : nullptr;
    if (tr && tid == 0) tr[0] = gtime();
    if (warp == 0)
      for (int o = 0; o < kStages; ++o) bwd_stage(sm.head[o], g, g.P - 1 - o, lane);
    for (int i = tid; i < kMaxRB; i += kThr) sm.cnt[i] = 0;
    for (int w = 0; w < kBulk; ++w)
      for (int i = tid; i < 32 * g.P; i += kThr) acc[w * 32 * pmax + i] = 0.0;
    if (tid == 0) sm.xdone = 0;
    // z_q = w_q / d_q for the pivots (the forward result, final)
    for (int q = tid; q < g.k; q += kThr) X[q] = __ldg(w + g.c0 + q) / __ldg(d + g.c0 + q);
    // the parent's solution rows
    const int par = __ldg(td.par + li);
    if (tid == 0 && par >= 0) gwait_ge(td.flags + par, 2);
    __syncthreads();
    if (tr && tid == 0) tr[1] = gtime();
    {
      const int* rows = sd.rows + __ldg(sd.rows_ptr + g.s);
      for (int r = g.k + tid; r < g.f; r += kThr) X[r] = __ldcg(x + __ldg(rows + r));
    }
    __syncthreads();
    if (tr && tid == 0) tr[2] = gtime();
    if (warp == 0)
      bwd_chain(g, X, acc, pmax, x, sm);
    else
      bwd_bulk(g, warp - 1, X, acc + (warp - 1) * 32 * pmax, sm);
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release(td.flags + g.s, 2);
      if (tr) tr[3] = gtime();
    }
  }
}

}  // namespace

size_t fwd_tree_smem(int fmax) { return (sizeof(FwdSmem) + 7) / 8 * 8 + sizeof(double) * fmax; }
size_t bwd_tree_smem(int fmax, int pmax) {
  return (sizeof(BwdSmem) + 7) / 8 * 8 + sizeof(double) * (kBulk * 32 * pmax + fmax);
}

static void tree_init() {
  static PerDeviceOnce once;
  once([] {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncSetAttribute(k_fwd_tree, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    cudaFuncSetAttribute(k_bwd_tree, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
  });
}

// resident CTAs per SM for both directions at these sizes (0: does not fit)
int tree_ctas_per_sm(int fmax, int pmax) {
  tree_init();
  if (fmax > kTreeMaxF || (fmax + 31) / 32 + 2 > kMaxRB) return 0;
  int a = 0, b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_fwd_tree, kThr, fwd_tree_smem(fmax)) !=
          cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_bwd_tree, kThr, bwd_tree_smem(fmax, pmax)) !=
          cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return a < b ? a : b;
}

void launch_fwd_tree(const SnDev& sd, const TreeDev& td, const double* lval, double* w, double* uvec,
                     int grid, int fmax, cudaStream_t st) {
  tree_init();
  k_fwd_tree<<<grid, kThr, fwd_tree_smem(fmax), st>>>(sd, td, lval, w, uvec);
}

void launch_bwd_tree(const SnDev& sd, const TreeDev& td, const double* lval, const double* d,
                     const double* w, double* x, int grid, int fmax, int pmax, cudaStream_t st) {
  tree_init();
  k_bwd_tree<<<grid, kThr, bwd_tree_smem(fmax, pmax), st>>>(sd, td, lval, d, w, x, pmax);
}

}  // namespace nclb
