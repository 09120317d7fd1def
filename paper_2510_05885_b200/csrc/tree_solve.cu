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
// (backward), through one flag per front (a CTA or cluster barrier, then
// st.release.gpu by one thread / relaxed polls + one ld.acquire.gpu).  Every CTA runs its positions in list order, so a
// front is only ever waited on by CTAs holding later positions: no deadlock
// while all CTAs are resident (grid <= resident CTAs).
//
// Inside a front (one CTA, 8 warps):
//   warp 0 ("chain")  -- the 32-pivot substitution chains, block by block; its
//                        L data (the 32x32 diagonal block and the 32x32 block
//                        next to it) is staged in shared memory by cp.async
//                        two blocks ahead, so the chain never waits on L2;
//   warps 1-7 ("bulk") -- apply every solved block to the rest of the front
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
//
// Big fronts (the top levels: a few fronts of hundreds of rows, ~1-2 MB of L
// each) are bandwidth-bound on one SM, so those levels run as a second
// launch of the same kernels with thread-block clusters of C CTAs per front:
// rank 0 keeps the chain and the pivot rows, ranks 1..C-1 split the update
// rows (the bulk of L).  Forward, a rank reads each solved block from rank
// 0's shared memory (DSMEM) and finishes its update rows itself; backward, a
// rank sums its update rows' contributions per pivot column block and sends
// the partial to rank 0, which adds the ranks' partials in rank order.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "cuda_util.hpp"
#include "device.cuh"
#include "launch.hpp"
#include "layout.hpp"

namespace cg = cooperative_groups;

namespace nclb {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kBulk = 7;                   // bulk warps (8 warps: up to 255 registers)
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
__device__ __forceinline__ void cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sptr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sptr(dst)), "l"(src) : "memory");
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
// cluster scope (generic addresses: local or another rank's shared memory)
__device__ __forceinline__ void st_rel_cl(int* p, int v) {
  asm volatile("st.release.cluster.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acq_cl(const int* p) {
  int v;
  asm volatile("ld.acquire.cluster.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel_cl(int* p, int v) {
  asm volatile("red.release.cluster.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int atom_add_acqrel_cta(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.s32 %0, [%1], %2;"
               : "=r"(old)
               : "r"(sptr(p)), "r"(v)
               : "memory");
  return old;
}
__device__ __forceinline__ void wait_ge_cl(const int* p, int v) {
  while (ld_acq_cl(p) < v) __nanosleep(32);
}
__device__ __forceinline__ void wait_ge(const int* p, int v) {
  while (ld_acq_cta(p) < v) __nanosleep(16);
}
// a flag of another CTA (gpu scope): relaxed polls, then one acquire read of
// it (device.cuh flag_acquire; the caller's barrier carries the edge to the
// other threads)
__device__ __forceinline__ void gwait_ge(const int* p, int v) {
  if (ld_relaxed(p) < v) {
    unsigned ns = 32;
    while (ld_relaxed(p) < v) {
      __nanosleep(ns);
      if (ns < 256) ns <<= 1;
    }
  }
  flag_acquire(p);
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
  int rlo, rhi;  // row blocks whose bulk work this CTA owns (forward) / update blocks (backward)
  size_t ld;
  const double* L;
};

// update blocks [j0, j1) (indices from 0 at row k) of rank r >= 1 of C
__device__ __forceinline__ void rank_share(int U, int C, int r, int& j0, int& j1) {
  j0 = static_cast<int>((static_cast<long long>(r - 1) * U) / (C - 1));
  j1 = static_cast<int>((static_cast<long long>(r) * U) / (C - 1));
}

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
  g.rlo = 0;
  g.rhi = g.NR;
  return g;
}


// ---------------------------------------------------------------------------
// forward
constexpr int kGMax = 2048;  // children's update entries staged for a front's gather
struct FwdSmem {
  double head[kStages][32 * kHeadSL];  // rows [32b, 32b+64) x the 32 columns of block b
  double first[kBulk][32 * 33];        // per bulk warp: its first item's L block, row-major (staged)
  int grel[kGMax];                     // gather: the children's entries in child order --
  int gsrc[kGMax];                     //   destination row, update-vector offset
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
    if (lane == 0) st_rel_cl(&sm.xdone, b + 1);  // cluster scope: other ranks read the block
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

// bulk items (c, R): panel c applied to row block R in [rlo, rhi), R owned by
// this warp ((R - rlo) % kBulk == wb), in (c, R) order; pivot blocks take
// panels c <= R-2 (panel R-1 is the chain warp's), update blocks every panel
__device__ __forceinline__ bool fwd_valid(const FrontGeo& g, int c, int R) {
  return R < g.P ? R >= c + 2 : true;
}
__device__ __forceinline__ bool fwd_next(const FrontGeo& g, int wb, int& c, int& R) {
  for (;;) {
    R += kBulk;
    if (R >= g.rhi) {
      if (++c >= g.P) return false;
      R = g.rlo + wb;
    }
    if (R < g.rhi && fwd_valid(g, c, R)) return true;
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
// T: this CTA's rows; X0/xd0: rank 0's front vector and progress (REMOTE: a
// rank >= 1 reading them through DSMEM)
template <bool REMOTE>
__device__ __forceinline__ void fwd_apply(const double (&v)[32], const FrontGeo& g, int c, int R,
                                          double* T, const double* X0, const int* xd0, int* cnt,
                                          int lane) {
  const int q0 = 32 * c, nq = min(32, g.k - q0);
  double a0 = 0.0, a1 = 0.0;
  if (REMOTE) {
    wait_ge_cl(xd0, c + 1);
    const double xl = lane < nq ? X0[q0 + lane] : 0.0;
#pragma unroll
    for (int q = 0; q < 32; q += 2) {
      a0 = fma(v[q], __shfl_sync(kFull, xl, q), a0);
      a1 = fma(v[q + 1], __shfl_sync(kFull, xl, q + 1), a1);
    }
  } else {
    wait_ge(xd0, c + 1);
#pragma unroll
    for (int q = 0; q < 32; q += 2) {
      a0 = fma(v[q], q < nq ? X0[q0 + q] : 0.0, a0);
      a1 = fma(v[q + 1], q + 1 < nq ? X0[q0 + q + 1] : 0.0, a1);
    }
  }
  const int r0 = rb_start(g.k, g.P, R), nr = rb_size(g.k, g.f, g.P, R);
  if (lane < nr) T[r0 + lane] -= a0 + a1;
  __syncwarp();
  if (!REMOTE && lane == 0 && R < g.P) st_rel_cta(&cnt[R], c + 1);
}

// the first item of bulk warp wb: (c, R) and whether there is one
__device__ __forceinline__ bool fwd_first(const FrontGeo& g, int wb, int& c, int& R) {
  c = 0;
  R = g.rlo + wb;
  if (R >= g.rhi || g.P == 0) return false;
  return fwd_valid(g, c, R) || fwd_next(g, wb, c, R);
}
// fwd_load's block into a row-major staging block (row lane at S[lane * 33])
// by cp.async: issued before the children are awaited (L is static)
__device__ __forceinline__ void fwd_stage_first(double* S, const FrontGeo& g, int c, int R, int lane) {
  const int r0 = rb_start(g.k, g.P, R), nr = rb_size(g.k, g.f, g.P, R);
  const int q0 = 32 * c, nq = min(32, g.k - q0);
  const double* src = g.L + r0 + lane + static_cast<size_t>(q0) * g.ld;
  const bool ok = lane < nr;
#pragma unroll 8
  for (int q = 0; q < 32; ++q) {
    if (ok && q < nq)
      cp8(S + lane * 33 + q, src + q * g.ld);
    else
      S[lane * 33 + q] = 0.0;
  }
  cp_commit();
}

template <bool REMOTE>
__device__ __forceinline__ void fwd_bulk(const FrontGeo& g, int wb, double* T, const double* X0,
                                         const int* xd0, int* cnt, const double* first) {
  const int lane = threadIdx.x & 31;
  __syncwarp();  // the warp enters converged (the CTA's tid-0 branches)
  int c, R;
  if (!fwd_first(g, wb, c, R)) return;
  double A[32], B[32];
  cp_wait<0>();  // the first item's block, staged before the children were awaited
  __syncwarp();
#pragma unroll
  for (int q = 0; q < 32; ++q) A[q] = first[lane * 33 + q];
  for (;;) {
    int cb = c, Rb = R;
    const bool hb = fwd_next(g, wb, cb, Rb);
    if (hb) fwd_load(B, g, cb, Rb, lane);
    fwd_apply<REMOTE>(A, g, c, R, T, X0, xd0, cnt, lane);
    if (!hb) break;
    c = cb;
    R = Rb;
    const bool ha = fwd_next(g, wb, cb, Rb);
    if (ha) fwd_load(A, g, cb, Rb, lane);
    fwd_apply<REMOTE>(B, g, c, R, T, X0, xd0, cnt, lane);
    if (!ha) break;
    c = cb;
    R = Rb;
  }
}

// C = 1: one CTA per front.  C > 1: a cluster of C CTAs per front (grid =
// clusters x C, cluster i takes list positions i, i + #clusters, ...)
template <int C>
__global__ void __launch_bounds__(kThr, 1)
k_fwd_tree(SnDev sd, TreeDev td, const double* __restrict__ lval, double* w, double* uvec) {
  extern __shared__ __align__(16) double dyn[];
  FwdSmem& sm = *reinterpret_cast<FwdSmem*>(dyn);
  double* T = dyn + (sizeof(FwdSmem) + 7) / 8;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = C > 1 ? static_cast<int>(cl.block_rank()) : 0;
  const int team = C > 1 ? blockIdx.x / C : blockIdx.x, nteams = C > 1 ? gridDim.x / C : gridDim.x;
  const double* T0 = C > 1 ? cl.map_shared_rank(T, 0) : T;
  const int* xd0 = C > 1 ? cl.map_shared_rank(&sm.xdone, 0) : &sm.xdone;
  unsigned long long ph[5] = {0, 0, 0, 0, 0};  // trace: SM clocks per phase, summed over the fronts
  for (int li = team; li < td.n; li += nteams) {
    FrontGeo g = front_geo(sd, lval, __ldg(td.list + li));
    int row_lo = 0, row_hi = g.f;  // the front rows this CTA gathers and writes
    if (C > 1) {
      if (rank == 0) {
        g.rhi = g.P;
        row_hi = g.k;
      } else {
        int j0, j1;
        rank_share(g.NR - g.P, C, rank, j0, j1);
        g.rlo = g.P + j0;
        g.rhi = g.P + j1;
        row_lo = g.k + 32 * j0;
        row_hi = min(g.f, g.k + 32 * j1);
      }
    }
    const bool tr = td.trace && tid == 0 && rank == 0;
    unsigned long long t0 = tr ? gtime() : 0, t1 = 0, t2 = 0, t3 = 0;
    if (warp == 0 && rank == 0)  // the chain's first L blocks do not depend on anything
      for (int b = 0; b < kStages; ++b) fwd_stage(sm.head[b], g, b, lane);
    for (int i = tid; i < kMaxRB; i += kThr) sm.cnt[i] = 0;
    if (tid == 0) sm.xdone = 0;
    // gather: T_r = w_r (pivot rows) + the children's entries in child order.
    // Its static part before the children are awaited (off the critical
    // path; cold index loads after the step's L2 flush): this CTA's pivot
    // rows of w (final before the launch) and every child's destination rows
    for (int r = row_lo + tid; r < row_hi; r += kThr) T[r] = r < g.k ? __ldcg(w + g.c0 + r) : 0.0;
    const int ch0 = __ldg(sd.ch_ptr + g.s), ch1 = __ldg(sd.ch_ptr + g.s + 1);
    int gtot = td.stage ? 0 : -1;  // entries staged (-1: more than kGMax, gathered directly)
    for (int cc = ch0; cc < ch1 && gtot >= 0; ++cc) {
      const int c = __ldg(sd.ch + cc);
      const int rp = __ldg(sd.rel_ptr + c), fu = __ldg(sd.rel_ptr + c + 1) - rp;
      if (gtot + fu > kGMax) {
        gtot = -1;
        break;
      }
      for (int i = tid; i < fu; i += kThr) {
        cp4(&sm.grel[gtot + i], sd.rel + rp + i);
        sm.gsrc[gtot + i] = rp + i;
      }
      gtot += fu;
    }
    cp_commit();
    if (warp > 0) {  // the bulk warps' first L blocks (static), before the children are awaited
      int c1, R1;
      if (fwd_first(g, warp - 1, c1, R1)) fwd_stage_first(sm.first[warp - 1], g, c1, R1, lane);
    }
    if (C > 1) cl.sync();  // rank 0's progress is reset before any rank reads it
    // children's update vectors: wide children in the list publish flags
    if (warp == 1) {
      const int e0 = __ldg(td.wait_ptr + li), e1 = __ldg(td.wait_ptr + li + 1);
      for (int e = e0 + lane; e < e1; e += 32) gwait_ge(td.flags + __ldg(td.wait + e), 1);
    }
    __syncthreads();
    if (tr) t1 = gtime();
    if (gtot >= 0) {  // every child's update entries in one round trip, then child by child
      cp_wait<0>();
      __syncthreads();  // grel / gsrc staged
      constexpr int kJ = kGMax / kThr;
      double v[kJ];
#pragma unroll
      for (int j = 0; j < kJ; ++j) {
        const int e = tid + j * kThr;
        v[j] = e < gtot ? __ldcg(uvec + sm.gsrc[e]) : 0.0;
      }
      for (int cc = ch0, o = 0; cc < ch1; ++cc) {
        const int c = __ldg(sd.ch + cc);
        const int o1 = o + __ldg(sd.rel_ptr + c + 1) - __ldg(sd.rel_ptr + c);
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
          const int e = tid + j * kThr;
          if (e >= o && e < o1) {
            const int dr = sm.grel[e];
            if (dr >= row_lo && dr < row_hi) T[dr] += v[j];
          }
        }
        o = o1;
        __syncthreads();
      }
    } else {  // child by child, a CTA barrier between children
      cp_wait<0>();
      __syncthreads();
      for (int cc = ch0; cc < ch1; ++cc) {
        const int c = __ldg(sd.ch + cc);
        const int rp = __ldg(sd.rel_ptr + c), fu = __ldg(sd.rel_ptr + c + 1) - rp;
        for (int i = tid; i < fu; i += kThr) {
          const int dr = __ldg(sd.rel + rp + i);
          const double u = __ldcg(uvec + rp + i);
          if (dr >= row_lo && dr < row_hi) T[dr] += u;
        }
        __syncthreads();
      }
    }
    if (tr) t2 = gtime();
    if (rank == 0) {
      if (warp == 0)
        fwd_chain(g, T, sm);
      else
        fwd_bulk<false>(g, warp - 1, T, T, &sm.xdone, sm.cnt, sm.first[warp - 1]);
    } else if (warp > 0) {
      fwd_bulk<true>(g, warp - 1, T, T0, xd0, sm.cnt, sm.first[warp - 1]);
    }
    __syncthreads();
    if (tr) t3 = gtime();
    double* u = uvec + __ldg(sd.rel_ptr + g.s);
    for (int r = row_lo + tid; r < row_hi; r += kThr) {
      if (r < g.k)
        w[g.c0 + r] = T[r];
      else
        u[r - g.k] = T[r];
    }
    if (C > 1) {
      cl.sync();  // every rank's rows are out (and rank 0's T is no longer read)
    } else {
      __syncthreads();
    }
    if (tid == 0 && rank == 0)  // the barrier above orders every thread's (rank's) writes before it
      st_release(td.flags + g.s, 1);
    if (tr) {  // per phase: wait, gather, solve, write-out + publish
      const unsigned long long t4 = gtime();
      ph[0] += t1 - t0;
      ph[1] += t2 - t1;
      ph[2] += t3 - t2;
      ph[3] += t4 - t3;
      ph[4] += 1;
    }
  }
  if (td.trace && tid == 0 && rank == 0)
    for (int i = 0; i < 5; ++i) td.trace[8 * static_cast<size_t>(blockIdx.x) + i] = ph[i];
}

// ---------------------------------------------------------------------------
// backward
struct BwdSmem {
  // chain head of block b: rows [32b, 32b+64) x block b's columns; column q,
  // 16-byte chunk c at chunk index q*32 + (c ^ (q & 7)) (lane = column reads)
  double head[kStages][32 * 64];
  double Ts[kBulk][32 * kTsSL];  // per bulk warp: one 32x32 block, row-major
  int grow[kTreeMaxF];           // x positions of this CTA's update rows (staged)
  int xdone;                     // pivot blocks solved, counted from the last
  int cnt[kMaxRB];               // per column block: contributions applied
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

// the chain of block b needs nexp contributions: its own CTA's items (C = 1:
// every update block and pivot blocks b+2..P-1; C > 1: the pivot blocks) and,
// C > 1, one partial per rank that owns update blocks
__device__ __forceinline__ void bwd_chain(const FrontGeo& g, double* X, const double* acc, int slots,
                                          int pstride, int nrem, double* x, BwdSmem& sm) {
  const int lane = threadIdx.x & 31;
  __syncwarp();  // the warp enters converged (the CTA's tid-0 branches)
  const int U1 = g.rhi - g.rlo;
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
    wait_ge(&sm.cnt[b], U1 + max(0, g.P - 2 - b) + nrem);
    double sb = 0.0;
    for (int sl = 0; sl < slots; ++sl) sb += acc[(sl * pstride + b) * 32 + lane];
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

// bulk items (R, b): row block R applied to column block b.  Phase 1 -- this
// CTA's update blocks [rlo, rhi), known from the start: items
// t = (P-1-b) * U1 + (R-rlo) (column blocks from the last, where the chain
// starts) dealt round-robin over the bulk warps; phase 2 (the chain's CTA) --
// pivot blocks R = P-1 .. 2 as the chain solves them, items b <= R-2 with
// b % kBulk == wb, from b = R-2 down (the one the chain needs next first).
struct BwdIt {
  int t, R, b;
};
__device__ __forceinline__ bool bwd_phase2_from(const FrontGeo& g, int wb, BwdIt& it, int R,
                                                bool ph2) {
  it.t = 0x7fffffff;
  if (!ph2) return false;
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
  const int U1 = g.rhi - g.rlo;
  if (it.t >= g.P * U1) return false;
  it.b = g.P - 1 - it.t / U1;
  it.R = g.rlo + it.t % U1;
  return true;
}
__device__ __forceinline__ bool bwd_first(const FrontGeo& g, int wb, BwdIt& it, bool ph2) {
  it.t = wb;
  if (bwd_set1(g, it)) return true;
  return bwd_phase2_from(g, wb, it, g.P - 1, ph2);
}
__device__ __forceinline__ bool bwd_next(const FrontGeo& g, int wb, BwdIt& it, bool ph2) {
  if (it.t != 0x7fffffff) {
    it.t += kBulk;
    if (bwd_set1(g, it)) return true;
    return bwd_phase2_from(g, wb, it, g.P - 1, ph2);
  }
  it.b -= kBulk;
  if (it.b >= 0) return true;
  return bwd_phase2_from(g, wb, it, it.R - 1, ph2);
}
__device__ __forceinline__ void bwd_load(double (&v)[32], const FrontGeo& g, int R, int b, int lane) {
  const int r0 = rb_start(g.k, g.P, R), nr = rb_size(g.k, g.f, g.P, R);
  const int q0 = 32 * b, nq = min(32, g.k - q0);
  const double* src = g.L + r0 + lane + static_cast<size_t>(q0) * g.ld;
  const bool ok = lane < nr;
#pragma unroll
  for (int q = 0; q < 32; ++q) v[q] = (ok && q < nq) ? __ldg(src + q * g.ld) : 0.0;
}
// bwd_load's block straight into the warp's transpose buffer Ts (row lane,
// column q at Ts[lane * kTsSL + q]) by cp.async: no registers held
__device__ __forceinline__ void bwd_stage_ts(double* Ts, const FrontGeo& g, int R, int b, int lane) {
  const int r0 = rb_start(g.k, g.P, R), nr = rb_size(g.k, g.f, g.P, R);
  const int q0 = 32 * b, nq = min(32, g.k - q0);
  const double* src = g.L + r0 + lane + static_cast<size_t>(q0) * g.ld;
  const bool ok = lane < nr;
#pragma unroll 8
  for (int q = 0; q < 32; ++q) {
    if (ok && q < nq)
      cp8(Ts + lane * kTsSL + q, src + q * g.ld);
    else
      Ts[lane * kTsSL + q] = 0.0;
  }
  cp_commit();
}
__device__ __forceinline__ void red_rel_cta(int* p, int v) {
  asm volatile("red.release.cta.shared::cta.add.s32 [%0], %1;" ::"r"(sptr(p)), "r"(v) : "memory");
}

// remote rank (C > 1, rank >= 1): partial sums of its update rows per column
// block, summed over its bulk warps in warp order when the block's last item
// lands, then sent to rank 0's slot `rank` with one release add on rank 0's
// counter
struct BwdRemote {
  double* acc0;  // rank 0's partial slots (DSMEM)
  int* cnt0;     // rank 0's counters (DSMEM)
  const double* accw_all;  // this rank's per-warp partials
  int pstride, rank;
};

template <bool REMOTE>
__device__ __forceinline__ void bwd_apply(const double (&v)[32], const FrontGeo& g, int R, int b,
                                          const double* X, double* accw, double* Ts, BwdSmem& sm,
                                          const BwdRemote& rm, int lane) {
  if (R < g.P) wait_ge(&sm.xdone, g.P - R);
  const int r0 = rb_start(g.k, g.P, R), nr = rb_size(g.k, g.f, g.P, R);
  __syncwarp();  // every lane's reads of the previous item's Ts are done
#pragma unroll
  for (int q = 0; q < 32; ++q) Ts[lane * kTsSL + q] = v[q];
  __syncwarp();
  double a = accw[32 * b + lane];
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i < nr) a = fma(Ts[i * kTsSL + lane], X[r0 + i], a);
  accw[32 * b + lane] = a;
  __syncwarp();
  if (!REMOTE) {
    if (lane == 0) red_rel_cta(&sm.cnt[b], 1);
    return;
  }
  int last = 0;
  if (lane == 0) last = atom_add_acqrel_cta(&sm.cnt[b], 1) == (g.rhi - g.rlo) - 1;
  last = __shfl_sync(kFull, last, 0);
  if (!last) return;
  __syncwarp();
  double s = 0.0;
  for (int w = 0; w < kBulk; ++w) s += rm.accw_all[(w * rm.pstride + b) * 32 + lane];
  rm.acc0[(rm.rank * rm.pstride + b) * 32 + lane] = s;
  __syncwarp();
  if (lane == 0) red_rel_cl(rm.cnt0 + b, 1);
}

// the warp's first item was staged into Ts before the parent was awaited
// (k_bwd_tree: L is static); the later ones go through registers, one ahead
template <bool REMOTE>
__device__ __forceinline__ void bwd_bulk(const FrontGeo& g, int wb, const double* X, double* accw,
                                         BwdSmem& sm, bool ph2, const BwdRemote& rm) {
  const int lane = threadIdx.x & 31;
  __syncwarp();  // the warp enters converged (the CTA's tid-0 branches)
  BwdIt it;
  if (!bwd_first(g, wb, it, ph2)) return;
  double* Ts = sm.Ts[wb];
  double A[32], B[32];
  cp_wait<0>();  // the first item's block, staged into Ts before the parent was awaited
  __syncwarp();
#pragma unroll
  for (int q = 0; q < 32; ++q) A[q] = Ts[lane * kTsSL + q];
  for (;;) {
    BwdIt nx = it;
    const bool hb = bwd_next(g, wb, nx, ph2);
    if (hb) bwd_load(B, g, nx.R, nx.b, lane);
    bwd_apply<REMOTE>(A, g, it.R, it.b, X, accw, Ts, sm, rm, lane);
    if (!hb) break;
    it = nx;
    const bool ha = bwd_next(g, wb, nx, ph2);
    if (ha) bwd_load(A, g, nx.R, nx.b, lane);
    bwd_apply<REMOTE>(B, g, it.R, it.b, X, accw, Ts, sm, rm, lane);
    if (!ha) break;
    it = nx;
  }
}

// partial slots: C = 1, one per bulk warp; C > 1, rank 0 keeps slot 0 for its
// pivot-row items (each column block belongs to one warp there) and slot r
// for rank r's partials, ranks >= 1 one per bulk warp
template <int C>
__global__ void __launch_bounds__(kThr, 1)
k_bwd_tree(SnDev sd, TreeDev td, const double* __restrict__ lval, const double* __restrict__ d,
           const double* __restrict__ w, double* x, int pmax) {
  extern __shared__ __align__(16) double dyn[];
  BwdSmem& sm = *reinterpret_cast<BwdSmem*>(dyn);
  constexpr int kSlots = C > kBulk ? C : kBulk;
  double* acc = dyn + (sizeof(BwdSmem) + 7) / 8;  // kSlots x pmax x 32
  double* X = acc + kSlots * 32 * pmax;            // front rows
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = C > 1 ? static_cast<int>(cl.block_rank()) : 0;
  const int team = C > 1 ? blockIdx.x / C : blockIdx.x, nteams = C > 1 ? gridDim.x / C : gridDim.x;
  BwdRemote rm{};
  if (C > 1) {
    rm.acc0 = cl.map_shared_rank(acc, 0);
    rm.cnt0 = cl.map_shared_rank(sm.cnt, 0);
    rm.accw_all = acc;
    rm.pstride = pmax;
    rm.rank = rank;
  }
  unsigned long long ph[5] = {0, 0, 0, 0, 0};  // trace: SM clocks per phase, summed over the fronts
  for (int i = tid; i < kMaxRB; i += kThr) sm.cnt[i] = 0;
  for (int i = tid; i < kSlots * 32 * pmax; i += kThr) acc[i] = 0.0;
  if (tid == 0) sm.xdone = 0;
  if (C > 1)
    cl.sync();  // every rank's slots are zero before any rank adds to rank 0's
  else
    __syncthreads();
  for (int li0 = team; li0 < td.n; li0 += nteams) {
    const int li = td.n - 1 - li0;
    FrontGeo g = front_geo(sd, lval, __ldg(td.list + li));
    const int U = g.NR - g.P;
    int nrem = 0;
    if (C > 1) {
      for (int r = 1; r < C; ++r) {
        int j0, j1;
        rank_share(U, C, r, j0, j1);
        nrem += j1 > j0;
      }
      if (rank == 0) {
        g.rlo = g.rhi = g.P;  // no update rows
      } else {
        int j0, j1;
        rank_share(U, C, rank, j0, j1);
        g.rlo = g.P + j0;
        g.rhi = g.P + j1;
      }
    } else {
      g.rlo = g.P;
      g.rhi = g.NR;
    }
    const bool tr = td.trace && tid == 0 && rank == 0;
    unsigned long long t0 = tr ? gtime() : 0, t1 = 0, t2 = 0, t3 = 0;
    if (warp == 0 && rank == 0)
      for (int o = 0; o < kStages; ++o) bwd_stage(sm.head[o], g, g.P - 1 - o, lane);
    // the slots and counters are zero here: zeroed before the loop and after
    // every front (before its closing barrier), so no cluster barrier is
    // needed before the other ranks add to rank 0's
    // z_q = w_q / d_q for the pivots (the forward result, final)
    if (rank == 0)
      for (int q = tid; q < g.k; q += kThr) X[q] = __ldg(w + g.c0 + q) / __ldg(d + g.c0 + q);
    // the bulk warps' first item (static L) into their transpose buffers
    // before the parent is awaited: the other ranks' first partials are what
    // rank 0's chain waits for at every front
    if (warp > 0) {
      BwdIt it0;
      if (bwd_first(g, warp - 1, it0, rank == 0)) bwd_stage_ts(sm.Ts[warp - 1], g, it0.R, it0.b, lane);
    }
    // the x positions of this CTA's update rows: static, staged before the
    // parent is awaited (cold index loads off the critical path)
    const int ur0 = g.rhi > g.rlo ? rb_start(g.k, g.P, g.rlo) : 0;
    const int ur1 = g.rhi > g.rlo ? min(g.f, rb_start(g.k, g.P, g.rhi - 1) + 32) : 0;
    {
      const int* rows = sd.rows + __ldg(sd.rows_ptr + g.s);
      for (int r = ur0 + tid; r < ur1; r += kThr) cp4(&sm.grow[r], rows + r);
      cp_commit();
    }
    // the parent's solution rows (the CTAs that own update rows)
    const int par = __ldg(td.par + li);
    if (tid == 0 && par >= 0 && g.rhi > g.rlo) gwait_ge(td.flags + par, 2);
    cp_wait<0>();
    __syncthreads();
    if (tr) t1 = gtime();
    for (int r = ur0 + tid; r < ur1; r += kThr) X[r] = __ldcg(x + sm.grow[r]);
    __syncthreads();
    if (tr) t2 = gtime();
    if (rank == 0) {
      if (warp == 0)
        bwd_chain(g, X, acc, C > 1 ? C : kBulk, pmax, C > 1 ? nrem : 0, x, sm);
      else
        bwd_bulk<false>(g, warp - 1, X, C > 1 ? acc : acc + (warp - 1) * 32 * pmax, sm, true, rm);
    } else if (warp > 0) {
      bwd_bulk<true>(g, warp - 1, X, acc + (warp - 1) * 32 * pmax, sm, false, rm);
    }
    if (tr) t3 = gtime();
    __syncthreads();  // this CTA is done with its slots and counters (rank 0: every partial consumed)
    for (int i = tid; i < kMaxRB; i += kThr) sm.cnt[i] = 0;
    for (int sl = 0; sl < kSlots; ++sl)
      for (int i = tid; i < 32 * g.P; i += kThr) acc[sl * 32 * pmax + i] = 0.0;
    if (tid == 0) sm.xdone = 0;
    if (C > 1) {
      cl.sync();  // every rank's x rows are out and slots reset
    } else {
      __syncthreads();
    }
    if (tid == 0 && rank == 0) st_release(td.flags + g.s, 2);
    if (tr) {
      const unsigned long long t4 = gtime();
      ph[0] += t1 - t0;
      ph[1] += t2 - t1;
      ph[2] += t3 - t2;
      ph[3] += t4 - t3;
      ph[4] += 1;
    }
  }
  if (td.trace && tid == 0 && rank == 0)
    for (int i = 0; i < 5; ++i) td.trace[8 * static_cast<size_t>(gridDim.x + blockIdx.x) + i] = ph[i];
}

}  // namespace

static size_t fwd_tree_smem(int fmax) { return (sizeof(FwdSmem) + 7) / 8 * 8 + sizeof(double) * fmax; }
static size_t bwd_tree_smem(int fmax, int pmax, int C) {
  const int slots = C > kBulk ? C : kBulk;
  return (sizeof(BwdSmem) + 7) / 8 * 8 + sizeof(double) * (static_cast<size_t>(slots) * 32 * pmax + fmax);
}

template <int C>
static void tree_init_c(int optin) {
  cudaFuncSetAttribute(k_fwd_tree<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
  cudaFuncSetAttribute(k_bwd_tree<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
}

static void tree_init() {
  static PerDeviceOnce once;
  once([] {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    tree_init_c<1>(optin);
    tree_init_c<kTreeCluster>(optin);
  });
}

// resident teams (C = 1: CTAs, C > 1: clusters) for both directions at these
// sizes (0: does not fit)
int tree_teams(int C, int fmax, int pmax) {
  tree_init();
  if (fmax > kTreeMaxF || (fmax + 31) / 32 + 2 > kMaxRB) return 0;
  if (C != 1 && C != kTreeCluster) return 0;
  int res[2] = {0, 0};
  for (int dir = 0; dir < 2; ++dir) {
    const void* fn = C == 1 ? (dir ? reinterpret_cast<const void*>(k_bwd_tree<1>)
                                   : reinterpret_cast<const void*>(k_fwd_tree<1>))
                            : (dir ? reinterpret_cast<const void*>(k_bwd_tree<kTreeCluster>)
                                   : reinterpret_cast<const void*>(k_fwd_tree<kTreeCluster>));
    const size_t smem = dir ? bwd_tree_smem(fmax, pmax, C) : fwd_tree_smem(fmax);
    if (C == 1) {
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res[dir], fn, kThr, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
      }
      int dev = 0, sms = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      res[dir] *= sms;
    } else {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(static_cast<unsigned>(C));
      cfg.blockDim = dim3(kThr);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = static_cast<unsigned>(C);
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      if (cudaOccupancyMaxActiveClusters(&res[dir], fn, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
      }
    }
  }
  return res[0] < res[1] ? res[0] : res[1];
}

template <class Kern, class... Args>
static void launch_c(Kern kern, int C, int teams, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(teams * C));
  cfg.blockDim = dim3(kThr);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(C);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, kern, args...));
}

void launch_fwd_tree(const SnDev& sd, const TreeDev& td, const double* lval, double* w, double* uvec,
                     int C, int teams, int fmax, cudaStream_t st) {
  tree_init();
  if (C == 1)
    launch_c(k_fwd_tree<1>, 1, teams, fwd_tree_smem(fmax), st, sd, td, lval, w, uvec);
  else
    launch_c(k_fwd_tree<kTreeCluster>, kTreeCluster, teams, fwd_tree_smem(fmax), st, sd, td, lval, w, uvec);
}

void launch_bwd_tree(const SnDev& sd, const TreeDev& td, const double* lval, const double* d,
                     const double* w, double* x, int C, int teams, int fmax, int pmax, cudaStream_t st) {
  tree_init();
  if (C == 1)
    launch_c(k_bwd_tree<1>, 1, teams, bwd_tree_smem(fmax, pmax, 1), st, sd, td, lval, d, w, x, pmax);
  else
    launch_c(k_bwd_tree<kTreeCluster>, kTreeCluster, teams, bwd_tree_smem(fmax, pmax, kTreeCluster), st,
             sd, td, lval, d, w, x, pmax);
}

}  // namespace nclb
