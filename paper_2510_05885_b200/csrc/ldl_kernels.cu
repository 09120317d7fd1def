// Static-pivot supernodal multifrontal LDL^T and its triangular solves for
// sm_100a.  Numeric semantics follow proj/src/sparse.cpp:182-276: pivots in
// the fixed (AMD) order, |d| < eps replaced by sign(d)*eps (exact zero -> +eps)
// and counted, inertia from the signs of D, ok = false on a non-finite or
// zero pivot or a non-finite L entry.
//
// Two tiers (see symbolic.hpp):
//  * warp tier  -- fronts of <= 32 rows.  One persistent kernel; each warp
//    pulls a heavy path of the supernodal elimination tree from a global
//    counter and walks it bottom-up (factor, forward solve) or top-down
//    (backward solve) with the front in shared memory, one front row per
//    lane.  Light children are other warps' paths that precede it in the
//    path order, so a warp only ever spins on work that an already-running
//    warp owns: no deadlock, no per-level launches, and long chains
//    (ring-shaped power grids) run at on-chip latency.
//  * wide tier  -- fronts above 32 rows and all their ancestors:
//    wide_kernels.cu (factorization) and wide_solve.cu (solves).
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#include "cuda_util.hpp"
#include "device.cuh"
#include "launch.hpp"

namespace nclb {

constexpr int kWF = 32;       // warp-tier front limit (rows)
constexpr int kFLD = 33;      // padded leading dimension of a warp front
constexpr int kWarpsPerCta = 4;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int next_path(int* counter, int lane) {
  int pi = 0;
  if (lane == 0) pi = atomicAdd(counter, 1);
  return __shfl_sync(0xffffffffu, pi, 0);
}

// spin on a flag with exponential back-off: a waiting warp then hardly takes
// issue slots (or L2 bandwidth) from the warp it waits for on the same SM
__device__ __forceinline__ void wait_flag(const int* flag, int epoch) {
  unsigned ns = 32;
  while (ld_relaxed(flag) != epoch) {
    __nanosleep(ns);
    if (ns < 512) ns <<= 1;
  }
}

// Publish a node: every lane's stores, then the flag.  __syncwarp orders the
// lanes' stores before lane 0's (bar.warp.sync is a memory-ordering barrier
// among its threads) and lane 0's st.release.gpu makes everything that
// happens-before it visible at gpu scope before the flag (release is
// cumulative) -- no per-lane fence.sc (__threadfence: MEMBAR.SC + L1
// invalidation, ~0.2 us per node on a chain).
__device__ __forceinline__ void publish(int* flag, int epoch, int lane) {
  __syncwarp();
  if (lane == 0) st_release(flag, epoch);
}

// ---------------------------------------------------------------------------
// warp-tier numeric factorization.  A warp walks its path bottom-up.  Each
// front is assembled in shared memory (lane = front row) and then factored
// in registers: lane i holds row i of the front, pivot p broadcasts column p
// by shuffles and every lane applies its rank-1 row update -- no shared
// memory round trip per update.  The update block is then scattered straight
// into the (zeroed) shared front of the next node on the path, the parent;
// only a path top writes its update block and flag to global memory, since
// every other node's parent is the same warp.  The assembly loads that do
// not depend on other warps -- the A entries (kLtA chunks in registers), the
// light children's extend-add chunks (symbolic.hpp lt_ent: destinations
// distinct within a chunk, so a chunk is one parallel step) -- are issued
// before the light children's flags are awaited.  Order of the sums: heavy
// child, A entries, light children in child order.
// Phase timers of the warp-tier factorization.  NCL_WTRACE builds print the
// cycles the longest path's warp spends per phase (diagnostic, NCL_NO_GRAPH=1).
// Default builds keep the same code with a condition that is never true at
// run time: the dead blocks split the node loop into basic blocks that ptxas
// schedules separately, and that keeps each phase's loads issued ahead of
// their uses -- measured on the 3927-node spine of opf_toy 78484: 19.8 ms
// without the blocks, 14.2 ms with them.
#ifndef NCL_WTRACE
#define NCL_WTRACE_DEAD
#endif
#if defined(NCL_WTRACE) || defined(NCL_WTRACE_DEAD)
__device__ unsigned long long g_wtrace[11];
__device__ unsigned long long g_ftrace[5];  // forward solve: flags, gather, substitute, prefetch, store
__device__ unsigned long long g_wtime[4];  // kernel start (min), spine start/end, last other path end (max)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif
constexpr int kLtR = 6;   // light-child chunks held in registers
constexpr int kLtA = 2;   // A-entry chunks held in registers
constexpr long long kSrcMask = (1LL << 48) - 1;
constexpr int kCB = kWF + 2;  // pivot-column broadcast buffer (x2 per warp)
constexpr size_t kWarpFactorDoubles = 2 * kWF * kFLD + 2 * kCB;
constexpr size_t kWarpFactorBytes = sizeof(double) * kWarpFactorDoubles;

// The k pivots of a warp-tier front held as register rows (fr[j] = row
// `lane`, column p + j while pivot p is processed: the row shifts down one
// column per pivot, so every register index is static).  NC = register
// columns kept live (>= f).  Pivot p's column is broadcast through shared
// memory (cb, two alternating buffers, one warp barrier per pivot), the next
// pivot is shuffled out as soon as its column is updated, and l = u * (1/d)
// with the wide tier's reciprocal.  l is written to column p of the shared
// front F, d stays in lane p (myd, perturbed flag mypf).
template <int NC, int BATCH>
__device__ __forceinline__ void warp_pivots(double (&fr)[kWF + 1], double* F, double* cb, int k, int f,
                                            double eps, int lane, double& myd, bool& mypf, int& fail) {
  double dnext = __shfl_sync(0xffffffffu, fr[0], 0);
  for (int p = 0; p < k; ++p) {
    double dp = dnext;
    const bool pf = fabs(dp) < eps;
    if (pf) dp = (dp >= 0.0) ? eps : -eps;
    myd = lane == p ? dp : myd;
    mypf = lane == p ? pf : mypf;
    const bool mine = lane > p && lane < f;
    const double u = fr[0];
    double* cbp = cb + (p & 1) * kCB;
    if (lane >= p) cbp[lane - p] = u;
    // row p+1's entry in column p+1, shuffled while 1/d is formed: with
    // u(p+1) from the broadcast column every lane forms the next pivot itself
    // (row p+1's own operations: the same value) -- no shuffle on the chain
    const double a11 = __shfl_sync(0xffffffffu, fr[1], (p + 1) & 31);
    const double r = rcp_nr(dp);
    const double l = mine ? u * r : 0.0;
    if (mine) F[p * kFLD + lane] = l;
    fail |= !isfinite(l);
    __syncwarp();
    // column values in batches of BATCH (128-bit loads): bounded registers
    constexpr int B = NC < BATCH ? NC : BATCH;
#pragma unroll
    for (int j0 = 0; j0 < NC; j0 += B) {
      double2 v[B / 2];  // issued before the dependent chain of the batch
#pragma unroll
      for (int j = 0; j < B; j += 2) v[j / 2] = *reinterpret_cast<const double2*>(cbp + j0 + j);
      if (j0 == 0) {  // the next pivot's column first
        fr[0] = fr[1] - l * v[0].y;
        const double u1 = v[0].y;  // u of row p+1 (0 past the front)
        dnext = (p + 1 < f) ? a11 - ((u1 * r) * u1) : fr[0];
      }
#pragma unroll
      for (int j = (j0 == 0 ? 2 : 0); j < B; j += 2) {
        fr[j0 + j - 1] = fr[j0 + j] - l * v[j / 2].x;
        fr[j0 + j] = fr[j0 + j + 1] - l * v[j / 2].y;
      }
    }
    fr[NC - 1] = 0.0;
  }
}

// static description of the node at one path position (symbolic.hpp prec)
struct WRec {
  int s, c0, k, f, chb, che, lb, le, ab, ae, relp, rowsp, lsb, lse, spar;
  long long loff, uoff;
};

__device__ __forceinline__ WRec load_rec(const SnDev& sd, int q) {
  const int4 a = ldg_pin(sd.prec + 4 * q), b = ldg_pin(sd.prec + 4 * q + 1);
  const int4 c = ldg_pin(sd.prec + 4 * q + 2), d = ldg_pin(sd.prec + 4 * q + 3);
  const longlong2 o = ldg_pin(sd.poff + q);
  return WRec{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w, d.x, d.y, d.z, o.x, o.y};
}

// the factorization's index loads for one node (no values)
struct FIdx {
  long long ent[kLtR];  // light-child chunks
  int ap[kLtA], as[kLtA];  // A entries: front position, value slot
  int chid;             // this lane's child (first 32)
  int myrel;            // parent position of front row `lane` (rows below)
};

__device__ __forceinline__ void load_fidx(const SnDev& sd, const WRec& R, int lane, FIdx& X) {
#pragma unroll
  for (int t = 0; t < kLtR; ++t) X.ent[t] = (R.lb + t * 32 < R.le) ? ldg_pin(sd.lt_ent + R.lb + t * 32 + lane) : -1;
#pragma unroll
  for (int t = 0; t < kLtA; ++t) {
    const int a = R.ab + t * 32 + lane;
    X.ap[t] = a < R.ae ? ldg_pin(sd.asm_pos + a) : -1;
    X.as[t] = a < R.ae ? ldg_pin(sd.asm_slot + a) : 0;
  }
  X.chid = R.chb + lane < R.che ? ldg_pin(sd.ch + R.chb + lane) : -1;
  X.myrel = (lane >= R.k && lane < R.f) ? ldg_pin(sd.rel + R.relp + lane - R.k) : 0;
}

// PIPE: the software pipeline along the path (long chains: latency-bound).
// !PIPE: each node's index words loaded at its start, fewer registers and
// three CTAs per SM (many short paths: throughput-bound, e.g. SCOPF blocks).
template <bool PIPE>
__global__ void __launch_bounds__(kWarpsPerCta * 32, PIPE ? 0 : 3)
k_factor_warp(SnDev sd, FactorDev fd, const double* __restrict__ kval,
              int* flags, int epoch, int* counter, int npaths, double eps) {
  extern __shared__ double wsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int npos = 0, nneg = 0, pert = 0, fail = 0;
  double* F = wsm + static_cast<size_t>(wid) * kWarpFactorDoubles;
  double* N = F + kWF * kFLD;
  double* cb = N + kWF * kFLD;
#ifdef NCL_WTRACE
  if (lane == 0) atomicMin(&g_wtime[0], gtimer());
#endif
  cb[lane] = 0.0;
  cb[kCB + lane] = 0.0;
  if (lane < 2) cb[32 + lane] = cb[kCB + 32 + lane] = 0.0;
  for (;;) {
    const int pi = next_path(counter, lane);
    if (pi >= npaths) break;
    const int pb = sd.path_ptr[pi], pe = sd.path_ptr[pi + 1];
    // software pipeline along the path: node q+1's record, index loads and
    // light-child flags are issued while node q is factored
    WRec R = load_rec(sd, pb);
    FIdx X;
    load_fidx(sd, R, lane, X);
    int fl = X.chid >= 0 ? ld_relaxed(flags + X.chid) : epoch;
    double av[kLtA];  // A values (kval is an input: prefetched a node ahead)
#pragma unroll
    for (int t = 0; t < kLtA; ++t) av[t] = X.ap[t] >= 0 ? ldg_pin(kval + X.as[t]) : 0.0;
    for (int c = 0; c < R.f; ++c) F[c * kFLD + lane] = 0.0;
    int heavy = -1;
#if defined(NCL_WTRACE) || defined(NCL_WTRACE_DEAD)
#ifdef NCL_WTRACE
    const bool trc = PIPE && pi == 0;  // the longest root path is handed out first
#else
    const bool trc = PIPE && pi == 0 && epoch == 0x7fffffff;
#endif
    if (trc && lane == 0) g_wtime[1] = gtimer();
    unsigned long long tph[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long tq = clock64();
#define WT(i)                       \
  if (trc) {                        \
    const long long tn = clock64(); \
    tph[i] += tn - tq;              \
    tq = tn;                        \
  }
#else
#define WT(i)
#endif
    for (int q = pb; q < pe; ++q) {
      const bool top = q == pe - 1;
      const int k = R.k, f = R.f;
      WRec Rn = R;
      if (!top) Rn = load_rec(sd, q + 1);
      if (!PIPE && q > pb) {
        load_fidx(sd, R, lane, X);
        fl = (X.chid >= 0 && X.chid != heavy) ? ld_relaxed(flags + X.chid) : epoch;
#pragma unroll
        for (int t = 0; t < kLtA; ++t) av[t] = X.ap[t] >= 0 ? ldg_pin(kval + X.as[t]) : 0.0;
      }
      WT(0);
      if (X.chid >= 0 && X.chid != heavy) {
        if (fl != epoch) wait_flag(flags + X.chid, epoch);
        flag_acquire(flags + X.chid);
      }
      for (int c = R.chb + 32 + lane; c < R.che; c += 32) {
        const int ch = sd.ch[c];
        if (ch != heavy) {
          wait_flag(flags + ch, epoch);
          flag_acquire(flags + ch);
        }
      }
      __syncwarp();
      WT(1);
      double lv[kLtR];
#pragma unroll
      for (int t = 0; t < kLtR; ++t) lv[t] = X.ent[t] >= 0 ? __ldcg(fd.upd + (X.ent[t] & kSrcMask)) : 0.0;
#pragma unroll
      for (int t = 0; t < kLtA; ++t)
        if (X.ap[t] >= 0) F[(X.ap[t] >> 16) * kFLD + (X.ap[t] & 0xffff)] += av[t];
      for (int a = R.ab + kLtA * 32 + lane; a < R.ae; a += 32) {
        const int pos = sd.asm_pos[a];
        F[(pos >> 16) * kFLD + (pos & 0xffff)] += __ldg(kval + sd.asm_slot[a]);
      }
      __syncwarp();
      WT(2);
#pragma unroll
      for (int t = 0; t < kLtR; ++t) {
        if (R.lb + t * 32 < R.le) {
          if (X.ent[t] >= 0) {
            const int dst = static_cast<int>(X.ent[t] >> 48);
            F[(dst >> 5) * kFLD + (dst & 31)] += lv[t];
          }
          __syncwarp();
        }
      }
      for (int e = R.lb + kLtR * 32; e < R.le; e += 32) {
        const long long x = __ldg(sd.lt_ent + e + lane);
        if (x >= 0) {
          const int dst = static_cast<int>(x >> 48);
          F[(dst >> 5) * kFLD + (dst & 31)] += __ldcg(fd.upd + (x & kSrcMask));
        }
        __syncwarp();
      }
      WT(3);
      double fr[kWF + 1];
#pragma unroll
      for (int j = 0; j < kWF; ++j) fr[j] = (j < f && lane < f) ? F[j * kFLD + lane] : 0.0;
      fr[kWF] = 0.0;
      const int myrel = X.myrel;
      // node q+1's index loads, in flight during the pivots
      WT(6);
      if (PIPE && !top) load_fidx(sd, Rn, lane, X);
      WT(7);
      double myd = 0.0;
      bool mypf = false;
      // (the pipelined walk loads a pivot's whole column at once; the lean
      // one in halves, to stay within three CTAs' registers)
      constexpr int kBatch = PIPE ? kWF : 16;
      if (f <= 8)
        warp_pivots<8, kBatch>(fr, F, cb, k, f, eps, lane, myd, mypf, fail);
      else if (f <= 16)
        warp_pivots<16, kBatch>(fr, F, cb, k, f, eps, lane, myd, mypf, fail);
      else
        warp_pivots<kWF, kBatch>(fr, F, cb, k, f, eps, lane, myd, mypf, fail);
      WT(8);
      // node q+1's light-child flags (its heavy child is this node)
      if (PIPE && !top) {
        fl = (X.chid >= 0 && X.chid != R.s) ? ld_relaxed(flags + X.chid) : epoch;
#pragma unroll
        for (int t = 0; t < kLtA; ++t) av[t] = X.ap[t] >= 0 ? ldg_pin(kval + X.as[t]) : 0.0;
      }
      __syncwarp();
      WT(9);
      {
        // the f x k L block is contiguous: coalesced linear stores (entries
        // on or above the diagonal written as zero)
        double* Lb = fd.lval + R.loff;
        const int nl = f * k;
        const float rf = 1.0f / static_cast<float>(f);
#pragma unroll 4
        for (int idx = lane; idx < nl; idx += 32) {
          int col = __float2int_rd((static_cast<float>(idx) + 0.5f) * rf);
          int row = idx - col * f;
          if (row >= f) {
            row -= f;
            ++col;
          } else if (row < 0) {
            row += f;
            --col;
          }
          Lb[idx] = row > col ? F[col * kFLD + row] : 0.0;
        }
        WT(10);
        const bool piv = lane < k;
        if (piv) fd.d[R.c0 + lane] = myd;
        fail |= piv && (!isfinite(myd) || myd == 0.0);
        const unsigned pos = __ballot_sync(0xffffffffu, piv && myd > 0.0);
        const unsigned neg = __ballot_sync(0xffffffffu, piv && !(myd > 0.0));
        const unsigned prt = __ballot_sync(0xffffffffu, piv && mypf);
        npos += __popc(pos);
        nneg += __popc(neg);
        pert += __popc(prt);
      }
      WT(4);
      if (top) {
        const int fu = f - k;
        double* Us = fd.upd + R.uoff;
        if (lane >= k && lane < f) {
#pragma unroll
          for (int j = 0; j < kWF; ++j)
            if (j < fu && j <= lane - k) Us[(lane - k) + static_cast<size_t>(j) * fu] = fr[j];
        }
        publish(flags + R.s, epoch, lane);
      } else {
        // update block -> the parent's (zeroed) shared front
        int cj[kWF];
#pragma unroll
        for (int j = 0; j < kWF; ++j) cj[j] = __shfl_sync(0xffffffffu, myrel, (j + k) & 31);
        for (int c = 0; c < Rn.f; ++c) N[c * kFLD + lane] = 0.0;
        __syncwarp();
        const int fu = f - k;
#pragma unroll
        for (int j = 0; j < kWF; ++j)
          if (j < fu && lane >= j + k && lane < f) N[cj[j] * kFLD + myrel] = fr[j];
        __syncwarp();
        double* t = F;
        F = N;
        N = t;
        heavy = R.s;
        R = Rn;
      }
      WT(5);
    }
#if defined(NCL_WTRACE) || defined(NCL_WTRACE_DEAD)
    if (trc && lane == 0) {
      for (int i = 0; i < 11; ++i) g_wtrace[i] = tph[i];
      g_wtime[2] = gtimer();
    }
#ifdef NCL_WTRACE
    if (!trc && lane == 0) atomicMax(&g_wtime[3], gtimer());
#endif
#endif
  }
  fail = __any_sync(0xffffffffu, fail);
  if (lane == 0) {
    if (npos) atomicAdd(fd.stats + 0, npos);
    if (nneg) atomicAdd(fd.stats + 1, nneg);
    if (pert) atomicAdd(fd.stats + 2, pert);
    if (fail) atomicOr(fd.stats + 3, 1);
  }
}

// ---------------------------------------------------------------------------
// forward solve L w = b (in place on the permuted vector w); update vectors of
// the multifrontal solve live at uvec + rel_ptr[s] (f - k entries).  The L
// block's column entries of a lane's row are all loaded before the
// substitution chain; the heavy child's update vector stays in shared memory
// along the path (path tops write theirs for other readers) and the light
// children's entries arrive as chunks with distinct destinations (ls_ent),
// their index words loaded before the children's flags are awaited.
constexpr int kLsR = 4;  // light-child solve chunks held in registers

template <bool PIPE>
__global__ void __launch_bounds__(kWarpsPerCta * 32, PIPE ? 0 : 6)
k_fwd_warp(SnDev sd, const double* __restrict__ lval, double* w, double* uvec,
           int* flags, int epoch, int* counter, int npaths) {
  __shared__ double Ts[kWarpsPerCta][kWF];
  __shared__ double Hs[kWarpsPerCta][kWF];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* T = Ts[wid];
  double* Hv = Hs[wid];
  for (;;) {
    const int pi = next_path(counter, lane);
    if (pi >= npaths) break;
    const int pb = sd.path_ptr[pi], pe = sd.path_ptr[pi + 1];
    // software pipeline: node q+1's record, L block, rhs and index words are
    // loaded while node q is substituted
    WRec R = load_rec(sd, pb);
    double lv[kWF];  // L(lane, p), p < lane
    double wv;
    long long ent[kLsR];
    int chid;
    auto load_node = [&](const WRec& Q) {
      const double* Lb = lval + Q.loff;
#pragma unroll
      for (int p = 0; p < kWF; ++p)
        lv[p] = (p < Q.k && lane > p && lane < Q.f) ? ldg_pin(Lb + lane + static_cast<size_t>(p) * Q.f) : 0.0;
      wv = (lane < Q.k) ? ldcg_pin(w + Q.c0 + lane) : 0.0;
    };
    auto load_idx = [&](const WRec& Q) {
#pragma unroll
      for (int t = 0; t < kLsR; ++t)
        ent[t] = (Q.lsb + t * 32 < Q.lse) ? ldg_pin(sd.ls_ent + Q.lsb + t * 32 + lane) : -1;
      chid = Q.chb + lane < Q.che ? ldg_pin(sd.ch + Q.chb + lane) : -1;
    };
    load_node(R);
    load_idx(R);
    int fl = chid >= 0 ? ld_relaxed(flags + chid) : epoch;  // polled a node ahead
    int heavy = -1, hfu = 0, hri = 0;
#if defined(NCL_WTRACE) || defined(NCL_WTRACE_DEAD)
#ifdef NCL_WTRACE
    const bool trc = PIPE && pi == 0;
#else
    const bool trc = PIPE && pi == 0 && epoch == 0x7fffffff;
#endif
    unsigned long long tph[6] = {0, 0, 0, 0, 0, 0};
    long long tq = clock64();
#endif
    for (int q = pb; q < pe; ++q) {
      const bool top = q == pe - 1;
      const int k = R.k, f = R.f;
      WRec Rn = R;
      if (!top) Rn = load_rec(sd, q + 1);
      if (!PIPE && q > pb) {
        load_node(R);
        load_idx(R);
        fl = (chid >= 0 && chid != heavy) ? ld_relaxed(flags + chid) : epoch;
      }
      if (chid >= 0 && chid != heavy) {
        if (fl != epoch) wait_flag(flags + chid, epoch);
        flag_acquire(flags + chid);
      }
      for (int c = R.chb + 32 + lane; c < R.che; c += 32) {
        const int ch = sd.ch[c];
        if (ch != heavy) {
          wait_flag(flags + ch, epoch);
          flag_acquire(flags + ch);
        }
      }
      __syncwarp();
      WT(0);
      double uv[kLsR];
#pragma unroll
      for (int t = 0; t < kLsR; ++t) uv[t] = ent[t] >= 0 ? __ldcg(uvec + (ent[t] & kSrcMask)) : 0.0;
      T[lane] = wv;
      __syncwarp();
      if (lane < hfu) T[hri] += Hv[lane];
      __syncwarp();
#pragma unroll
      for (int t = 0; t < kLsR; ++t) {
        if (R.lsb + t * 32 < R.lse) {
          if (ent[t] >= 0) T[ent[t] >> 48] += uv[t];
          __syncwarp();
        }
      }
      for (int e = R.lsb + kLsR * 32; e < R.lse; e += 32) {
        const long long x = __ldg(sd.ls_ent + e + lane);
        if (x >= 0) T[x >> 48] += __ldcg(uvec + (x & kSrcMask));
        __syncwarp();
      }
      WT(1);
      if (PIPE && !top) load_idx(Rn);  // node q+1's index words, in flight during the substitution
      double t = (lane < f) ? T[lane] : 0.0;
#pragma unroll
      for (int p = 0; p < kWF; ++p) {
        if (p < k) {
          const double wp = __shfl_sync(0xffffffffu, t, p);
          t -= lv[p] * wp;
        }
      }
      WT(2);
      const int hri_n = (!top && lane < f - k) ? ldg_pin(sd.rel + R.relp + lane) : 0;
      if (PIPE && !top) {
        load_node(Rn);
        fl = (chid >= 0 && chid != R.s) ? ld_relaxed(flags + chid) : epoch;
      }
      WT(3);
      __syncwarp();
      if (lane >= k && lane < f) Hv[lane - k] = t;
      if (lane < k)
        w[R.c0 + lane] = t;
      else if (lane < f && top)
        uvec[R.relp + lane - k] = t;
      if (top) publish(flags + R.s, epoch, lane);
      heavy = R.s;
      hfu = f - k;
      hri = hri_n;
      R = Rn;
      __syncwarp();
      WT(4);
    }
#if defined(NCL_WTRACE) || defined(NCL_WTRACE_DEAD)
    if (trc && lane == 0)
      for (int i = 0; i < 5; ++i) g_ftrace[i] = tph[i];
#endif
  }
}

// backward solve L^T x = D^-1 w, paths taken in reverse order, top-down.
// Lane q owns pivot q and its L column; the rows below the block enter
// through one shuffle-broadcast dot product per lane, then the pivots
// resolve last-first with one shuffle + FMA each.  Along a path the parent's
// front values (its pivots' x and the rows below it) stay in registers, lane
// i holding front row i, and the child reads its rows below through rel with
// a shuffle; only a path's top node reads x from memory, and only nodes with
// light children (other paths' tops) publish a flag.  Node q-1's record, L
// columns, w, d and rel are loaded while node q is solved.
template <bool PIPE>  // !PIPE: trees of short paths, register-capped for 6 CTAs per SM
__global__ void __launch_bounds__(kWarpsPerCta * 32, PIPE ? 0 : 6)
k_bwd_warp(SnDev sd, const double* __restrict__ lval, const double* __restrict__ d,
           const double* __restrict__ w, double* x, int* flags, int epoch,
           const int8_t* __restrict__ wide, int* counter, int npaths) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    const int pj = next_path(counter, lane);
    if (pj >= npaths) break;
    const int pi = __ldg(sd.bwd_path + pj);
    const int pb = sd.path_ptr[pi], pe = sd.path_ptr[pi + 1];
    WRec R = load_rec(sd, pe - 1);
    double lc[kWF];  // L(r, lane), r > lane
    double wd;       // w / d of pivot `lane`
    auto load_node = [&](const WRec& Q) {
      const double* Lb = lval + Q.loff;
#pragma unroll
      for (int r = 0; r < kWF; ++r)
        lc[r] = (lane < Q.k && r > lane && r < Q.f) ? ldg_pin(Lb + r + static_cast<size_t>(lane) * Q.f) : 0.0;
      wd = (lane < Q.k) ? ldcg_pin(w + Q.c0 + lane) / ldg_pin(d + Q.c0 + lane) : 0.0;
    };
    load_node(R);
    double xr;
    {
      const int par = R.spar;
      const int row = (lane >= R.k && lane < R.f) ? __ldg(sd.rows + R.rowsp + lane) : 0;
      if (par >= 0 && !wide[par] && lane == 0) {
        wait_flag(flags + par, epoch);
        flag_acquire(flags + par);
      }
      __syncwarp();
      xr = (lane >= R.k && lane < R.f) ? __ldcg(x + row) : 0.0;
    }
    for (int q = pe - 1; q >= pb; --q) {
      const int k = R.k, f = R.f;
      WRec Rn = R;
      if (q > pb) Rn = load_rec(sd, q - 1);
      double z = wd;
#pragma unroll
      for (int r = 0; r < kWF; ++r) {
        if (r >= k && r < f) {
          const double xv = __shfl_sync(0xffffffffu, xr, r);
          z -= lc[r] * xv;
        }
      }
      // the next (child) node's rows below as positions in this front
      const int myrel = (q > pb && lane >= Rn.k && lane < Rn.f) ? ldg_pin(sd.rel + Rn.relp + lane - Rn.k) : 0;
#pragma unroll
      for (int p = kWF - 1; p >= 0; --p) {
        if (p < k) {
          const double xp = __shfl_sync(0xffffffffu, z, p);
          if (lane < p) z -= lc[p] * xp;
        }
      }
      if (lane < k) x[R.c0 + lane] = z;
      const double pv = lane < k ? z : xr;  // this front's row `lane`
      if (R.lse > R.lsb) publish(flags + R.s, epoch, lane);  // light children wait
      if (q > pb) {
        load_node(Rn);
        xr = __shfl_sync(0xffffffffu, pv, myrel);
        if (!(lane >= Rn.k && lane < Rn.f)) xr = 0.0;
      }
      R = Rn;
    }
  }
}

__global__ void k_permute_in(int n, const int* __restrict__ perm,
                             const double* __restrict__ b, double* w) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) w[i] = b[perm[i]];
}

__global__ void k_permute_out(int n, const int* __restrict__ perm,
                              const double* __restrict__ xp, double* x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[perm[i]] = xp[i];
}

// ---------------------------------------------------------------------------
// launch helpers (host)
void launch_factor_warp(const SnDev& sd, const FactorDev& fd, const double* kval,
                        int* flags, int epoch, int* counter, int npaths,
                        double eps, int grid, bool pipe, cudaStream_t st) {
  if (npaths == 0) return;
  static PerDeviceOnce init;
  init([] {
    cudaFuncSetAttribute(k_factor_warp<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kWarpsPerCta * kWarpFactorBytes));
    cudaFuncSetAttribute(k_factor_warp<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kWarpsPerCta * kWarpFactorBytes));
  });
  if (pipe)
    k_factor_warp<true><<<grid, kWarpsPerCta * 32, kWarpsPerCta * kWarpFactorBytes, st>>>(
        sd, fd, kval, flags, epoch, counter, npaths, eps);
  else
    k_factor_warp<false><<<grid, kWarpsPerCta * 32, kWarpsPerCta * kWarpFactorBytes, st>>>(
        sd, fd, kval, flags, epoch, counter, npaths, eps);
#ifdef NCL_WTRACE  // diagnostic build: phase cycles of the last path's warp (NCL_NO_GRAPH=1)
  {
    unsigned long long t[11], tt[4];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(t, g_wtrace, sizeof(t));
    cudaMemcpyFromSymbol(tt, g_wtime, sizeof(tt));
    std::fprintf(stderr, "[ncl wtime] spine starts %.3f ms, ends %.3f ms, other paths end %.3f ms\n",
                 (tt[1] - tt[0]) * 1e-6, (tt[2] - tt[0]) * 1e-6, (tt[3] - tt[0]) * 1e-6);
    const unsigned long long init2[4] = {~0ull, 0, 0, 0};
    cudaMemcpyToSymbol(g_wtime, init2, sizeof(init2));
    std::fprintf(stderr,
                 "[ncl wtrace] static %llu flags %llu A %llu light %llu fr %llu fidx %llu pivots %llu "
                 "flagpf %llu Lstore %llu d+stats %llu next %llu\n",
                 t[0], t[1], t[2], t[3], t[6], t[7], t[8], t[9], t[10], t[4], t[5]);
  }
#endif
}

void launch_fwd_warp(const SnDev& sd, const double* lval, double* w, double* uvec,
                     int* flags, int epoch, int* counter, int npaths, int grid, bool pipe,
                     cudaStream_t st) {
  if (npaths == 0) return;
  if (pipe)
    k_fwd_warp<true><<<grid, kWarpsPerCta * 32, 0, st>>>(sd, lval, w, uvec, flags, epoch, counter, npaths);
  else
    k_fwd_warp<false><<<grid, kWarpsPerCta * 32, 0, st>>>(sd, lval, w, uvec, flags, epoch, counter, npaths);
#ifdef NCL_WTRACE
  {
    unsigned long long t[5];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(t, g_ftrace, sizeof(t));
    std::fprintf(stderr, "[ncl ftrace] flags %llu gather %llu substitute %llu prefetch %llu store %llu\n", t[0],
                 t[1], t[2], t[3], t[4]);
  }
#endif
}

void launch_bwd_warp(const SnDev& sd, const double* lval, const double* d,
                     const double* w, double* x, int* flags, int epoch,
                     const int8_t* wide, int* counter, int npaths, int grid, bool pipe,
                     cudaStream_t st) {
  if (npaths == 0) return;
  if (pipe)
    k_bwd_warp<true><<<grid, kWarpsPerCta * 32, 0, st>>>(sd, lval, d, w, x, flags, epoch, wide, counter, npaths);
  else
    k_bwd_warp<false><<<grid, kWarpsPerCta * 32, 0, st>>>(sd, lval, d, w, x, flags, epoch, wide, counter, npaths);
}

void launch_permute_in(int n, const int* perm, const double* b, double* w,
                       cudaStream_t st) {
  if (n == 0) return;
  k_permute_in<<<(n + 255) / 256, 256, 0, st>>>(n, perm, b, w);
}

void launch_permute_out(int n, const int* perm, const double* xp, double* x,
                        cudaStream_t st) {
  if (n == 0) return;
  k_permute_out<<<(n + 255) / 256, 256, 0, st>>>(n, perm, xp, x);
}

int warp_tier_grid(int which) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (which == 3) {  // lean solves
    int a = 0, b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_fwd_warp<false>, kWarpsPerCta * 32, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_bwd_warp<false>, kWarpsPerCta * 32, 0);
    per_sm = a < b ? a : b;
  } else if (which == 1) {
    int a = 0, b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_fwd_warp<true>, kWarpsPerCta * 32, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_bwd_warp<true>, kWarpsPerCta * 32, 0);
    per_sm = a < b ? a : b;
  } else {
    const size_t smem = kWarpsPerCta * kWarpFactorBytes;
    if (which == 0) {
      cudaFuncSetAttribute(k_factor_warp<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_factor_warp<true>, kWarpsPerCta * 32, smem);
    } else {
      cudaFuncSetAttribute(k_factor_warp<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_factor_warp<false>, kWarpsPerCta * 32, smem);
    }
  }
  if (per_sm < 1) per_sm = 1;
  return sms * per_sm;
}

}  // namespace nclb
