// Wide-tier numeric factorization (fronts above 32 rows and their ancestors).
//
// A wide front is f x f column-major with leading dimension ld = wide_ld(f)
// (even: every column starts 16-byte aligned), resident in HBM/L2 inside the
// L buffer; its first k columns are the L block, the trailing (f-k)^2 corner
// the update matrix the parent extend-adds from.
//
// Data movement: every block a kernel computes on is staged into shared
// memory with 16-byte cp.async copies.  Measured on B200 (tools/ubench_ld.cu),
// one warp pulls a 32x32 FP64 block out of L2 in ~1.2K cycles that way versus
// 3.3-7K cycles with register loads (too few loads in flight per warp) -- the
// difference between a latency-bound and a DMMA-bound trailing update.
//
// Building blocks:
//   assemble_col  -- (WARP) one front column: zero, scatter A, extend-add the
//                    children's columns that land in it, child by child
//                    (deterministic order), accumulated in shared memory;
//   diag_block    -- (WARP) static-pivot LDL^T of a <=32-pivot diagonal block
//                    (sparse.cpp:235-247 pivot rule, inertia, perturbed
//                    counts); a lane owns one row in registers, rotated one
//                    column per pivot (static register indices, compact loop);
//   trsm_rows     -- (THREAD per row) the rows below the block, in lockstep
//                    with diag_block through a shared-memory progress flag;
//   group_tile    -- (4 WARPS) F22 -= L21 D L21^T on a 32x32 tile: A, B, C
//                    staged by cp.async, each warp an 8-row slice on FP64
//                    tensor cores (mma.sync.m8n8k4.f64 = DMMA).
// k_wide_front runs a whole tree level in ONE launch: one thread-block
// cluster (1..16 CTAs) per front walks assembly -> panels with one panel of
// lookahead (see the panel loop).  Levels holding huge fronts use the
// multi-kernel path (k_wide_assemble, then per panel k_wide_panel /
// k_wide_update) so one front spreads over every SM.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdlib>
#include <stdint.h>

#include "cuda_util.hpp"
#include "device.cuh"
#include "launch.hpp"
#include "layout.hpp"
#include "symbolic.hpp"
#include "dag.hpp"

namespace cg = cooperative_groups;

namespace nclb {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kGroups = kWarps / 4;   // 4-warp tile groups
constexpr int kSL = 40;               // smem column stride of a staged 32-row block
constexpr int kTrsRows = 96;          // rows per TRSM round (warps 1..3)
constexpr int kSLT = kTrsRows + 2;    // smem column stride of the TRSM stage
constexpr int kHugeRows = kPanelRows + 32;  // threads per huge-path panel CTA: diag warp + 96 TRSM
constexpr unsigned kFull = 0xffffffffu;

// Us[p][j] = unscaled u = F(p0+p+1+j, p0+p) after the first p pivots (zero
// past the block); row p is what every row below subtracts at pivot p.
struct PanelSmem {
  double Us[kWidePanel][kWidePanel];
  double rinv[kWidePanel];
  double Lsh[kWidePanel][kWidePanel + 1];  // scaled L11 (published late)
  int prog;                                // pivots of the block published
  int qctr;                                // deferred-update tile queue
  int gq[kGroups];                         // per-group dequeued tile
};

struct GroupSmem {
  double A[kWidePanel * kSL], B[kWidePanel * kSL], C[kWidePanel * kSL];
  double d[kWidePanel];
};

struct RowSmem {  // per-group buffers of groups 1..3
  GroupSmem g;
};

// dynamic shared memory of k_wide_front (the assembly accumulators alias it).
// Group 0 (warps 0-3) computes phase-B tiles in the diagonal / TRSM stage,
// which is idle then; groups 1-3 have their own tile buffers.
struct StageSmem {
  union {
    struct {
      double D[kWidePanel * kSL];    // diagonal block
      double TR[kWidePanel * kSLT];  // TRSM rows
    } p;
    GroupSmem g0;
  } u;
  RowSmem r[kGroups - 1];
};



__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// diagnostic (NCL_PANEL_TRACE): per huge-path panel g, 8 %globaltimer stamps
// (latest over the CTAs) -- panel entry, after the programmatic wait, staged, strip applied,
// diagonal block done, panel end (last CTA), rest update start, rest end
// Compiled in only with -DNCL_PANEL_TRACE (make EXTRA=-DNCL_PANEL_TRACE): even
// never taken, the stamps cost the panel kernel 16 registers and ~0.9 us per
// launch (ncu launch list, same box).
#ifdef NCL_PANEL_TRACE
__device__ unsigned long long* g_ptrace = nullptr;
__device__ __forceinline__ void ptrace_max(int g, int i) {
  if (g >= 0 && g_ptrace) atomicMax(g_ptrace + 8 * g + i, globaltimer());
}
#else
__device__ __forceinline__ void ptrace_max(int, int) {}
#endif

__device__ __forceinline__ void cp16(void* dst, const void* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp4(void* dst, const void* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait_group() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// rows [r0, r0+nr) x columns [c0, c0+nc) of the column-major M (ld even, base
// 16-byte aligned) -> S with column stride SL: element (r0+i, c0+j) lands at
// S[j*SL + i + sh], sh = r0 & 1.  Every column copies NR2 16-byte chunks from
// the even row below r0 (a compile-time count: no integer division in the
// issue loop; rows past the block are harmless reads -- the L buffer is
// padded at its end).  Issued by thread t of nthr; completion: cp_wait_all /
// cp_wait_group + a barrier.
template <int NR2>
__device__ __forceinline__ int stage_block(double* S, int SL, const double* M, size_t ld, int r0,
                                           int c0, int nc, int t, int nthr) {
  const int a = r0 & ~1;
  const double* src = M + a + c0 * ld;
  for (int idx = t; idx < NR2 * nc; idx += nthr) {
    const int j = idx / NR2, ch = idx - j * NR2;
    cp16(S + j * SL + 2 * ch, src + 2 * ch + j * ld);
  }
  return r0 - a;
}
constexpr int kNR2 = (kUpdTile + 2) / 2;  // 32 rows + shift -> 17 chunks

// progress flag in shared memory: release by the diagonal warp, acquire by
// the lockstep TRSM warps (no MEMBAR.SC / system-scope generic stores)
__device__ __forceinline__ void st_release_smem(int* p, int v) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_smem(const int* p) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
  int v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}

// lower-triangular tile index -> (row block, col block), row >= col
__device__ __forceinline__ void tri_decode(int t, int& i, int& j) {
  int r = static_cast<int>((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
  while (r * (r + 1) / 2 > t) --r;
  while ((r + 1) * (r + 2) / 2 <= t) ++r;
  i = r;
  j = t - r * (r + 1) / 2;
}

// ---------------------------------------------------------------------------
// assembly of front column J (one warp).  acc: f doubles of shared memory
// private to this warp, or nullptr to accumulate in place (huge fronts).
// Index words are static: ColMeta (the column's contribution and A-entry
// ranges) can be loaded a column ahead (assemble_cols), and the first A chunk
// and children group are issued before the zero fill.
struct ColMeta {
  int e0, e1, a0, a1;
};
__device__ __forceinline__ ColMeta col_meta(const SnDev& sd, int s, int c0, int k, int J) {
  const int cb = sd.cc_off[s] + J;
  return ColMeta{ldg_pin(sd.cc_ptr + cb), ldg_pin(sd.cc_ptr + cb + 1), J < k ? ldg_pin(sd.asm_cp + c0 + J) : 0,
                 J < k ? ldg_pin(sd.asm_cp + c0 + J + 1) : 0};
}
constexpr int kColG = 4;  // children per contribution group
struct ColPre {  // the first children group's index words
  int cw0[kColG], rb0[kColG];
  long long ub0[kColG];
};
// the column's static part: zero fill and A entries (kval is an input)
__device__ __forceinline__ void col_static(const SnDev& sd, const double* __restrict__ kval, int f, int J,
                                           double* a, const ColMeta& m, ColPre& p) {
  const int lane = threadIdx.x & 31;
  const int qa = m.a0 + lane;
  const int ap0 = qa < m.a1 ? ldg_pin(sd.asm_pos + qa) : 0, as0 = qa < m.a1 ? ldg_pin(sd.asm_slot + qa) : 0;
#pragma unroll
  for (int t = 0; t < kColG; ++t) {
    const bool in = m.e0 + t < m.e1;
    p.cw0[t] = in ? ldg_pin(sd.cc_cnt + m.e0 + t) : 0;
    p.ub0[t] = in ? ldg_pin(sd.cc_ubase + m.e0 + t) : 0;
    p.rb0[t] = in ? ldg_pin(sd.cc_rbase + m.e0 + t) : 0;
  }
  for (int r = J + lane; r < f; r += 32) a[r] = 0.0;
  __syncwarp();
  if (qa < m.a1) a[ap0 & 0xffff] += __ldg(kval + as0);
  for (int q = qa + 32; q < m.a1; q += 32) a[sd.asm_pos[q] & 0xffff] += __ldg(kval + sd.asm_slot[q]);
  __syncwarp();
}
// the children's contributions (the previous level's update blocks), then
// the column out of acc
__device__ __forceinline__ void col_children(const SnDev& sd, const FactorDev& fd, int s, int f, double* F,
                                             size_t ld, int J, double* acc, const ColMeta& m, const ColPre& p) {
  constexpr int G = kColG;
  const int lane = threadIdx.x & 31;
  double* col = F + J * ld;
  double* a = acc ? acc : col;
  const int e0 = m.e0, e1 = m.e1;
  const int* cw0 = p.cw0;
  const int* rb0 = p.rb0;
  const long long* ub0 = p.ub0;
  const int ng = sd.split_ng[s];
  if (ng) {  // group sums of the contributions (split.cu), in group order
    const double* P = fd.ccpart + sd.split_off[s] + static_cast<size_t>(J) * ng * f;
    for (int r = J + lane; r < f; r += 32) {
      double v = a[r];
#pragma unroll 8
      for (int g = 0; g < ng; ++g) v += __ldcg(P + static_cast<size_t>(g) * f + r);
      a[r] = v;
    }
    __syncwarp();
  } else {
    // contributions in groups of four: the four children's column segments
    // are loaded together, then added one child after the other (a warp
    // barrier each); per position the order is fixed by (32-row chunk, child),
    // so sums are deterministic, though not child by child for columns
    // taller than 32 rows
    for (int eg = e0; eg < e1; eg += G) {
      const double* U[G];
      const int* rel[G];
      int cnt[G], mc = 0;
#pragma unroll
      for (int t = 0; t < G; ++t) {
        const int e = eg + t;
        cnt[t] = 0;
        U[t] = nullptr;
        rel[t] = nullptr;
        if (e < e1) {
          const int cw = eg == e0 ? cw0[t] : sd.cc_cnt[e];
          cnt[t] = cw & ((1 << 30) - 1);
          U[t] = ((cw >> 30) ? fd.lval : fd.upd) + (eg == e0 ? ub0[t] : sd.cc_ubase[e]);
          rel[t] = sd.rel + (eg == e0 ? rb0[t] : sd.cc_rbase[e]);
          mc = max(mc, cnt[t]);
        }
      }
      // four 32-row chunks per batch: every load of the batch is issued
      // before the first add (the adds go through a pointer the compiler
      // cannot tell apart from the loads, so it would not hoist them), the
      // adds in the (chunk, child) order of a chunk-by-chunk pass
      constexpr int B = 4;
      for (int i0 = lane; i0 < mc; i0 += 32 * B) {
        double v[B][G];
        int r[B][G];
#pragma unroll
        for (int b = 0; b < B; ++b)
#pragma unroll
          for (int t = 0; t < G; ++t) {
            const int i = i0 + 32 * b;
            v[b][t] = i < cnt[t] ? __ldcg(U[t] + i) : 0.0;
            r[b][t] = i < cnt[t] ? rel[t][i] : -1;
          }
#pragma unroll
        for (int b = 0; b < B; ++b)
#pragma unroll
          for (int t = 0; t < G; ++t) {
            if (r[b][t] >= 0) a[r[b][t]] += v[b][t];
            __syncwarp(__activemask());
          }
      }
      __syncwarp();
    }
  }
  if (acc)
    for (int r = J + lane; r < f; r += 32) col[r] = a[r];
}
__device__ __forceinline__ void assemble_col_m(const SnDev& sd, const FactorDev& fd,
                                               const double* __restrict__ kval, int s, int f, double* F,
                                               size_t ld, int J, double* acc, const ColMeta& m) {
  ColPre p;
  col_static(sd, kval, f, J, acc ? acc : F + J * ld, m, p);
  col_children(sd, fd, s, f, F, ld, J, acc, m, p);
}
__device__ __noinline__ void assemble_col(const SnDev& sd, const FactorDev& fd,
                                          const double* __restrict__ kval, int s, int c0, int k,
                                          int f, double* F, size_t ld, int J, double* acc) {
  assemble_col_m(sd, fd, kval, s, f, F, ld, J, acc, col_meta(sd, s, c0, k, J));
}
// columns J, J + Js, ... of the front on one warp, the next column's ColMeta
// in flight while a column is assembled
__device__ __noinline__ void assemble_cols(const SnDev& sd, const FactorDev& fd,
                                           const double* __restrict__ kval, int s, int c0, int k,
                                           int f, double* F, size_t ld, int J, int Js, double* acc) {
  if (J >= f) return;
  ColMeta m = col_meta(sd, s, c0, k, J);
  for (;;) {
    const int Jn = J + Js;
    ColMeta mn{0, 0, 0, 0};
    if (Jn < f) mn = col_meta(sd, s, c0, k, Jn);
    assemble_col_m(sd, fd, kval, s, f, F, ld, J, acc, m);
    if (Jn >= f) break;
    J = Jn;
    m = mn;
  }
}

// 1/d without the branchy slow path of __drcp_rn (which splits the pivot loop
// into basic blocks the scheduler cannot interleave across): MUFU.RCP64H
// seed + two Newton steps, within 1 ulp for the pivot magnitudes static
// pivoting admits (|d| >= eps; NaN/Inf propagate and are flagged).

// ---------------------------------------------------------------------------
// Pivots [pb, pe) of the diagonal block with a rotation width of W registers:
// after p pivots only columns p..31 of the block are live, so the later
// quarters rotate 24 / 16 / 8 registers instead of 32.  Branch-free: lanes
// that are not below the pivot write zeros to slots nobody reads.
template <int W>
__device__ __forceinline__ void diag_pivot(int p, int nb, double eps, double (&a)[kWidePanel],
                                           double& dnext, double& myd, int& pf, int& bad, int lane,
                                           PanelSmem& sm) {
  double dp = dnext;
  const bool small = fabs(dp) < eps;
  dp = small ? (dp >= 0.0 ? eps : -eps) : dp;
  const bool below = lane > p && lane < nb;
  const double u = below ? a[0] : 0.0;
  const double u1 = __shfl_sync(kFull, u, (p + 1) & 31);      // u of row p+1
  const double a11 = __shfl_sync(kFull, a[1], (p + 1) & 31);  // its entry in column p+1
  const double rp = rcp_nr(dp);
  const double l = u * rp;
  const double n0 = a[1] - l * u1;  // this row's entry in column p+1
  // the next pivot on every lane: row p+1's n0 by the same operations (the
  // same value) without a shuffle on the chain (~7 % fewer cycles per block,
  // tools/ubench_diag.cu)
  dnext = a11 - (u1 * rp) * u1;
  sm.Us[p][below ? lane - p - 1 : kWidePanel - 1] = u;  // slot 31 stays zero
  sm.Lsh[lane][p] = l;
  sm.rinv[p] = rp;
  myd = lane == p ? dp : myd;
  pf |= (lane == p) & small;
  bad |= !isfinite(l);
  __syncwarp();
  const double2* up = reinterpret_cast<const double2*>(sm.Us[p]);
  a[0] = n0;
  {
    const double2 v = up[0];
    a[1] = a[2] - l * v.y;
  }
#pragma unroll
  for (int j = 2; j < W; j += 2) {
    const double2 v = up[j >> 1];
    a[j] = a[j + 1] - l * v.x;
    a[j + 1] = (j + 2 < W ? a[j + 2] : 0.0) - l * v.y;
  }
}

// Pivots [pb, pe) with rotation width W, four per straight-line block so the
// scheduler overlaps pivot p+1's chain with pivot p's row update; the
// lockstep TRSM is released after every four pivots.
template <int W>
__device__ __forceinline__ void diag_steps(int pb, int pe, int nb, double eps, double (&a)[kWidePanel],
                                           double& dnext, double& myd, int& pf, int& bad, int lane,
                                           PanelSmem& sm, int* prog) {
  int p = pb;
#pragma unroll 1
  for (; p + 4 <= pe; p += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) diag_pivot<W>(p + u, nb, eps, a, dnext, myd, pf, bad, lane, sm);
    if (prog && lane == 0) st_release_smem(prog, p + 4);
  }
#pragma unroll 1
  for (; p < pe; ++p) {
    diag_pivot<W>(p, nb, eps, a, dnext, myd, pf, bad, lane, sm);
    if (prog && lane == 0) st_release_smem(prog, p + 1);
  }
}

// static-pivot LDL^T of the nb-pivot diagonal block at p0 (one warp), staged
// through D (32 x kSL doubles).  Fills sm.Us / sm.rinv / sm.Lsh and, when
// `prog` is given, publishes pivot p by setting *prog = p + 1 (threads running
// trsm_rows in lockstep wait on it).  With `dout` (publisher only) writes D
// and adds the inertia / perturbed / failure counts.
//
// The pivot chain is d_p -> 1/d_p -> next diagonal
// a' = a(p+1, p+1) - (u(p+1) / d_p) u(p+1), formed on every lane from
// a(p+1, p+1) and u(p+1) shuffled from lane p+1 while 1/d_p is computed, so
// no shuffle or shared-memory round trip is serial; the rest of the row
// update overlaps the chain.
__device__ __noinline__ void diag_block(const double* F, size_t ld, int p0, int nb, double eps,
                                        PanelSmem& sm, double* D, double* dout, int* stats,
                                        int* prog, bool staged = false) {
  const int lane = threadIdx.x & 31;
  // staged: D already holds the block (p0 is even: no shift)
  const int sh = staged ? 0 : stage_block<kNR2>(D, kSL, F, ld, p0, p0, nb, lane, 32);
  double* us = &sm.Us[0][0];
  for (int i = lane; i < kWidePanel * kWidePanel; i += 32) us[i] = 0.0;
  cp_wait_all();
  __syncwarp();
  double a[kWidePanel];  // a[j] = current F(p0+lane, p0+p+j)
#pragma unroll
  for (int j = 0; j < kWidePanel; ++j) a[j] = (lane < nb && j <= lane) ? D[j * kSL + lane + sh] : 0.0;
  double myd = 0.0;  // lane p keeps d_p
  int pf = 0, bad = 0;
  double dnext = __shfl_sync(kFull, a[0], 0);
  // two rotation widths: fewer code bodies (instruction fetch) than four
  // narrowing ones outweigh the extra zero updates (tools/ubench_diag.cu:
  // ~16 % fewer cycles per block)
  diag_steps<32>(0, min(nb, 16), nb, eps, a, dnext, myd, pf, bad, lane, sm, prog);
  diag_steps<16>(16, nb, nb, eps, a, dnext, myd, pf, bad, lane, sm, prog);
  __syncwarp();
  if (dout && lane < nb) dout[lane] = myd;
  if (stats) {
    const bool mine = lane < nb;
    const unsigned pos = __ballot_sync(kFull, mine && myd > 0.0);
    const unsigned neg = __ballot_sync(kFull, mine && !(myd > 0.0));
    const unsigned per = __ballot_sync(kFull, mine && pf);
    const bool fail = __any_sync(kFull, bad || (mine && (!isfinite(myd) || myd == 0.0)));
    if (lane == 0) {
      if (pos) atomicAdd(stats + 0, __popc(pos));
      if (neg) atomicAdd(stats + 1, __popc(neg));
      if (per) atomicAdd(stats + 2, __popc(per));
      if (fail) atomicOr(stats + 3, 1);
    }
  }
}

// TRSM pivots [pb, pe) for one row with rotation width W (see diag_steps)
template <int W>
__device__ __forceinline__ void trsm_steps(int pb, int pe, double (&x)[kWidePanel], double* row,
                                           size_t ld, const double* us, const double* rinv,
                                           const int* prog, bool& bad) {
#pragma unroll 1
  for (int p = pb; p < pe; ++p) {
    if (prog)  // back off between polls: the diagonal warp shares the LSU
      while (ld_acquire_smem(prog) <= p) __nanosleep(64);
    const double l = x[0] * rinv[p];
    row[p * ld] = l;
    bad |= !isfinite(l);
    const double2* up = reinterpret_cast<const double2*>(us + p * kWidePanel);
#pragma unroll
    for (int j = 0; j < W; j += 2) {
      const double2 v = up[j >> 1];
      x[j] = x[j + 1] - l * v.x;
      x[j + 1] = (j + 2 < W ? x[j + 2] : 0.0) - l * v.y;
    }
  }
}

// rows [row_lo, row_hi) of panel columns [p0, p0+nb): L(r, :) from the
// unscaled diagonal columns us (32x32) and 1/d.  nthr threads (named barrier
// `bar`), this one number vt; rows are staged nthr at a time into TR (column
// stride SLT >= nthr + 2).  With `prog`, pivot p is used as soon as
// *prog > p (lockstep with diag_block in the same CTA).
template <int NTHR>
__device__ __noinline__ void trsm_rows(double* F, size_t ld, int p0, int nb, int row_lo,
                                       int row_hi, const double* us, const double* rinv,
                                       int* stats, int vt, double* TR, const int* prog, int bar,
                                       bool staged = false) {
  constexpr int nthr = NTHR, SLT = NTHR + 2;
  bool bad = false;
  // staged: TR already holds the rows (one round: row_hi - row_lo <= NTHR)
  for (int base = row_lo; base < row_hi; base += nthr) {
    const int nr = min(nthr, row_hi - base);
    const int sh = staged ? (base & 1) : stage_block<(NTHR + 2) / 2>(TR, SLT, F, ld, base, p0, nb, vt, nthr);
    if (!staged) cp_wait_all();
    named_bar(bar, nthr);
    if (vt < nr) {
      double x[kWidePanel];
#pragma unroll
      for (int q = 0; q < kWidePanel; ++q) x[q] = q < nb ? TR[q * SLT + vt + sh] : 0.0;
      double* row = F + base + vt + p0 * ld;
      trsm_steps<32>(0, min(nb, 8), x, row, ld, us, rinv, prog, bad);
      trsm_steps<24>(8, min(nb, 16), x, row, ld, us, rinv, prog, bad);
      trsm_steps<16>(16, min(nb, 24), x, row, ld, us, rinv, prog, bad);
      trsm_steps<8>(24, nb, x, row, ld, us, rinv, prog, bad);
    }
    named_bar(bar, nthr);  // TR is reused by the next round
  }
  if (bad) atomicOr(stats + 3, 1);
}

__device__ __forceinline__ void dmma_m8n8k4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// DMMA core shared by the tile routines: rows gw*8..+8 of a 32x32 tile from
// staged A (shift shA), B (shB), scaled by d, minus into C (shC) -> F.
__device__ __forceinline__ void tile_mma_store(double* F, size_t ld, const double* A, int shA,
                                               const double* Bs, int shB, const double* Cs, int shC,
                                               const double* d, int nb, int r0, int nr, int q0,
                                               int nc, int gt) {
  const int lane = gt & 31, gw = gt >> 5, g = lane >> 2, tq = lane & 3;
  const int rr = gw * 8 + g;
  double acc[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < kWidePanel / 4; ++kk) {
    const int q = kk * 4 + tq;
    const bool qv = q < nb;
    const double a = (qv && rr < nr) ? A[q * kSL + rr + shA] : 0.0;
    const double dq = qv ? d[q] : 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cc = j * 8 + g;
      const double b = (qv && cc < nc) ? Bs[q * kSL + cc + shB] * dq : 0.0;
      dmma_m8n8k4(acc[j][0], acc[j][1], a, b);
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = j * 8 + tq * 2 + e;
      if (rr < nr && c < nc && r0 + rr >= q0 + c)
        F[(r0 + rr) + (q0 + c) * ld] = Cs[c * kSL + rr + shC] - acc[j][e];
    }
}

// 4 warps (128 threads, named barrier `bar`; gt = thread in group): the
// trailing-update tile F[r0:r0+32, q0:q0+32] -= L21_r D L21_q^T for panel
// columns [p0, p0+nb) (lower part only).  Warp gw computes rows gw*8..+8.
__device__ __noinline__ void group_tile(double* F, size_t ld, int f, const double* __restrict__ dv,
                                        int p0, int nb, int r0, int q0, GroupSmem& G, int gt,
                                        int bar) {
  const int nr = min(kUpdTile, f - r0), nc = min(kUpdTile, f - q0);
  const bool dg = r0 == q0;
  const int shA = stage_block<kNR2>(G.A, kSL, F, ld, r0, p0, nb, gt, 128);
  const int shB = dg ? shA : stage_block<kNR2>(G.B, kSL, F, ld, q0, p0, nb, gt, 128);
  const int shC = stage_block<kNR2>(G.C, kSL, F, ld, r0, q0, nc, gt, 128);
  if (gt < nb) G.d[gt] = __ldcg(dv + gt);
  cp_wait_all();
  named_bar(bar, 128);
  tile_mma_store(F, ld, G.A, shA, dg ? G.A : G.B, shB, G.C, shC, G.d, nb, r0, nr, q0, nc, gt);
  named_bar(bar, 128);  // G is reused by the group's next tile
}

// the trailing update of panel [p0, p0+nb) on the grid from p1 (T blocks),
// tiles (i, j) with 1 <= j <= i: this CTA takes tiles rank, rank + C, ...
// from its queue, groups 1..3 pull (the group buffers overlay RowSmem)
__device__ __forceinline__ void rest_update(double* F, size_t ld, int f, const double* dv, int p0,
                                            int nb, int p1, int T, int rank, int C, StageSmem& st,
                                            PanelSmem& sm, int grp, int gt) {
  const int ntiles = T * (T - 1) / 2;
  GroupSmem& G = *reinterpret_cast<GroupSmem*>(&st.r[grp - 1]);
  for (;;) {
    if (gt == 0) sm.gq[grp] = atomicAdd(&sm.qctr, 1);
    named_bar(1 + grp, 128);
    const int t = rank + sm.gq[grp] * C;
    if (t >= ntiles) break;
    int i, j;
    tri_decode(t, i, j);
    group_tile(F, ld, f, dv, p0, nb, p1 + (i + 1) * kUpdTile, p1 + (j + 1) * kUpdTile, G, gt, 1 + grp);
  }
}

// ---------------------------------------------------------------------------
// one launch per level, one cluster per front.
// trace (optional, diagnostic): per front, timestamps (ns) after assembly
// and after every panel / update phase, recorded by cluster rank 0
__global__ void __launch_bounds__(kThreads, 1)
k_wide_front(SnDev sd, FactorDev fd, const double* __restrict__ kval,
             const int* __restrict__ nodes, double eps, int acc_f, unsigned long long* trace) {
  __shared__ PanelSmem sm;
  extern __shared__ __align__(16) double dyn_smem[];
  StageSmem& st = *reinterpret_cast<StageSmem*>(dyn_smem);
  cg::cluster_group cl = cg::this_cluster();
  const int C = static_cast<int>(cl.num_blocks());
  const int rank = static_cast<int>(cl.block_rank());
  const int fi = blockIdx.x / C;
  const int s = nodes[fi];
  const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
  const size_t ld = wide_ld(f);
  double* F = fd.lval + sd.l_off[s];
  pdl_launch_dependents();
  pdl_wait();  // the children's update blocks (previous level)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = warp >> 2, gt = threadIdx.x & 127;
  const bool tr = trace && rank == 0 && threadIdx.x == 0;
  int ti = 0;
  if (threadIdx.x == 0) {
    sm.prog = 0;
    sm.qctr = 0;
  }
  if (tr) trace[fi * 128 + ti++] = globaltimer();
  {
    double* acc = dyn_smem + static_cast<size_t>(warp) * acc_f;
    assemble_cols(sd, fd, kval, s, c0, k, f, F, ld, rank * kWarps + warp, C * kWarps, acc);
  }
  cl.sync();
  if (tr) trace[fi * 128 + ti++] = globaltimer();
  // Panel loop with one panel of lookahead.  The trailing update of panel p
  // is split: its first column block (the next panel's columns) is applied
  // right away (phase B, all four groups); the rest is deferred into phase A
  // of panel p+1, where groups 1..3 run it while warp 0 factors the next
  // diagonal block and warps 1..3 solve the rows below it in lockstep.  Every
  // trailing tile still receives its updates in panel order (the phases are
  // separated by cluster barriers).
  int pend_p0 = 0, pend_p1 = 0, pend_nb = 0, pend_T = 0;  // deferred update
  const int kp = s == sd.schur ? 0 : k;  // Schur mode: the coupling front is only assembled
  for (int p0 = 0; p0 < kp; p0 += kWidePanel) {
    const int p1 = min(p0 + kWidePanel, k), nb = p1 - p0;
    const int rows = f - p1;
    const int chunk = (rows + C - 1) / C;
    const int lo = p1 + rank * chunk, hi = min(f, lo + chunk);
    // detailed stamps of the second panel (the first when k <= 32)
    unsigned long long* dt = (tr && p0 == (k > kWidePanel ? kWidePanel : 0)) ? trace + fi * 128 + 120
                                                                             : nullptr;
    if (dt) dt[0] = globaltimer();
    // phase A.  Every CTA factors the diagonal block itself (no extra
    // cluster barrier); rank 0 publishes D and the counts now, L11 after the
    // barrier (other CTAs may still be reading the unfactored block).
    if (warp == 0) {
      diag_block(F, ld, p0, nb, eps, sm, st.u.p.D, rank == 0 ? fd.d + c0 + p0 : nullptr,
                 rank == 0 ? fd.stats : nullptr, &sm.prog);
      if (dt) dt[1] = globaltimer();
    } else if (grp == 0) {
      trsm_rows<kTrsRows>(F, ld, p0, nb, lo, max(lo, hi), &sm.Us[0][0], sm.rinv, fd.stats,
                          threadIdx.x - 32, st.u.p.TR, &sm.prog, 1 + kGroups);
    } else if (pend_T > 1) {
      // deferred tiles (i, j), j >= 1, of the previous panel
      rest_update(F, ld, f, fd.d + c0 + pend_p0, pend_p0, pend_nb, pend_p1, pend_T, rank, C, st, sm,
                  grp, gt);
    }
    __syncthreads();
    if (dt) dt[2] = globaltimer();
    if (threadIdx.x == 0) {
      sm.prog = 0;
      sm.qctr = 0;
    }
    if (dt) dt[3] = globaltimer();
    cl.sync();
    if (dt) dt[4] = globaltimer();
    if (tr && ti < 119) trace[fi * 128 + ti++] = globaltimer();
    if (rank == 0)  // L11 (scaled) from shared memory, one column per warp
      for (int p = warp; p < nb; p += kWarps)
        if (lane > p && lane < nb) F[(p0 + lane) + (p0 + p) * ld] = sm.Lsh[lane][p];
    if (dt) dt[5] = globaltimer();
    // phase B: the next panel's column block now, the rest deferred; after
    // the last panel, the whole trailing update
    const int T = (rows + kUpdTile - 1) / kUpdTile;
    const bool last = p1 >= k;
    {
      GroupSmem& G = grp == 0 ? st.u.g0 : *reinterpret_cast<GroupSmem*>(&st.r[grp - 1]);
      for (int t = rank * kGroups + grp; t < T; t += C * kGroups)
        group_tile(F, ld, f, fd.d + c0 + p0, p0, nb, p1 + t * kUpdTile, p1, G, gt, 1 + grp);
    }
    if (last && T > 1) {  // no next panel: the rest of the update now
      if (threadIdx.x == 0) sm.qctr = 0;
      __syncthreads();
      if (grp > 0)
        rest_update(F, ld, f, fd.d + c0 + p0, p0, nb, p1, T, rank, C, st, sm, grp, gt);
    }
    pend_p0 = p0;
    pend_p1 = p1;
    pend_nb = nb;
    pend_T = last ? 0 : T;
    if (dt) dt[6] = globaltimer();
    cl.sync();
    if (dt) dt[7] = globaltimer();
    if (tr && ti < 119) trace[fi * 128 + ti++] = globaltimer();
  }
}

// ---------------------------------------------------------------------------
// multi-kernel path for levels with huge fronts
// a warp per front column, accumulated in the warp's shared-memory column
// (acc_f doubles) and written to the front once: in place in global memory
// the zero fill, the A entries and every child's adds were L2
// read-modify-write round trips on the critical path of each huge level
__global__ void __launch_bounds__(256)
k_wide_assemble(SnDev sd, FactorDev fd, const double* __restrict__ kval,
                const int4* __restrict__ tasks, int acc_f) {
  extern __shared__ __align__(16) double asm_acc[];
  const int4 t = tasks[blockIdx.x];
  const int s = t.x, J = t.y + (threadIdx.x >> 5);
  pdl_launch_dependents();
  const int c0 = sd.first[s], f = sd.f[s], k = sd.first[s + 1] - c0;
  const bool mine = J < min(f, t.y + kAsmCols);
  double* acc = asm_acc + static_cast<size_t>(threadIdx.x >> 5) * acc_f;
  ColMeta m{0, 0, 0, 0};
  ColPre p;
  // the static part (index words, zero fill, A entries) before the wait
  if (mine) {
    m = col_meta(sd, s, c0, k, J);
    col_static(sd, kval, f, J, acc, m, p);
  }
  pdl_wait();  // the previous level (programmatic launch)
  if (mine) col_children(sd, fd, s, f, fd.lval + sd.l_off[s], wide_ld(f), J, acc, m, p);
}

// one CTA per (front, 128-row block below the panel): warp 0 factors the
// diagonal block (every CTA redundantly: no extra launch), warps 1..3 solve
// the block's rows in lockstep with it.  The CTA of row block 0 publishes D
// and the counts, and leaves the scaled L11 in the scratch slot of its front;
// k_wide_update writes it into the front (other CTAs of this launch may
// still be reading the unfactored diagonal block).
__global__ void __launch_bounds__(kHugeRows)
k_wide_panel(SnDev sd, FactorDev fd, const int4* __restrict__ tasks, int panel, double eps) {
  __shared__ PanelSmem sm;
  __shared__ __align__(16) double D[kWidePanel * kSL];
  extern __shared__ __align__(16) double TR[];  // kWidePanel * (kTrsRows + 2)
  const int4 task = tasks[blockIdx.x];
  const int s = task.x, rb = task.y;
  const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
  const size_t ld = wide_ld(f);
  const int p0 = panel * kWidePanel, p1 = min(p0 + kWidePanel, k), nb = p1 - p0;
  double* F = fd.lval + sd.l_off[s];
  const int lo = p1 + rb * kPanelRows, hi = min(f, lo + kPanelRows);
  if (threadIdx.x == 0) sm.prog = 0;
  pdl_launch_dependents();
  pdl_wait();  // the previous panel's strip update (programmatic launch)
  __syncthreads();
  if (threadIdx.x < 32) {
    diag_block(F, ld, p0, nb, eps, sm, D, rb == 0 ? fd.d + c0 + p0 : nullptr,
               rb == 0 ? fd.stats : nullptr, &sm.prog);
    if (rb == 0) {
      double* scr = fd.dscr + static_cast<size_t>(task.z) * (kWidePanel * kWidePanel);
      for (int i = threadIdx.x; i < kWidePanel * kWidePanel; i += 32)
        scr[i] = sm.Lsh[i / kWidePanel][i % kWidePanel];
    }
  } else {
    trsm_rows<kTrsRows>(F, ld, p0, nb, lo, max(lo, hi), &sm.Us[0][0], sm.rinv, fd.stats,
                        threadIdx.x - 32, TR, &sm.prog, 1);
  }
}

// C (shared memory, column stride SC, row shift shC) -= A diag(d) B^T for a
// 32x32 tile over the 32 columns of the previous panel (A, B staged with
// column stride kSL); 4 warps, warp gw rows gw*8..+8, on DMMA
__device__ __forceinline__ void strip_mma(double* Cs, int SC, int shC, const double* A, int shA,
                                          const double* Bs, int shB, const double* d, int gt) {
  const int lane = gt & 31, gw = gt >> 5, g = lane >> 2, tq = lane & 3;
  const int rr = gw * 8 + g;
  double acc[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < kWidePanel / 4; ++kk) {
    const int q = kk * 4 + tq;
    const double a = A[q * kSL + rr + shA];
    const double dq = d[q];
#pragma unroll
    for (int j = 0; j < 4; ++j) dmma_m8n8k4(acc[j][0], acc[j][1], a, Bs[q * kSL + j * 8 + g + shB] * dq);
  }
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) Cs[(j * 8 + tq * 2 + e) * SC + rr + shC] -= acc[j][e];
}

// strip_mma for a whole 32x32 tile on ONE warp (lane layout as above): 16
// independent 8x8 accumulators, so the DMMA latency overlaps; per element
// the same k order as strip_mma (bitwise the same result)
__device__ __forceinline__ void strip_mma_warp(double* Cs, int SC, int shC, const double* A, int shA,
                                               const double* Bs, int shB, const double* d, int lane) {
  const int g = lane >> 2, tq = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < kWidePanel / 4; ++kk) {
    const int q = kk * 4 + tq;
    const double dq = d[q];
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = A[q * kSL + i * 8 + g + shA];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = Bs[q * kSL + j * 8 + g + shB] * dq;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_m8n8k4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) Cs[(j * 8 + tq * 2 + e) * SC + i * 8 + g + shC] -= acc[i][j][e];
}

// k_wide_panel with the lookahead strip folded in: for panel g >= 1 the CTA
// first applies panel g-1's update to panel g's columns -- of the diagonal
// rows (every CTA, like the diagonal block itself; all four warps) and of its
// own rows (each TRSM warp its 32 rows, while warp 0 factors the diagonal
// block: factor 2.41 -> 2.34 ms on the mesh against all strips first) --
// straight into shared memory (DMMA), and factors / solves from there.  The
// previous panel's L is final in the front (its kernel completed: this launch
// follows it on the stream), and every earlier panel's update of these
// columns is in (the host orders this launch after the rest update of panel
// g-2).  The scaled L11 goes to the scratch slot `scr` (the rest-update
// launch of this panel writes it into the front).
// one panel task (front s, row block rb below the panel; di: the front's
// scratch slot): the body of k_wide_panel_f, shared with k_huge_level.  The
// caller has completed the previous panel and every earlier update of this
// panel's columns; returns after a CTA barrier.
struct PanelTaskSmem {  // cp.async destinations 16-byte aligned
  PanelSmem sm;
  alignas(16) double D[kWidePanel * kSL];
  alignas(16) double TR[kWidePanel * kSLT];
  alignas(16) double A[4 * kWidePanel * kSL];
  double dv[kWidePanel];
};
static_assert(offsetof(PanelTaskSmem, D) % 16 == 0 && offsetof(PanelTaskSmem, TR) % 16 == 0 &&
                  offsetof(PanelTaskSmem, A) % 16 == 0, "PanelTaskSmem alignment");
// a front's static geometry (loaded before the programmatic wait: after it
// the panel's first loads are the staging of its blocks, one round trip)
struct PanelGeo {
  int c0, k, f;
  long long loff;
};
__device__ __forceinline__ PanelGeo panel_geo(const SnDev& sd, int s) {
  const int c0 = sd.first[s];
  return PanelGeo{c0, sd.first[s + 1] - c0, sd.f[s], sd.l_off[s]};
}
__device__ __forceinline__ void panel_task(const SnDev& sd, const FactorDev& fd, int4 task, int panel,
                                           double eps, double* scr_base, PanelTaskSmem& P, const PanelGeo& geo,
                                           long long* stamp = nullptr, int gtr = -1) {
  PanelSmem& sm = P.sm;
  double* D = P.D;
  double* TR = P.TR;
  double* A = P.A;
  double* dv = P.dv;
  const int rb = task.y;
  const int c0 = geo.c0, k = geo.k, f = geo.f;
  const size_t ld = wide_ld(f);
  const int p0 = panel * kWidePanel, p1 = min(p0 + kWidePanel, k), nb = p1 - p0;
  double* F = fd.lval + geo.loff;
  const int lo = p1 + rb * kPanelRows, hi = min(f, lo + kPanelRows);
  const int nrow = max(0, hi - lo);
  const int t = threadIdx.x;
  if (t == 0) sm.prog = 0;
  // the strip is the whole 32-column block: on a front's last (partial)
  // panel its columns [p1, p0+32) are trailing entries, updated here and
  // written back by the TRSM warps (rows >= p1 are this CTA's rows: each
  // entry once)
  const int q0 = p0 - kWidePanel;  // panel g-1: 32 columns (not a front's last panel)
  const int ncs = min(kWidePanel, f - p0);
  if (panel > 0) {
    // only the diagonal rows' strip is on the critical path: cp.async group 0
    // (every thread) stages them, group 1 (the TRSM warps) this CTA's rows,
    // whose strip the TRSM warps apply while warp 0 factors the diagonal block
    stage_block<kNR2>(D, kSL, F, ld, p0, p0, nb, t, kHugeRows);
    stage_block<kNR2>(A, kSL, F, ld, p0, q0, kWidePanel, t, kHugeRows);
    cp_commit();
    if (t >= 32) {
      if (nrow > 0) stage_block<(kTrsRows + 2) / 2>(TR, kSLT, F, ld, lo, p0, ncs, t - 32, kTrsRows);
      for (int j = 0; 32 * j < nrow; ++j)
        stage_block<kNR2>(A + (j + 1) * kWidePanel * kSL, kSL, F, ld, lo + 32 * j, q0, kWidePanel, t - 32,
                          kTrsRows);
      cp_commit();
    }
    if (t < kWidePanel) dv[t] = __ldcg(fd.d + c0 + q0 + t);
    if (t < 32)
      cp_wait_all();
    else
      cp_wait_group<1>();
    __syncthreads();
    if (t == 0) ptrace_max(gtr, 2);
    strip_mma(D, kSL, 0, A, 0, A, 0, dv, t);
  }
  __syncthreads();
  if (stamp && t == 0) stamp[1] = clock64();
  if (t == 0) {
    if (panel == 0) ptrace_max(gtr, 2);
    ptrace_max(gtr, 3);
  }
  if (t < 32) {
    diag_block(F, ld, p0, nb, eps, sm, D, rb == 0 ? fd.d + c0 + p0 : nullptr,
               rb == 0 ? fd.stats : nullptr, &sm.prog, panel > 0);
    if (stamp && t == 0) stamp[2] = clock64();
    if (t == 0) ptrace_max(gtr, 4);
    if (rb == 0) {
      double* scr = scr_base + static_cast<size_t>(task.z) * (kWidePanel * kWidePanel);
      for (int i = t; i < kWidePanel * kWidePanel; i += 32) scr[i] = sm.Lsh[i / kWidePanel][i % kWidePanel];
    }
  } else {
    if (panel > 0) {
      cp_wait_all();
      named_bar(1, kTrsRows);
      const int w = (t >> 5) - 1, lane = t & 31, sh = lo & 1;  // warp w: rows [32w, 32w+32)
      if (32 * w < nrow) {
        strip_mma_warp(TR + 32 * w, kSLT, sh, A + (w + 1) * kWidePanel * kSL, sh, A, 0, dv, lane);
        __syncwarp();
        for (int c = nb; c < ncs; ++c)
          for (int i = 32 * w + lane; i < min(nrow, 32 * w + 32); i += 32)
            if (lo + i >= p0 + c) F[(lo + i) + static_cast<size_t>(p0 + c) * ld] = TR[c * kSLT + i + sh];
      }
    }
    trsm_rows<kTrsRows>(F, ld, p0, nb, lo, max(lo, hi), &sm.Us[0][0], sm.rinv, fd.stats, t - 32, TR,
                        &sm.prog, 1, panel > 0);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kHugeRows)
k_wide_panel_f(SnDev sd, FactorDev fd, const int4* __restrict__ tasks, int panel, double eps,
               double* scr_base, int gtr) {
  extern __shared__ __align__(16) double dyn_smem[];
  PanelTaskSmem& P = *reinterpret_cast<PanelTaskSmem*>(dyn_smem);
  const int4 task = tasks[blockIdx.x];
  const PanelGeo geo = panel_geo(sd, task.x);  // static: before the wait
  if (threadIdx.x == 0) ptrace_max(gtr, 0);
  pdl_launch_dependents();
  pdl_wait();  // the previous panel (programmatic launch)
  if (threadIdx.x == 0) ptrace_max(gtr, 1);
  panel_task(sd, fd, task, panel, eps, scr_base, P, geo, nullptr, gtr);
  if (threadIdx.x == 0) ptrace_max(gtr, 5);
}

// ---------------------------------------------------------------------------
// A whole huge level as ONE persistent launch (the per-panel launches of
// k_wide_panel_f / k_wide_update cost a launch gap each and start on SMs
// whose instruction caches are cold for an 86 KB kernel).  CTAs [0, npc)
// run the panel tasks of every panel in order (task j of panel g on CTA
// j % npc); the others run the trailing-update tiles of panel g plus one
// L11 write-back item.  Dependencies are the stream schedule's, through
// per-panel completion counters (zeroed before the launch): panel g waits for
// panel g-1 and the rest update of g-2; the rest update of g for panel g and
// the rest update of g-1 (every tile still sees the panels in order).  Each
// CTA runs its items in that order and waits only on earlier items, and the
// grid is resident (HugeDev.ctas <= resident CTAs): no deadlock.
__device__ __forceinline__ void huge_wait(const int* p, int v) {
  if (ld_relaxed(p) < v) {
    unsigned ns = 32;
    while (ld_relaxed(p) < v) {
      __nanosleep(ns);
      if (ns < 256) ns <<= 1;
    }
  }
  flag_acquire(p);  // the caller's CTA barrier carries it to the other threads
}
__device__ __forceinline__ void huge_done(int* p) {
  __syncthreads();  // every thread's writes before thread 0's release
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(p) : "memory");
}

__global__ void __launch_bounds__(kHugeRows)
k_huge_level(SnDev sd, FactorDev fd, HugeDev h, double eps) {
  extern __shared__ __align__(16) double dyn_smem[];
  const int t = threadIdx.x;
  pdl_launch_dependents();
  pdl_wait();  // the level's assembly
  const int ng = h.g1 - h.g0;
  auto np = [&](int g) { return h.pn_ptr[g + 1] - h.pn_ptr[g]; };
  auto nr = [&](int g) { return h.tl_ptr[g + 1] - h.tl_ptr[g] + 1; };  // tiles + the L11 item
  if (static_cast<int>(blockIdx.x) < h.npc) {
    PanelTaskSmem& P = *reinterpret_cast<PanelTaskSmem*>(dyn_smem);
    for (int gi = 0; gi < ng; ++gi) {
      const int g = h.g0 + gi;
      double* scr = h.scr + static_cast<size_t>(gi & 1) * h.max_dg * (kWidePanel * kWidePanel);
      for (int j = blockIdx.x; j < np(g); j += h.npc) {
        if (t == 0) {
          if (h.trace) h.trace[5 * static_cast<size_t>(h.pn_ptr[g] + j)] = clock64();
          if (gi >= 1) huge_wait(h.pc + g - 1, np(g - 1));
          if (gi >= 2) huge_wait(h.rc + g - 2, nr(g - 2));
        }
        __syncthreads();
        long long* stamp = h.trace ? h.trace + 5 * static_cast<size_t>(h.pn_ptr[g] + j) : nullptr;
        if (stamp && t == 0) stamp[4] = clock64();
        const int4 task = h.pn[h.pn_ptr[g] + j];
        panel_task(sd, fd, task, gi, eps, scr, P, panel_geo(sd, task.x), stamp);
        if (stamp && t == 0) stamp[3] = clock64();
        huge_done(h.pc + g);
      }
    }
    return;
  }
  GroupSmem& G = *reinterpret_cast<GroupSmem*>(dyn_smem);
  const int nrc = gridDim.x - h.npc, r = blockIdx.x - h.npc;
  for (int gi = 0; gi < ng; ++gi) {
    const int g = h.g0 + gi;
    const double* scr = h.scr + static_cast<size_t>(gi & 1) * h.max_dg * (kWidePanel * kWidePanel);
    const int ntl = nr(g) - 1;
    for (int j = r; j < ntl + 1; j += nrc) {
      if (t == 0) {
        huge_wait(h.pc + g, np(g));
        if (gi >= 1) huge_wait(h.rc + g - 1, nr(g - 1));
      }
      __syncthreads();
      if (j < ntl) {
        const int4 tl = h.tiles[h.tl_ptr[g] + j];
        const int s = tl.x;
        const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
        const int p0 = tl.w * kWidePanel, p1 = min(p0 + kWidePanel, k);
        group_tile(fd.lval + sd.l_off[s], wide_ld(f), f, fd.d + c0 + p0, p0, p1 - p0, tl.y, tl.z, G, t, 1);
      } else {  // the panel's L11 blocks from the scratch slots
        for (int di = 0; di < h.dg_ptr[g + 1] - h.dg_ptr[g]; ++di) {
          const int s = h.dg[h.dg_ptr[g] + di];
          const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
          const size_t ld = wide_ld(f);
          const int p0 = gi * kWidePanel, nb = min(p0 + kWidePanel, k) - p0;
          const double* sc = scr + static_cast<size_t>(di) * (kWidePanel * kWidePanel);
          double* F = fd.lval + sd.l_off[s];
          for (int idx = t; idx < kWidePanel * kWidePanel; idx += kHugeRows) {
            const int i = idx / kWidePanel, p = idx % kWidePanel;
            if (i > p && i < nb) F[(p0 + i) + (p0 + p) * ld] = sc[idx];
          }
        }
      }
      huge_done(h.rc + g);
    }
  }
}

// one 4-warp group (CTA) per 32x32 tile; block 0 also writes the panel's L11
// blocks from the scratch slots of the nd fronts
__global__ void __launch_bounds__(128)
k_wide_update(SnDev sd, FactorDev fd, const int4* __restrict__ tiles, int count,
              const int* __restrict__ fronts, int nd, int panel, const double* scr_base, int gtr) {
  __shared__ __align__(16) GroupSmem G;
  pdl_launch_dependents();
  pdl_wait();  // the panel kernel (programmatic launch on the main stream)
  if (threadIdx.x == 0) ptrace_max(gtr, 6);
  if (blockIdx.x == 0) {
    for (int di = 0; di < nd; ++di) {
      const int s = fronts[di];
      const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
      const size_t ld = wide_ld(f);
      const int p0 = panel * kWidePanel, nb = min(p0 + kWidePanel, k) - p0;
      const double* scr = scr_base + static_cast<size_t>(di) * (kWidePanel * kWidePanel);
      double* F = fd.lval + sd.l_off[s];
      for (int idx = threadIdx.x; idx < kWidePanel * kWidePanel; idx += blockDim.x) {
        const int i = idx / kWidePanel, p = idx % kWidePanel;
        if (i > p && i < nb) F[(p0 + i) + (p0 + p) * ld] = scr[idx];
      }
    }
  }
  if (static_cast<int>(blockIdx.x) < count) {
    const int4 t = tiles[blockIdx.x];
    const int s = t.x;
    const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
    const int p0 = t.w * kWidePanel, p1 = min(p0 + kWidePanel, k);
    group_tile(fd.lval + sd.l_off[s], wide_ld(f), f, fd.d + c0 + p0, p0, p1 - p0, t.y, t.z, G,
               threadIdx.x, 1);
  }
#ifdef NCL_PANEL_TRACE
  if (gtr >= 0) {
    __syncthreads();
    if (threadIdx.x == 0) ptrace_max(gtr, 7);
  }
#endif
}

// ---------------------------------------------------------------------------
// The rest update as 64x64 tiles (fused path): one 16-warp CTA per tile, warp
// w rows 8(w mod 8).. x one 32-column half; A and B (the panel's L rows of the tile's
// row and column blocks) are staged once for what four 32x32 tiles stage
// twice each.  Per element the same DMMA sequence as tile_mma_store (k in
// chunks of four, accumulated, then subtracted from C): bitwise the same.
constexpr int kT64 = 2 * kUpdTile;
constexpr int kSL64 = 72;  // column stride of a staged 64-row block (66 rows with the shift)
struct Group64Smem {
  double A[kWidePanel * kSL64], B[kWidePanel * kSL64], C[kT64 * kSL64];
  double d[kWidePanel];
};
static_assert(offsetof(Group64Smem, B) % 16 == 0 && offsetof(Group64Smem, C) % 16 == 0, "Group64Smem alignment");
__global__ void __launch_bounds__(512)
k_wide_update64(SnDev sd, FactorDev fd, const int4* __restrict__ tiles, int count,
                const int* __restrict__ fronts, int nd, int panel, const double* scr_base) {
  extern __shared__ __align__(16) double g64_smem[];
  Group64Smem& G = *reinterpret_cast<Group64Smem*>(g64_smem);
  pdl_launch_dependents();
  pdl_wait();  // the panel kernel
  const int tid = threadIdx.x;
  if (blockIdx.x == 0) {  // the panel's L11 blocks from the scratch slots (as k_wide_update)
    for (int di = 0; di < nd; ++di) {
      const int s = fronts[di];
      const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
      const size_t ld = wide_ld(f);
      const int p0 = panel * kWidePanel, nb = min(p0 + kWidePanel, k) - p0;
      const double* scr = scr_base + static_cast<size_t>(di) * (kWidePanel * kWidePanel);
      double* F = fd.lval + sd.l_off[s];
      for (int idx = tid; idx < kWidePanel * kWidePanel; idx += blockDim.x) {
        const int i = idx / kWidePanel, p = idx % kWidePanel;
        if (i > p && i < nb) F[(p0 + i) + (p0 + p) * ld] = scr[idx];
      }
    }
  }
  if (static_cast<int>(blockIdx.x) >= count) return;
  const int4 t = tiles[blockIdx.x];
  const int s = t.x, r0 = t.y, q0 = t.z;
  const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
  const size_t ld = wide_ld(f);
  const int p0 = t.w * kWidePanel, nb = min(p0 + kWidePanel, k) - p0;
  const int nr = min(kT64, f - r0), nc = min(kT64, f - q0);
  const bool dg = r0 == q0;
  double* F = fd.lval + sd.l_off[s];
  constexpr int NR2 = (kT64 + 2) / 2;
  const int shA = stage_block<NR2>(G.A, kSL64, F, ld, r0, p0, nb, tid, 512);
  const int shB = dg ? shA : stage_block<NR2>(G.B, kSL64, F, ld, q0, p0, nb, tid, 512);
  const int shC = stage_block<NR2>(G.C, kSL64, F, ld, r0, q0, nc, tid, 512);
  if (tid < nb) G.d[tid] = __ldcg(fd.d + c0 + p0 + tid);
  cp_wait_all();
  __syncthreads();
  const double* Bs = dg ? G.A : G.B;
  const int lane = tid & 31, g = lane >> 2, tq = lane & 3, w = tid >> 5;
  const int rr = (w & 7) * 8 + g, ch = (w >> 3) * 32;  // warp: 8 rows x one 32-column half
  double acc[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < kWidePanel / 4; ++kk) {
    const int q = kk * 4 + tq;
    const bool qv = q < nb;
    const double a = (qv && rr < nr) ? G.A[q * kSL64 + rr + shA] : 0.0;
    const double dq = qv ? G.d[q] : 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cc = ch + j * 8 + g;
      const double b = (qv && cc < nc) ? Bs[q * kSL64 + cc + shB] * dq : 0.0;
      dmma_m8n8k4(acc[j][0], acc[j][1], a, b);
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = ch + j * 8 + tq * 2 + e;
      if (rr < nr && c < nc && r0 + rr >= q0 + c)
        F[(r0 + rr) + static_cast<size_t>(q0 + c) * ld] = G.C[c * kSL64 + rr + shC] - acc[j][e];
    }
}

// ---------------------------------------------------------------------------
// Mid fronts: levels whose fronts all have at most kMidF rows and a single
// panel (k <= 32) -- on the 78k-bus mesh the 3,100 fronts of levels 0-4.
// k_wide_front gives such a front a 512-thread cluster CTA (one per SM) that
// round-trips every phase through L2 (assembled columns, the staged diagonal
// block and rows, three staged blocks per trailing tile) with a barrier
// between phases.  Here one 4-warp CTA keeps the whole front in shared memory
// (packed lower triangle: element (r, J) at S[cb[J] + r]) from the assembly
// to the single write-back: zero + A entries + the children one by one (the
// child's row map in shared memory, 16 of its entries per thread in flight),
// the diagonal block (diag_block, warp 0) with the rows below in lock-step
// (warps 1-3, trsm_steps), then the trailing update tile by tile on DMMA with
// the fragment layout and masking of tile_mma_store -- every entry gets
// bitwise the k_wide_front arithmetic.
constexpr int kMidF = 216;

constexpr int kMidCh = 16;    // children whose row maps are staged before the wait
constexpr int kMidRel = 1024;  // staged row-map entries (all children)
struct MidSmem {
  PanelSmem sm;
  alignas(16) double D[kWidePanel * kSL];
  double dv[kWidePanel];
  const double* chU[kMidCh];  // per child: its update block, rows, leading dimension
  int chfu[kMidCh], chld[kMidCh], chrp[kMidCh];
  int relall[kMidRel];  // the children's row maps into the front, child order
  int rel[kMidF];       // one child's row map (more than kMidCh children / kMidRel entries)
  int cb[kMidF];        // column bases of the packed front
};

// the front's tile (rows r0.., columns q0..; nr x nc; lower part only when
// `dg`) -= L(rows, 0:nb) diag(d) L(cols, 0:nb)^T, 4 warps, warp gw rows gw*8..+8
__device__ __forceinline__ void mid_tile(double* S, const int* cb, int r0, int q0, const double* d,
                                         int nb, int nr, int nc, bool dg, int gt) {
  const int lane = gt & 31, gw = gt >> 5, g = lane >> 2, tq = lane & 3;
  const int rr = gw * 8 + g;
  double acc[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < kWidePanel / 4; ++kk) {
    const int q = kk * 4 + tq;
    const bool qv = q < nb;
    const int bq = qv ? cb[q] : 0;
    const double a = (qv && rr < nr) ? S[bq + r0 + rr] : 0.0;
    const double dq = qv ? d[q] : 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cc = j * 8 + g;
      const double b = (qv && cc < nc) ? S[bq + q0 + cc] * dq : 0.0;
      dmma_m8n8k4(acc[j][0], acc[j][1], a, b);
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = j * 8 + tq * 2 + e;
      if (rr < nr && c < nc && (!dg || rr >= c)) {
        double* x = S + cb[q0 + c] + r0 + rr;
        *x = *x - acc[j][e];
      }
    }
}

// trsm_steps for one row r of the packed front: L(r, p) = x_p / d_p stored at
// S[cb[p] + r]
template <int W>
__device__ __forceinline__ void mid_trsm_steps(int pb, int pe, double (&x)[kWidePanel], double* S,
                                               const int* cb, int r, const double* us, const double* rinv,
                                               const int* prog, bool& bad) {
#pragma unroll 1
  for (int p = pb; p < pe; ++p) {
    while (ld_acquire_smem(prog) <= p) __nanosleep(64);
    const double l = x[0] * rinv[p];
    S[cb[p] + r] = l;
    bad |= !isfinite(l);
    const double2* up = reinterpret_cast<const double2*>(us + p * kWidePanel);
#pragma unroll
    for (int j = 0; j < W; j += 2) {
      const double2 v = up[j >> 1];
      x[j] = x[j + 1] - l * v.x;
      x[j + 1] = (j + 2 < W ? x[j + 2] : 0.0) - l * v.y;
    }
  }
}

// NT threads: 128 (fronts up to 128 rows, several CTAs per SM) or 256 (two
// 4-warp tile groups, wider assembly and row rounds for the bigger fronts)
template <int NT>
__global__ void __launch_bounds__(NT, NT == 128 ? 4 : 1)
k_mid_front(SnDev sd, FactorDev fd, const double* __restrict__ kval, const int* __restrict__ nodes,
            double eps, int stage) {
  extern __shared__ __align__(16) double dyn_smem[];
  MidSmem& M = *reinterpret_cast<MidSmem*>(dyn_smem);
  double* S = dyn_smem + (sizeof(MidSmem) + 7) / 8;  // the front, packed lower triangle
  const int* cb = M.cb;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int s = nodes[blockIdx.x];
  const int c0 = sd.first[s], k = sd.first[s + 1] - c0, f = sd.f[s];
  const size_t ld = wide_ld(f);
  double* F = fd.lval + sd.l_off[s];
  pdl_launch_dependents();
  // column J: rows J..f-1 after the columns before it
  for (int J = t; J < f; J += NT) M.cb[J] = J * f - (J * (J - 1)) / 2 - J;
  // assembly: zero, the A entries, then the children in child order (per
  // position the order of the column pass of assemble_col).  Everything but
  // the children's update values is static (kval is complete before the
  // level launches), so it is done before the programmatic wait: the first
  // wave overlaps the previous level and no CTA waits on index loads after it
  const int ntri = f * (f + 1) / 2;
  for (int i = t; i < ntri; i += NT) S[i] = 0.0;
  if (t == 0) M.sm.prog = 0;
  const int ch0 = sd.ch_ptr[s], nch = sd.ch_ptr[s + 1] - ch0;
  const bool chpre = stage && nch <= kMidCh;  // stage = 0: the per-child path (tests)
  if (chpre && t < nch) {
    const int c = sd.ch[ch0 + t];
    M.chfu[t] = f_minus_k(sd, c);
    M.chld[t] = sd.u_ld[c];
    M.chrp[t] = sd.rel_ptr[c];
    M.chU[t] = (sd.wide[c] ? fd.lval : fd.upd) + sd.u_off[c];
  }
  __syncthreads();
  for (int q = sd.asm_ptr[s] + t; q < sd.asm_ptr[s + 1]; q += NT) {
    const int pos = sd.asm_pos[q];
    S[cb[pos >> 16] + (pos & 0xffff)] += __ldg(kval + sd.asm_slot[q]);
  }
  int nrel = 0;  // row-map entries staged (-1: too many, staged per child)
  if (chpre) {
    for (int ci = 0; ci < nch; ++ci) {
      const int fu = M.chfu[ci];
      if (nrel + fu > kMidRel) {
        nrel = -1;
        break;
      }
      for (int i = t; i < fu; i += NT) cp4(&M.relall[nrel + i], sd.rel + M.chrp[ci] + i);
      nrel += fu;
    }
  } else {
    nrel = -1;
  }
  cp_commit();
  cp_wait_all();
  pdl_wait();  // the children (previous level)
  __syncthreads();
  // a child at a time: its entries (i, j), i >= j, in batches of 16 per thread
  // with every load of a batch in flight (entries of one child land on
  // distinct positions)
  for (int ci = 0, ro = 0; ci < nch; ++ci) {
    int fu, uld;
    const double* U;
    const int* rel;
    if (nrel >= 0) {
      fu = M.chfu[ci];
      uld = M.chld[ci];
      U = M.chU[ci];
      rel = M.relall + ro;
      ro += fu;
    } else {
      const int c = sd.ch[ch0 + ci];
      fu = f_minus_k(sd, c);
      uld = sd.u_ld[c];
      U = (sd.wide[c] ? fd.lval : fd.upd) + sd.u_off[c];
      const int* grel = sd.rel + sd.rel_ptr[c];
      for (int i = t; i < fu; i += NT) M.rel[i] = __ldg(grel + i);
      __syncthreads();
      rel = M.rel;
    }
    const int n2 = fu * fu;
    const float rfu = 1.0f / static_cast<float>(fu);
    for (int e0 = 0; e0 < n2; e0 += NT * 16) {
      double v[16];
      int pos[16];
#pragma unroll
      for (int b = 0; b < 16; ++b) {
        const int e = e0 + b * NT + t;
        int j = __float2int_rz((static_cast<float>(e) + 0.5f) * rfu), i = e - j * fu;  // e = j fu + i
        if (i < 0) {
          --j;
          i += fu;
        } else if (i >= fu) {
          ++j;
          i -= fu;
        }
        const bool ok = e < n2 && i >= j;
        pos[b] = ok ? cb[rel[j]] + rel[i] : -1;
        v[b] = ok ? __ldcg(U + i + static_cast<size_t>(j) * uld) : 0.0;
      }
#pragma unroll
      for (int b = 0; b < 16; ++b)
        if (pos[b] >= 0) S[pos[b]] += v[b];
    }
    __syncthreads();
  }
  // the panel: diagonal block on warp 0 (staged copy), the rows below in
  // lock-step on warps 1-3 (rounds of 96 rows; the first in lock-step)
  for (int i = t; i < kWidePanel * kWidePanel; i += NT) {
    const int q = i >> 5, r = i & 31;
    M.D[q * kSL + r] = (q < k && r < k && r >= q) ? S[cb[q] + r] : 0.0;
  }
  __syncthreads();
  if (warp == 0) {
    diag_block(nullptr, 0, 0, k, eps, M.sm, M.D, fd.d + c0, fd.stats, &M.sm.prog, true);
    for (int i = lane; i < kWidePanel * kWidePanel; i += 32) {
      const int r = i >> 5, q = i & 31;
      if (r > q && r < k) S[cb[q] + r] = M.sm.Lsh[r][q];
    }
  } else {
    bool bad = false;
    for (int r = k + t - 32; r < f; r += NT - 32) {
      double x[kWidePanel];
#pragma unroll
      for (int q = 0; q < kWidePanel; ++q) x[q] = q < k ? S[cb[q] + r] : 0.0;
      const double* us = &M.sm.Us[0][0];
      mid_trsm_steps<32>(0, min(k, 8), x, S, cb, r, us, M.sm.rinv, &M.sm.prog, bad);
      mid_trsm_steps<24>(8, min(k, 16), x, S, cb, r, us, M.sm.rinv, &M.sm.prog, bad);
      mid_trsm_steps<16>(16, min(k, 24), x, S, cb, r, us, M.sm.rinv, &M.sm.prog, bad);
      mid_trsm_steps<8>(24, k, x, S, cb, r, us, M.sm.rinv, &M.sm.prog, bad);
    }
    if (bad) atomicOr(fd.stats + 3, 1);
  }
  __syncthreads();
  if (t < kWidePanel) M.dv[t] = t < k ? __ldcg(fd.d + c0 + t) : 0.0;
  __syncthreads();
  // trailing update: tiles (ti >= tj) of rows / columns [k, f), in place; the
  // operands (the L columns) and the tiles are disjoint
  const int T = (f - k + kUpdTile - 1) / kUpdTile;
  for (int tl = t >> 7; tl < T * (T + 1) / 2; tl += NT / 128) {  // a 4-warp group per tile
    int ti, tj;
    tri_decode(tl, ti, tj);
    const int r0 = k + ti * kUpdTile, q0 = k + tj * kUpdTile;
    mid_tile(S, cb, r0, q0, M.dv, k, min(kUpdTile, f - r0), min(kUpdTile, f - q0), ti == tj, t & 127);
  }
  __syncthreads();
  for (int J = warp; J < f; J += NT / 32)
    for (int r = J + lane; r < f; r += 32) F[r + J * ld] = S[cb[J] + r];
}

// ---------------------------------------------------------------------------
thread_local const char* wide_last_error = "";

static void wide_init() {
  static PerDeviceOnce once;
  once([] {
  cudaFuncSetAttribute(k_wide_front, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa = {};
  cudaFuncGetAttributes(&fa, k_wide_front);
  cudaFuncSetAttribute(k_wide_front, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       optin - static_cast<int>(fa.sharedSizeBytes));
  cudaGetLastError();
  });
}

int wide_front_smem(int max_f) {
  const size_t acc = sizeof(double) * kWarps * static_cast<size_t>(max_f > 0 ? max_f : 1);
  return static_cast<int>(acc > sizeof(StageSmem) ? acc : sizeof(StageSmem));
}

int launch_wide_front(const SnDev& sd, const FactorDev& fd, const double* kval, const int* nodes,
                      int count, int cluster, int max_f, double eps, cudaStream_t st,
                      unsigned long long* trace) {
  if (!count) return cluster;
  wide_init();
  for (; cluster >= 1; cluster >>= 1) {  // largest cluster the device can place
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(count * cluster));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = static_cast<size_t>(wide_front_smem(max_f));
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(cluster);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // device: pdl_wait()
    attr[1].val.programmaticStreamSerializationAllowed = std::getenv("NCL_NO_PDL") == nullptr ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    int nclusters = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, k_wide_front, &cfg);
    if (e != cudaSuccess || nclusters < 1) {
      wide_last_error = e != cudaSuccess ? cudaGetErrorString(e) : "occupancy 0";
      cudaGetLastError();
      continue;
    }
    e = cudaLaunchKernelEx(&cfg, k_wide_front, sd, fd, kval, nodes, eps, max_f, trace);
    if (e == cudaSuccess) return cluster;
    wide_last_error = cudaGetErrorString(e);
    cudaGetLastError();
  }
  return 0;
}

// ordinary launch, or programmatic dependent launch (the kernel waits in
// pdl_wait() for its predecessor on the stream); NCL_NO_PDL=1 turns it off
template <typename Kern, typename... Args>
static void launch_pdl(Kern kern, int grid, int block, size_t smem, cudaStream_t st, bool pdl, Args... args) {
  static const bool allowed = std::getenv("NCL_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(static_cast<unsigned>(block));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (pdl && allowed) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, args...);
}

void launch_wide_assemble(const SnDev& sd, const FactorDev& fd, const double* kval,
                          const int4* tasks, int count, int max_f, cudaStream_t st) {
  static PerDeviceOnce init;
  init([] {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncSetAttribute(k_wide_assemble, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
  });
  const int acc_f = max_f < 1 ? 1 : max_f;
  const size_t smem = sizeof(double) * kAsmCols * static_cast<size_t>(acc_f);
  if (count) launch_pdl(k_wide_assemble, count, 256, smem, st, true, sd, fd, kval, tasks, acc_f);
}

void launch_wide_panel(const SnDev& sd, const FactorDev& fd, const int4* tasks, int count,
                       int panel, double eps, cudaStream_t st) {
  static PerDeviceOnce init;
  constexpr int tr_bytes = static_cast<int>(sizeof(double)) * kWidePanel * (kTrsRows + 2);
  init([] { cudaFuncSetAttribute(k_wide_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, tr_bytes); });
  if (count) launch_pdl(k_wide_panel, count, kHugeRows, tr_bytes, st, true, sd, fd, tasks, panel, eps);
}

void launch_wide_update(const SnDev& sd, const FactorDev& fd, const int4* tiles, int count,
                        const int* fronts, int nd, int panel, cudaStream_t st, bool pdl,
                        const double* scr, int gtr) {
  const int blocks = count > 0 ? count : (nd > 0 ? 1 : 0);
  if (blocks)
    launch_pdl(k_wide_update, blocks, 128, 0, st, pdl, sd, fd, tiles, count, fronts, nd, panel,
               scr ? scr : static_cast<const double*>(fd.dscr), gtr);
}

void launch_wide_update64(const SnDev& sd, const FactorDev& fd, const int4* tiles, int count,
                          const int* fronts, int nd, int panel, cudaStream_t st, bool pdl, const double* scr) {
  static PerDeviceOnce init;
  constexpr int bytes = static_cast<int>(sizeof(Group64Smem));
  init([] { cudaFuncSetAttribute(k_wide_update64, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); });
  const int blocks = count > 0 ? count : (nd > 0 ? 1 : 0);
  if (blocks)
    launch_pdl(k_wide_update64, blocks, 512, bytes, st, pdl, sd, fd, tiles, count, fronts, nd, panel, scr);
}

void launch_wide_panel_f(const SnDev& sd, const FactorDev& fd, const int4* tasks, int count, int panel,
                         double eps, double* scr, cudaStream_t st, int gtr) {
  static PerDeviceOnce init;
  constexpr int bytes = static_cast<int>(sizeof(PanelTaskSmem));
  init([] { cudaFuncSetAttribute(k_wide_panel_f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); });
  if (count) launch_pdl(k_wide_panel_f, count, kHugeRows, bytes, st, true, sd, fd, tasks, panel, eps, scr, gtr);
}

bool set_panel_trace(unsigned long long* p) {
#ifdef NCL_PANEL_TRACE
  cudaMemcpyToSymbol(g_ptrace, &p, sizeof(p));
  return true;
#else
  (void)p;
  return false;
#endif
}

static constexpr int huge_smem() {
  return static_cast<int>(sizeof(PanelTaskSmem) > sizeof(GroupSmem) ? sizeof(PanelTaskSmem) : sizeof(GroupSmem));
}

int huge_level_ctas() {  // resident CTAs of k_huge_level on this device
  static PerDeviceOnce init;
  init([] { cudaFuncSetAttribute(k_huge_level, cudaFuncAttributeMaxDynamicSharedMemorySize, huge_smem()); });
  int per = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_huge_level, kHugeRows, huge_smem()) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return per * sms;
}

void launch_huge_level(const SnDev& sd, const FactorDev& fd, const HugeDev& h, double eps, cudaStream_t st) {
  huge_level_ctas();  // the shared-memory opt-in on this device
  launch_pdl(k_huge_level, h.ctas, kHugeRows, static_cast<size_t>(huge_smem()), st, true, sd, fd, h, eps);
}

// ---------------------------------------------------------------------------
// Tile dataflow over a segment of wide levels (dag.hpp): one persistent
// launch, one 128-thread worker per CTA running its task list in order.
// Waits: warp 0's lanes poll the tile states a task needs (ld.acquire.gpu,
// back-off), then a CTA barrier; publication: CTA barrier, then one thread's
// st.release.gpu (cumulative over the CTA's writes ordered by the barrier).
struct DagSmem {
  PanelSmem pm;
  union alignas(16) {  // cp.async destinations: 16-byte aligned
    GroupSmem g;
    struct {
      double D[kWidePanel * kSL];
      double TR[kWidePanel * (kWidePanel + 2)];
    } t;
  } u;
};

static_assert(offsetof(DagSmem, u) % 16 == 0 && sizeof(PanelSmem) % 8 == 0, "DagSmem alignment");

__device__ __forceinline__ void dag_wait(const int* p, int v) {
  if (ld_acquire(p) >= v) return;
  unsigned ns = 32;
  while (ld_acquire(p) < v) {
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
  }
}

__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int dag_tri(int i, int j) { return i * (i + 1) / 2 + j; }

__global__ void __launch_bounds__(128, 4)
k_front_dag(SnDev sd, FactorDev fd, const double* __restrict__ kval, DagDev g, double eps) {
  extern __shared__ __align__(16) double dyn_smem[];
  DagSmem& S = *reinterpret_cast<DagSmem*>(dyn_smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_launch_dependents();
  pdl_wait();  // the previous kernels (warp tier, earlier levels)
  const int t0 = g.w_ptr[blockIdx.x], t1 = g.w_ptr[blockIdx.x + 1];
  for (int ti = t0; ti < t1; ++ti) {
    const int4 tk = g.tasks[ti];
    const DagFront& Fr = g.fronts[tk.x];
    const int type = tk.y >> 24, i = tk.y & 0xfff, j = (tk.y >> 12) & 0xfff, p = tk.z;
    const int k = Fr.k, f = Fr.f, P = Fr.P, NB = Fr.NB, c0 = Fr.c0;
    int* stf = g.st + Fr.st_off;
    double* F = fd.lval + Fr.loff;
    const size_t ld = wide_ld(f);
    unsigned long long tw = 0;
    if (g.trace && tid == 0) tw = globaltimer();
    // ---- waits
    if (warp == 0) {
      if (type == kDagAsm) {
        for (int q = Fr.ch_b + lane; q < Fr.ch_e; q += 32) {
          const int c = g.ch[q];
          dag_wait(g.done + c, g.fronts[c].ntrail);
        }
      } else if (type == kDagDiag) {
        if (lane == 0) dag_wait(stf + dag_tri(p, p), p + 1);
      } else if (type == kDagTrsm) {
        if (lane == 0) dag_wait(stf + dag_tri(i, p), p + 1);
        if (lane == 1) dag_wait(stf + dag_tri(p, p), p + 2);
      } else {
        if (lane == 0) dag_wait(stf + dag_tri(i, p), p + 2);
        if (lane == 1) dag_wait(stf + dag_tri(j, p), p + 2);
        if (lane == 2) dag_wait(stf + dag_tri(i, j), p + 1);
      }
    }
    __syncthreads();
    unsigned long long tb = 0;
    if (g.trace && tid == 0) tb = globaltimer();
    // ---- work
    if (type == kDagAsm) {
      const int j0 = dag_block_start(k, P, j), nb = dag_block_size(k, f, P, j);
      for (int J = j0 + warp; J < j0 + nb; J += 4)
        assemble_col(sd, fd, kval, Fr.s, c0, k, f, F, ld, J, nullptr);
    } else if (type == kDagDiag) {
      const int p0 = 32 * p, nb = min(32, k - p0);
      if (warp == 0)
        diag_block(F, ld, p0, nb, eps, S.pm, S.u.t.D, fd.d + c0 + p0, fd.stats, nullptr);
      __syncthreads();
      double* scr = g.scr + static_cast<size_t>(Fr.scr_off + p) * kDagScr;
      for (int x = tid; x < kWidePanel * kWidePanel; x += 128) {
        const int r = x >> 5, q = x & 31;
        scr[x] = (&S.pm.Us[0][0])[x];
        if (r > q && r < nb) F[(p0 + r) + (p0 + q) * ld] = S.pm.Lsh[r][q];
      }
      if (tid < 32) scr[kWidePanel * kWidePanel + tid] = S.pm.rinv[tid];
    } else if (type == kDagTrsm) {
      const int p0 = 32 * p, nb = min(32, k - p0);
      const int r0 = dag_block_start(k, P, i), nr = dag_block_size(k, f, P, i);
      const double* scr = g.scr + static_cast<size_t>(Fr.scr_off + p) * kDagScr;
      double* us = &S.pm.Us[0][0];
      for (int x = tid; x < kDagScr / 2; x += 128) {
        double* dst = x < 512 ? us + 2 * x : S.pm.rinv + 2 * (x - 512);
        cp16(dst, scr + 2 * x);
      }
      cp_wait_all();
      __syncthreads();
      if (warp == 0)
        trsm_rows<32>(F, ld, p0, nb, r0, r0 + nr, us, S.pm.rinv, fd.stats, lane, S.u.t.TR, nullptr, 1);
    } else {
      const int p0 = 32 * p, nb = min(32, k - p0);
      const int ri = dag_block_start(k, P, i), nr = dag_block_size(k, f, P, i);
      const int rj = dag_block_start(k, P, j), nc = dag_block_size(k, f, P, j);
      GroupSmem& G = S.u.g;
      const bool dg = i == j;
      const int shA = stage_block<kNR2>(G.A, kSL, F, ld, ri, p0, nb, tid, 128);
      const int shB = dg ? shA : stage_block<kNR2>(G.B, kSL, F, ld, rj, p0, nb, tid, 128);
      const int shC = stage_block<kNR2>(G.C, kSL, F, ld, ri, rj, nc, tid, 128);
      if (tid < nb) G.d[tid] = __ldcg(fd.d + c0 + p0 + tid);
      cp_wait_all();
      __syncthreads();
      tile_mma_store(F, ld, G.A, shA, dg ? G.A : G.B, shB, G.C, shC, G.d, nb, ri, nr, rj, nc, tid);
    }
    __syncthreads();  // the task's writes, then its state (and the smem reuse)
    // ---- publish
    if (type == kDagAsm) {
      for (int a = j + tid; a < NB; a += 128) st_release(stf + dag_tri(a, j), 1);
    } else if (tid == 0) {
      st_release(stf + dag_tri(i, type == kDagUpd ? j : p), p + 2);
      if (type == kDagUpd && j >= P && p == P - 1) red_release_add(g.done + tk.x, 1);
    }
    if (g.trace && tid == 0) {
      unsigned long long* tr = g.trace + 4 * static_cast<size_t>(ti);
      tr[0] = tw;
      tr[1] = tb;
      tr[2] = globaltimer();
      tr[3] = blockIdx.x;
    }
  }
}

int dag_smem_bytes() { return static_cast<int>(sizeof(DagSmem)); }

int dag_workers_per_sm() {
  static PerDeviceOnce init;
  init([] {
    cudaFuncSetAttribute(k_front_dag, cudaFuncAttributeMaxDynamicSharedMemorySize, dag_smem_bytes());
  });
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_front_dag, 128, dag_smem_bytes());
  cudaGetLastError();
  return per_sm;
}

void launch_front_dag(const SnDev& sd, const FactorDev& fd, const double* kval, const DagDev& g,
                      int workers, double eps, cudaStream_t st) {
  dag_workers_per_sm();  // the smem opt-in on this device
  launch_pdl(k_front_dag, workers, 128, static_cast<size_t>(dag_smem_bytes()), st, true, sd, fd, kval, g,
             eps);
}

int mid_front_limit() { return kMidF; }

void launch_mid_front(const SnDev& sd, const FactorDev& fd, const double* kval, const int* nodes, int count,
                      int fmax, double eps, cudaStream_t st, bool stage) {
  static PerDeviceOnce init;
  init([] {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncSetAttribute(k_mid_front<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    cudaFuncSetAttribute(k_mid_front<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
  });
  const int fm = fmax < 1 ? 1 : fmax;
  const size_t smem = (sizeof(MidSmem) + 7) / 8 * 8 + sizeof(double) * (static_cast<size_t>(fm) * (fm + 1) / 2);
  if (!count) return;
  if (fm <= 128)
    launch_pdl(k_mid_front<128>, count, 128, smem, st, true, sd, fd, kval, nodes, eps, stage ? 1 : 0);
  else
    launch_pdl(k_mid_front<256>, count, 256, smem, st, true, sd, fd, kval, nodes, eps, stage ? 1 : 0);
}

}  // namespace nclb
