// Device-side views shared by the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace nclb {

// Supernodal structure on the device (see symbolic.hpp).
struct SnDev {
  int nsn;
  const int* first;     // nsn+1
  const int* f;         // nsn
  const int* sparent;   // nsn
  const int* rows_ptr;  // nsn+1
  const int* rows;
  const long long* l_off;  // nsn+1
  const long long* u_off;  // nsn
  const int* u_ld;         // nsn (f - k)
  const int* asm_ptr;
  const int* asm_pos;
  const int* asm_slot;
  const int* asm_cp;    // N+1: asm entries of (permuted) pivot column c
  const int* cc_off;    // nsn: wide front -> offset into cc_ptr (-1 narrow)
  const int* cc_ptr;
  const long long* cc_ubase;  // U_c(j, j) offset (lval if wide, else upd)
  const int* cc_rbase;        // rel index of child row j
  const int* cc_cnt;          // fu_c - j | (child wide) << 30
  const int* ch_ptr;
  const int* ch;
  const int* rel_ptr;  // also the offsets of the forward-solve update vectors
  const int* rel;
  const int* path_ptr;
  const int* path_nodes;
  const int* bwd_path;       // backward-solve path order
  const int* lt_ptr;         // nsn+1: light-child factor extend-add chunks
  const long long* lt_ent;   //   src | dst << 48 (symbolic.hpp)
  const int* ls_ptr;         // nsn+1: light-child solve chunks
  const long long* ls_ent;
  const int4* prec;          // 4 per path position (symbolic.hpp)
  const longlong2* poff;     // 1 per path position: {l_off, u_off}
  const int* split_ng;       // per front: factorization extend-add groups (0: unsplit)
  const long long* split_off;
  const int* usplit_ng;      // per front: forward-solve gather groups (0: unsplit)
  const long long* usplit_off;
  double* uvpart;            // forward-solve group sums (split.cu)
  const int8_t* wide;        // 1: wide-tier front (stored f x f in lval)
  int schur;                 // Schur-mode coupling supernode (assembled only), or -1
};

__device__ __forceinline__ int f_minus_k(const SnDev& sd, int s) {
  return sd.f[s] - (sd.first[s + 1] - sd.first[s]);
}

// numeric factor storage
struct FactorDev {
  double* lval;   // l_off[nsn]: warp-tier L blocks and whole wide fronts
  double* d;      // N (permuted order)
  double* upd;    // u_total: warp-tier update blocks
  int* stats;     // [0] n_pos [1] n_neg [2] perturbed [3] fail
  double* dscr;   // huge-front path: per diag task {Us[32][32], rinv[32]}
  double* ccpart; // split extend-add group sums (split.cu)
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Flag polling of the warp tier.  A relaxed load (no L1 invalidation, which
// ld.acquire.gpu costs: CCTL.IVALL after every poll, and with it the L1 hits
// of all static index data).  Ordering: the producer's lanes store their data,
// meet at a warp barrier and lane 0 releases the flag (st.release.gpu,
// ldl_kernels.cu publish).  The consumer polls relaxed and, once per flag
// after its last poll, reads the flag with ld.acquire.gpu (flag_acquire), so
// the producer's release synchronizes-with it and the __syncwarp that follows
// carries the edge to every lane.  Its loads of the produced data are L2
// loads (ld.global.cg) issued after that.
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Read-only loads issued exactly where written (asm volatile): the software
// pipelines of the warp tier issue a node ahead, and the compiler would
// otherwise sink plain __ldg loads down to their first use.
__device__ __forceinline__ int ldg_pin(const int* p) {
  int v;
  asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ long long ldg_pin(const long long* p) {
  long long v;
  asm volatile("ld.global.nc.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ldg_pin(const double* p) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int4 ldg_pin(const int4* p) {
  int4 v;
  asm volatile("ld.global.nc.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ longlong2 ldg_pin(const longlong2* p) {
  longlong2 v;
  asm volatile("ld.global.nc.v2.s64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ double ldcg_pin(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// Programmatic dependent launch (launches with
// cudaLaunchAttributeProgrammaticStreamSerialization): let the next kernel of
// the stream be scheduled now, and wait here until the previous kernel has
// completed and its writes are visible (no-ops for ordinary launches)
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// The acquire half of a flag wait, per flag: the lane that observed `flag` at
// its epoch (relaxed polls) reads it once more with ld.acquire.gpu (LDG.STRONG
// + L1 invalidation) -- the producer's st.release synchronizes-with that read,
// and a __syncwarp after carries the edge to the other lanes.  Cheaper than
// fence.acq_rel.gpu (MEMBAR.ALL.GPU + ERRBAR: waits for every outstanding
// access of the warp; 10 % of the warp-tier factorization's stall samples),
// and nodes without a flag to wait for pay nothing.
__device__ __forceinline__ void flag_acquire(const int* flag) { (void)ld_acquire(flag); }

__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// 1/d: MUFU approximation + two Newton steps (|d| >= the pivot eps)
__device__ __forceinline__ double rcp_nr(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

// max of non-negative doubles (NaN skipped, like std::max(acc, nan) == acc)
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  if (!(v >= 0.0)) return;
  atomicMax(reinterpret_cast<unsigned long long*>(addr),
            static_cast<unsigned long long>(__double_as_longlong(v)));
}

}  // namespace nclb
