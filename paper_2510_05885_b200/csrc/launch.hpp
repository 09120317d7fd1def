// Host-callable launchers of the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "device.cuh"
#include "kkt_plan.hpp"

namespace nclb {

struct AsmDev {
  int nnz;
  const int* c_ptr;
  const uint32_t* c_code;
  const int* pair_row;
  const int* pair_pa;
  const int* pair_pb;
  const int* long_slots;  // slots with more than kLongSum contributions (k_assemble_long)
  int nlong;
};

constexpr int kLongSum = 64;  // in-order sums longer than this: a warp each

// ldl_kernels.cu
void launch_factor_warp(const SnDev& sd, const FactorDev& fd, const double* kval,
                        int* flags, int epoch, int* counter, int npaths,
                        double eps, int grid, bool pipe, cudaStream_t st);
// wide_kernels.cu
// returns the cluster size used (0: launch impossible); max_f = largest
// front of the level (sizes the per-warp assembly accumulators)
int launch_wide_front(const SnDev& sd, const FactorDev& fd, const double* kval, const int* nodes,
                      int count, int cluster, int max_f, double eps, cudaStream_t st,
                      unsigned long long* trace = nullptr);
extern thread_local const char* wide_last_error;
// tile-dataflow segment of wide levels (dag.hpp): one persistent launch of
// `workers` resident CTAs
struct DagFront;
struct DagDev {
  const DagFront* fronts;
  const int* ch;
  const int4* tasks;  // per worker, in order: w_ptr
  const int* w_ptr;
  int* st;            // tile states (zeroed before the launch)
  int* done;          // per front: final trailing tiles (zeroed)
  double* scr;        // DIAG pivots, kDagScr per diagonal tile
  unsigned long long* trace;  // optional: 4 words per task
};
int dag_workers_per_sm();
void launch_front_dag(const SnDev& sd, const FactorDev& fd, const double* kval, const DagDev& g,
                      int workers, double eps, cudaStream_t st);
// max_f: the level's largest front (per-warp shared accumulators)
void launch_wide_assemble(const SnDev& sd, const FactorDev& fd, const double* kval,
                          const int4* tasks, int count, int max_f, cudaStream_t st);
void launch_wide_panel(const SnDev& sd, const FactorDev& fd, const int4* tasks, int count,
                       int panel, double eps, cudaStream_t st);
// scr: the scaled L11 blocks of the nd fronts (nullptr: fd.dscr)
void launch_wide_update(const SnDev& sd, const FactorDev& fd, const int4* tiles, int count,
                        const int* fronts, int nd, int panel, cudaStream_t st, bool pdl,
                        const double* scr = nullptr, int gtr = -1);
// the fused path's rest updates as 64x64 tiles (symbolic tiles64)
void launch_wide_update64(const SnDev& sd, const FactorDev& fd, const int4* tiles, int count,
                          const int* fronts, int nd, int panel, cudaStream_t st, bool pdl, const double* scr);
// a huge level's panels and trailing updates as one persistent launch
// (wide_kernels.cu k_huge_level): global panels [g0, g1) of the schedule
struct HugeDev {
  const int4* pn;       // panel tasks, pn_ptr per global panel
  const int* pn_ptr;
  const int4* tiles;    // rest-update tiles, tl_ptr per global panel
  const int* tl_ptr;
  const int* dg;        // fronts of each panel, dg_ptr per global panel (L11 write-back)
  const int* dg_ptr;
  int g0, g1;
  int* pc;              // per global panel: panel tasks done
  int* rc;              // per global panel: rest items done (tiles + 1)
  double* scr;          // L11 scratch, 2 x max_dg slots (panel parity)
  int max_dg;
  int npc;              // CTAs [0, npc) run panel tasks, the rest tiles
  int ctas;             // grid (<= resident CTAs)
  long long* trace;     // diagnostic: 5 SM-clock stamps per panel task
};
int huge_level_ctas();
void launch_huge_level(const SnDev& sd, const FactorDev& fd, const HugeDev& h, double eps, cudaStream_t st);
// k_wide_panel with the previous panel's strip update folded in (scr: this
// panel's L11 scratch slots)
void launch_wide_panel_f(const SnDev& sd, const FactorDev& fd, const int4* tasks, int count, int panel,
                         double eps, double* scr, cudaStream_t st, int gtr = -1);
// diagnostic: device buffer of 8 stamps per huge-path panel (nullptr: off);
// gtr above is the panel's global index in it
// false: the library was built without -DNCL_PANEL_TRACE
bool set_panel_trace(unsigned long long* p);
void launch_fwd_warp(const SnDev& sd, const double* lval, double* w, double* uvec,
                     int* flags, int epoch, int* counter, int npaths, int grid, bool pipe,
                     cudaStream_t st);
void launch_bwd_warp(const SnDev& sd, const double* lval, const double* d,
                     const double* w, double* x, int* flags, int epoch,
                     const int8_t* wide, int* counter, int npaths, int grid, bool pipe,
                     cudaStream_t st);
// wide_kernels.cu: levels of single-panel fronts (k <= 32) of at most
// mid_front_limit() rows, one 4-warp CTA per front kept in shared memory
int mid_front_limit();
void launch_mid_front(const SnDev& sd, const FactorDev& fd, const double* kval, const int* nodes, int count,
                      int fmax, double eps, cudaStream_t st, bool stage = true);
// small_front.cu: levels whose fronts all have <= small_*_limit() rows, one
// warp per front (factorization; forward and backward solve)
int small_factor_limit();
int small_solve_limit();
void launch_small_front(const SnDev& sd, const FactorDev& fd, const double* kval, const int* nodes,
                        int count, int fmax, double eps, cudaStream_t st);
void launch_fwd_small(const SnDev& sd, const double* lval, double* w, double* uvec,
                      const int* nodes, int count, int fmax, cudaStream_t st);
void launch_bwd_small(const SnDev& sd, const double* lval, const double* d, const double* w,
                      double* x, const int* nodes, int count, int fmax, cudaStream_t st);
// wide_solve.cu: one cluster per front of a level; return the cluster used
int launch_fwd_front(const SnDev& sd, const double* lval, double* w, double* uvec,
                     const int* nodes, int count, int cluster, int max_f, bool par,
                     cudaStream_t st);
// scr: 16 x 32 doubles per front of the level (cluster-parallel L11^T partials)
int launch_bwd_front(const SnDev& sd, const double* lval, const double* d, const double* w,
                     double* x, const int* nodes, int count, int cluster, int max_f, double* scr,
                     bool par, cudaStream_t st);
int solve_par_k();  // pivot count from which a front's L11 solve is cluster-parallel
// tree_solve.cu: the wide-tier solves of a run of levels as one persistent
// dataflow launch per direction (one CTA per front, per-front flags)
struct TreeDev {
  const int* list;      // wide fronts in topological order (children first)
  int n;
  const int* wait_ptr;  // forward: per list position, its children in the list
  const int* wait;
  const int* par;       // backward: per list position, the parent if in the list, else -1
  int* flags;           // per supernode: 1 forward done, 2 backward done
  unsigned long long* trace;  // diagnostic (NCL_TREE_TRACE): phase clocks per team and direction
  int stage;            // 0: the forward gather's direct loop only (NCL_NO_STAGED_GATHER, tests)
};
constexpr int kTreeMaxF = 2048;
constexpr int kTreeCluster = 8;  // CTAs per front in the cluster launch (top levels)
constexpr int kTreeClusterF = 256;  // ... for levels whose fronts reach this many rows
// resident teams (C = 1: CTAs; C = kTreeCluster: clusters), 0 if it does not fit
int tree_teams(int C, int fmax, int pmax);
void launch_fwd_tree(const SnDev& sd, const TreeDev& td, const double* lval, double* w, double* uvec,
                     int C, int teams, int fmax, cudaStream_t st);
void launch_bwd_tree(const SnDev& sd, const TreeDev& td, const double* lval, const double* d,
                     const double* w, double* x, int C, int teams, int fmax, int pmax, cudaStream_t st);
void launch_permute_in(int n, const int* perm, const double* b, double* w,
                       cudaStream_t st);
void launch_permute_out(int n, const int* perm, const double* xp, double* x,
                        cudaStream_t st);
int warp_tier_grid(int which);  // resident CTAs: 0 factor (pipelined), 1 solves, 2 factor (lean)
void launch_cc_partial(const SnDev& sd, const FactorDev& fd, int s, int f, int ng, cudaStream_t st);
void launch_uv_partial(const SnDev& sd, const double* uvec, int s, int f, int ng, cudaStream_t st);  // resident CTAs of the factor / solve kernels

// kkt_kernels.cu
void launch_assemble(const AsmDev& a, int form, int m, int m_eq, int nt,
                     const double* hval, const double* jval, const double* sigma,
                     double* wrow, double rho, double delta, double* kval,
                     cudaStream_t st);
void launch_absmax2(int n1, const double* a, int n2, const double* b, double* out,
                    cudaStream_t st);
void launch_rhs(const KktPlan& P, const int* jt_ptr, const int* jt_row, const int* jt_slot,
                const double* jval, const double* sigma, const double* r1,
                const double* r2, const double* r3, double rho, double delta, double* v,
                double* wk, double* rs, double* pk, double* rhs, const int* long_cols, int nlong_cols,
                cudaStream_t st);
void launch_recover(const KktPlan& P, const int* jp_ptr, const int* jp_idx,
                    const double* jval, const double* sol, const double* v,
                    const double* rs, const double* pk, const double* r2, double rho,
                    double delta, double* dx, double* dr, double* dy, cudaStream_t st);
void launch_nonfinite(int n, const double* a, int* flag, cudaStream_t st);
// dx[n], dr[m], dy[m] in one pass
void launch_nonfinite3(int n, const double* a, int m, const double* b, const double* c, int* flag,
                       cudaStream_t st);
void launch_residual(int N, const int* fr_ptr, const int* fr_col, const int* fr_slot,
                     const double* kval, const double* x, const double* b, double* r,
                     double* norm, const int* long_rows, int nlong_rows, cudaStream_t st);
void launch_axpy_to(int n, const double* x, const double* dx, double* out, cudaStream_t st);

}  // namespace nclb
