// Host orchestration of the sm_100a Newton-step path and its C ABI
// (include/ncl_b200.h).
//
//   LdlSystem  -- symbolic-once / numeric-per-call static-pivot LDL^T on the
//                 device: factorize (sparse.cpp:182-256), ldl_solve
//                 (sparse.cpp:258-276), solve_refined (sparse.cpp:278-322).
//   KktSystem  -- KktContext (kkt.cpp:41-314): bit-exact refill, delta loop
//                 with inertia control, rhs, refined solve, recovery.
// One CUDA stream per context; host synchronisation points are exactly the
// scalars the reference branches on (inertia / perturbed / ok per attempt,
// residual norms per refinement step).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ncl_b200.h"
#include "cuda_util.hpp"
#include "dag.hpp"
#include "kkt_plan.hpp"
#include "launch.hpp"
#include "layout.hpp"

namespace nclb {

// the wide-tier staging copies whole 34-row column chunks: pad the L buffer
constexpr size_t kLvalPad = 256;

std::string& last_error() {
  static thread_local std::string e;
  return e;
}

namespace {

struct Scalars {
  int stats[4];   // n_pos, n_neg, perturbed, fail
  int nonfinite;
  int pad;
  double hmax;
  double norm[4];  // [0] max|b| [1] residual
};

}  // namespace

struct FactorInfo {
  bool ok = false;
  int n_pos = 0, n_neg = 0, perturbed = 0;
};

// ---------------------------------------------------------------------------
constexpr int kSmallSolveMinFronts = 8;

class LdlSystem {
 public:
  // S: the reference's symbolic analysis (exposed, and the layout factors()
  // returns).  The numeric work uses the same elimination tree re-postordered
  // with the tallest child last (S2_): identical factor entries, but chains
  // occupy consecutive columns and collapse into relaxed supernodes.
  LdlSystem(const LowerCsc& K, const Symbolic& S, cudaStream_t st, int schur_n0 = 0)
      : K_(K), S_(S), st_(st) {
    S2_ = analyze_with_permutation(K_, tallest_child_last(K_, S_.perm));
    sn_ = build_supernodal(K_, S2_, schur_n0);
    N_ = K_.n;
    upload();
  }

  int n() const { return N_; }
  const Symbolic& sym() const { return S_; }
  const Supernodal& sn() const { return sn_; }
  const LowerCsc& pattern() const { return K_; }
  Scalars* host_scalars() { return hs_; }
  Scalars* dev_scalars() { return ds_.p; }
  cudaStream_t stream() const { return st_; }

  ~LdlSystem() {
    if (ptrace_.p) dump_panel_trace();
    if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
    if (solve_exec_) cudaGraphExecDestroy(solve_exec_);
    for (auto e : evs_) cudaEventDestroy(e);
    if (st2_) cudaStreamDestroy(st2_);
    if (hs_) cudaFreeHost(hs_);
  }

  // numeric factorization of the values kval (device, lower-CSC slot order);
  // the stats land in dev_scalars()->stats (not synchronised)
  // The launch sequence is fixed by the symbolic analysis, so from the second
  // factorization on it is replayed as one CUDA graph (~230 launches for the
  // 78k-bus mesh: per-launch overhead off the critical path).  The warp tier's
  // flags are cleared in the sequence and the factorization always uses epoch
  // 1 (solves use epochs >= 2), so the graph has no per-call arguments.
  void factorize_async(const double* kval, double eps) {
    if (graph_exec_ && kval == g_kval_ && eps == g_eps_) {
      CK(cudaGraphLaunch(graph_exec_, st_));
      launches_ += g_launches_;
      return;
    }
    const bool capture = use_graph_ && nfact_ >= 1 && !graph_exec_ && trace_level_ < 0;
    ++nfact_;
    if (capture && cudaStreamBeginCapture(st_, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
      cudaGetLastError();
      use_graph_ = false;
      factorize_direct(kval, eps);
      return;
    }
    const long long l0 = launches_;
    factorize_direct(kval, eps);
    if (!capture) return;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ex = nullptr;
    cudaError_t e = cudaStreamEndCapture(st_, &g);
    if (e == cudaSuccess) e = cudaGraphInstantiate(&ex, g, 0);
    if (g) cudaGraphDestroy(g);
    if (e != cudaSuccess) {  // fall back to direct launches for good
      cudaGetLastError();
      use_graph_ = false;
      factorize_direct(kval, eps);
      return;
    }
    graph_exec_ = ex;
    g_kval_ = kval;
    g_eps_ = eps;
    g_launches_ = launches_ - l0;
    CK(cudaGraphLaunch(graph_exec_, st_));
  }

  void factorize_direct(const double* kval, double eps) {
    CK(cudaMemsetAsync(ds_.p, 0, sizeof(int) * 4, st_));
    if (huge_ctas_ > 0) CK(cudaMemsetAsync(hcnt_.p, 0, sizeof(int) * hcnt_.n, st_));
    FactorDev fd = factor_dev();
    if (sn_.path_ptr.size() > 1) {
      CK(cudaMemsetAsync(counter_.p, 0, sizeof(int), st_));
      CK(cudaMemsetAsync(flags_.p, 0, sizeof(int) * flags_.n, st_));
      launch_factor_warp(sd_, fd, kval, flags_.p, 1, counter_.p, npaths(), eps,
                         pipe_ ? grid_ : lgrid_, pipe_, st_);
    }
    launches_ += npaths() > 0 ? 1 : 0;
    const auto& T = sn_;
    // diagnostic (NCL_LEVEL_TIMES=1, with NCL_NO_GRAPH=1): device time per level
    static const bool lvl_times = std::getenv("NCL_LEVEL_TIMES") != nullptr;
    std::vector<cudaEvent_t> lev;
    if (lvl_times) {
      lev.resize(static_cast<size_t>(nlevels()) + 1);
      for (auto& e : lev) CK(cudaEventCreate(&e));
      CK(cudaEventRecord(lev[0], st_));
    }
    g_kval_cur_ = kval;
    for (int l = 0; l < nlevels(); ++l) {
      if (lvl_times && l > 0) CK(cudaEventRecord(lev[l], st_));
      if (lvl_dag_[l] == -2) continue;  // inside a tile-dataflow segment
      if (lvl_dag_[l] >= 0) {
        launch_dag(lvl_dag_[l], eps);
        continue;
      }
      for (int s : lvl_split_[l]) {  // fronts with very many children: group sums first
        launch_cc_partial(sd_, fd, s, T.f[s], T.split_ng[s], st_);
        launches_ += 1;
      }
      if (mid_level(l)) {  // a 4-warp CTA per front, the front in shared memory
        launch_mid_front(sd_, fd, kval, mid_nodes_.p + T.lvl_ptr[l], T.lvl_ptr[l + 1] - T.lvl_ptr[l],
                         lvl_fmax_[l], eps, st_, stage_gather_);
        launches_ += 1;
        continue;
      }
      if (lvl_fmax_[l] <= small_factor_limit()) {  // a warp per front
        launch_small_front(sd_, fd, kval, lvl_nodes_.p + T.lvl_ptr[l], T.lvl_ptr[l + 1] - T.lvl_ptr[l],
                           lvl_fmax_[l], eps, st_);
        launches_ += 1;
        continue;
      }
      if (lvl_cluster_[l] > 0) {  // one launch, one cluster per front
        unsigned long long* tr = (l == trace_level_) ? trace_.p : nullptr;
        const int used = launch_wide_front(sd_, fd, kval, lvl_nodes_.p + T.lvl_ptr[l],
                                           T.lvl_ptr[l + 1] - T.lvl_ptr[l], lvl_cluster_[l],
                                           lvl_fmax_[l], eps, st_, tr);
        if (tr) dump_trace(l);
        if (used == 0)
          throw CudaError(std::string("k_wide_front: no cluster configuration fits: ") +
                          wide_last_error);
        lvl_cluster_[l] = used;
        launches_ += 1;
        continue;
      }
      const int na = T.asm_task_ptr[l + 1] - T.asm_task_ptr[l];
      launch_wide_assemble(sd_, fd, kval, asm_task_.p + T.asm_task_ptr[l], na, lvl_fmax_[l], st_);
      launches_ += na > 0;
      // one panel of lookahead across two streams: the panel kernel of g+1
      // runs as soon as the strip update of g is in, the rest of g's update
      // overlaps it on st2_ (every tile still sees the panels in order: the
      // strip of g waits for the rest of g-1, the panel of g for the rest of g-2)
      const int g0 = T.lp_ptr[l], g1 = T.lp_ptr[l + 1];
      if (huge_ctas_ > 0) {  // the level's panels as one persistent launch
        HugeDev h{pn_tasks_.p, pn_ptr_.p, tiles_.p, tl_ptr_.p, dg_nodes_.p, dg_ptr_.p, g0, g1,
                  hcnt_.p, hcnt_.p + T.lp_ptr.back(), dscr_.p, std::max(1, T.max_dg), 0, huge_ctas_,
                  htrace_.p};
        int mp = 1;
        for (int g = g0; g < g1; ++g) mp = std::max(mp, T.pn_ptr[g + 1] - T.pn_ptr[g]);
        h.npc = std::min(mp, huge_ctas_ / 2);
        launch_huge_level(sd_, fd, h, eps, st_);
        launches_ += 1;
        if (htrace_.p && l == nlevels() - 1) {  // diagnostic: mean clocks per panel task phase, per level
          std::vector<long long> hs(htrace_.n);
          CK(cudaMemcpyAsync(hs.data(), htrace_.p, hs.size() * 8, cudaMemcpyDeviceToHost, st_));
          CK(cudaStreamSynchronize(st_));
          for (int l2 = 0; l2 < nlevels(); ++l2) {
            double w = 0, a = 0, dg = 0, tr = 0;
            int c = 0;
            for (int g = T.lp_ptr[l2]; g < T.lp_ptr[l2 + 1]; ++g)
              for (int q = T.pn_ptr[g]; q < T.pn_ptr[g + 1]; ++q) {
                const long long* x = &hs[5 * q];
                w += x[4] - x[0];
                a += x[1] - x[4];
                dg += x[2] - x[1];
                tr += x[3] - x[2];
                ++c;
              }
            if (c)
              std::fprintf(stderr, "[ncl huge trace] level %d: %d panels, per task us: wait %.2f stage+strip %.2f "
                           "diag %.2f trsm-tail %.2f\n", l2, T.lp_ptr[l2 + 1] - T.lp_ptr[l2], w / c / 1965.0,
                           a / c / 1965.0, dg / c / 1965.0, tr / c / 1965.0);
          }
        }
        continue;
      }
      if (fused_panel_) {
        const bool ptr = ptrace_.p != nullptr;  // diagnostic: NCL_PANEL_TRACE
        if (ptr && l == first_huge_) CK(cudaMemsetAsync(ptrace_.p, 0, ptrace_.n * 8, st_));
        // the strip update of panel g-1 runs inside panel g's kernel; panel g
        // waits for the rest update of g-2, the rest update of g (stream 2,
        // also writing panel g's L11) for panel g; L11 scratch by parity
        for (int g = g0; g < g1; ++g) {
          const int nd = T.dg_ptr[g + 1] - T.dg_ptr[g];
          const int np = T.pn_ptr[g + 1] - T.pn_ptr[g];
          // 64x64 tiles where the update is latency-bound (up to ~two waves
          // of 32x32 tile CTAs: the mesh, bearing); the 32x32 kernel's
          // parallelism where it is throughput-bound (elec's 3000-row front's
          // early panels)
          const bool t64 = use_t64_ && T.tl_ptr[g + 1] - T.tl_ptr[g] <= kT64MaxTiles;
          const int nt = t64 ? T.tl64_ptr[g + 1] - T.tl64_ptr[g] : T.tl_ptr[g + 1] - T.tl_ptr[g];
          auto rest = [&](cudaStream_t s2, bool pdl, double* sc) {
            if (t64)
              launch_wide_update64(sd_, fd, tiles64_.p + T.tl64_ptr[g], nt, dg_nodes_.p + T.dg_ptr[g], nd, g - g0,
                                   s2, pdl, sc);
            else
              launch_wide_update(sd_, fd, tiles_.p + T.tl_ptr[g], nt, dg_nodes_.p + T.dg_ptr[g], nd, g - g0, s2,
                                 pdl, sc, ptrace_.p ? g : -1);
          };
          double* scr = dscr_.p + static_cast<size_t>((g - g0) & 1) * std::max(1, T.max_dg) * (kWidePanel * kWidePanel);
          if (g - 2 >= g0) CK(cudaStreamWaitEvent(st_, ev_rest(g - 2), 0));
          launch_wide_panel_f(sd_, fd, pn_tasks_.p + T.pn_ptr[g], np, g - g0, eps, scr, st_, ptr ? g : -1);
          if (g == g1 - 1) {
            // the level's last rest update (the update matrices the next
            // level's assembly reads) on the main stream as a programmatic
            // launch: no launch gap behind the last panel, and the next
            // assembly's static part overlaps it (factor -16 us on the mesh)
            if (g - 1 >= g0) CK(cudaStreamWaitEvent(st_, ev_rest(g - 1), 0));
            rest(st_, true, scr);
          } else {
            CK(cudaEventRecord(ev_panel(g), st_));
            CK(cudaStreamWaitEvent(st2_, ev_panel(g), 0));
            rest(st2_, false, scr);
            CK(cudaEventRecord(ev_rest(g), st2_));
          }
          launches_ += (np > 0) + (nt > 0 || nd > 0);
        }
        continue;
      }
      for (int g = g0; g < g1; ++g) {
        const int nd = T.dg_ptr[g + 1] - T.dg_ptr[g];
        const int np = T.pn_ptr[g + 1] - T.pn_ptr[g];
        const int nt = T.tl_ptr[g + 1] - T.tl_ptr[g];
        const int ns = T.ts_ptr[g + 1] - T.ts_ptr[g];
        if (g - 2 >= g0) CK(cudaStreamWaitEvent(st_, ev_rest(g - 2), 0));
        launch_wide_panel(sd_, fd, pn_tasks_.p + T.pn_ptr[g], np, g - g0, eps, st_);
        CK(cudaEventRecord(ev_panel(g), st_));
        if (g - 1 >= g0) CK(cudaStreamWaitEvent(st_, ev_rest(g - 1), 0));
        launch_wide_update(sd_, fd, tiles_s_.p + T.ts_ptr[g], ns, dg_nodes_.p + T.dg_ptr[g], nd,
                           g - g0, st_, true);
        CK(cudaStreamWaitEvent(st2_, ev_panel(g), 0));
        launch_wide_update(sd_, fd, tiles_.p + T.tl_ptr[g], nt, nullptr, 0, g - g0, st2_, false);
        CK(cudaEventRecord(ev_rest(g), st2_));
        launches_ += (np > 0) + (ns > 0 || nd > 0) + (nt > 0);
      }
      if (g1 > g0) CK(cudaStreamWaitEvent(st_, ev_rest(g1 - 1), 0));  // join before the next level
    }
    if (lvl_times) {
      CK(cudaEventRecord(lev[nlevels()], st_));
      CK(cudaStreamSynchronize(st_));
      std::fprintf(stderr, "[ncl level times] us:");
      for (int l = 0; l < nlevels(); ++l) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, lev[l], lev[l + 1]));
        std::fprintf(stderr, " %d:%.0f", l, ms * 1e3f);
      }
      std::fprintf(stderr, "\n");
      for (auto& e : lev) cudaEventDestroy(e);
    }
    CK(cudaGetLastError());
  }

  // diagnostic (NCL_PANEL_TRACE=1, library built with make EXTRA=-DNCL_PANEL_TRACE):
  // per huge level of the last factorization,
  // printed when the context is destroyed, the mean per panel of: launch gap
  // (previous panel's end -> this panel past its programmatic wait), staging,
  // strip, diagonal block, TRSM tail; and how often the rest update of g-2
  // ended after panel g-1 (it gated panel g)
  DBuf<unsigned long long> ptrace_;
  int first_huge_ = -1;
  void dump_panel_trace() {
    std::vector<unsigned long long> h(ptrace_.n);
    CK(cudaStreamSynchronize(st_));
    CK(cudaStreamSynchronize(st2_));
    CK(cudaMemcpy(h.data(), ptrace_.p, h.size() * 8, cudaMemcpyDeviceToHost));
    const auto& T = sn_;
    double tot[6] = {0, 0, 0, 0, 0, 0};
    for (int l = 0; l < nlevels(); ++l) {
      const int g0 = T.lp_ptr[l], g1 = T.lp_ptr[l + 1];
      if (g1 <= g0) continue;
      double a[6] = {0, 0, 0, 0, 0, 0};
      int late = 0;
      for (int g = g0; g < g1; ++g) {
        const unsigned long long* x = &h[8 * static_cast<size_t>(g)];
        const double prev_end = g > g0 ? static_cast<double>(h[8 * static_cast<size_t>(g - 1) + 5]) : static_cast<double>(x[0]);
        a[0] += (static_cast<double>(x[1]) - prev_end) * 1e-3;
        a[1] += (static_cast<double>(x[2]) - static_cast<double>(x[1])) * 1e-3;
        a[2] += (static_cast<double>(x[3]) - static_cast<double>(x[2])) * 1e-3;
        a[3] += (static_cast<double>(x[4]) - static_cast<double>(x[3])) * 1e-3;
        a[4] += (static_cast<double>(x[5]) - static_cast<double>(x[4])) * 1e-3;
        a[5] += (static_cast<double>(x[5]) - static_cast<double>(x[1])) * 1e-3;
        if (g - 2 >= g0 && h[8 * static_cast<size_t>(g - 2) + 7] > h[8 * static_cast<size_t>(g - 1) + 5]) ++late;
      }
      const int n = g1 - g0;
      for (int i = 0; i < 6; ++i) tot[i] += a[i];
      std::fprintf(stderr, "[ncl panel trace] level %d: %d panels, per panel us: gap %.2f stage %.2f strip %.2f "
                   "diag %.2f tail %.2f (body %.2f); rest g-2 late %d; level span %.1f\n", l, n, a[0] / n, a[1] / n,
                   a[2] / n, a[3] / n, a[4] / n, a[5] / n, late,
                   (static_cast<double>(h[8 * static_cast<size_t>(g1 - 1) + 7]) - static_cast<double>(h[8 * static_cast<size_t>(g0)])) * 1e-3);
    }
    std::fprintf(stderr, "[ncl panel trace] total us: gap %.1f stage %.1f strip %.1f diag %.1f tail %.1f\n", tot[0],
                 tot[1], tot[2], tot[3], tot[4]);
    set_panel_trace(nullptr);
    std::fflush(stderr);
  }
  // diagnostic: NCL_WIDE_TRACE=<level> prints per-phase timestamps of the
  // first front of that wide level (cluster rank 0, %globaltimer) to stderr
  void dump_trace(int l) {
    std::vector<unsigned long long> h(128);
    CK(cudaMemcpyAsync(h.data(), trace_.p, 128 * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    const int s = sn_.lvl_nodes[sn_.lvl_ptr[l]];
    std::fprintf(stderr, "[ncl trace] level %d front %d f=%d k=%d cluster=%d:", l, s, sn_.f[s],
                 sn_.first[s + 1] - sn_.first[s], lvl_cluster_[l]);
    for (int i = 1; i < 120 && h[i] > h[0]; ++i)
      std::fprintf(stderr, " %.1f", (h[i] - h[i - 1]) / 1e3);
    std::fprintf(stderr, " (us per phase); panel detail:");
    const char* nm[7] = {"diag", "bar", "trsm", "csync", "l11", "tiles", "csync"};
    for (int i = 0; i < 7; ++i) std::fprintf(stderr, " %s %.2f", nm[i], (h[121 + i] - h[120 + i]) / 1e3);
    std::fprintf(stderr, " us\n");
    CK(cudaMemsetAsync(trace_.p, 0, 128 * sizeof(unsigned long long), st_));
  }

  int nlevels() const { return static_cast<int>(sn_.lvl_ptr.size()) - 1; }
  // single-panel levels of fronts that fit in one CTA's shared memory, without
  // Schur / split fronts (NCL_NO_MID=1: the small-front / cluster kernels)
  bool use_mid_ = std::getenv("NCL_NO_MID") == nullptr;
  bool mid_level(int l) const {
    if (!use_mid_ || lvl_fmax_[l] > mid_front_limit() || lvl_kmax_[l] > kWidePanel) return false;
    for (int q = sn_.lvl_ptr[l]; q < sn_.lvl_ptr[l + 1]; ++q) {
      const int s = sn_.lvl_nodes[q];
      if (s == sn_.schur || sn_.split_ng[s]) return false;
    }
    return true;
  }
  // a warp per front for levels of many small fronts; a level of a few
  // fronts (the dense Schur system: one 118-row front) takes the cluster
  // solve, which spreads each front over up to 16 CTAs
  bool small_solve(int l) const {
    return lvl_fmax_[l] <= small_solve_limit() &&
           (lvl_fmax_[l] <= 32 || sn_.lvl_ptr[l + 1] - sn_.lvl_ptr[l] >= kSmallSolveMinFronts);
  }
  long long launches() const { return launches_; }

  FactorInfo read_factor_info() {
    CK(cudaMemcpyAsync(hs_, ds_.p, sizeof(Scalars), cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    FactorInfo fi;
    fi.n_pos = hs_->stats[0];
    fi.n_neg = hs_->stats[1];
    fi.perturbed = hs_->stats[2];
    fi.ok = hs_->stats[3] == 0;
    return fi;
  }

  // Solves.  Epochs are fixed (forward 2, backward 3; the factorization uses
  // 1) and the warp-tier flags are cleared at the start of every forward
  // pass, so a whole solve is one argument-free CUDA graph from the second
  // call on; the caller's vectors are copied in / out around it.
  // NCL_LEVEL_TIMES diagnostic: events between the phases of a sequence
  struct PhaseTimer {
    bool on;
    cudaStream_t st;
    std::vector<cudaEvent_t> ev;
    explicit PhaseTimer(cudaStream_t s) : on(std::getenv("NCL_LEVEL_TIMES") != nullptr), st(s) { mark(); }
    void mark() {
      if (!on) return;
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      CK(cudaEventRecord(e, st));
      ev.push_back(e);
    }
    void report(const char* what) {
      if (!on) return;
      mark();
      CK(cudaStreamSynchronize(st));
      std::fprintf(stderr, "[ncl %s times] us:", what);
      for (size_t i = 0; i + 1 < ev.size(); ++i) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
        std::fprintf(stderr, " %.0f", ms * 1e3f);
      }
      std::fprintf(stderr, "\n");
      for (auto e : ev) cudaEventDestroy(e);
    }
  };

  void fwd_seq(const double* b) {
    PhaseTimer pt(st_);
    launch_permute_in(N_, perm_.p, b, wp_.p, st_);
    if (npaths()) {
      CK(cudaMemsetAsync(counter_.p, 0, sizeof(int), st_));
      CK(cudaMemsetAsync(flags_.p, 0, sizeof(int) * flags_.n, st_));
      launch_fwd_warp(sd_, lval_.p, wp_.p, uvec_.p, flags_.p, 2, counter_.p, npaths(),
                      pipe_ ? sgrid_ : fgrid_, pipe_, st_);
    }
    pt.mark();
    for (int l = 0; l < nlevels(); ++l) {
      if (l) pt.mark();
      if (l == tr_l0_ && tree_on()) {  // levels [tr_l0_, tr_l1_): dataflow launches
        CK(cudaMemsetAsync(tr_flags_.p, 0, sizeof(int) * tr_flags_.n, st_));
        for (auto& P : tp_)
          if (P.on()) launch_fwd_tree(sd_, P.td, lval_.p, wp_.p, uvec_.p, P.C, P.teams, P.fmax, st_);
        l = tr_l1_ - 1;
        continue;
      }
      for (int s : lvl_usplit_[l]) {
        launch_uv_partial(sd_, uvec_.p, s, sn_.f[s], sn_.usplit_ng[s], st_);
        launches_ += 1;
      }
      if (small_solve(l)) {
        launch_fwd_small(sd_, lval_.p, wp_.p, uvec_.p, lvl_nodes_.p + sn_.lvl_ptr[l],
                         sn_.lvl_ptr[l + 1] - sn_.lvl_ptr[l], lvl_fmax_[l], st_);
        continue;
      }
      const int used = launch_fwd_front(sd_, lval_.p, wp_.p, uvec_.p, lvl_nodes_.p + sn_.lvl_ptr[l],
                                        sn_.lvl_ptr[l + 1] - sn_.lvl_ptr[l], solve_cluster_[l],
                                        lvl_fmax_[l], lvl_kmax_[l] >= solve_par_k(), st_);
      if (used == 0) throw CudaError("k_fwd_front: no cluster configuration fits");
      solve_cluster_[l] = used;
    }
    pt.report("fwd (warp, levels)");
    launches_ += 1 + (npaths() > 0 ? 1 : 0) + nlevels() - (tree_on() ? tr_l1_ - tr_l0_ - (tp_[0].on() + tp_[1].on()) : 0);
    CK(cudaGetLastError());
  }
  void bwd_seq(double* x) {
    PhaseTimer pt(st_);
    for (int l = nlevels() - 1; l >= 0; --l) {
      if (l < nlevels() - 1) pt.mark();
      if (l == tr_l1_ - 1 && tree_on()) {
        for (int pi = 1; pi >= 0; --pi)
          if (tp_[pi].on())
            launch_bwd_tree(sd_, tp_[pi].td, lval_.p, d_.p, wp_.p, xp_.p, tp_[pi].C, tp_[pi].teams,
                            tp_[pi].fmax, tp_[pi].pmax, st_);
        if (tr_dump_) dump_tree_trace();
        l = tr_l0_;
        continue;
      }
      if (small_solve(l)) {
        launch_bwd_small(sd_, lval_.p, d_.p, wp_.p, xp_.p, lvl_nodes_.p + sn_.lvl_ptr[l],
                         sn_.lvl_ptr[l + 1] - sn_.lvl_ptr[l], lvl_fmax_[l], st_);
        continue;
      }
      const int used = launch_bwd_front(sd_, lval_.p, d_.p, wp_.p, xp_.p,
                                        lvl_nodes_.p + sn_.lvl_ptr[l],
                                        sn_.lvl_ptr[l + 1] - sn_.lvl_ptr[l], solve_cluster_[l],
                                        lvl_fmax_[l], bscr_.p, lvl_kmax_[l] >= solve_par_k(), st_);
      if (used == 0) throw CudaError("k_bwd_front: no cluster configuration fits");
      solve_cluster_[l] = used;
    }
    pt.mark();
    if (npaths()) {
      CK(cudaMemsetAsync(counter_.p, 0, sizeof(int), st_));
      launch_bwd_warp(sd_, lval_.p, d_.p, wp_.p, xp_.p, flags_.p, 3, wide_.p, counter_.p,
                      npaths(), pipe_ ? sgrid_ : fgrid_, pipe_, st_);
    }
    launch_permute_out(N_, perm_.p, xp_.p, x, st_);
    pt.report("bwd (levels top-down, warp)");
    launches_ += 1 + (npaths() > 0 ? 1 : 0) + nlevels() - (tree_on() ? tr_l1_ - tr_l0_ - (tp_[0].on() + tp_[1].on()) : 0);
    CK(cudaGetLastError());
  }

  // Schur mode: the forward half (b -> permuted w, coupling rows assembled
  // at the tail of wp) and the backward half (coupling solution at the tail
  // of xp -> x)
  void solve_fwd_async(const double* b) { fwd_seq(b); }
  void solve_bwd_async(double* x) { bwd_seq(x); }
  int schur_n0() const { return sn_.schur >= 0 ? N_ - sn_.first[sn_.schur] : 0; }
  const double* schur_front() const { return lval_.p + sn_.l_off[sn_.schur]; }
  double* w_tail() { return wp_.p + (N_ - schur_n0()); }
  double* x_tail() { return xp_.p + (N_ - schur_n0()); }

  // x = P^T L^-T D^-1 L^-1 P b (device vectors, async)
  void solve_async(const double* b, double* x) {
    if (!use_graph_ || trace_level_ >= 0) {
      fwd_seq(b);
      bwd_seq(x);
      return;
    }
    CK(cudaMemcpyAsync(bin_.p, b, sizeof(double) * N_, cudaMemcpyDeviceToDevice, st_));
    if (!solve_exec_ && nsolve_ >= 1) {  // capture the second solve
      if (cudaStreamBeginCapture(st_, cudaStreamCaptureModeRelaxed) == cudaSuccess) {
        const long long l0 = launches_;
        fwd_seq(bin_.p);
        bwd_seq(xout_.p);
        cudaGraph_t g = nullptr;
        cudaError_t e = cudaStreamEndCapture(st_, &g);
        if (e == cudaSuccess) e = cudaGraphInstantiate(&solve_exec_, g, 0);
        if (g) cudaGraphDestroy(g);
        if (e != cudaSuccess) {
          cudaGetLastError();
          solve_exec_ = nullptr;
          use_graph_ = false;
        }
        s_launches_ = launches_ - l0;
        launches_ = l0;
      } else {
        cudaGetLastError();
        use_graph_ = false;
      }
    }
    ++nsolve_;
    if (solve_exec_) {
      CK(cudaGraphLaunch(solve_exec_, st_));
      launches_ += s_launches_;
    } else {
      fwd_seq(bin_.p);
      bwd_seq(xout_.p);
    }
    CK(cudaMemcpyAsync(x, xout_.p, sizeof(double) * N_, cudaMemcpyDeviceToDevice, st_));
  }

  // r = b - A x; norm slot (device) receives max|r| (must be zeroed by caller)
  void residual_async(const double* kval, const double* x, const double* b, double* r,
                      double* norm) {
    launch_residual(N_, fr_ptr_.p, fr_col_.p, fr_slot_.p, kval, x, b, r, norm, long_rows_.p,
                    static_cast<int>(long_rows_.n), st_);
    launches_ += 1;
  }

  // solve_refined (sparse.cpp:278-322).  b on device; solution in x_out
  // (device).  Returns steps; rel/conv through pointers.
  int solve_refined(const double* kval, const double* b, int max_ref, double tol,
                    double* x_out, double* rel_out, int* conv_out) {
    double* x = rx_.p;
    double* r = rr_.p;
    double* dx = rdx_.p;
    double* xn = rxn_.p;
    double* rn = rrn_.p;
    solve_async(b, x);
    CK(cudaMemsetAsync(&ds_.p->norm[0], 0, sizeof(double) * 2, st_));
    launch_absmax2(N_, b, 0, nullptr, &ds_.p->norm[0], st_);
    launches_ += 1;
    residual_async(kval, x, b, r, &ds_.p->norm[1]);
    CK(cudaMemcpyAsync(&hs_->norm[0], &ds_.p->norm[0], sizeof(double) * 2,
                       cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    const double bnorm = hs_->norm[0];
    const double denom = bnorm > 0.0 ? bnorm : 1.0;
    double res = hs_->norm[1];
    double prev = res;
    int stagnant = 0, steps = 0;
    while (steps < max_ref && res > tol * denom) {
      solve_async(r, dx);
      launch_axpy_to(N_, x, dx, xn, st_);
      launches_ += 1;
      CK(cudaMemsetAsync(&ds_.p->norm[1], 0, sizeof(double), st_));
      residual_async(kval, xn, b, rn, &ds_.p->norm[1]);
      CK(cudaMemcpyAsync(&hs_->norm[1], &ds_.p->norm[1], sizeof(double),
                         cudaMemcpyDeviceToHost, st_));
      CK(cudaStreamSynchronize(st_));
      const double res_new = hs_->norm[1];
      if (!std::isfinite(res_new) || res_new >= res) break;
      std::swap(x, xn);
      std::swap(r, rn);
      steps++;
      stagnant = (res_new > 0.5 * prev) ? stagnant + 1 : 0;
      prev = res_new;
      res = res_new;
      if (stagnant >= 2) break;
    }
    CK(cudaMemcpyAsync(x_out, x, sizeof(double) * N_, cudaMemcpyDeviceToDevice, st_));
    if (rel_out) *rel_out = res / denom;
    if (conv_out) *conv_out = res <= tol * denom;
    return steps;
  }

  // host copy of the factors in the reference's LdlFactors layout
  void factors_host(int* lcol_ptr, int* lrow_ind, double* lval, double* d) const {
    const int nsn = sn_.nsn;
    std::vector<double> lv(static_cast<size_t>(sn_.l_off[nsn]));
    std::vector<double> dv(static_cast<size_t>(N_));
    if (!lv.empty())
      CK(cudaMemcpy(lv.data(), lval_.p, lv.size() * sizeof(double), cudaMemcpyDeviceToHost));
    if (N_) CK(cudaMemcpy(dv.data(), d_.p, dv.size() * sizeof(double), cudaMemcpyDeviceToHost));
    // reference column j <-> internal column S2_.iperm[S_.perm[j]]
    std::vector<int> in(static_cast<size_t>(N_));
    for (int j = 0; j < N_; ++j) in[j] = S2_.iperm[S_.perm[j]];
    if (lcol_ptr) std::copy(S_.lcol_ptr.begin(), S_.lcol_ptr.end(), lcol_ptr);
    if (d)
      for (int j = 0; j < N_; ++j) d[j] = dv[in[j]];
    if (!lrow_ind && !lval) return;
    // the reference's L pattern; each value from its position in the internal
    // front (relaxed supernodes hold explicit zeros, columns are reordered)
    const std::vector<int> lri = l_row_pattern(K_, S_);
    std::vector<int> col2sn(static_cast<size_t>(N_));
    for (int s = 0; s < nsn; ++s)
      for (int c = sn_.first[s]; c < sn_.first[s + 1]; ++c) col2sn[c] = s;
    for (int j = 0; j < N_; ++j) {
      const int jj = in[j], s = col2sn[jj];
      const int c0 = sn_.first[s], f = sn_.f[s], p = jj - c0;
      const long long ld = sn_.wide[s] ? wide_ld(f) : f;
      const int* rows = sn_.rows.data() + sn_.rows_ptr[s];  // ascending internal rows
      for (int q = S_.lcol_ptr[j]; q < S_.lcol_ptr[j + 1]; ++q) {
        if (lrow_ind) lrow_ind[q] = lri[q];
        if (lval) {
          const int r = static_cast<int>(std::lower_bound(rows, rows + f, in[lri[q]]) - rows);
          lval[q] = lv[static_cast<size_t>(sn_.l_off[s] + r + p * ld)];
        }
      }
    }
  }

  // y += A x on the host pattern (diagnostic)
  int npaths() const { return static_cast<int>(sn_.path_ptr.size()) - 1; }

 private:
  FactorDev factor_dev() {
    FactorDev fd;
    fd.lval = lval_.p;
    fd.d = d_.p;
    fd.upd = upd_.p;
    fd.stats = ds_.p->stats;
    fd.dscr = dscr_.p;
    fd.ccpart = ccpart_.p;
    return fd;
  }

  void upload() {
    const Supernodal& T = sn_;
    first_.upload(T.first);
    f_.upload(T.f);
    sparent_.upload(T.sparent);
    rows_ptr_.upload(T.rows_ptr);
    rows_.upload(T.rows);
    l_off_.upload(T.l_off);
    u_off_.upload(T.u_off);
    u_ld_.upload(T.u_ld);
    asm_ptr_.upload(T.asm_ptr);
    asm_pos_.upload(T.asm_pos);
    asm_slot_.upload(T.asm_slot);
    ch_ptr_.upload(T.ch_ptr);
    ch_.upload(T.ch);
    rel_ptr_.upload(T.rel_ptr);
    rel_.upload(T.rel);
    path_ptr_.upload(T.path_ptr);
    path_nodes_.upload(T.path_nodes);
    bwd_path_.upload(T.bwd_path);
    lt_ptr_.upload(T.lt_ptr);
    lt_ent_.upload(T.lt_ent);
    ls_ptr_.upload(T.ls_ptr);
    ls_ent_.upload(T.ls_ent);
    {
      std::vector<int4> pr(T.prec.size() / 4);
      for (size_t i = 0; i < pr.size(); ++i)
        pr[i] = make_int4(T.prec[4 * i], T.prec[4 * i + 1], T.prec[4 * i + 2], T.prec[4 * i + 3]);
      prec_.upload(pr);
      std::vector<longlong2> po(T.poff.size() / 2);
      for (size_t i = 0; i < po.size(); ++i) {
        po[i].x = T.poff[2 * i];
        po[i].y = T.poff[2 * i + 1];
      }
      poff_.upload(po);
    }
    lvl_nodes_.upload(T.lvl_nodes);
    {  // mid-front launches: each level's fronts largest first (the last wave
       // is then the small fronts; fronts of a level are independent)
      std::vector<int> mn(T.lvl_nodes);
      for (size_t l = 0; l + 1 < T.lvl_ptr.size(); ++l)
        std::stable_sort(mn.begin() + T.lvl_ptr[l], mn.begin() + T.lvl_ptr[l + 1],
                         [&](int a, int b) { return T.f[a] > T.f[b]; });
      mid_nodes_.upload(mn);
    }
    std::vector<int8_t> wide(T.wide.begin(), T.wide.end());
    wide_.upload(wide);
    std::vector<int4> at(T.asm_task.size());
    for (size_t i = 0; i < at.size(); ++i)
      at[i] = make_int4(T.asm_task[i][0], T.asm_task[i][1], T.asm_task[i][2], T.asm_task[i][3]);
    asm_task_.upload(at);
    std::vector<int4> pt(T.pn_tasks.size());
    for (size_t i = 0; i < pt.size(); ++i)
      pt[i] = make_int4(T.pn_tasks[i][0], T.pn_tasks[i][1], T.pn_tasks[i][2], T.pn_tasks[i][3]);
    pn_tasks_.upload(pt);
    dg_nodes_.upload(T.dg_nodes);
    dscr_.alloc(2 * static_cast<size_t>(std::max(1, T.max_dg)) * (kWidePanel * kWidePanel));
    split_ng_.upload(T.split_ng);
    split_off_.upload(T.split_off);
    usplit_ng_.upload(T.usplit_ng);
    usplit_off_.upload(T.usplit_off);
    ccpart_.alloc(static_cast<size_t>(std::max(1LL, T.split_total)));
    uvpart_.alloc(static_cast<size_t>(std::max(1LL, T.usplit_total)));
    asm_cp_.upload(T.asm_cp);
    cc_off_.upload(T.cc_off);
    cc_ptr_.upload(T.cc_ptr);
    cc_ubase_.upload(T.cc_ubase);
    cc_rbase_.upload(T.cc_rbase);
    cc_cnt_.upload(T.cc_cnt);
    {
      std::vector<int4> ts(T.tiles_s.size());
      for (size_t i = 0; i < ts.size(); ++i)
        ts[i] = make_int4(T.tiles_s[i][0], T.tiles_s[i][1], T.tiles_s[i][2], T.tiles_s[i][3]);
      tiles_s_.upload(ts);
      const int ng = T.lp_ptr.empty() ? 0 : T.lp_ptr.back();
      evs_.resize(static_cast<size_t>(2 * ng));
      for (auto& e : evs_) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      CK(cudaStreamCreateWithFlags(&st2_, cudaStreamNonBlocking));
    }
    std::vector<int4> tl(T.tiles.size());
    for (size_t i = 0; i < tl.size(); ++i)
      tl[i] = make_int4(T.tiles[i][0], T.tiles[i][1], T.tiles[i][2], T.tiles[i][3]);
    tiles_.upload(tl);
    {
      std::vector<int4> t64(T.tiles64.size());
      for (size_t i = 0; i < t64.size(); ++i)
        t64[i] = make_int4(T.tiles64[i][0], T.tiles64[i][1], T.tiles64[i][2], T.tiles64[i][3]);
      tiles64_.upload(t64);
    }
    // per level: cluster size of the fused launch, or 0 = huge-front path
    int sms = 148;
    {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    lvl_cluster_.assign(static_cast<size_t>(nlevels()), 0);
    lvl_split_.assign(static_cast<size_t>(nlevels()), {});
    lvl_usplit_.assign(static_cast<size_t>(nlevels()), {});
    for (int l = 0; l < nlevels(); ++l)
      for (int q = T.lvl_ptr[l]; q < T.lvl_ptr[l + 1]; ++q) {
        const int s = T.lvl_nodes[q];
        if (T.split_ng[s]) lvl_split_[l].push_back(s);
        if (T.usplit_ng[s]) lvl_usplit_[l].push_back(s);
      }
    lvl_fmax_.assign(static_cast<size_t>(nlevels()), 0);
    lvl_kmax_.assign(static_cast<size_t>(nlevels()), 0);
    solve_cluster_.assign(static_cast<size_t>(nlevels()), 1);
    for (int l = 0; l < nlevels(); ++l) {
      int fmax = 0;
      const int nf = T.lvl_ptr[l + 1] - T.lvl_ptr[l];
      for (int q = T.lvl_ptr[l]; q < T.lvl_ptr[l + 1]; ++q) fmax = std::max(fmax, T.f[T.lvl_nodes[q]]);
      lvl_fmax_[l] = fmax;
      for (int q = T.lvl_ptr[l]; q < T.lvl_ptr[l + 1]; ++q)
        lvl_kmax_[l] = std::max(lvl_kmax_[l], T.first[T.lvl_nodes[q] + 1] - T.first[T.lvl_nodes[q]]);
      {
        int c = 16;
        while (c > 1 && nf * c > 2 * sms) c >>= 1;
        solve_cluster_[l] = c;
      }
      if (level_is_huge(fmax, nf)) continue;  // multi-kernel path
      // one wave: k_wide_front holds one CTA per SM (its staging shared
      // memory), so a level's clusters should fit the SMs at once
      // (mesh levels 5-6: 276 -> 250 us against sizing for two CTAs per SM)
      int c = 16;
      while (c > 1 && nf * c > sms) c >>= 1;
      lvl_cluster_[l] = c;
    }
    build_dag_segments(sms);
    // opt-in (NCL_HUGE_LEVEL=1): measured slower than the per-panel launches
    // on the 78k-bus mesh (2.43 vs 2.15 ms per factorization with the acquire
    // reads of this round; 3.28 vs 2.80 ms with fence.acq_rel: a flag hop per
    // panel instead of the programmatic launch, staging unchanged)
    if (std::getenv("NCL_HUGE_LEVEL") && T.lp_ptr.back() > 0) {
      huge_ctas_ = huge_level_ctas();
      if (huge_ctas_ < 2) huge_ctas_ = 0;
      pn_ptr_.upload(T.pn_ptr);
      tl_ptr_.upload(T.tl_ptr);
      dg_ptr_.upload(T.dg_ptr);
      hcnt_.alloc(2 * static_cast<size_t>(T.lp_ptr.back()));
      if (std::getenv("NCL_HUGE_TRACE")) {
        htrace_.alloc(5 * T.pn_tasks.size());
        htrace_.zero(st_);
      }
    }
    if (std::getenv("NCL_PANEL_TRACE") && T.lp_ptr.back() > 0) {
      ptrace_.alloc(8 * static_cast<size_t>(T.lp_ptr.back()));
      if (!set_panel_trace(ptrace_.p)) {
        std::fprintf(stderr, "[ncl] NCL_PANEL_TRACE: library built without -DNCL_PANEL_TRACE\n");
        ptrace_.alloc(0);
      }
      for (int l = 0; l < nlevels() && first_huge_ < 0; ++l)
        if (T.lp_ptr[l + 1] > T.lp_ptr[l]) first_huge_ = l;
    }
    build_tree(sms);
    if (std::getenv("NCL_LEVEL_STATS")) {  // diagnostic: split fronts
      int ns = 0, nu = 0;
      for (int q = 0; q < T.nsn; ++q) {
        ns += T.split_ng[q] > 0;
        nu += T.usplit_ng[q] > 0;
      }
      std::fprintf(stderr, "[ncl split] fronts with split extend-add: %d (factor), %d (forward gather)\n", ns, nu);
      if (T.schur >= 0) {
        const int sc = T.schur;
        int maxc = 0;
        for (int J = 0; J < T.f[sc]; ++J)
          maxc = std::max(maxc, T.cc_ptr[T.cc_off[sc] + J + 1] - T.cc_ptr[T.cc_off[sc] + J]);
        std::fprintf(stderr, "[ncl split] coupling front: f %d, children %d, most contributions per column %d\n",
                     T.f[sc], T.ch_ptr[sc + 1] - T.ch_ptr[sc], maxc);
      }
    }
    if (std::getenv("NCL_LEVEL_STATS")) {  // diagnostic: warp-tier paths, wide-tier levels
      int longest = 0, lp = -1;
      for (int p = 0; p + 1 < static_cast<int>(T.path_ptr.size()); ++p)
        if (T.path_ptr[p + 1] - T.path_ptr[p] > longest) longest = T.path_ptr[p + 1] - T.path_ptr[p], lp = p;
      if (lp >= 0) {
        double sk = 0, sf = 0, sch = 0, slt = 0, sasm = 0;
        for (int q = T.path_ptr[lp]; q < T.path_ptr[lp + 1]; ++q) {
          const int s = T.path_nodes[q];
          sk += T.first[s + 1] - T.first[s];
          sf += T.f[s];
          sch += T.ch_ptr[s + 1] - T.ch_ptr[s];
          slt += T.lt_ptr[s + 1] - T.lt_ptr[s];
          sasm += T.asm_ptr[s + 1] - T.asm_ptr[s];
        }
        std::fprintf(stderr,
                     "[ncl paths] %d paths, sn_height %d, longest %d: mean k %.1f f %.1f children %.1f "
                     "light entries %.1f A entries %.1f\n",
                     static_cast<int>(T.path_ptr.size()) - 1, T.sn_height, longest, sk / longest, sf / longest,
                     sch / longest, slt / longest, sasm / longest);
      }
      for (int l = 0; l < nlevels(); ++l) {
        int fmax = 0, kmax = 0;
        double fl = 0;
        for (int q = T.lvl_ptr[l]; q < T.lvl_ptr[l + 1]; ++q) {
          const int s = T.lvl_nodes[q], f = T.f[s], k = T.first[s + 1] - T.first[s];
          fmax = std::max(fmax, f);
          kmax = std::max(kmax, k);
          for (int j = 0; j < k; ++j) fl += double(f - j - 1) * (f - j + 1);
        }
        std::fprintf(stderr, "[ncl level] %d fronts %d fmax %d kmax %d flops %.3g cluster %d\n", l,
                     T.lvl_ptr[l + 1] - T.lvl_ptr[l], fmax, kmax, fl, lvl_cluster_[l]);
      }
    }
    if (const char* e = std::getenv("NCL_WIDE_TRACE")) {
      trace_level_ = std::atoi(e);
      trace_.alloc(128 * static_cast<size_t>(std::max(1, T.lvl_ptr.empty() ? 1 : T.nsn)));
      trace_.zero(st_);
    }
    perm_.upload(S2_.perm);
    lval_.alloc(static_cast<size_t>(T.l_off[T.nsn]) + kLvalPad);
    lval_.zero(st_);
    d_.alloc(static_cast<size_t>(N_));
    upd_.alloc(static_cast<size_t>(T.u_total));
    uvec_.alloc(static_cast<size_t>(T.rel_ptr[T.nsn]));
    {
      int maxw = 1;
      for (int l = 0; l < nlevels(); ++l) maxw = std::max(maxw, T.lvl_ptr[l + 1] - T.lvl_ptr[l]);
      bscr_.alloc(static_cast<size_t>(maxw) * 16 * 32);
    }
    flags_.alloc(static_cast<size_t>(std::max(T.nsn, 1)));
    flags_.zero(st_);
    counter_.alloc(1);
    wp_.alloc(static_cast<size_t>(N_));
    bin_.alloc(static_cast<size_t>(N_));
    xout_.alloc(static_cast<size_t>(N_));
    xp_.alloc(static_cast<size_t>(N_));
    rx_.alloc(static_cast<size_t>(N_));
    rr_.alloc(static_cast<size_t>(N_));
    rdx_.alloc(static_cast<size_t>(N_));
    rxn_.alloc(static_cast<size_t>(N_));
    rrn_.alloc(static_cast<size_t>(N_));
    ds_.alloc(1);
    ds_.zero(st_);
    CK(cudaMallocHost(&hs_, sizeof(Scalars)));
    // full symmetric row pattern for the residual matvec
    std::vector<int> cnt(static_cast<size_t>(N_) + 1, 0);
    for (int j = 0; j < N_; ++j)
      for (int p = K_.col_ptr[j]; p < K_.col_ptr[j + 1]; ++p) {
        cnt[K_.row_ind[p] + 1]++;
        if (K_.row_ind[p] != j) cnt[j + 1]++;
      }
    for (int i = 0; i < N_; ++i) cnt[i + 1] += cnt[i];
    std::vector<int> fcol(static_cast<size_t>(cnt[N_])), fslot(static_cast<size_t>(cnt[N_]));
    std::vector<int> nx(cnt.begin(), cnt.end() - 1);
    // columns ascending within each row: upper part (cols > i) comes from
    // column i itself, lower part (cols < i) from earlier columns
    for (int j = 0; j < N_; ++j)
      for (int p = K_.col_ptr[j]; p < K_.col_ptr[j + 1]; ++p) {
        const int i = K_.row_ind[p];
        if (i != j) {
          fcol[nx[i]] = j;
          fslot[nx[i]++] = p;
        }
      }
    for (int j = 0; j < N_; ++j)
      for (int p = K_.col_ptr[j]; p < K_.col_ptr[j + 1]; ++p) {
        fcol[nx[j]] = K_.row_ind[p];
        fslot[nx[j]++] = p;
      }
    fr_ptr_.upload(cnt);
    {
      std::vector<int> lr;
      for (int i = 0; i < N_; ++i)
        if (cnt[i + 1] - cnt[i] > 256) lr.push_back(i);  // kkt_kernels.cu kLongRow
      long_rows_.upload(lr);
    }
    fr_col_.upload(fcol);
    fr_slot_.upload(fslot);
    sd_.nsn = T.nsn;
    sd_.first = first_.p;
    sd_.f = f_.p;
    sd_.sparent = sparent_.p;
    sd_.rows_ptr = rows_ptr_.p;
    sd_.rows = rows_.p;
    sd_.l_off = l_off_.p;
    sd_.u_off = u_off_.p;
    sd_.u_ld = u_ld_.p;
    sd_.asm_ptr = asm_ptr_.p;
    sd_.asm_pos = asm_pos_.p;
    sd_.asm_slot = asm_slot_.p;
    sd_.asm_cp = asm_cp_.p;
    sd_.cc_off = cc_off_.p;
    sd_.cc_ptr = cc_ptr_.p;
    sd_.cc_ubase = cc_ubase_.p;
    sd_.cc_rbase = cc_rbase_.p;
    sd_.cc_cnt = cc_cnt_.p;
    sd_.ch_ptr = ch_ptr_.p;
    sd_.ch = ch_.p;
    sd_.rel_ptr = rel_ptr_.p;
    sd_.rel = rel_.p;
    sd_.path_ptr = path_ptr_.p;
    sd_.path_nodes = path_nodes_.p;
    sd_.bwd_path = bwd_path_.p;
    sd_.lt_ptr = lt_ptr_.p;
    sd_.lt_ent = lt_ent_.p;
    sd_.ls_ptr = ls_ptr_.p;
    sd_.ls_ent = ls_ent_.p;
    sd_.prec = prec_.p;
    sd_.split_ng = split_ng_.p;
    sd_.split_off = split_off_.p;
    sd_.usplit_ng = usplit_ng_.p;
    sd_.usplit_off = usplit_off_.p;
    sd_.uvpart = uvpart_.p;
    sd_.poff = poff_.p;
    sd_.wide = wide_.p;
    sd_.schur = T.schur;
    grid_ = warp_tier_grid(0);
    sgrid_ = warp_tier_grid(1);
    lgrid_ = warp_tier_grid(2);
    fgrid_ = warp_tier_grid(3);
    {  // long chains: the pipelined walk; only short paths: the lean one
      int longest = 0;
      for (size_t p = 0; p + 1 < T.path_ptr.size(); ++p)
        longest = std::max(longest, T.path_ptr[p + 1] - T.path_ptr[p]);
      pipe_ = longest >= kFrontPathLen;
    }
    CK(cudaStreamSynchronize(st_));
  }

  // tree-dataflow solves (tree_solve.cu): the wide levels [tr_l0_, tr_l1_)
  // -- from the first level that is not a small-front level up to the first
  // one holding a Schur / split-gather front, a front above kTreeMaxF rows or
  // one with cluster-parallel pivot blocks -- as one launch per direction of
  // one CTA per front for [tr_l0_, tr_l2_) and one of a cluster per front for
  // the top levels [tr_l2_, tr_l1_) (few big fronts: one SM's bandwidth is
  // too little for them).  NCL_NO_TREE=1 keeps the per-level kernels;
  // NCL_TREE_C=1 runs every tree level one CTA per front.
  struct TreePart {
    int l0 = 0, l1 = 0, C = 1, teams = 0, fmax = 0, pmax = 0;
    DBuf<int> list, wptr, wait, par;
    std::vector<int> lvl;  // per list position: level (trace)
    TreeDev td{};
    bool on() const { return l1 > l0; }
  };
  int tr_l0_ = 0, tr_l1_ = 0;
  TreePart tp_[2];  // [0] one CTA per front (lower levels), [1] clusters (top levels)
  DBuf<int> tr_flags_;
  DBuf<unsigned long long> tr_trace_[2];
  bool tr_dump_ = false;
  bool tree_on() const { return tr_l1_ > tr_l0_; }
  bool build_tree_part(TreePart& P, int l0, int l1, int C, int trmode, int idx) {
    const auto& T = sn_;
    std::vector<int> list, pos(static_cast<size_t>(T.nsn), -1);
    int fmax = 0, pmax = 0;
    for (int q = T.lvl_ptr[l0]; q < T.lvl_ptr[l1]; ++q) {
      const int s = T.lvl_nodes[q];
      list.push_back(s);
      fmax = std::max(fmax, T.f[s]);
      pmax = std::max(pmax, (T.first[s + 1] - T.first[s] + 31) / 32);
    }
    // each level's fronts largest first (fronts of a level are independent:
    // the list stays topological; the teams start on the long fronts)
    for (int l = l0; l < l1; ++l)
      std::stable_sort(list.begin() + (T.lvl_ptr[l] - T.lvl_ptr[l0]), list.begin() + (T.lvl_ptr[l + 1] - T.lvl_ptr[l0]),
                       [&](int a, int b) { return T.f[a] > T.f[b]; });
    for (size_t i = 0; i < list.size(); ++i) pos[list[i]] = static_cast<int>(i);
    const int teams = tree_teams(C, fmax, pmax);
    if (teams < 1) return false;
    std::vector<int> wptr{0}, wait, par;
    for (int s : list) {
      for (int q = T.ch_ptr[s]; q < T.ch_ptr[s + 1]; ++q)
        if (pos[T.ch[q]] >= 0) wait.push_back(T.ch[q]);
      wptr.push_back(static_cast<int>(wait.size()));
      const int p = T.sparent[s];
      par.push_back(p >= 0 && pos[p] >= 0 ? p : -1);
    }
    P.list.upload(list);
    P.wptr.upload(wptr);
    P.wait.upload(wait.empty() ? std::vector<int>{0} : wait);
    P.par.upload(par);
    if (trmode) {
      tr_trace_[idx].alloc(16 * static_cast<size_t>(std::max<int>(static_cast<int>(list.size()), teams * C)));
      tr_trace_[idx].zero(st_);
    }
    P.td = TreeDev{P.list.p, static_cast<int>(list.size()), P.wptr.p, P.wait.p, P.par.p,
                   tr_flags_.p, trmode == 3 ? nullptr : tr_trace_[idx].p, stage_gather_ ? 1 : 0};
    P.lvl.assign(list.size(), 0);
    for (int l = l0; l < l1; ++l)
      for (int q = T.lvl_ptr[l]; q < T.lvl_ptr[l + 1]; ++q) P.lvl[pos[T.lvl_nodes[q]]] = l;
    P.l0 = l0;
    P.l1 = l1;
    P.C = C;
    P.teams = std::min(static_cast<int>(list.size()), teams);
    P.fmax = fmax;
    P.pmax = pmax;
    if (std::getenv("NCL_LEVEL_STATS")) {
      long long nch = 0, nent = 0;
      int mch = 0;
      for (int s : list) {
        const int c = T.ch_ptr[s + 1] - T.ch_ptr[s];
        nch += c;
        mch = std::max(mch, c);
        for (int q = T.ch_ptr[s]; q < T.ch_ptr[s + 1]; ++q) nent += T.rel_ptr[T.ch[q] + 1] - T.rel_ptr[T.ch[q]];
      }
      std::fprintf(stderr, "[ncl tree] levels %d-%d: %zu fronts on %d teams of %d CTAs (fmax %d); children per "
                   "front mean %.1f max %d, update entries per front %.0f\n", l0, l1 - 1, list.size(), P.teams, C,
                   fmax, static_cast<double>(nch) / list.size(), mch, static_cast<double>(nent) / list.size());
    }
    return true;
  }
  void build_tree(int /*sms*/) {
    if (std::getenv("NCL_NO_TREE")) return;
    const auto& T = sn_;
    const int nl = nlevels();
    int l0 = 0;
    while (l0 < nl && small_solve(l0)) ++l0;
    auto eligible = [&](int l) {
      if (lvl_fmax_[l] > kTreeMaxF || lvl_kmax_[l] >= solve_par_k()) return false;
      for (int q = T.lvl_ptr[l]; q < T.lvl_ptr[l + 1]; ++q) {
        const int s = T.lvl_nodes[q];
        if (s == T.schur || T.usplit_ng[s]) return false;
      }
      return true;
    };
    int l1 = l0;
    while (l1 < nl && eligible(l1)) ++l1;
    if (const char* e = std::getenv("NCL_TREE_L1")) l1 = std::min(l1, std::atoi(e));  // experiments
    if (l1 - l0 < 2) return;
    // top levels for the cluster launch: a suffix of levels of at most
    // `teams` fronts of >= kTreeClusterF rows (each front gets its cluster)
    const int cteams = std::getenv("NCL_TREE_C") && std::atoi(std::getenv("NCL_TREE_C")) == 1
                           ? 0
                           : tree_teams(kTreeCluster, lvl_fmax_[l1 - 1], 1);
    int l2 = l1;
    while (l2 > l0 && cteams > 0 && T.lvl_ptr[l2] - T.lvl_ptr[l2 - 1] <= cteams &&
           lvl_fmax_[l2 - 1] >= kTreeClusterF)
      --l2;
    if (const char* e = std::getenv("NCL_TREE_L2")) l2 = std::max(l0, std::min(l1, std::atoi(e)));
    const int trmode = std::getenv("NCL_TREE_TRACE") ? std::atoi(std::getenv("NCL_TREE_TRACE")) : 0;
    tr_dump_ = trmode == 1 || trmode == 3;
    tr_flags_.alloc(static_cast<size_t>(T.nsn));
    tr_flags_.zero(st_);
    bool ok = true;
    if (l2 > l0) ok = build_tree_part(tp_[0], l0, l2, 1, trmode, 0);
    if (ok && l1 > l2) ok = build_tree_part(tp_[1], l2, l1, kTreeCluster, trmode, 1);
    if (!ok) {
      tp_[0].l1 = tp_[0].l0;
      tp_[1].l1 = tp_[1].l0;
      return;
    }
    tr_l0_ = l0;
    tr_l1_ = l1;
  }
  // diagnostic (NCL_TREE_TRACE=1): per launch and direction, the mean SM
  // clocks (us at 1.965 GHz) per front of each phase, from each team's rank 0:
  // wait (reset, cluster barrier, children / parent flags), gather, solve,
  // write-out + publish
  void dump_tree_trace() {
    for (int pi = 0; pi < 2; ++pi) {
      const TreePart& P = tp_[pi];
      if (!P.on() || !tr_trace_[pi].p) continue;
      std::vector<unsigned long long> h(tr_trace_[pi].n);
      CK(cudaMemcpyAsync(h.data(), tr_trace_[pi].p, h.size() * 8, cudaMemcpyDeviceToHost, st_));
      CK(cudaStreamSynchronize(st_));
      const int grid = P.teams * P.C;
      for (int dir = 0; dir < 2; ++dir) {
        double sum[4] = {0, 0, 0, 0}, cnt = 0;
        for (int b = 0; b < grid; ++b) {
          const unsigned long long* x = &h[8 * static_cast<size_t>(dir * grid + b)];
          for (int i = 0; i < 4; ++i) sum[i] += static_cast<double>(x[i]);
          cnt += static_cast<double>(x[4]);
        }
        const double us = 1.0 / 1965.0 / std::max(1.0, cnt);
        std::fprintf(stderr, "[ncl tree trace] C=%d %s: %.0f fronts, per front us: wait %.2f gather %.2f solve %.2f "
                     "out %.2f\n", P.C, dir ? "bwd" : "fwd", cnt, sum[0] * us, sum[1] * us, sum[2] * us, sum[3] * us);
      }
    }
  }

  // tile-dataflow segments (dag.hpp): maximal runs of wide levels that are
  // not small-front levels, hold no split extend-add and no Schur front;
  // NCL_NO_DAG=1 keeps the level-synchronous kernels
  struct DagSeg {
    DagSegment g;
    DBuf<DagFront> fronts;
    DBuf<int> ch, w_ptr, st;  // st: tile states, then per-front done counters
    DBuf<int4> tasks;
    DBuf<double> scr;
    DBuf<unsigned long long> trace;
    DagDev dev{};
  };
  std::vector<std::unique_ptr<DagSeg>> dag_;
  std::vector<int> lvl_dag_;  // per level: segment starting here, or -1 (-2: inside one)

  void build_dag_segments(int sms) {
    lvl_dag_.assign(static_cast<size_t>(nlevels()), -1);
    if (!std::getenv("NCL_DAG")) return;  // opt-in while the level kernels are faster
    const int per_sm = dag_workers_per_sm();
    if (per_sm < 1) return;
    const int workers = per_sm * sms;
    const bool trace = std::getenv("NCL_DAG_TRACE") != nullptr;
    for (const auto& run : dag_level_runs(sn_, small_factor_limit())) {
      const int l = run[0], e = run[1];
      auto seg = std::make_unique<DagSeg>();
      seg->g = build_dag_segment(sn_, l, e, workers);
      const DagSegment& G = seg->g;
      seg->fronts.upload(G.fronts);
      seg->ch.upload(G.ch.empty() ? std::vector<int>{0} : G.ch);
      seg->w_ptr.upload(G.w_ptr);
      std::vector<int4> tk(G.tasks.size());
      for (size_t q = 0; q < tk.size(); ++q)
        tk[q] = make_int4(G.tasks[q][0], G.tasks[q][1], G.tasks[q][2], G.tasks[q][3]);
      seg->tasks.upload(tk);
      seg->st.alloc(static_cast<size_t>(G.nstate) + G.fronts.size());
      seg->scr.alloc(static_cast<size_t>(std::max(1, G.nscr)) * kDagScr);
      if (trace) seg->trace.alloc(4 * std::max<size_t>(1, G.tasks.size()));
      seg->dev = DagDev{seg->fronts.p, seg->ch.p, seg->tasks.p, seg->w_ptr.p, seg->st.p,
                        seg->st.p + G.nstate, seg->scr.p, trace ? seg->trace.p : nullptr};
      if (std::getenv("NCL_LEVEL_STATS"))
        std::fprintf(stderr, "[ncl dag] levels %d-%d: %zu fronts, %zu tasks on %d workers, "
                     "simulated %.1f us (critical path %.1f us)\n", l, e - 1, G.fronts.size(),
                     G.tasks.size(), workers, G.makespan_us, G.crit_us);
      lvl_dag_[l] = static_cast<int>(dag_.size());
      for (int q = l + 1; q < e; ++q) lvl_dag_[q] = -2;
      dag_.push_back(std::move(seg));
    }
  }
  void launch_dag(int si, double eps) {
    DagSeg& D = *dag_[si];
    CK(cudaMemsetAsync(D.st.p, 0, D.st.n * sizeof(int), st_));
    launch_front_dag(sd_, factor_dev(), g_kval_cur_, D.dev, D.g.workers, eps, st_);
    launches_ += 1;
    if (D.dev.trace && std::getenv("NCL_DAG_TRACE")) dump_dag_trace(D);
  }
  // diagnostic (NCL_DAG_TRACE=1, with NCL_NO_GRAPH=1): per task type the
  // mean wait and work time, and the segment's span
  void dump_dag_trace(DagSeg& D) {
    const size_t nt = D.g.tasks.size();
    std::vector<unsigned long long> h(4 * nt);
    CK(cudaMemcpyAsync(h.data(), D.trace.p, h.size() * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    unsigned long long t0 = ~0ull, t1 = 0;
    double wsum[4] = {0, 0, 0, 0}, xsum[4] = {0, 0, 0, 0};
    int cnt[4] = {0, 0, 0, 0};
    for (size_t q = 0; q < nt; ++q) {
      const int type = D.g.tasks[q][1] >> 24;
      t0 = std::min(t0, h[4 * q]);
      t1 = std::max(t1, h[4 * q + 2]);
      wsum[type] += (h[4 * q + 1] - h[4 * q]) * 1e-3;
      xsum[type] += (h[4 * q + 2] - h[4 * q + 1]) * 1e-3;
      cnt[type]++;
    }
    const char* nm[4] = {"asm", "diag", "trsm", "upd"};
    std::fprintf(stderr, "[ncl dag trace] levels %d-%d span %.1f us (simulated %.1f):", D.g.l0, D.g.l1 - 1,
                 (t1 - t0) * 1e-3, D.g.makespan_us);
    for (int c = 0; c < 4; ++c)
      if (cnt[c])
        std::fprintf(stderr, " %s n=%d wait %.2f work %.2f us;", nm[c], cnt[c], wsum[c] / cnt[c],
                     xsum[c] / cnt[c]);
    std::fprintf(stderr, "\n");
    if (const char* path = std::getenv("NCL_DAG_TRACE_FILE")) {
      if (FILE* fp = std::fopen(path, "a")) {
        for (size_t q = 0; q < nt; ++q)
          std::fprintf(fp, "%d %d %d %d %d %llu %llu %llu %llu\n", D.g.l0, D.g.tasks[q][0],
                       D.g.tasks[q][1], D.g.tasks[q][2], D.g.tasks[q][3], h[4 * q] - t0,
                       h[4 * q + 1] - t0, h[4 * q + 2] - t0, h[4 * q + 3]);
        std::fclose(fp);
      }
    }
  }
  const double* g_kval_cur_ = nullptr;

  LowerCsc K_;
  Symbolic S_, S2_;
  Supernodal sn_;
  cudaStream_t st_;
  int N_ = 0;
  int grid_ = 1, sgrid_ = 1, lgrid_ = 1, fgrid_ = 1;  // warp-tier factor / solve / lean-factor grids (resident CTAs)
  bool pipe_ = true;                       // pipelined warp-tier factor walk (long chains)
  int epoch_ = 1;  // the factorization uses epoch 1, solves 2, 3, ...
  bool use_graph_ = std::getenv("NCL_NO_GRAPH") == nullptr;
  // huge levels: strip update folded into the panel kernel (NCL_NO_FUSED_PANEL=1: separate launch)
  bool fused_panel_ = std::getenv("NCL_NO_FUSED_PANEL") == nullptr;
  // the fused path's rest updates as 64x64 tiles (NCL_UPD32=1: 32x32, k_wide_update)
  bool use_t64_ = std::getenv("NCL_UPD32") == nullptr;
  // 32x32 tiles per launch up to which 64x64 tiles are used: ~two waves of
  // 32x32 tile CTAs (7 per SM x 148); measured: mesh indifferent above 1000,
  // bearing best near 2000-3000, elec worse above 2000
  static constexpr int kT64MaxTiles = 2000;
  // NCL_NO_STAGED_GATHER=1 (tests): the mid-front assembly and the tree forward
  // gather take their unstaged fallback paths (more children / entries than
  // the staging buffers hold)
  bool stage_gather_ = std::getenv("NCL_NO_STAGED_GATHER") == nullptr;
  // huge levels as one persistent launch (opt-in NCL_HUGE_LEVEL=1)
  int huge_ctas_ = 0;
  DBuf<int> hcnt_, pn_ptr_, tl_ptr_, dg_ptr_;
  DBuf<long long> htrace_;
  int nfact_ = 0;
  cudaGraphExec_t graph_exec_ = nullptr;
  const double* g_kval_ = nullptr;
  double g_eps_ = 0.0;
  long long g_launches_ = 0;
  cudaGraphExec_t solve_exec_ = nullptr;
  int nsolve_ = 0;
  long long s_launches_ = 0;
  DBuf<double> bin_, xout_;
  long long launches_ = 0;
  std::vector<int> lvl_cluster_, lvl_fmax_, lvl_kmax_, solve_cluster_;
  std::vector<std::vector<int>> lvl_split_, lvl_usplit_;  // per level: fronts with split extend-adds
  int trace_level_ = -1;
  DBuf<unsigned long long> trace_;
  SnDev sd_{};
  DBuf<int> first_, f_, sparent_, rows_ptr_, rows_, u_ld_, asm_ptr_, asm_pos_, asm_slot_,
      ch_ptr_, ch_, rel_ptr_, rel_, path_ptr_, path_nodes_, lvl_nodes_, perm_, flags_,
      counter_, fr_ptr_, fr_col_, fr_slot_, long_rows_, dg_nodes_, asm_cp_, cc_off_, cc_ptr_, cc_rbase_,
      cc_cnt_, lt_ptr_, ls_ptr_, bwd_path_, split_ng_, usplit_ng_;
  DBuf<long long> cc_ubase_, lt_ent_, ls_ent_, split_off_, usplit_off_;
  DBuf<double> dscr_, ccpart_, uvpart_;
  DBuf<int8_t> wide_;
  DBuf<int4> asm_task_, prec_;
  DBuf<longlong2> poff_;
  DBuf<int4> pn_tasks_;
  DBuf<int4> tiles_, tiles_s_;
  DBuf<int4> tiles64_;  // the fused path's rest updates, 64x64 tiles
  DBuf<int> mid_nodes_;  // lvl_nodes with each level's fronts largest first (mid-front launches)
  cudaStream_t st2_ = nullptr;        // huge-level lookahead stream
  std::vector<cudaEvent_t> evs_;      // per huge panel: panel done, rest done
  cudaEvent_t ev_panel(int g) { return evs_[2 * g]; }
  cudaEvent_t ev_rest(int g) { return evs_[2 * g + 1]; }
  DBuf<long long> l_off_, u_off_;
  DBuf<double> lval_, d_, upd_, uvec_, wp_, xp_, rx_, rr_, rdx_, rxn_, rrn_, bscr_;
  DBuf<Scalars> ds_;
  Scalars* hs_ = nullptr;
};

// ---------------------------------------------------------------------------
class KktSystem {
 public:
  KktSystem(KktPlan plan, const ncl_kkt_opts& opt)
      : P_(std::move(plan)), opt_(opt) {
    CK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&cst_, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&rev_, cudaEventDisableTiming));
    ldl_ = std::make_unique<LdlSystem>(
        P_.K, P_.sym, st_, P_.sn.schur >= 0 ? P_.N - P_.sn.first[P_.sn.schur] : 0);
    c_ptr_.upload(P_.c_ptr);
    c_code_.upload(P_.c_code);
    pair_row_.upload(P_.pair_row);
    pair_pa_.upload(P_.pair_pa);
    pair_pb_.upload(P_.pair_pb);
    jp_ptr_.upload(P_.jp_ptr);
    jp_idx_.upload(P_.jp_idx);
    jt_ptr_.upload(P_.jt_ptr);
    jt_row_.upload(P_.jt_row);
    jt_slot_.upload(P_.jt_slot);
    const size_t n = static_cast<size_t>(P_.n), m = static_cast<size_t>(P_.m);
    hval_.alloc(P_.hp_idx.size());
    jval_.alloc(P_.jp_idx.size());
    sigma_.alloc(n);
    r1_.alloc(n);
    r2_.alloc(m);
    r3_.alloc(m);
    dx_.alloc(n);
    dr_.alloc(m);
    dy_.alloc(m);
    kval_.alloc(static_cast<size_t>(P_.K.nnz()));
    kval_.zero(st_);
    wrow_.alloc(m);
    v_.alloc(m);
    wk_.alloc(static_cast<size_t>(P_.m_ineq));
    rs_.alloc(static_cast<size_t>(P_.m_ineq));
    pk_.alloc(static_cast<size_t>(P_.m_ineq));
    rhs_.alloc(static_cast<size_t>(P_.N));
    sol_.alloc(static_cast<size_t>(P_.N));
    asm_.nnz = P_.K.nnz();
    asm_.c_ptr = c_ptr_.p;
    asm_.c_code = c_code_.p;
    asm_.pair_row = pair_row_.p;
    asm_.pair_pa = pair_pa_.p;
    asm_.pair_pb = pair_pb_.p;
    {  // long in-order sums get a warp each (kkt_kernels.cu)
      std::vector<int> ls, lc;
      for (int q = 0; q < P_.K.nnz(); ++q)
        if (P_.c_ptr[q + 1] - P_.c_ptr[q] > kLongSum) ls.push_back(q);
      for (int c = 0; c < P_.nt; ++c)
        if (P_.jt_ptr[c + 1] - P_.jt_ptr[c] > kLongSum) lc.push_back(c);
      long_slots_.upload(ls);
      long_cols_.upload(lc);
      asm_.long_slots = long_slots_.p;
      asm_.nlong = static_cast<int>(ls.size());
    }
    CK(cudaStreamSynchronize(st_));
  }

  ~KktSystem() {
    ldl_.reset();
    for (auto& e : pool_) cudaEventDestroy(e);
    if (rev_) cudaEventDestroy(rev_);
    if (cst_) cudaStreamDestroy(cst_);
    if (st_) cudaStreamDestroy(st_);
  }

  const KktPlan& plan() const { return P_; }
  LdlSystem& ldl() { return *ldl_; }
  cudaStream_t stream() const { return st_; }

  void refill_async(const double* hv, const double* jv, const double* sg, double rho,
                    double delta) {
    launch_assemble(asm_, P_.form, P_.m, P_.m_eq, P_.nt, hv, jv, sg, wrow_.p, rho, delta,
                    kval_.p, st_);
  }

  void refill_host(const double* hv, const double* jv, const double* sg, double rho,
                   double delta) {
    upload_inputs(hv, jv, sg, nullptr, nullptr, nullptr);
    refill_async(hval_.p, jval_.p, sigma_.p, rho, delta);
    CK(cudaStreamSynchronize(st_));
  }

  void upload_inputs(const double* hv, const double* jv, const double* sg, const double* r1,
                     const double* r2, const double* r3) {
    auto h2d = [&](double* dst, const double* src, size_t k) {
      if (k) CK(cudaMemcpyAsync(dst, src, k * sizeof(double), cudaMemcpyHostToDevice, st_));
    };
    h2d(hval_.p, hv, hval_.n);
    h2d(jval_.p, jv, jval_.n);
    h2d(sigma_.p, sg, sigma_.n);
    // the right-hand sides are first read after the factorization: their
    // copies overlap the refill and the factorization on a copy stream
    CK(cudaEventRecord(rev_, st_));  // the previous solve is done with r1..r3
    CK(cudaStreamWaitEvent(cst_, rev_, 0));
    auto h2dc = [&](double* dst, const double* src, size_t k) {
      if (k && src) CK(cudaMemcpyAsync(dst, src, k * sizeof(double), cudaMemcpyHostToDevice, cst_));
    };
    h2dc(r1_.p, r1, r1_.n);
    h2dc(r2_.p, r2, r2_.n);
    h2dc(r3_.p, r3, r3_.n);
    CK(cudaEventRecord(rev_, cst_));
    r_pending_ = true;
  }

  // KktContext::solve (kkt.cpp:266-314) on device-resident inputs
  void solve_device(const double* hv, const double* jv, const double* sg, const double* r1,
                    const double* r2, const double* r3, double rho, double warm, double* dx,
                    double* dr, double* dy, ncl_kkt_stats* st) {
    std::memset(st, 0, sizeof(*st));
    std::fill(std::begin(ms_), std::end(ms_) - 1, 0.0);
    Scalars* ds = ldl_->dev_scalars();
    Scalars* hs = ldl_->host_scalars();
    // max(|H|, |sigma|) is only read for the first delta after a rejected
    // unregularised attempt without a warm start (kkt.cpp:273-313): computed
    // then, not on every call
    double delta = 0.0;
    bool first = true;
    const int* tgt = P_.inertia_target;
    for (;;) {
      st->factor_attempts++;
      const int e0 = tick();
      refill_async(hv, jv, sg, rho, delta);
      launches_ += P_.form == kK1s ? 2 : 1;
      const int e1 = tick();
      ldl_->factorize_async(kval_.p, opt_.pivot_eps);
      const int e2 = tick();
      span(0, e0, e1);
      span(1, e1, e2);
      const FactorInfo F = ldl_->read_factor_info();
      if (F.ok && F.n_pos == tgt[0] && F.n_neg == tgt[1]) {
        const int e3 = tick();
        if (r_pending_) {  // host-buffer call: the right-hand sides' copies
          CK(cudaStreamWaitEvent(st_, rev_, 0));
          r_pending_ = false;
        }
        launch_rhs(P_, jt_ptr_.p, jt_row_.p, jt_slot_.p, jv, sg, r1, r2, r3, rho, delta, v_.p,
                   wk_.p, rs_.p, pk_.p, rhs_.p, long_cols_.p, static_cast<int>(long_cols_.n), st_);
        launches_ += P_.form == kK1s ? 2 : 1;
        double rel = 0.0;
        int conv = 0;
        const int steps = ldl_->solve_refined(kval_.p, rhs_.p, opt_.max_refine,
                                              opt_.refine_tol, sol_.p, &rel, &conv);
        const int e4 = tick();
        span(2, e3, e4);
        // bn = ||rhs||_inf was read inside solve_refined
        const double bn = hs->norm[0];
        const double abs_res = rel * (bn > 0.0 ? bn : 1.0);
        const bool accept =
            F.perturbed == 0 || abs_res <= opt_.accept_tol * std::max(1.0, bn);
        if (accept) {
          st->accepted = 1;
          st->delta = delta;
          st->refine_steps = steps;
          st->perturbed_pivots = F.perturbed;
          st->rel_residual = rel;
          const int e5 = tick();
          launch_recover(P_, jp_ptr_.p, jp_idx_.p, jv, sol_.p, v_.p, rs_.p, pk_.p, r2, rho,
                         delta, dx, dr, dy, st_);
          CK(cudaMemsetAsync(&ds->nonfinite, 0, sizeof(int), st_));
          launch_nonfinite3(P_.n, dx, P_.m, dr, dy, &ds->nonfinite, st_);
          launches_ += 2;
          CK(cudaMemcpyAsync(&hs->nonfinite, &ds->nonfinite, sizeof(int),
                             cudaMemcpyDeviceToHost, st_));
          const int e6 = tick();
          span(3, e5, e6);
          CK(cudaStreamSynchronize(st_));
          st->ok = hs->nonfinite == 0;
          finish_timing();
          return;
        }
      }
      if (first) {
        if (warm > 0.0) {
          delta = std::max(1e-20, warm / 3.0);
        } else {
          CK(cudaMemsetAsync(&ds->hmax, 0, sizeof(double), st_));
          launch_absmax2(static_cast<int>(hval_.n), hv, P_.n, sg, &ds->hmax, st_);
          launches_ += 1;
          CK(cudaMemcpyAsync(&hs->hmax, &ds->hmax, sizeof(double), cudaMemcpyDeviceToHost, st_));
          CK(cudaStreamSynchronize(st_));
          delta = 1e-8 * std::max(1.0, hs->hmax);
        }
        first = false;
      } else {
        delta *= 8.0;
      }
      if (delta > opt_.delta_max) {
        st->ok = 0;
        finish_timing();
        return;
      }
    }
  }

  void solve_host(const double* hv, const double* jv, const double* sg, const double* r1,
                  const double* r2, const double* r3, double rho, double warm, double* dx,
                  double* dr, double* dy, ncl_kkt_stats* st) {
    upload_inputs(hv, jv, sg, r1, r2, r3);
    solve_device(hval_.p, jval_.p, sigma_.p, r1_.p, r2_.p, r3_.p, rho, warm, dx_.p, dr_.p,
                 dy_.p, st);
    auto d2h = [&](double* dst, const double* src, size_t k) {
      if (k && dst) CK(cudaMemcpyAsync(dst, src, k * sizeof(double), cudaMemcpyDeviceToHost, st_));
    };
    if (st->accepted) {
      d2h(dx, dx_.p, dx_.n);
      d2h(dr, dr_.p, dr_.n);
      d2h(dy, dy_.p, dy_.n);
    }
    if (r_pending_) {  // no attempt reached the right-hand sides: still join their copies
      CK(cudaStreamWaitEvent(st_, rev_, 0));
      r_pending_ = false;
    }
    CK(cudaStreamSynchronize(st_));
  }

  // pieces of solve_device for the distributed (Schur-mode) driver
  double* kval() { return kval_.p; }
  void rhs_async(const double* jv, const double* sg, const double* r1, const double* r2,
                 const double* r3, double rho, double delta, double* out) {
    launch_rhs(P_, jt_ptr_.p, jt_row_.p, jt_slot_.p, jv, sg, r1, r2, r3, rho, delta, v_.p, wk_.p,
               rs_.p, pk_.p, out, long_cols_.p, static_cast<int>(long_cols_.n), st_);
    launches_ += P_.form == kK1s ? 2 : 1;
  }
  void recover_async(const double* jv, const double* sol, const double* r2, double rho,
                     double delta, double* dx, double* dr, double* dy) {
    launch_recover(P_, jp_ptr_.p, jp_idx_.p, jv, sol, v_.p, rs_.p, pk_.p, r2, rho, delta, dx, dr,
                   dy, st_);
    launches_ += 1;
  }

  void matrix(int* cp, int* ri, double* val) const {
    if (cp) std::copy(P_.K.col_ptr.begin(), P_.K.col_ptr.end(), cp);
    if (ri) std::copy(P_.K.row_ind.begin(), P_.K.row_ind.end(), ri);
    if (val && kval_.n)
      CK(cudaMemcpy(val, kval_.p, kval_.n * sizeof(double), cudaMemcpyDeviceToHost));
  }

  void set_timing(bool on) { timing_ = on; }
  void timing(double* out) const { std::copy(std::begin(ms_), std::end(ms_), out); }
  long long launches() const { return launches_ + ldl_->launches(); }

 private:
  // sync-free phase timing: events are recorded on the context stream and
  // only read after the solve's final synchronisation
  int tick() {
    if (!timing_) return -1;
    if (nev_ == pool_.size()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      pool_.push_back(e);
    }
    CK(cudaEventRecord(pool_[nev_], st_));
    return static_cast<int>(nev_++);
  }
  void span(int phase, int a, int b) {
    if (timing_) spans_.push_back({phase, a, b});
  }
  void finish_timing() {
    if (timing_) {
      CK(cudaStreamSynchronize(st_));
      for (const auto& s : spans_) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, pool_[s[1]], pool_[s[2]]));
        ms_[s[0]] += ms;
      }
    }
    spans_.clear();
    nev_ = 0;
    ms_[4] = ms_[0] + ms_[1] + ms_[2] + ms_[3];
    ms_[5] += 1.0;
  }

  KktPlan P_;
  ncl_kkt_opts opt_;
  cudaStream_t st_ = nullptr;
  std::unique_ptr<LdlSystem> ldl_;
  AsmDev asm_{};
  DBuf<int> long_slots_, long_cols_;
  cudaStream_t cst_ = nullptr;  // host-buffer calls: copy stream of the right-hand sides
  cudaEvent_t rev_ = nullptr;
  bool r_pending_ = false;
  DBuf<int> c_ptr_, pair_row_, pair_pa_, pair_pb_, jp_ptr_, jp_idx_, jt_ptr_, jt_row_,
      jt_slot_;
  DBuf<uint32_t> c_code_;
  DBuf<double> hval_, jval_, sigma_, r1_, r2_, r3_, dx_, dr_, dy_, kval_, wrow_, v_, wk_, rs_,
      pk_, rhs_, sol_;
  std::vector<cudaEvent_t> pool_;
  size_t nev_ = 0;
  std::vector<std::array<int, 3>> spans_;
  bool timing_ = false;
  double ms_[6] = {0, 0, 0, 0, 0, 0};
  long long launches_ = 0;
};

// ---------------------------------------------------------------------------
// Schur-mode KKT of one rank's share of a block-arrowhead problem (SCOPF,
// SURVEY.md 8(e)).  The rank's sub-problem (coupling variables first, then
// its contingency blocks) is assembled with the ordinary bit-exact refill;
// the multifrontal factorization eliminates the blocks and leaves the
// assembled coupling front -- the rank's Schur contribution
// S_g = A00_g - sum_k A0k Akk^-1 Ak0 -- which the caller sums over ranks
// (NCCL allreduce); every rank then factors the dense S the same way.
__global__ void k_front_to_dense(int n0, size_t ld, const double* __restrict__ F, double* S) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i < n0) S[i + static_cast<size_t>(j) * n0] = i >= j ? F[i + j * ld] : 0.0;
}
__global__ void k_dense_to_slots(int n0, const double* __restrict__ S, const int* __restrict__ cp,
                                 double shift, double* kv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i < n0 && i >= j)
    kv[cp[j] + (i - j)] = S[i + static_cast<size_t>(j) * n0] + (i == j ? shift : 0.0);
}

class SchurSystem {
 public:
  SchurSystem(KktPlan plan, const ncl_kkt_opts& opt) : ks_(std::move(plan), opt), opt_(opt) {
    n0_ = ks_.ldl().schur_n0();
    if (n0_ <= 0) throw std::invalid_argument("schur: no coupling variables");
    LowerCsc D;
    D.n = n0_;
    D.col_ptr.assign(static_cast<size_t>(n0_) + 1, 0);
    for (int j = 0; j < n0_; ++j) {
      for (int i = j; i < n0_; ++i) D.row_ind.push_back(i);
      D.col_ptr[j + 1] = static_cast<int>(D.row_ind.size());
    }
    std::vector<int> id(static_cast<size_t>(n0_));
    for (int i = 0; i < n0_; ++i) id[i] = i;
    dense_ = std::make_unique<LdlSystem>(D, analyze_with_permutation(D, id), ks_.stream());
    dcp_.upload(D.col_ptr);
    dkval_.alloc(static_cast<size_t>(D.nnz()));
    norm_.alloc(2);
    CK(cudaStreamSynchronize(ks_.stream()));
  }
  KktSystem& kkt() { return ks_; }
  int n0() const { return n0_; }
  cudaStream_t stream() { return ks_.stream(); }

  // refill + local factorization; stats4 = n_pos, n_neg, perturbed, fail of
  // the block pivots; S (device, n0 x n0, lower filled, upper zero)
  void factor(const double* hv, const double* jv, const double* sg, double rho, double delta,
              int* stats4, double* S) {
    cudaStream_t st = stream();
    ks_.refill_async(hv, jv, sg, rho, delta);
    ks_.ldl().factorize_async(ks_.kval(), opt_.pivot_eps);
    const size_t ld = wide_ld(n0_);
    k_front_to_dense<<<dim3((n0_ + 127) / 128, n0_), 128, 0, st>>>(n0_, ld, ks_.ldl().schur_front(),
                                                                    S);
    const FactorInfo F = ks_.ldl().read_factor_info();  // synchronises
    stats4[0] = F.n_pos;
    stats4[1] = F.n_neg;
    stats4[2] = F.perturbed;
    stats4[3] = F.ok ? 0 : 1;
  }
  void factor_dense(const double* S, double shift, int* stats4) {
    cudaStream_t st = stream();
    k_dense_to_slots<<<dim3((n0_ + 127) / 128, n0_), 128, 0, st>>>(n0_, S, dcp_.p, shift,
                                                                    dkval_.p);
    dense_->factorize_async(dkval_.p, opt_.pivot_eps);
    const FactorInfo F = dense_->read_factor_info();
    stats4[0] = F.n_pos;
    stats4[1] = F.n_neg;
    stats4[2] = F.perturbed;
    stats4[3] = F.ok ? 0 : 1;
  }
  void forward(const double* b, double* b0) {
    ks_.ldl().solve_fwd_async(b);
    CK(cudaMemcpyAsync(b0, ks_.ldl().w_tail(), sizeof(double) * n0_, cudaMemcpyDeviceToDevice,
                       stream()));
    CK(cudaStreamSynchronize(stream()));
  }
  void solve0(const double* b0, double* x0) {
    dense_->solve_async(b0, x0);
    CK(cudaStreamSynchronize(stream()));
  }
  void backward(const double* x0, double* x) {
    CK(cudaMemcpyAsync(ks_.ldl().x_tail(), x0, sizeof(double) * n0_, cudaMemcpyDeviceToDevice,
                       stream()));
    ks_.ldl().solve_bwd_async(x);
    CK(cudaStreamSynchronize(stream()));
  }
  // r = b - K_g x (local matrix of the last refill)
  void residual(const double* x, const double* b, double* r) {
    CK(cudaMemsetAsync(norm_.p, 0, sizeof(double), stream()));
    ks_.ldl().residual_async(ks_.kval(), x, b, r, norm_.p);
    CK(cudaStreamSynchronize(stream()));
  }
  void rhs(const double* jv, const double* sg, const double* r1, const double* r2, const double* r3,
           double rho, double delta, double* b) {
    ks_.rhs_async(jv, sg, r1, r2, r3, rho, delta, b);
    CK(cudaStreamSynchronize(stream()));
  }
  void recover(const double* jv, const double* sol, const double* r2, double rho, double delta,
               double* dx, double* dr, double* dy) {
    ks_.recover_async(jv, sol, r2, rho, delta, dx, dr, dy);
    CK(cudaStreamSynchronize(stream()));
  }
  long long launches() { return ks_.launches() + dense_->launches(); }

 private:
  KktSystem ks_;
  ncl_kkt_opts opt_;
  int n0_ = 0;
  std::unique_ptr<LdlSystem> dense_;
  DBuf<int> dcp_;
  DBuf<double> dkval_, norm_;
};


// ---------------------------------------------------------------------------
// plain sparse system (sparse.hpp API on the device LDL^T)
class SparseSystem {
 public:
  SparseSystem(int n, const std::vector<int>& rows, const std::vector<int>& cols,
               const std::vector<double>& vals, const int* perm) {
    std::vector<int> slot;
    K_ = sym_lower_from_pattern(n, rows, cols, &slot);
    // values summed in sorted (stable) order like sym_from_triplets
    std::vector<int> order(rows.size());
    for (size_t k = 0; k < order.size(); ++k) order[k] = static_cast<int>(k);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return slot[a] < slot[b]; });
    val_.assign(static_cast<size_t>(K_.nnz()), 0.0);
    std::vector<char> seen(static_cast<size_t>(K_.nnz()), 0);
    for (int k : order) {
      if (!seen[slot[k]]) {
        val_[slot[k]] = vals[k];
        seen[slot[k]] = 1;
      } else {
        val_[slot[k]] += vals[k];
      }
    }
    std::vector<int> pm = perm ? std::vector<int>(perm, perm + n) : amd_order(K_);
    S_ = analyze_with_permutation(K_, pm);
    CK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    ldl_ = std::make_unique<LdlSystem>(K_, S_, st_);
    kval_.upload(val_);
    b_.alloc(static_cast<size_t>(n));
    x_.alloc(static_cast<size_t>(n));
  }
  ~SparseSystem() {
    ldl_.reset();
    if (st_) cudaStreamDestroy(st_);
  }
  LdlSystem& ldl() { return *ldl_; }
  const LowerCsc& K() const { return K_; }
  const std::vector<double>& val() const { return val_; }
  FactorInfo factorize(double eps) {
    ldl_->factorize_async(kval_.p, eps);
    return ldl_->read_factor_info();
  }
  void solve(const double* b, double* x) {
    const int n = K_.n;
    if (!n) return;
    CK(cudaMemcpyAsync(b_.p, b, sizeof(double) * n, cudaMemcpyHostToDevice, st_));
    ldl_->solve_async(b_.p, x_.p);
    CK(cudaMemcpyAsync(x, x_.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
  }
  int solve_refined(const double* b, int max_ref, double tol, double* x, double* rel,
                    int* conv) {
    const int n = K_.n;
    if (!n) {
      if (rel) *rel = 0.0;
      if (conv) *conv = 1;
      return 0;
    }
    CK(cudaMemcpyAsync(b_.p, b, sizeof(double) * n, cudaMemcpyHostToDevice, st_));
    const int steps = ldl_->solve_refined(kval_.p, b_.p, max_ref, tol, x_.p, rel, conv);
    CK(cudaMemcpyAsync(x, x_.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    return steps;
  }
  const Symbolic& sym() const { return S_; }

 private:
  LowerCsc K_;
  Symbolic S_;
  std::vector<double> val_;
  cudaStream_t st_ = nullptr;
  std::unique_ptr<LdlSystem> ldl_;
  DBuf<double> kval_, b_, x_;
};

// ---------------------------------------------------------------------------
// init_multipliers (solver.cpp:43-91) without the O(m^2) row-pair loop: the
// candidate pairs are the rows that share a Jacobian column (host, once per
// pattern), their dots run on the device one pair per thread with the
// reference's ascending-column merge and separate rounding of every product
// and sum (__dmul_rn/__dadd_rn: bit-identical to the -ffp-contract=off
// reference), exact-zero dots are dropped as the reference drops them, and
// the system goes through the same static-pivot LDL^T (eps 1e-14, no
// refinement, sparse.cpp:182-276) on the device.
__global__ void k_jjt_dots(long long npairs, const int* __restrict__ pi, const int* __restrict__ pj,
                           const int* __restrict__ jp_ptr, const int* __restrict__ jp_idx,
                           const double* __restrict__ jv, int m_eq, double* out) {
  const long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (q >= npairs) return;
  const int i = pi[q], j = pj[q];
  double dot = 0.0;
  int pa = jp_ptr[i], pb = jp_ptr[j];
  const int ea = jp_ptr[i + 1], eb = jp_ptr[j + 1];
  while (pa < ea && pb < eb) {
    const int ca = jp_idx[pa], cb = jp_idx[pb];
    if (ca < cb) {
      ++pa;
    } else if (ca > cb) {
      ++pb;
    } else {
      dot = __dadd_rn(dot, __dmul_rn(jv[pa], jv[pb]));
      ++pa;
      ++pb;
    }
  }
  if (i == j) {
    if (i >= m_eq) dot = __dadd_rn(dot, 1.0);  // slack column
    dot = __dadd_rn(dot, 1e-8);
  }
  out[q] = dot;
}

// rows sharing a column with row i, j <= i, ascending (rows of J^T merged)
void jjt_candidates(int m, int nt, const int* jp_ptr, const int* jp_idx, std::vector<int>& pi,
                    std::vector<int>& pj) {
  std::vector<int> cnt(static_cast<size_t>(nt) + 1, 0);
  for (int p = 0; p < jp_ptr[m]; ++p) cnt[jp_idx[p] + 1]++;
  for (int c = 0; c < nt; ++c) cnt[c + 1] += cnt[c];
  std::vector<int> rows(static_cast<size_t>(cnt[nt]));
  std::vector<int> nx(cnt.begin(), cnt.end() - 1);
  for (int i = 0; i < m; ++i)
    for (int p = jp_ptr[i]; p < jp_ptr[i + 1]; ++p) rows[nx[jp_idx[p]]++] = i;
  std::vector<int> mark(static_cast<size_t>(m), -1), tmp;
  pi.clear();
  pj.clear();
  for (int i = 0; i < m; ++i) {
    tmp.clear();
    mark[i] = i;
    tmp.push_back(i);  // the diagonal is always kept
    for (int p = jp_ptr[i]; p < jp_ptr[i + 1]; ++p) {
      const int c = jp_idx[p];
      for (int q = cnt[c]; q < cnt[c + 1]; ++q) {
        const int j = rows[q];
        if (j > i) break;  // rows of a column ascend
        if (mark[j] != i) {
          mark[j] = i;
          tmp.push_back(j);
        }
      }
    }
    std::sort(tmp.begin(), tmp.end());
    for (int j : tmp) {
      pi.push_back(i);
      pj.push_back(j);
    }
  }
}

struct InitMultipliersTiming {
  double pairs = 0, dots = 0, symbolic = 0, numeric = 0;
};

void init_multipliers(int m, int m_eq, int nt, const int* jp_ptr, const int* jp_idx,
                      const double* jv, const double* g, double* y, InitMultipliersTiming* tm) {
  using clk = std::chrono::steady_clock;
  auto secs = [](clk::time_point a, clk::time_point b) {
    return std::chrono::duration<double>(b - a).count();
  };
  if (m == 0) return;
  const auto t0 = clk::now();
  std::vector<int> pi, pj;
  jjt_candidates(m, nt, jp_ptr, jp_idx, pi, pj);
  const auto t1 = clk::now();
  const long long np = static_cast<long long>(pi.size());
  const int nnzj = jp_ptr[m];
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  std::vector<double> dots(static_cast<size_t>(np));
  {
    DBuf<int> dpi, dpj, dptr, didx;
    DBuf<double> djv, dout;
    dpi.upload(pi);
    dpj.upload(pj);
    dptr.upload(std::vector<int>(jp_ptr, jp_ptr + m + 1));
    didx.upload(std::vector<int>(jp_idx, jp_idx + nnzj));
    djv.upload(std::vector<double>(jv, jv + nnzj));
    dout.alloc(static_cast<size_t>(np));
    k_jjt_dots<<<static_cast<unsigned>((np + 255) / 256), 256, 0, st>>>(np, dpi.p, dpj.p, dptr.p, didx.p,
                                                                       djv.p, m_eq, dout.p);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(dots.data(), dout.p, sizeof(double) * np, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  CK(cudaStreamDestroy(st));
  std::vector<int> rows, cols;
  std::vector<double> vals;
  for (long long q = 0; q < np; ++q)
    if (pi[q] == pj[q] || dots[q] != 0.0) {
      rows.push_back(pi[q]);
      cols.push_back(pj[q]);
      vals.push_back(dots[q]);
    }
  const auto t2 = clk::now();
  SparseSystem A(m, rows, cols, vals, nullptr);
  const auto t3 = clk::now();
  A.factorize(1e-14);
  std::vector<double> rhs(static_cast<size_t>(m), 0.0);
  for (int i = 0; i < m; ++i)
    for (int p = jp_ptr[i]; p < jp_ptr[i + 1]; ++p) rhs[i] += jv[p] * g[jp_idx[p]];
  A.solve(rhs.data(), y);
  for (int i = 0; i < m; ++i) y[i] = std::min(1e3, std::max(-1e3, y[i]));
  const auto t4 = clk::now();
  if (tm) {
    tm->pairs = secs(t0, t1);
    tm->dots = secs(t1, t2);
    tm->symbolic = secs(t2, t3);
    tm->numeric = secs(t3, t4);
  }
}

}  // namespace nclb

// ===========================================================================
// C ABI
struct ncl_kkt {
  std::unique_ptr<nclb::KktSystem> sys;
};
struct ncl_sparse {
  std::unique_ptr<nclb::SparseSystem> sys;
};
struct ncl_schur {
  std::unique_ptr<nclb::SchurSystem> sys;
};
struct ncl_plan {
  nclb::KktPlan plan;
};

namespace {

using nclb::guard;

ncl_kkt_opts default_opts() {
  ncl_kkt_opts o;
  o.pivot_eps = 1e-10;
  o.max_refine = 10;
  o.refine_tol = 1e-12;
  o.delta_max = 1e40;
  o.accept_tol = 1e-8;
  return o;
}

}  // namespace

extern "C" {

const char* ncl_last_error(void) { return nclb::last_error().c_str(); }

int ncl_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int ncl_kkt_create(int nt, const int* hp_ptr, const int* hp_idx, int m, const int* jp_ptr,
                   const int* jp_idx, int ns, int m_eq, int form, const ncl_kkt_opts* opt,
                   ncl_kkt** out) {
  if (!out || !hp_ptr || !jp_ptr) {
    nclb::last_error() = "ncl_kkt_create: null argument";
    return NCL_EINVAL;
  }
  *out = nullptr;
  return guard([&] {
    nclb::KktPlan plan =
        nclb::make_kkt_plan(nt, hp_ptr, hp_idx, m, jp_ptr, jp_idx, ns, m_eq, form, 0, false);
    auto* c = new ncl_kkt;
    try {
      c->sys = std::make_unique<nclb::KktSystem>(std::move(plan), opt ? *opt : default_opts());
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

void ncl_kkt_destroy(ncl_kkt* ctx) { delete ctx; }

int ncl_kkt_solve(ncl_kkt* ctx, const double* hval, const double* jval, const double* sigma,
                  const double* rbar1, const double* rbar2, const double* rbar3, double rho,
                  double warm_delta, double* dx, double* dr, double* dy,
                  ncl_kkt_stats* stats) {
  if (!ctx || !stats) return NCL_EINVAL;
  return guard([&] {
    ctx->sys->solve_host(hval, jval, sigma, rbar1, rbar2, rbar3, rho, warm_delta, dx, dr, dy,
                         stats);
  });
}

int ncl_kkt_solve_device(ncl_kkt* ctx, const double* hval, const double* jval,
                         const double* sigma, const double* rbar1, const double* rbar2,
                         const double* rbar3, double rho, double warm_delta, double* dx,
                         double* dr, double* dy, ncl_kkt_stats* stats) {
  if (!ctx || !stats) return NCL_EINVAL;
  return guard([&] {
    ctx->sys->solve_device(hval, jval, sigma, rbar1, rbar2, rbar3, rho, warm_delta, dx, dr, dy,
                           stats);
  });
}

int ncl_kkt_info_get(const ncl_kkt* ctx, ncl_kkt_info* info) {
  if (!ctx || !info) return NCL_EINVAL;
  const auto& P = ctx->sys->plan();
  const auto& T = ctx->sys->ldl().sn();
  info->n = P.N;
  info->nnz = P.K.nnz();
  info->l_nnz = P.sym.l_nnz();
  info->flops = T.flops;
  info->n_supernodes = T.nsn;
  info->sn_height = T.sn_height;
  info->n_paths = static_cast<int>(T.path_ptr.size()) - 1;
  info->n_wide = static_cast<int>(T.lvl_nodes.size());
  info->n_levels = static_cast<int>(T.lvl_ptr.size()) - 1;
  info->max_front = T.max_f;
  info->npairs = static_cast<long long>(P.pair_slot.size());
  return NCL_OK;
}

int ncl_kkt_inertia_target(const ncl_kkt* ctx, int* tgt3) {
  if (!ctx || !tgt3) return NCL_EINVAL;
  for (int i = 0; i < 3; ++i) tgt3[i] = ctx->sys->plan().inertia_target[i];
  return NCL_OK;
}

int ncl_kkt_symbolic(const ncl_kkt* ctx, int* perm, int* parent, int* lcol_ptr) {
  if (!ctx) return NCL_EINVAL;
  const auto& S = ctx->sys->plan().sym;
  if (perm) std::copy(S.perm.begin(), S.perm.end(), perm);
  if (parent) std::copy(S.parent.begin(), S.parent.end(), parent);
  if (lcol_ptr) std::copy(S.lcol_ptr.begin(), S.lcol_ptr.end(), lcol_ptr);
  return NCL_OK;
}

int ncl_kkt_matrix(const ncl_kkt* ctx, int* col_ptr, int* row_ind, double* val) {
  if (!ctx) return NCL_EINVAL;
  return guard([&] { ctx->sys->matrix(col_ptr, row_ind, val); });
}

int ncl_kkt_refill(ncl_kkt* ctx, const double* hval, const double* jval, const double* sigma,
                   double rho, double delta) {
  if (!ctx) return NCL_EINVAL;
  return guard([&] {
    ctx->sys->refill_host(hval, jval, sigma, rho, delta);
  });
}

int ncl_kkt_factors(const ncl_kkt* ctx, int* lcol_ptr, int* lrow_ind, double* lval, double* d,
                    int* info4) {
  if (!ctx) return NCL_EINVAL;
  return guard([&] {
    auto& L = ctx->sys->ldl();
    L.factors_host(lcol_ptr, lrow_ind, lval, d);
    if (info4) {
      nclb::Scalars* hs = L.host_scalars();
      CK(cudaMemcpy(hs, L.dev_scalars(), sizeof(nclb::Scalars), cudaMemcpyDeviceToHost));
      info4[0] = hs->stats[3] == 0;
      info4[1] = hs->stats[0];
      info4[2] = hs->stats[1];
      info4[3] = hs->stats[2];
    }
  });
}

int ncl_kkt_last_timing(const ncl_kkt* ctx, double* ms6) {
  if (!ctx || !ms6) return NCL_EINVAL;
  ctx->sys->timing(ms6);
  return NCL_OK;
}

int ncl_kkt_get_stream(const ncl_kkt* ctx, void** stream) {
  if (!ctx || !stream) return NCL_EINVAL;
  *stream = static_cast<void*>(ctx->sys->stream());
  return NCL_OK;
}

int ncl_kkt_launch_count(const ncl_kkt* ctx, long long* count) {
  if (!ctx || !count) return NCL_EINVAL;
  *count = ctx->sys->launches();
  return NCL_OK;
}

int ncl_kkt_set_timing(ncl_kkt* ctx, int enable) {
  if (!ctx) return NCL_EINVAL;
  ctx->sys->set_timing(enable != 0);
  return NCL_OK;
}

// ---- host-only plan ---------------------------------------------------------
int ncl_plan_create(int nt, const int* hp_ptr, const int* hp_idx, int m, const int* jp_ptr,
                    const int* jp_idx, int ns, int m_eq, int form, ncl_plan** out) {
  if (!out || !hp_ptr || !jp_ptr) return NCL_EINVAL;
  *out = nullptr;
  return guard([&] {
    auto* p = new ncl_plan;
    try {
      p->plan = nclb::make_kkt_plan(nt, hp_ptr, hp_idx, m, jp_ptr, jp_idx, ns, m_eq, form);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

void ncl_plan_destroy(ncl_plan* plan) { delete plan; }

int ncl_plan_info(const ncl_plan* plan, ncl_kkt_info* info) {
  if (!plan || !info) return NCL_EINVAL;
  const auto& P = plan->plan;
  const auto& T = P.sn;
  info->n = P.N;
  info->nnz = P.K.nnz();
  info->l_nnz = P.sym.l_nnz();
  info->flops = T.flops;
  info->n_supernodes = T.nsn;
  info->sn_height = T.sn_height;
  info->n_paths = static_cast<int>(T.path_ptr.size()) - 1;
  info->n_wide = static_cast<int>(T.lvl_nodes.size());
  info->n_levels = static_cast<int>(T.lvl_ptr.size()) - 1;
  info->max_front = T.max_f;
  info->npairs = static_cast<long long>(P.pair_slot.size());
  return NCL_OK;
}

int ncl_plan_symbolic(const ncl_plan* plan, int* perm, int* parent, int* lcol_ptr) {
  if (!plan) return NCL_EINVAL;
  const auto& S = plan->plan.sym;
  if (perm) std::copy(S.perm.begin(), S.perm.end(), perm);
  if (parent) std::copy(S.parent.begin(), S.parent.end(), parent);
  if (lcol_ptr) std::copy(S.lcol_ptr.begin(), S.lcol_ptr.end(), lcol_ptr);
  return NCL_OK;
}

int ncl_plan_pattern(const ncl_plan* plan, int* col_ptr, int* row_ind) {
  if (!plan) return NCL_EINVAL;
  const auto& K = plan->plan.K;
  if (col_ptr) std::copy(K.col_ptr.begin(), K.col_ptr.end(), col_ptr);
  if (row_ind) std::copy(K.row_ind.begin(), K.row_ind.end(), row_ind);
  return NCL_OK;
}

int ncl_plan_check_schedule(const ncl_plan* plan, int internal) {
  if (!plan) return NCL_EINVAL;
  return guard([&] {
    const auto& P = plan->plan;
    const int n0 = P.sn.schur >= 0 ? P.N - P.sn.first[P.sn.schur] : 0;
    std::string err;
    if (internal) {  // the structure LdlSystem factors (context.cu: LdlSystem::LdlSystem)
      const nclb::Symbolic S2 = nclb::analyze_with_permutation(P.K, nclb::tallest_child_last(P.K, P.sym.perm));
      err = nclb::check_warp_schedule(nclb::build_supernodal(P.K, S2, n0));
    } else {
      err = nclb::check_warp_schedule(P.sn);
    }
    if (!err.empty()) throw std::logic_error("warp schedule: " + err);
  });
}

int ncl_plan_check_dag(const ncl_plan* plan, int workers, double* stats4) {
  if (!plan || workers < 1) return NCL_EINVAL;
  return guard([&] {
    const auto& P = plan->plan;
    const int n0 = P.sn.schur >= 0 ? P.N - P.sn.first[P.sn.schur] : 0;
    const nclb::Symbolic S2 = nclb::analyze_with_permutation(P.K, nclb::tallest_child_last(P.K, P.sym.perm));
    const nclb::Supernodal T = nclb::build_supernodal(P.K, S2, n0);
    double st[4] = {0, 0, 0, 0};
    for (const auto& run : nclb::dag_level_runs(T, nclb::small_factor_limit())) {
      const nclb::DagSegment G = nclb::build_dag_segment(T, run[0], run[1], workers);
      const std::string err = nclb::check_dag_segment(T, G);
      if (!err.empty()) throw std::logic_error("dag schedule: " + err);
      st[0] += 1;
      st[1] += static_cast<double>(G.tasks.size());
      st[2] += G.makespan_us;
      st[3] += G.crit_us;
    }
    if (stats4) std::copy(st, st + 4, stats4);
  });
}

int ncl_amd_full_pattern(int n, const int* Ap, const int* Ai, int* perm) {
  if (n < 0 || !Ap || !perm) return NCL_EINVAL;
  return guard([&] {
    const std::vector<int> p = nclb::amd_full_pattern(
        n, std::vector<int>(Ap, Ap + n + 1), std::vector<int>(Ai, Ai + Ap[n]));
    std::copy(p.begin(), p.end(), perm);
  });
}

int ncl_analyze_host(int n, int ntrip, const int* rows, const int* cols, const int* perm_in,
                     int* perm, int* parent, int* lcol_ptr) {
  if (n < 0 || ntrip < 0) return NCL_EINVAL;
  return guard([&] {
    const nclb::LowerCsc K = nclb::sym_lower_from_pattern(
        n, std::vector<int>(rows, rows + ntrip), std::vector<int>(cols, cols + ntrip));
    const std::vector<int> pm =
        perm_in ? std::vector<int>(perm_in, perm_in + n) : nclb::amd_order(K);
    const nclb::Symbolic S = nclb::analyze_with_permutation(K, pm);
    if (perm) std::copy(S.perm.begin(), S.perm.end(), perm);
    if (parent) std::copy(S.parent.begin(), S.parent.end(), parent);
    if (lcol_ptr) std::copy(S.lcol_ptr.begin(), S.lcol_ptr.end(), lcol_ptr);
  });
}

// ---- sparse layer ---------------------------------------------------------
int ncl_sparse_create(int n, int ntrip, const int* rows, const int* cols, const double* vals,
                      const int* perm, ncl_sparse** out) {
  if (!out || n < 0 || ntrip < 0) return NCL_EINVAL;
  *out = nullptr;
  return guard([&] {
    std::vector<int> r(rows, rows + ntrip), c(cols, cols + ntrip);
    std::vector<double> v(vals, vals + ntrip);
    auto* s = new ncl_sparse;
    try {
      s->sys = std::make_unique<nclb::SparseSystem>(n, r, c, v, perm);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

void ncl_sparse_destroy(ncl_sparse* sp) { delete sp; }

int ncl_sparse_nnz(const ncl_sparse* sp, int* nnz, long long* l_nnz) {
  if (!sp) return NCL_EINVAL;
  if (nnz) *nnz = sp->sys->K().nnz();
  if (l_nnz) *l_nnz = sp->sys->sym().l_nnz();
  return NCL_OK;
}

int ncl_sparse_symbolic(const ncl_sparse* sp, int* perm, int* parent, int* lcol_ptr) {
  if (!sp) return NCL_EINVAL;
  const auto& S = sp->sys->sym();
  if (perm) std::copy(S.perm.begin(), S.perm.end(), perm);
  if (parent) std::copy(S.parent.begin(), S.parent.end(), parent);
  if (lcol_ptr) std::copy(S.lcol_ptr.begin(), S.lcol_ptr.end(), lcol_ptr);
  return NCL_OK;
}

int ncl_sparse_factorize(ncl_sparse* sp, double pivot_eps, int* info4) {
  if (!sp) return NCL_EINVAL;
  return guard([&] {
    const nclb::FactorInfo fi = sp->sys->factorize(pivot_eps);
    if (info4) {
      info4[0] = fi.ok;
      info4[1] = fi.n_pos;
      info4[2] = fi.n_neg;
      info4[3] = fi.perturbed;
    }
  });
}

int ncl_sparse_factors(const ncl_sparse* sp, int* lcol_ptr, int* lrow_ind, double* lval,
                       double* d) {
  if (!sp) return NCL_EINVAL;
  return guard([&] { sp->sys->ldl().factors_host(lcol_ptr, lrow_ind, lval, d); });
}

int ncl_sparse_ldl_solve(ncl_sparse* sp, const double* b, double* x) {
  if (!sp) return NCL_EINVAL;
  return guard([&] { sp->sys->solve(b, x); });
}

int ncl_sparse_solve_refined(ncl_sparse* sp, const double* b, int max_ref, double tol,
                             double* x, int* steps, double* rel_residual, int* converged) {
  if (!sp) return NCL_EINVAL;
  return guard([&] {
    const int s = sp->sys->solve_refined(b, max_ref, tol, x, rel_residual, converged);
    if (steps) *steps = s;
  });
}

int ncl_sparse_matvec(ncl_sparse* sp, const double* x, double* y) {
  if (!sp) return NCL_EINVAL;
  const auto& K = sp->sys->K();
  const auto& v = sp->sys->val();
  for (int j = 0; j < K.n; ++j)
    for (int p = K.col_ptr[j]; p < K.col_ptr[j + 1]; ++p) {
      const int i = K.row_ind[p];
      y[i] += v[p] * x[j];
      if (i != j) y[j] += v[p] * x[i];
    }
  return NCL_OK;
}

/* ---- Schur mode (block-arrowhead sub-problems) ---------- */
int ncl_schur_create(int nt, const int* hp_ptr, const int* hp_idx, int m, const int* jp_ptr,
                     const int* jp_idx, int ns, int m_eq, int n0, const ncl_kkt_opts* opt,
                     ncl_schur** out) {
  if (!out || !hp_ptr || !jp_ptr || n0 <= 0) {
    nclb::last_error() = "ncl_schur_create: invalid argument";
    return NCL_EINVAL;
  }
  *out = nullptr;
  return guard([&] {
    nclb::KktPlan plan = nclb::make_kkt_plan(nt, hp_ptr, hp_idx, m, jp_ptr, jp_idx, ns, m_eq,
                                             nclb::kK1s, n0);
    auto* c = new ncl_schur;
    try {
      c->sys = std::make_unique<nclb::SchurSystem>(std::move(plan), opt ? *opt : default_opts());
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

void ncl_schur_destroy(ncl_schur* h) { delete h; }

int ncl_schur_info(const ncl_schur* h, ncl_kkt_info* info) {
  if (!h || !info) return NCL_EINVAL;
  auto& K = h->sys->kkt();
  const auto& P = K.plan();
  const auto& T = K.ldl().sn();
  info->n = P.N;
  info->nnz = P.K.nnz();
  info->l_nnz = P.sym.l_nnz();
  info->flops = T.flops;
  info->n_supernodes = T.nsn;
  info->sn_height = T.sn_height;
  info->n_paths = static_cast<int>(T.path_ptr.size()) - 1;
  info->n_wide = static_cast<int>(T.lvl_nodes.size());
  info->n_levels = static_cast<int>(T.lvl_ptr.size()) - 1;
  info->max_front = T.max_f;
  info->npairs = static_cast<long long>(P.pair_slot.size());
  return NCL_OK;
}

int ncl_schur_n0(const ncl_schur* h) { return h ? h->sys->n0() : NCL_EINVAL; }

int ncl_schur_factor(ncl_schur* h, const double* hval, const double* jval, const double* sigma,
                     double rho, double delta, int* stats4, double* S) {
  if (!h || !stats4 || !S) return NCL_EINVAL;
  return guard([&] { h->sys->factor(hval, jval, sigma, rho, delta, stats4, S); });
}

int ncl_schur_factor_dense(ncl_schur* h, const double* S, double diag_shift, int* stats4) {
  if (!h || !stats4 || !S) return NCL_EINVAL;
  return guard([&] { h->sys->factor_dense(S, diag_shift, stats4); });
}

int ncl_schur_rhs(ncl_schur* h, const double* jval, const double* sigma, const double* rbar1,
                  const double* rbar2, const double* rbar3, double rho, double delta, double* b) {
  if (!h || !b) return NCL_EINVAL;
  return guard([&] { h->sys->rhs(jval, sigma, rbar1, rbar2, rbar3, rho, delta, b); });
}

int ncl_schur_forward(ncl_schur* h, const double* b, double* b0) {
  if (!h || !b || !b0) return NCL_EINVAL;
  return guard([&] { h->sys->forward(b, b0); });
}

int ncl_schur_solve0(ncl_schur* h, const double* b0, double* x0) {
  if (!h || !b0 || !x0) return NCL_EINVAL;
  return guard([&] { h->sys->solve0(b0, x0); });
}

int ncl_schur_backward(ncl_schur* h, const double* x0, double* x) {
  if (!h || !x0 || !x) return NCL_EINVAL;
  return guard([&] { h->sys->backward(x0, x); });
}

int ncl_schur_residual(ncl_schur* h, const double* x, const double* b, double* r) {
  if (!h || !x || !b || !r) return NCL_EINVAL;
  return guard([&] { h->sys->residual(x, b, r); });
}

int ncl_schur_recover(ncl_schur* h, const double* jval, const double* sol, const double* rbar2,
                      double rho, double delta, double* dx, double* dr, double* dy) {
  if (!h || !sol) return NCL_EINVAL;
  return guard([&] { h->sys->recover(jval, sol, rbar2, rho, delta, dx, dr, dy); });
}

int ncl_schur_launch_count(const ncl_schur* h, long long* count) {
  if (!h || !count) return NCL_EINVAL;
  *count = h->sys->launches();
  return NCL_OK;
}


/* ---- init_multipliers (solver.cpp:43-91) --------------------------------- */
int ncl_init_multipliers(int m, int m_eq, int nt, const int* jp_ptr, const int* jp_idx,
                         const double* jval, const double* grad, double* y, double* seconds4) {
  if (m < 0 || m_eq < 0 || m_eq > m || (m > 0 && (!jp_ptr || !y))) return NCL_EINVAL;
  return guard([&] {
    nclb::InitMultipliersTiming tm;
    nclb::init_multipliers(m, m_eq, nt, jp_ptr, jp_idx, jval, grad, y, &tm);
    if (seconds4) {
      seconds4[0] = tm.pairs;
      seconds4[1] = tm.dots;
      seconds4[2] = tm.symbolic;
      seconds4[3] = tm.numeric;
    }
  });
}

int ncl_jjt_candidates(int m, int nt, const int* jp_ptr, const int* jp_idx, long long cap,
                       long long* count, int* pi, int* pj) {
  if (!jp_ptr || !count || m < 0) return NCL_EINVAL;
  return guard([&] {
    std::vector<int> a, b;
    nclb::jjt_candidates(m, nt, jp_ptr, jp_idx, a, b);
    *count = static_cast<long long>(a.size());
    if (pi && pj && cap >= *count) {
      std::copy(a.begin(), a.end(), pi);
      std::copy(b.begin(), b.end(), pj);
    }
  });
}

}  // extern "C"
