// Tile-dataflow schedule of the wide-front tier: task graph + list
// scheduling (see dag.hpp).
#include "dag.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <queue>
#include <string>

#include "layout.hpp"

namespace nclb {

namespace {

// cost model (us), calibrated on the B200 with NCL_DAG_TRACE: a 32-pivot
// diagonal tile is a dependent chain; TRSM / UPD / ASM are dominated by
// their L2 round trips; a dependency between two workers costs a flag hop
struct Cost {
  double diag0 = 0.8, diag_per = 0.16, trsm = 1.6, upd = 1.2, asm0 = 1.2, asm_per = 0.002,
         hop = 1.0;
  Cost() {
    if (const char* e = std::getenv("NCL_DAG_COST")) {  // diag0,diag_per,trsm,upd,asm0,hop
      std::sscanf(e, "%lf,%lf,%lf,%lf,%lf,%lf", &diag0, &diag_per, &trsm, &upd, &asm0, &hop);
    }
  }
};

struct Task {
  int fr, type, i, j, p;
};

inline int tri(int i, int j) { return i * (i + 1) / 2 + j; }

}  // namespace

DagSegment build_dag_segment(const Supernodal& T, int l0, int l1, int workers) {
  const Cost C;
  DagSegment G;
  G.l0 = l0;
  G.l1 = l1;
  G.workers = workers;
  // fronts in level order (children before parents)
  std::vector<int> loc(static_cast<size_t>(T.nsn), -1);
  for (int q = T.lvl_ptr[l0]; q < T.lvl_ptr[l1]; ++q) {
    const int s = T.lvl_nodes[q];
    DagFront F{};
    F.s = s;
    F.loff = T.l_off[s];
    F.c0 = T.first[s];
    F.k = T.first[s + 1] - T.first[s];
    F.f = T.f[s];
    F.P = (F.k + 31) / 32;
    const int NT = (F.f - F.k + 31) / 32;
    F.NB = F.P + NT;
    F.st_off = G.nstate;
    G.nstate += F.NB * (F.NB + 1) / 2;
    F.ntrail = NT * (NT + 1) / 2;
    F.scr_off = G.nscr;
    G.nscr += F.P;
    loc[s] = static_cast<int>(G.fronts.size());
    G.fronts.push_back(F);
  }
  for (auto& F : G.fronts) {
    F.ch_b = static_cast<int>(G.ch.size());
    for (int q = T.ch_ptr[F.s]; q < T.ch_ptr[F.s + 1]; ++q)
      if (loc[T.ch[q]] >= 0) G.ch.push_back(loc[T.ch[q]]);
    F.ch_e = static_cast<int>(G.ch.size());
  }
  // tasks in a topological order: fronts children first; per front all ASM,
  // then per panel DIAG, TRSMs, UPDs
  std::vector<Task> tk;
  std::vector<int> base(G.fronts.size());  // first task of each front
  for (int fi = 0; fi < static_cast<int>(G.fronts.size()); ++fi) {
    const DagFront& F = G.fronts[fi];
    base[fi] = static_cast<int>(tk.size());
    for (int jb = 0; jb < F.NB; ++jb) tk.push_back({fi, kDagAsm, 0, jb, 0});
    for (int p = 0; p < F.P; ++p) {
      tk.push_back({fi, kDagDiag, p, p, p});
      for (int i = p + 1; i < F.NB; ++i) tk.push_back({fi, kDagTrsm, i, p, p});
      for (int j = p + 1; j < F.NB; ++j)
        for (int i = j; i < F.NB; ++i) tk.push_back({fi, kDagUpd, i, j, p});
    }
  }
  const int nt = static_cast<int>(tk.size());
  // task id lookups (per front, computed from the generation order)
  auto panel_base = [&](const DagFront& F, int fi, int p) {
    // tasks of panels < p: per panel q: 1 + (NB-q-1) + (NB-q-1)(NB-q)/2
    int b = base[fi] + F.NB;
    for (int q = 0; q < p; ++q) {
      const int r = F.NB - q - 1;
      b += 1 + r + r * (r + 1) / 2;
    }
    return b;
  };
  // per front, per panel base ids
  std::vector<std::vector<int>> pb(G.fronts.size());
  for (int fi = 0; fi < static_cast<int>(G.fronts.size()); ++fi) {
    const DagFront& F = G.fronts[fi];
    pb[fi].resize(static_cast<size_t>(F.P) + 1);
    for (int p = 0; p <= F.P; ++p) pb[fi][p] = panel_base(F, fi, p);
  }
  auto id_asm = [&](int fi, int jb) { return base[fi] + jb; };
  auto id_diag = [&](int fi, int p) { return pb[fi][p]; };
  auto id_trsm = [&](int fi, int i, int p) { return pb[fi][p] + 1 + (i - p - 1); };
  auto id_upd = [&](int fi, int i, int j, int p) {
    const DagFront& F = G.fronts[fi];
    const int r = F.NB - p - 1;
    // columns j = p+1.. in order, rows i = j..NB-1
    int off = 0;
    for (int jj = p + 1; jj < j; ++jj) off += F.NB - jj;
    return pb[fi][p] + 1 + r + off + (i - j);
  };
  auto id_lready = [&](int fi, int i, int p) { return i == p ? id_diag(fi, p) : id_trsm(fi, i, p); };
  // dependencies
  std::vector<int> dptr(static_cast<size_t>(nt) + 1, 0);
  std::vector<int> dep;
  std::vector<int> final_upd;  // per front: ids of the trailing tiles' last updates
  std::vector<int> fu_ptr(G.fronts.size() + 1, 0);
  for (int fi = 0; fi < static_cast<int>(G.fronts.size()); ++fi) {
    const DagFront& F = G.fronts[fi];
    for (int j = F.P; j < F.NB; ++j)
      for (int i = j; i < F.NB; ++i) final_upd.push_back(id_upd(fi, i, j, F.P - 1));
    fu_ptr[fi + 1] = static_cast<int>(final_upd.size());
  }
  for (int t = 0; t < nt; ++t) {
    const Task& a = tk[t];
    const DagFront& F = G.fronts[a.fr];
    switch (a.type) {
      case kDagAsm:
        for (int q = F.ch_b; q < F.ch_e; ++q) {
          const int c = G.ch[q];
          for (int x = fu_ptr[c]; x < fu_ptr[c + 1]; ++x) dep.push_back(final_upd[x]);
        }
        break;
      case kDagDiag:
        dep.push_back(a.p ? id_upd(a.fr, a.p, a.p, a.p - 1) : id_asm(a.fr, a.p));
        break;
      case kDagTrsm:
        dep.push_back(id_diag(a.fr, a.p));
        dep.push_back(a.p ? id_upd(a.fr, a.i, a.p, a.p - 1) : id_asm(a.fr, a.p));
        break;
      default:
        dep.push_back(id_lready(a.fr, a.i, a.p));
        if (a.j != a.i) dep.push_back(id_lready(a.fr, a.j, a.p));
        dep.push_back(a.p ? id_upd(a.fr, a.i, a.j, a.p - 1) : id_asm(a.fr, a.j));
    }
    dptr[t + 1] = static_cast<int>(dep.size());
  }
  // successors
  std::vector<int> sptr(static_cast<size_t>(nt) + 1, 0), suc(dep.size());
  for (int t = 0; t < nt; ++t)
    for (int q = dptr[t]; q < dptr[t + 1]; ++q) sptr[dep[q] + 1]++;
  for (int t = 0; t < nt; ++t) sptr[t + 1] += sptr[t];
  {
    std::vector<int> nx(sptr.begin(), sptr.end() - 1);
    for (int t = 0; t < nt; ++t)
      for (int q = dptr[t]; q < dptr[t + 1]; ++q) suc[nx[dep[q]]++] = t;
  }
  std::vector<double> cost(static_cast<size_t>(nt));
  for (int t = 0; t < nt; ++t) {
    const Task& a = tk[t];
    const DagFront& F = G.fronts[a.fr];
    switch (a.type) {
      case kDagAsm: {
        const int j0 = dag_block_start(F.k, F.P, a.j), nb = dag_block_size(F.k, F.f, F.P, a.j);
        long long ent = 0;
        const int cb = T.cc_off[F.s];
        for (int J = j0; J < j0 + nb; ++J) ent += T.cc_ptr[cb + J + 1] - T.cc_ptr[cb + J];
        cost[t] = C.asm0 + C.asm_per * static_cast<double>(ent) / 4.0;
        break;
      }
      case kDagDiag:
        cost[t] = C.diag0 + C.diag_per * dag_block_size(F.k, F.f, F.P, a.p);
        break;
      case kDagTrsm:
        cost[t] = C.trsm;
        break;
      default:
        cost[t] = C.upd;
    }
  }
  // upward ranks (generation order is topological: reverse it)
  std::vector<double> rank(static_cast<size_t>(nt), 0.0);
  for (int t = nt - 1; t >= 0; --t) {
    double m = 0.0;
    for (int q = sptr[t]; q < sptr[t + 1]; ++q) m = std::max(m, C.hop + rank[suc[q]]);
    rank[t] = cost[t] + m;
  }
  {  // critical path without flag hops: a lower bound of any schedule
    std::vector<double> r0(static_cast<size_t>(nt), 0.0);
    G.crit_us = 0.0;
    for (int t = nt - 1; t >= 0; --t) {
      double m = 0.0;
      for (int q = sptr[t]; q < sptr[t + 1]; ++q) m = std::max(m, r0[suc[q]]);
      r0[t] = cost[t] + m;
      G.crit_us = std::max(G.crit_us, r0[t]);
    }
  }
  std::vector<int> order(static_cast<size_t>(nt));
  for (int t = 0; t < nt; ++t) order[t] = t;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return rank[a] > rank[b]; });
  // list scheduling: each task on the worker (among the idlest one and its
  // dependencies' workers) where it finishes first
  std::vector<double> wfree(static_cast<size_t>(workers), 0.0), fin(static_cast<size_t>(nt), 0.0),
      start(static_cast<size_t>(nt), 0.0);
  std::vector<int> wk(static_cast<size_t>(nt), -1);
  using QE = std::pair<double, int>;
  std::priority_queue<QE, std::vector<QE>, std::greater<QE>> idle;
  for (int w = 0; w < workers; ++w) idle.push({0.0, w});
  std::vector<std::vector<int>> wl(static_cast<size_t>(workers));
  std::vector<int> cand;
  for (int t : order) {
    while (idle.top().first != wfree[idle.top().second]) idle.pop();  // stale entries
    cand.clear();
    cand.push_back(idle.top().second);
    for (int q = dptr[t]; q < dptr[t + 1]; ++q) cand.push_back(wk[dep[q]]);
    double best = 1e300, bst = 0.0;
    int bw = -1;
    for (int w : cand) {
      double ready = wfree[w];
      for (int q = dptr[t]; q < dptr[t + 1]; ++q) {
        const int d = dep[q];
        ready = std::max(ready, fin[d] + (wk[d] == w ? 0.0 : C.hop));
      }
      if (ready + cost[t] < best || (ready + cost[t] == best && w < bw)) {
        best = ready + cost[t];
        bst = ready;
        bw = w;
      }
    }
    wk[t] = bw;
    start[t] = bst;
    fin[t] = best;
    wfree[bw] = best;
    idle.push({best, bw});
    wl[bw].push_back(t);
  }
  G.makespan_us = 0.0;
  for (int w = 0; w < workers; ++w) G.makespan_us = std::max(G.makespan_us, wfree[w]);
  G.w_ptr.assign(static_cast<size_t>(workers) + 1, 0);
  G.tasks.reserve(static_cast<size_t>(nt));
  for (int w = 0; w < workers; ++w) {
    for (int t : wl[w]) {
      const Task& a = tk[t];
      G.tasks.push_back({a.fr, a.i | a.j << 12 | a.type << 24, a.p,
                         static_cast<int>(std::min(start[t] * 1e3, 2e9))});
    }
    G.w_ptr[w + 1] = static_cast<int>(G.tasks.size());
  }
  return G;
}

std::vector<std::array<int, 2>> dag_level_runs(const Supernodal& T, int small_limit) {
  const int nl = static_cast<int>(T.lvl_ptr.size()) - 1;
  auto ok = [&](int l) {
    int fmax = 0;
    for (int q = T.lvl_ptr[l]; q < T.lvl_ptr[l + 1]; ++q) {
      const int s = T.lvl_nodes[q];
      if (s == T.schur || T.split_ng[s]) return false;
      fmax = std::max(fmax, T.f[s]);
    }
    return fmax > small_limit;
  };
  std::vector<std::array<int, 2>> runs;
  for (int l = 0; l < nl;) {
    if (!ok(l)) {
      ++l;
      continue;
    }
    int e = l + 1;
    while (e < nl && ok(e)) ++e;
    runs.push_back({l, e});
    l = e;
  }
  return runs;
}

std::string check_dag_segment(const Supernodal& T, const DagSegment& G) {
  // replay the worker lists as the device would (a worker runs its next task
  // once the tile states it waits on are reached); every task must run and
  // the states must end where the factorization leaves them
  const int W = G.workers;
  std::vector<int> st(static_cast<size_t>(G.nstate), 0), done(G.fronts.size(), 0);
  std::vector<int> pos(G.w_ptr.begin(), G.w_ptr.end() - 1);
  long long left = static_cast<long long>(G.tasks.size());
  size_t want = 0;
  for (const auto& F : G.fronts) {
    want += static_cast<size_t>(F.NB);  // ASM
    for (int p = 0; p < F.P; ++p) {
      const int r = F.NB - p - 1;
      want += 1 + r + r * (r + 1) / 2;
    }
  }
  if (want != G.tasks.size()) return "task count " + std::to_string(G.tasks.size()) + " != " + std::to_string(want);
  (void)T;
  while (left > 0) {
    bool progress = false;
    for (int w = 0; w < W; ++w) {
      while (pos[w] < G.w_ptr[w + 1]) {
        const auto& t = G.tasks[pos[w]];
        const DagFront& F = G.fronts[t[0]];
        const int i = t[1] & 0xfff, j = (t[1] >> 12) & 0xfff, type = t[1] >> 24, p = t[2];
        auto S = [&](int a, int b) -> int& { return st[F.st_off + tri(a, b)]; };
        bool ok = true;
        switch (type) {
          case kDagAsm:
            for (int q = F.ch_b; q < F.ch_e; ++q)
              ok = ok && done[G.ch[q]] >= G.fronts[G.ch[q]].ntrail;
            break;
          case kDagDiag:
            ok = S(p, p) >= p + 1;
            break;
          case kDagTrsm:
            ok = S(i, p) >= p + 1 && S(p, p) >= p + 2;
            break;
          default:
            ok = S(i, p) >= p + 2 && S(j, p) >= p + 2 && S(i, j) >= p + 1;
        }
        if (!ok) break;
        switch (type) {
          case kDagAsm:
            for (int a = j; a < F.NB; ++a) {
              if (S(a, j) != 0) return "tile assembled twice";
              S(a, j) = 1;
            }
            break;
          case kDagDiag:
          case kDagTrsm:
            if (S(i, p) != p + 1) return "L block computed twice";
            S(i, p) = p + 2;
            break;
          default:
            if (S(i, j) != p + 1) return "update out of panel order";
            S(i, j) = p + 2;
            if (j >= F.P && p == F.P - 1) done[t[0]]++;
        }
        ++pos[w];
        --left;
        progress = true;
      }
    }
    if (!progress) return "deadlock with " + std::to_string(left) + " tasks left";
  }
  for (size_t fi = 0; fi < G.fronts.size(); ++fi) {
    const DagFront& F = G.fronts[fi];
    for (int j = 0; j < F.NB; ++j)
      for (int i = j; i < F.NB; ++i) {
        const int want_st = j < F.P ? j + 2 : F.P + 1;
        if (st[F.st_off + tri(i, j)] != want_st) return "tile state incomplete";
      }
  }
  return "";
}

}  // namespace nclb
