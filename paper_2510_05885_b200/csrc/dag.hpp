// Tile-dataflow schedule of the wide-front tier (host side, built once per
// KKT pattern next to the rest of the symbolic analysis).
//
// A run of consecutive wide levels (a "segment") is factored by ONE
// persistent launch (k_front_dag, wide_kernels.cu): every front is cut into
// 32-row blocks -- pivot blocks [32p, min(32p+32, k)) then trailing blocks
// [k + 32t, ...) -- and factored as a task graph over its lower tiles:
//   ASM(jb)      assemble column block jb (A entries + the children's update
//                matrices, assemble_col); waits for the wide children of the
//                segment to finish
//   DIAG(p)      static-pivot LDL^T of diagonal tile (p, p) (diag_block)
//   TRSM(i, p)   L(i, p) from tile (i, p) and DIAG(p)'s pivots (trsm_rows)
//   UPD(i, j, p) tile (i, j) -= L(i, p) D_p L(j, p)^T on FP64 tensor cores,
//                every tile receiving its panels in panel order
// Tiles carry a state word (0 = not assembled, 1 + updates applied, +1 when
// the tile's own TRSM / DIAG is done), so every wait is "state >= value" and
// the device needs no dependency lists.  Tasks are placed on workers (one
// resident 128-thread CTA each) by list scheduling (HEFT: tasks by
// decreasing upward rank, each on the worker that finishes it first under a
// cost model in which a dependency between workers costs one flag hop); a
// worker runs its list in order.  The per-worker order is the simulated start
// order, a topological order of the graph, so a grid whose workers are all
// resident cannot deadlock.  What changes against the level-synchronous
// kernels is only who computes a tile and when -- the arithmetic per tile
// (diag_block, trsm_rows, the DMMA tile update, assemble_col) and the panel
// order per tile are the same, so the factors are bitwise identical.
#pragma once

#include <array>
#include <string>
#include <vector>

#include "layout.hpp"
#include "symbolic.hpp"

namespace nclb {

enum DagType { kDagAsm = 0, kDagDiag = 1, kDagTrsm = 2, kDagUpd = 3 };

// task word: x = front (segment-local), y = i | j << 12 | type << 24, z = p,
// w = simulated start (ns, diagnostics)
struct DagFront {
  long long loff;  // front offset in lval (f x f, ld = wide_ld(f))
  int s, c0, k, f;
  int P, NB;       // pivot blocks, all blocks
  int st_off;      // tile states: st_off + i (i + 1) / 2 + j
  int ntrail;      // trailing tiles (final after P updates)
  int ch_b, ch_e;  // wide children inside the segment: dag_ch[ch_b..ch_e)
  int scr_off;     // DIAG(p) pivots published at scr + (scr_off + p) * kDagScr
};

constexpr int kDagScr = 32 * 32 + 32;  // Us[32][32], rinv[32] per diagonal tile

struct DagSegment {
  int l0 = 0, l1 = 0;  // wide levels [l0, l1)
  int workers = 0;
  std::vector<DagFront> fronts;
  std::vector<int> ch;                         // segment-local wide children
  std::vector<std::array<int, 4>> tasks;       // in worker order
  std::vector<int> w_ptr;                      // workers + 1
  int nstate = 0;                              // tile states
  int nscr = 0;                                // diagonal tiles
  double makespan_us = 0.0;                    // simulated
  double crit_us = 0.0;                        // critical path (no worker limit, no hops)
};

// block b of a front: start row and size
NCLB_HD inline int dag_block_start(int k, int P, int b) { return b < P ? 32 * b : k + 32 * (b - P); }
NCLB_HD inline int dag_block_size(int k, int f, int P, int b) {
  const int s0 = dag_block_start(k, P, b);
  const int e = b < P ? (32 * b + 32 < k ? 32 * b + 32 : k) : (s0 + 32 < f ? s0 + 32 : f);
  return e - s0;
}

// the segments: maximal runs of wide levels whose fronts all exceed the
// small-front limit and that hold no split extend-add and no Schur front
std::vector<std::array<int, 2>> dag_level_runs(const Supernodal& T, int small_limit);

// levels [l0, l1) of T as one segment on `workers` workers
DagSegment build_dag_segment(const Supernodal& T, int l0, int l1, int workers);

// "" when the worker lists form a valid schedule (every task once, each
// worker's list in a topological order consistent across workers), else the
// first violation -- test hook
std::string check_dag_segment(const Supernodal& T, const DagSegment& G);

}  // namespace nclb
