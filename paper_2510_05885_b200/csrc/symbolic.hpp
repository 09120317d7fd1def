// Host-side symbolic analysis for the sm_100a static-pivot LDL^T.
//
// Everything here runs once per KKT pattern (KktContext construction,
// proj/src/kkt.cpp:41-138) and is bit-exact with the reference where the
// reference defines a result:
//   sym_lower_from_pattern  == sym_from_triplets   (proj/src/sparse.cpp:33-68)
//   amd_order               == Eigen AMDOrdering    (proj/src/sparse.cpp:81-100)
//   analyze_with_permutation: perm/iperm/parent/lcol_ptr/a_map
//                                                  (proj/src/sparse.cpp:102-176)
// and adds the B200-side structures the reference does not have: the
// fundamental-supernode partition, front row lists, assembly / extend-add
// maps, the warp tier (fronts <= 32 rows) with its heavy-path schedule, and
// the level schedule of the wide-front tier.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

namespace nclb {

// lower CSC (row >= col, rows strictly increasing per column)
struct LowerCsc {
  int n = 0;
  std::vector<int> col_ptr, row_ind;
  int nnz() const { return col_ptr.empty() ? 0 : col_ptr[n]; }
};

// (rows, cols) triplets, upper mirrored, sorted by (col,row), duplicates
// merged; dup_of[k] = slot of triplet k.
LowerCsc sym_lower_from_pattern(int n, const std::vector<int>& rows,
                                const std::vector<int>& cols,
                                std::vector<int>* slot_of_triplet = nullptr);

std::vector<int> amd_order(const LowerCsc& A);
// minimum-degree core on a full symmetric pattern (CSC, rows sorted, the
// structural diagonal present where it exists) -- Eigen's entry point
std::vector<int> amd_full_pattern(int n, const std::vector<int>& Ap,
                                  const std::vector<int>& Ai);

struct Symbolic {
  int n = 0;
  std::vector<int> perm, iperm, parent, lcol_ptr;
  std::vector<int> a_map;  // orig lower slot -> permuted upper slot
  long long l_nnz() const { return lcol_ptr.empty() ? 0 : lcol_ptr[n]; }
};

// throws std::invalid_argument like the reference
Symbolic analyze_with_permutation(const LowerCsc& A,
                                  const std::vector<int>& perm);

// Supernodal structure consumed by the CUDA kernels (all indices in the
// permuted numbering).
struct Supernodal {
  int n = 0;
  int nsn = 0;
  std::vector<int> first;      // nsn+1: first pivot column of each supernode
  std::vector<int> f;          // front size (pivots + rows below)
  std::vector<int> sparent;    // supernodal parent, -1 for roots
  std::vector<int> rows_ptr;   // nsn+1
  std::vector<int> rows;       // front rows (global permuted ids)
  std::vector<long long> l_off;  // nsn+1: offset of the f x k column-major
                                 // L block (diag: unit, not stored; d apart)
  std::vector<long long> u_off;  // offset of the update block (ld u_ld)
  std::vector<int> u_ld;
  long long u_total = 0;
  // assembly of A into the front: packed (front_row | front_col << 16), slot
  std::vector<int> asm_ptr, asm_pos, asm_slot;
  std::vector<int> asm_cp;  // n+1: asm entries of pivot column c (global)
  // wide fronts, column-wise extend-add: for front column J of wide front s
  // the children's columns landing in it, in child order:
  // cc_ent[cc_ptr[cc_off[s] + J] .. cc_ptr[cc_off[s] + J + 1]) = {child, col}
  // entry = {element offset of U_c(j, j) in its buffer (lval if the child
  // is wide, else upd), rel index of row j, count fu_c - j, child is wide}
  std::vector<int> cc_off, cc_ptr;
  std::vector<long long> cc_ubase;
  std::vector<int> cc_rbase, cc_cnt;
  // children in increasing order and their update-row map into the parent
  std::vector<int> ch_ptr, ch;
  std::vector<int> rel_ptr, rel;  // indexed by child: f_c - k_c entries
  // tiers
  std::vector<int8_t> wide;  // 1: front > warp limit, or any descendant is
                             // (upward closed)
  // warp tier: heavy paths (bottom -> top), ordered so that every light
  // child's path precedes the path it hangs from
  std::vector<int> path_ptr, path_nodes;
  std::vector<int> bwd_path;  // backward-solve hand-out order (path indices)
  // warp tier: extend-add entries of the children that are not the node's
  // path predecessor ("light" children), in chunks of 32 with distinct
  // destinations: src | dst << 48, -1 = padding.  Factorization: src = upd
  // offset, dst = row | col << 5 of the front; solves: src = update-vector
  // offset, dst = front row.
  std::vector<int> lt_ptr, ls_ptr;
  std::vector<long long> lt_ent, ls_ent;
  // warp tier: one record per path position q (path_nodes order) so a warp
  // reaches everything static about its next node with one dependent load:
  // prec[4q..4q+3] = {s, first, k, f}, {ch_b, ch_e, lt_b, lt_e},
  // {asm_b, asm_e, rel_ptr, rows_ptr}, {ls_b, ls_e, sparent, 0};
  // poff[2q..2q+1] = {l_off, u_off}
  std::vector<int> prec;
  std::vector<long long> poff;
  // split extend-add of fronts with many children (symbolic.cpp): groups per
  // front (0 = none) and offsets of the group sums (factorization: ng x f x f
  // doubles; forward solve: ng x f)
  std::vector<int> split_ng, usplit_ng;
  std::vector<long long> split_off, usplit_off;
  long long split_total = 0, usplit_total = 0;
  // wide tier: level lists (level 0 = deepest wide fronts)
  std::vector<int> lvl_ptr, lvl_nodes;
  // huge-front (three-kernel) schedule: assembly tasks {front, first
  // column} per level (kAsmCols columns each); panels of level l are
  // lp_ptr[l]..lp_ptr[l+1]-1 (global panel index g); the fronts factoring
  // panel g are dg_nodes[dg_ptr[g]..]; TRSM tasks {front, row block, diag
  // task index} are pn_tasks[pn_ptr[g]..]; trailing-update tiles {front,
  // row0, col0, panel} are tiles[tl_ptr[g]..]
  std::vector<std::array<int, 4>> asm_task;  // {front, col0, 0, 0}
  std::vector<std::array<int, 4>> pn_tasks;
  std::vector<int> dg_nodes;
  // lookahead strip tiles (the next panel's column block) of panel g are
  // tiles_s[ts_ptr[g]..], the rest tiles[tl_ptr[g]..]
  std::vector<std::array<int, 4>> tiles_s;
  std::vector<int> asm_task_ptr, lp_ptr, pn_ptr, tl_ptr, ts_ptr, dg_ptr;
  // the same rest updates as 64x64 tiles {front, row0, col0, panel} for the
  // fused path's k_wide_update64: tiles64[tl64_ptr[g]..]
  std::vector<std::array<int, 4>> tiles64;
  std::vector<int> tl64_ptr;
  int max_dg = 0;  // most fronts in one huge panel launch
  std::vector<std::array<int, 4>> tiles;
  long long wide_update_flops = 0;
  int schur = -1;  // Schur mode: the coupling supernode (assembled, not factored)
  int max_f = 0, max_wide_f = 0;
  long long flops = 0;      // sum_j c_j (c_j + 2), the SURVEY 8(d) figure
  long long wide_front_elems = 0;
  int sn_height = 0;
};

constexpr int kWarpFront = 32;
constexpr int kSplitMin = 128;       // contributions (children) per column that trigger a split
constexpr int kSplitPerGroup = 64;   // contributions per group (8 warps x 8)
constexpr int kSplitMaxG = 64;
constexpr int kSplitMaxF = 512;
constexpr int kFrontPaths = 32;     // long root paths handed out first (symbolic.cpp)
constexpr int kFrontPathLen = 64;
constexpr int kWidePanel = 32;  // pivots per panel of a wide front
constexpr int kAsmCols = 8;     // front columns per assembly task (warp each)
constexpr int kUpdTile = 32;    // trailing-update tile edge (one warp)
constexpr int kPanelRows = 96;  // rows below a panel solved per CTA (huge path; 3 lockstep warps)
constexpr int kHugeFront = 1536;  // levels with a larger front use the
                                  // three-kernel (whole-GPU) path

// schur_n0 > 0 (Schur mode): the last schur_n0 columns of the elimination
// order form one supernode that is assembled (extend-add of every child) but
// not factored; its front is the local Schur complement.
Supernodal build_supernodal(const LowerCsc& A, const Symbolic& S, int schur_n0 = 0);

// the same elimination tree re-postordered with every node's tallest child
// last (same fill, same factor entries): chains become consecutive columns
// that (relaxed) supernodes can follow.  perm[k] = variable eliminated k-th.
std::vector<int> tallest_child_last(const LowerCsc& A, const std::vector<int>& perm);

// the reference's row indices of L (sparse.cpp:157-175 / factorize's
// ascending order per column): lrow_ind for lcol_ptr
std::vector<int> l_row_pattern(const LowerCsc& A, const Symbolic& S);

// invariants of the warp-tier schedule (paths, hand-out orders, chunk lists,
// records); "" when they hold, else the first violation
std::string check_warp_schedule(const Supernodal& T);

// wide levels factored by the multi-kernel path (one front over every SM):
// a front above kHugeFront, or at most kHugeMaxN fronts of kHugeMinF rows
// (NCL_HUGE_MIN_F overrides; measured on the 78,400-bus mesh: 7.02 ms per
// Newton step with the cluster kernel on those levels, 6.47 ms with this path)
constexpr int kHugeMinF = 256;
constexpr int kHugeMaxN = 24;
bool level_is_huge(int fmax, int nfronts);

}  // namespace nclb
