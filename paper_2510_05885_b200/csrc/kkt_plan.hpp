// KKT pattern plan: the symbolic-once half of KktContext
// (proj/src/kkt.cpp:41-138), re-expressed as per-slot gather lists so the
// numeric refill runs as one conflict-free, bit-exact gather kernel.
#pragma once

#include <cstdint>
#include <vector>

#include "symbolic.hpp"

namespace nclb {

enum Form { kK2 = 0, kK2r = 1, kK1s = 2 };

// contribution codes for the per-slot gather (type in the top 3 bits)
enum ContribType : uint32_t {
  kCH = 0,       // + hval[idx]
  kCDiag = 1,    // + (sigma[idx] + delta)
  kCPair = 2,    // + (w[row(idx)] * jv[pa(idx)]) * jv[pb(idx)]     (K1s)
  kCJ = 3,       // + jval[idx]                                    (K2/K2r)
  kCMinus1 = 4,  // + (-1.0)                                       (slacks)
  kCYdiag = 5,   // + (-1.0 / rho_hat)                             (K2r)
  kCRho = 6,     // + rho_hat                                      (K2)
  kCOne = 7,     // + 1.0                                          (K2)
};
constexpr int kTypeShift = 29;
constexpr uint32_t kIdxMask = (1u << kTypeShift) - 1;

struct KktPlan {
  int form = kK1s;
  int nt = 0, ns = 0, n = 0, m_eq = 0, m_ineq = 0, m = 0;
  int N = 0;
  std::vector<int> hp_ptr, hp_idx, jp_ptr, jp_idx;
  LowerCsc K;                      // pattern of the assembled matrix
  std::vector<int> h_slot, diag_slot, pair_slot, pair_ptr, j_slot,
      slack_slot, rdiag_slot, ry_slot, ydiag_slot;
  // per-slot contributions in the reference's accumulation order
  std::vector<int> c_ptr;          // nnz_K + 1
  std::vector<uint32_t> c_code;
  // K1s pairs: row of pair q, pa, pb (jp slots)
  std::vector<int> pair_row, pair_pa, pair_pb;
  // J transposed (column -> entries in increasing row), for Jt-gathers
  std::vector<int> jt_ptr, jt_row, jt_slot;
  Symbolic sym;
  Supernodal sn;
  int inertia_target[3] = {0, 0, 0};
};

// throws std::invalid_argument on inconsistent shapes (kkt.cpp:52-53)
// schur_n0 > 0 (K1s only): Schur mode for a block-arrowhead sub-problem whose
// first schur_n0 variables couple the blocks -- they are ordered last (AMD on
// the rest) and form the unfactored coupling supernode
// supernodal = false (non-Schur only): skip the plan's own supernodal
// structure (the device factorization builds its re-postordered one)
KktPlan make_kkt_plan(int nt, const int* hp_ptr, const int* hp_idx, int m,
                      const int* jp_ptr, const int* jp_idx, int ns, int m_eq,
                      int form, int schur_n0 = 0, bool supernodal = true);

}  // namespace nclb
