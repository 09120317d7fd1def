// KKT symbolic plan (see kkt_plan.hpp).
#include "kkt_plan.hpp"

#include <algorithm>
#include <stdexcept>

namespace nclb {

namespace {

// slot_of (proj/src/kkt.cpp:31-37)
int slot_of(const LowerCsc& A, int i, int j) {
  const auto b = A.row_ind.begin() + A.col_ptr[j];
  const auto e = A.row_ind.begin() + A.col_ptr[j + 1];
  const auto it = std::lower_bound(b, e, i);
  if (it == e || *it != i) throw std::logic_error("kkt: missing slot");
  return static_cast<int>(it - A.row_ind.begin());
}

}  // namespace

KktPlan make_kkt_plan(int nt, const int* hp_ptr, const int* hp_idx, int m,
                      const int* jp_ptr, const int* jp_idx, int ns, int m_eq,
                      int form, int schur_n0, bool supernodal) {
  KktPlan P;
  if (form < 0 || form > 2) throw std::invalid_argument("unknown kkt form");
  if (nt < 0 || m < 0 || ns < 0 || m_eq < 0 || m - m_eq != ns)
    throw std::invalid_argument("kkt: inconsistent problem shape");
  P.form = form;
  P.nt = nt;
  P.ns = ns;
  P.n = nt + ns;
  P.m_eq = m_eq;
  P.m_ineq = m - m_eq;
  P.m = m;
  P.hp_ptr.assign(hp_ptr, hp_ptr + nt + 1);
  P.hp_idx.assign(hp_idx, hp_idx + hp_ptr[nt]);
  P.jp_ptr.assign(jp_ptr, jp_ptr + m + 1);
  P.jp_idx.assign(jp_idx, jp_idx + jp_ptr[m]);
  for (int j = 0; j < nt; ++j)
    for (int p = hp_ptr[j]; p < hp_ptr[j + 1]; ++p)
      if (hp_idx[p] < j || hp_idx[p] >= nt)
        throw std::invalid_argument("kkt: hessian pattern not lower");
  for (int i = 0; i < m; ++i)
    for (int p = jp_ptr[i]; p < jp_ptr[i + 1]; ++p)
      if (jp_idx[p] < 0 || jp_idx[p] >= nt ||
          (p > jp_ptr[i] && jp_idx[p] <= jp_idx[p - 1]))
        throw std::invalid_argument("kkt: jacobian columns unsorted");
  const int n = P.n;
  const int N = form == kK2 ? n + 2 * m : (form == kK2r ? n + m : nt);
  P.N = N;
  // pattern triplets in the reference's order (kkt.cpp:63-91)
  std::vector<int> ri, ci;
  auto add = [&](int i, int j) {
    ri.push_back(i);
    ci.push_back(j);
  };
  for (int j = 0; j < nt; ++j)
    for (int p = hp_ptr[j]; p < hp_ptr[j + 1]; ++p) add(hp_idx[p], j);
  if (form == kK1s) {
    for (int i = 0; i < nt; ++i) add(i, i);
    for (int i = 0; i < m; ++i)
      for (int pa = jp_ptr[i]; pa < jp_ptr[i + 1]; ++pa)
        for (int pb = jp_ptr[i]; pb <= pa; ++pb) add(jp_idx[pa], jp_idx[pb]);
  } else {
    for (int i = 0; i < n; ++i) add(i, i);
    const int yb = (form == kK2) ? n + m : n;
    for (int i = 0; i < m; ++i)
      for (int p = jp_ptr[i]; p < jp_ptr[i + 1]; ++p) add(yb + i, jp_idx[p]);
    for (int k = 0; k < P.m_ineq; ++k) add(yb + m_eq + k, nt + k);
    if (form == kK2) {
      for (int i = 0; i < m; ++i) add(n + i, n + i);
      for (int i = 0; i < m; ++i) add(n + m + i, n + i);
    } else {
      for (int i = 0; i < m; ++i) add(n + i, n + i);
    }
  }
  P.K = sym_lower_from_pattern(N, ri, ci);
  const LowerCsc& K = P.K;
  // slot maps (kkt.cpp:95-137)
  for (int j = 0; j < nt; ++j)
    for (int p = hp_ptr[j]; p < hp_ptr[j + 1]; ++p)
      P.h_slot.push_back(slot_of(K, hp_idx[p], j));
  const int nd = form == kK1s ? nt : n;
  for (int i = 0; i < nd; ++i) P.diag_slot.push_back(slot_of(K, i, i));
  if (form == kK1s) {
    P.pair_ptr.assign(static_cast<size_t>(m) + 1, 0);
    for (int i = 0; i < m; ++i) {
      const int v = jp_ptr[i + 1] - jp_ptr[i];
      P.pair_ptr[i + 1] = P.pair_ptr[i] + v * (v + 1) / 2;
    }
    for (int i = 0; i < m; ++i)
      for (int pa = jp_ptr[i]; pa < jp_ptr[i + 1]; ++pa)
        for (int pb = jp_ptr[i]; pb <= pa; ++pb) {
          P.pair_slot.push_back(slot_of(K, jp_idx[pa], jp_idx[pb]));
          P.pair_row.push_back(i);
          P.pair_pa.push_back(pa);
          P.pair_pb.push_back(pb);
        }
  } else {
    const int yb = (form == kK2) ? n + m : n;
    for (int i = 0; i < m; ++i)
      for (int p = jp_ptr[i]; p < jp_ptr[i + 1]; ++p)
        P.j_slot.push_back(slot_of(K, yb + i, jp_idx[p]));
    for (int k = 0; k < P.m_ineq; ++k)
      P.slack_slot.push_back(slot_of(K, yb + m_eq + k, nt + k));
    if (form == kK2) {
      for (int i = 0; i < m; ++i) {
        P.rdiag_slot.push_back(slot_of(K, n + i, n + i));
        P.ry_slot.push_back(slot_of(K, n + m + i, n + i));
      }
    } else {
      for (int i = 0; i < m; ++i) P.ydiag_slot.push_back(slot_of(K, n + i, n + i));
    }
  }
  // per-slot contribution lists in refill order (kkt.cpp:149-186): all H
  // entries (k ascending), then the diagonal, then pairs / J / slacks / y
  // blocks, each in the reference's loop order
  const int nnz = K.nnz();
  std::vector<std::vector<uint32_t>> lists(static_cast<size_t>(nnz));
  auto code = [](uint32_t t, long long idx) {
    if (idx < 0 || idx > static_cast<long long>(kIdxMask))
      throw std::length_error("kkt: pattern too large for contribution codes");
    return (t << kTypeShift) | static_cast<uint32_t>(idx);
  };
  for (size_t k = 0; k < P.h_slot.size(); ++k)
    lists[P.h_slot[k]].push_back(code(kCH, static_cast<long long>(k)));
  for (int i = 0; i < nd; ++i) lists[P.diag_slot[i]].push_back(code(kCDiag, i));
  if (form == kK1s) {
    for (size_t q = 0; q < P.pair_slot.size(); ++q)
      lists[P.pair_slot[q]].push_back(code(kCPair, static_cast<long long>(q)));
  } else {
    for (size_t p = 0; p < P.j_slot.size(); ++p)
      lists[P.j_slot[p]].push_back(code(kCJ, static_cast<long long>(p)));
    for (int k = 0; k < P.m_ineq; ++k) lists[P.slack_slot[k]].push_back(code(kCMinus1, 0));
    if (form == kK2) {
      for (int i = 0; i < m; ++i) {
        lists[P.rdiag_slot[i]].push_back(code(kCRho, 0));
        lists[P.ry_slot[i]].push_back(code(kCOne, 0));
      }
    } else {
      for (int i = 0; i < m; ++i) lists[P.ydiag_slot[i]].push_back(code(kCYdiag, 0));
    }
  }
  P.c_ptr.assign(static_cast<size_t>(nnz) + 1, 0);
  for (int s = 0; s < nnz; ++s)
    P.c_ptr[s + 1] = P.c_ptr[s] + static_cast<int>(lists[s].size());
  P.c_code.reserve(static_cast<size_t>(P.c_ptr[nnz]));
  for (int s = 0; s < nnz; ++s)
    P.c_code.insert(P.c_code.end(), lists[s].begin(), lists[s].end());
  // J^T (entries of each column in increasing row order)
  P.jt_ptr.assign(static_cast<size_t>(nt) + 1, 0);
  for (int p = 0; p < jp_ptr[m]; ++p) P.jt_ptr[jp_idx[p] + 1]++;
  for (int c = 0; c < nt; ++c) P.jt_ptr[c + 1] += P.jt_ptr[c];
  P.jt_row.assign(static_cast<size_t>(jp_ptr[m]), 0);
  P.jt_slot.assign(static_cast<size_t>(jp_ptr[m]), 0);
  {
    std::vector<int> nx(P.jt_ptr.begin(), P.jt_ptr.end() - 1);
    for (int i = 0; i < m; ++i)
      for (int p = jp_ptr[i]; p < jp_ptr[i + 1]; ++p) {
        const int q = nx[jp_idx[p]]++;
        P.jt_row[q] = i;
        P.jt_slot[q] = p;
      }
  }
  // inertia target (kkt.cpp:140-147)
  if (form == kK2) {
    P.inertia_target[0] = n + m;
    P.inertia_target[1] = m;
  } else if (form == kK2r) {
    P.inertia_target[0] = n;
    P.inertia_target[1] = m;
  } else {
    P.inertia_target[0] = nt;
    P.inertia_target[1] = 0;
  }
  // symbolic analysis (kkt.cpp:94 -> sparse.cpp:178-180)
  if (schur_n0 > 0) {
    if (form != kK1s || schur_n0 > N) throw std::invalid_argument("schur: K1s and n0 <= N only");
    // AMD on the block part K[n0:, n0:], coupling columns last in their order
    LowerCsc B;
    B.n = N - schur_n0;
    B.col_ptr.assign(static_cast<size_t>(B.n) + 1, 0);
    for (int j = schur_n0; j < N; ++j) {
      for (int p = K.col_ptr[j]; p < K.col_ptr[j + 1]; ++p) B.row_ind.push_back(K.row_ind[p] - schur_n0);
      B.col_ptr[j - schur_n0 + 1] = static_cast<int>(B.row_ind.size());
    }
    std::vector<int> perm = amd_order(B);
    for (int& v : perm) v += schur_n0;
    for (int j = 0; j < schur_n0; ++j) perm.push_back(j);
    // the coupling columns stay last: they are the top of the tree
    perm = tallest_child_last(K, perm);
    P.sym = analyze_with_permutation(K, perm);
    P.sn = build_supernodal(K, P.sym, schur_n0);
  } else {
    P.sym = analyze_with_permutation(K, amd_order(K));
    if (supernodal) P.sn = build_supernodal(K, P.sym);
  }
  return P;
}

}  // namespace nclb
