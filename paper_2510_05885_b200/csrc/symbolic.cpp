// Host symbolic analysis (see symbolic.hpp).
#include "symbolic.hpp"
#include "layout.hpp"

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <numeric>
#include <stdexcept>

namespace nclb {

// ---------------------------------------------------------------------------
// sym_from_triplets (proj/src/sparse.cpp:33-68): mirror upper entries, sort by
// (col,row), merge duplicates.  Only the pattern is needed here: KktContext
// builds its matrix from zero-valued triplets (kkt.cpp:93).
LowerCsc sym_lower_from_pattern(int n, const std::vector<int>& rows,
                                const std::vector<int>& cols,
                                std::vector<int>* slot_of_triplet) {
  if (rows.size() != cols.size())
    throw std::invalid_argument("sym_from_triplets: length mismatch");
  const size_t nt = rows.size();
  std::vector<long long> key(nt);
  for (size_t k = 0; k < nt; ++k) {
    int i = rows[k], j = cols[k];
    if (i < 0 || i >= n || j < 0 || j >= n)
      throw std::invalid_argument("sym_from_triplets: index out of range");
    if (i < j) std::swap(i, j);
    key[k] = (static_cast<long long>(j) << 32) | static_cast<unsigned>(i);
  }
  std::vector<int> order(nt);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return key[a] < key[b]; });
  LowerCsc A;
  A.n = n;
  A.col_ptr.assign(static_cast<size_t>(n) + 1, 0);
  if (slot_of_triplet) slot_of_triplet->assign(nt, -1);
  long long prev = -1;
  for (size_t q = 0; q < nt; ++q) {
    const long long kq = key[order[q]];
    if (q == 0 || kq != prev) {
      A.col_ptr[static_cast<size_t>(kq >> 32) + 1]++;
      A.row_ind.push_back(static_cast<int>(kq & 0xffffffffLL));
      prev = kq;
    }
    if (slot_of_triplet)
      (*slot_of_triplet)[order[q]] = static_cast<int>(A.row_ind.size()) - 1;
  }
  for (int j = 0; j < n; ++j) A.col_ptr[j + 1] += A.col_ptr[j];
  return A;
}

// ---------------------------------------------------------------------------
// Approximate minimum degree, restating Eigen's AMDOrdering<int>
// (Eigen/src/OrderingMethods/Amd.h: internal::minimum_degree_ordering, a port
// of CSparse cs_amd) on the pattern of A^T + A with the diagonal kept, as
// proj/src/sparse.cpp:81-100 calls it.  Quotient-graph elimination with
// approximate external degrees, aggressive absorption, hash-based
// indistinguishable-node detection and mass elimination; Eigen's structural
// diagonal rule (a node without a diagonal entry, or denser than
// max(16, 10 sqrt n) capped at n-2, is absorbed into the dummy root n); the
// permutation is the postorder of the assembly tree.
namespace {

struct AmdState {
  int n;
  std::vector<int> Cp, Ci, len, nv, next, head, elen, degree, w, hhead, last;
};

inline int flip(int i) { return -i - 2; }

int wclear(int mark, int lemax, std::vector<int>& w, int n) {
  if (mark < 2 || (mark + lemax < 0)) {
    for (int k = 0; k < n; k++)
      if (w[k] != 0) w[k] = 1;
    mark = 2;
  }
  return mark;
}

int tdfs(int j, int k, std::vector<int>& head, const std::vector<int>& next,
         std::vector<int>& post, std::vector<int>& stack) {
  int top = 0;
  stack[0] = j;
  while (top >= 0) {
    const int p = stack[top];
    const int i = head[p];
    if (i == -1) {
      top--;
      post[k++] = p;
    } else {
      head[p] = next[i];
      stack[++top] = i;
    }
  }
  return k;
}

std::vector<int> min_degree(int n, const std::vector<int>& Ap,
                            const std::vector<int>& Ai) {
  std::vector<int> P(static_cast<size_t>(n) + 1, 0);
  if (n == 0) return {};
  int dense = std::max(16, static_cast<int>(10 * std::sqrt(static_cast<double>(n))));
  dense = std::min(n - 2, dense);
  int cnz = Ap[n];
  const int nzmax = cnz + cnz / 5 + 2 * n;
  std::vector<int> Cp(Ap.begin(), Ap.end());
  std::vector<int> Ci(static_cast<size_t>(nzmax), 0);
  std::copy(Ai.begin(), Ai.begin() + cnz, Ci.begin());
  const size_t n1 = static_cast<size_t>(n) + 1;
  std::vector<int> len(n1), nv(n1), next(n1), head(n1), elen(n1), degree(n1),
      w(n1), hhead(n1);
  std::vector<int>& last = P;
  for (int k = 0; k < n; k++) len[k] = Cp[k + 1] - Cp[k];
  len[n] = 0;
  for (int i = 0; i <= n; i++) {
    head[i] = -1;
    last[i] = -1;
    next[i] = -1;
    hhead[i] = -1;
    nv[i] = 1;
    w[i] = 1;
    elen[i] = 0;
    degree[i] = len[i];
  }
  int mark = wclear(0, 0, w, n);
  int nel = 0, mindeg = 0, lemax = 0;
  for (int i = 0; i < n; i++) {
    bool has_diag = false;
    for (int p = Cp[i]; p < Cp[i + 1]; ++p)
      if (Ci[p] == i) {
        has_diag = true;
        break;
      }
    const int d = degree[i];
    if (d == 1 && has_diag) {
      elen[i] = -2;
      nel++;
      Cp[i] = -1;
      w[i] = 0;
    } else if (d > dense || !has_diag) {
      nv[i] = 0;
      elen[i] = -1;
      nel++;
      Cp[i] = flip(n);
      nv[n]++;
    } else {
      if (head[d] != -1) last[head[d]] = i;
      next[i] = head[d];
      head[d] = i;
    }
  }
  elen[n] = -2;
  Cp[n] = -1;
  w[n] = 0;

  while (nel < n) {
    int k = -1;
    for (; mindeg < n && (k = head[mindeg]) == -1; mindeg++) {
    }
    if (next[k] != -1) last[next[k]] = -1;
    head[mindeg] = next[k];
    const int elenk = elen[k];
    int nvk = nv[k];
    nel += nvk;

    if (elenk > 0 && cnz + mindeg >= nzmax) {  // garbage collection
      for (int j = 0; j < n; j++) {
        int p;
        if ((p = Cp[j]) >= 0) {
          Cp[j] = Ci[p];
          Ci[p] = flip(j);
        }
      }
      int q = 0;
      for (int p = 0; p < cnz;) {
        int j;
        if ((j = flip(Ci[p++])) >= 0) {
          Ci[q] = Cp[j];
          Cp[j] = q++;
          for (int k3 = 0; k3 < len[j] - 1; k3++) Ci[q++] = Ci[p++];
        }
      }
      cnz = q;
    }

    int dk = 0;  // construct the new element
    nv[k] = -nvk;
    int p = Cp[k];
    const int pk1 = (elenk == 0) ? p : cnz;
    int pk2 = pk1;
    for (int k1 = 1; k1 <= elenk + 1; k1++) {
      int e, pj, ln;
      if (k1 > elenk) {
        e = k;
        pj = p;
        ln = len[k] - elenk;
      } else {
        e = Ci[p++];
        pj = Cp[e];
        ln = len[e];
      }
      for (int k2 = 1; k2 <= ln; k2++) {
        const int i = Ci[pj++];
        int nvi;
        if ((nvi = nv[i]) <= 0) continue;
        dk += nvi;
        nv[i] = -nvi;
        Ci[pk2++] = i;
        if (next[i] != -1) last[next[i]] = last[i];
        if (last[i] != -1)
          next[last[i]] = next[i];
        else
          head[degree[i]] = next[i];
      }
      if (e != k) {
        Cp[e] = flip(k);
        w[e] = 0;
      }
    }
    if (elenk != 0) cnz = pk2;
    degree[k] = dk;
    Cp[k] = pk1;
    len[k] = pk2 - pk1;
    elen[k] = -2;

    mark = wclear(mark, lemax, w, n);  // set differences |Le \ Lk|
    for (int pk = pk1; pk < pk2; pk++) {
      const int i = Ci[pk];
      const int eln = elen[i];
      if (eln <= 0) continue;
      const int nvi = -nv[i];
      const int wnvi = mark - nvi;
      for (p = Cp[i]; p <= Cp[i] + eln - 1; p++) {
        const int e = Ci[p];
        if (w[e] >= mark)
          w[e] -= nvi;
        else if (w[e] != 0)
          w[e] = degree[e] + wnvi;
      }
    }

    for (int pk = pk1; pk < pk2; pk++) {  // degree update
      const int i = Ci[pk];
      const int p1 = Cp[i];
      const int p2 = p1 + elen[i] - 1;
      int pn = p1;
      int h = 0, d = 0;
      for (p = p1; p <= p2; p++) {
        const int e = Ci[p];
        if (w[e] != 0) {
          const int dext = w[e] - mark;
          if (dext > 0) {
            d += dext;
            Ci[pn++] = e;
            h += e;
          } else {
            Cp[e] = flip(k);
            w[e] = 0;
          }
        }
      }
      elen[i] = pn - p1 + 1;
      const int p3 = pn;
      const int p4 = p1 + len[i];
      for (p = p2 + 1; p < p4; p++) {
        const int j = Ci[p];
        int nvj;
        if ((nvj = nv[j]) <= 0) continue;
        d += nvj;
        Ci[pn++] = j;
        h += j;
      }
      if (d == 0) {  // mass elimination
        Cp[i] = flip(k);
        const int nvi = -nv[i];
        dk -= nvi;
        nvk += nvi;
        nel += nvi;
        nv[i] = 0;
        elen[i] = -1;
      } else {
        degree[i] = std::min(degree[i], d);
        Ci[pn] = Ci[p3];
        Ci[p3] = Ci[p1];
        Ci[p1] = k;
        len[i] = pn - p1 + 1;
        h = ((h < 0) ? (-h) : h) % n;
        next[i] = hhead[h];
        hhead[h] = i;
        last[i] = h;
      }
    }
    degree[k] = dk;
    lemax = std::max(lemax, dk);
    mark = wclear(mark + lemax, lemax, w, n);

    for (int pk = pk1; pk < pk2; pk++) {  // supernode detection
      int i = Ci[pk];
      if (nv[i] >= 0) continue;
      const int h = last[i];
      i = hhead[h];
      hhead[h] = -1;
      for (; i != -1 && next[i] != -1; i = next[i], mark++) {
        const int ln = len[i];
        const int eln = elen[i];
        for (p = Cp[i] + 1; p <= Cp[i] + ln - 1; p++) w[Ci[p]] = mark;
        int jlast = i;
        for (int j = next[i]; j != -1;) {
          bool ok = (len[j] == ln) && (elen[j] == eln);
          for (p = Cp[j] + 1; ok && p <= Cp[j] + ln - 1; p++)
            if (w[Ci[p]] != mark) ok = false;
          if (ok) {
            Cp[j] = flip(i);
            nv[i] += nv[j];
            nv[j] = 0;
            elen[j] = -1;
            j = next[j];
            next[jlast] = j;
          } else {
            jlast = j;
            j = next[j];
          }
        }
      }
    }

    int pq = pk1;  // finalize the new element
    for (int pk = pk1; pk < pk2; pk++) {
      const int i = Ci[pk];
      int nvi;
      if ((nvi = -nv[i]) <= 0) continue;
      nv[i] = nvi;
      int d = degree[i] + dk - nvi;
      d = std::min(d, n - nel - nvi);
      if (head[d] != -1) last[head[d]] = i;
      next[i] = head[d];
      last[i] = -1;
      head[d] = i;
      mindeg = std::min(mindeg, d);
      degree[i] = d;
      Ci[pq++] = i;
    }
    nv[k] = nvk;
    if ((len[k] = pq - pk1) == 0) {
      Cp[k] = -1;
      w[k] = 0;
    }
    if (elenk != 0) cnz = pq;
  }

  for (int i = 0; i < n; i++) Cp[i] = flip(Cp[i]);  // postorder
  for (int j = 0; j <= n; j++) head[j] = -1;
  for (int j = n; j >= 0; j--) {
    if (nv[j] > 0) continue;
    next[j] = head[Cp[j]];
    head[Cp[j]] = j;
  }
  for (int e = n; e >= 0; e--) {
    if (nv[e] <= 0) continue;
    if (Cp[e] != -1) {
      next[e] = head[Cp[e]];
      head[Cp[e]] = e;
    }
  }
  std::vector<int> post(n1), stack(n1);
  for (int k = 0, i = 0; i <= n; i++)
    if (Cp[i] == -1) k = tdfs(i, k, head, next, post, stack);
  post.resize(static_cast<size_t>(n));
  return post;
}

}  // namespace

std::vector<int> amd_full_pattern(int n, const std::vector<int>& Ap,
                                  const std::vector<int>& Ai) {
  return min_degree(n, Ap, Ai);
}

std::vector<int> amd_order(const LowerCsc& A) {
  const int n = A.n;
  // full symmetric pattern, rows sorted (mirrored rows < j, then lower part)
  std::vector<int> cnt(static_cast<size_t>(n), 0);
  for (int j = 0; j < n; ++j)
    for (int p = A.col_ptr[j]; p < A.col_ptr[j + 1]; ++p) {
      cnt[j]++;
      if (A.row_ind[p] != j) cnt[A.row_ind[p]]++;
    }
  std::vector<int> Mp(static_cast<size_t>(n) + 1, 0);
  for (int j = 0; j < n; ++j) Mp[j + 1] = Mp[j] + cnt[j];
  std::vector<int> Mi(static_cast<size_t>(Mp[n]));
  std::vector<int> nx(Mp.begin(), Mp.end() - 1);
  for (int r = 0; r < n; ++r)
    for (int p = A.col_ptr[r]; p < A.col_ptr[r + 1]; ++p)
      if (A.row_ind[p] != r) Mi[nx[A.row_ind[p]]++] = r;
  for (int j = 0; j < n; ++j)
    for (int p = A.col_ptr[j]; p < A.col_ptr[j + 1]; ++p)
      Mi[nx[j]++] = A.row_ind[p];
  return min_degree(n, Mp, Mi);
}

// ---------------------------------------------------------------------------
// analyze_with_permutation (proj/src/sparse.cpp:102-176)
Symbolic analyze_with_permutation(const LowerCsc& A,
                                  const std::vector<int>& perm) {
  const int n = A.n;
  for (int j = 0; j < n; ++j) {
    if (A.col_ptr[j] > A.col_ptr[j + 1])
      throw std::invalid_argument("sparse: col_ptr not nondecreasing");
    for (int p = A.col_ptr[j]; p < A.col_ptr[j + 1]; ++p) {
      if (A.row_ind[p] < j || A.row_ind[p] >= n)
        throw std::invalid_argument("sparse: row index outside lower triangle");
      if (p > A.col_ptr[j] && A.row_ind[p] <= A.row_ind[p - 1])
        throw std::invalid_argument("sparse: rows not strictly increasing");
    }
  }
  if (static_cast<int>(perm.size()) != n)
    throw std::invalid_argument("analyze: permutation length mismatch");
  Symbolic S;
  S.n = n;
  S.perm = perm;
  S.iperm.assign(static_cast<size_t>(n), -1);
  for (int k = 0; k < n; ++k) {
    if (perm[k] < 0 || perm[k] >= n || S.iperm[perm[k]] != -1)
      throw std::invalid_argument("analyze: not a permutation");
    S.iperm[perm[k]] = k;
  }
  const int nnz = A.nnz();
  // permuted upper pattern by column; a_map = orig slot -> sorted slot
  std::vector<int> acp(static_cast<size_t>(n) + 1, 0);
  for (int j = 0; j < n; ++j)
    for (int p = A.col_ptr[j]; p < A.col_ptr[j + 1]; ++p)
      acp[std::max(S.iperm[A.row_ind[p]], S.iperm[j]) + 1]++;
  for (int c = 0; c < n; ++c) acp[c + 1] += acp[c];
  std::vector<long long> key(static_cast<size_t>(nnz));
  std::vector<int> nx(acp.begin(), acp.end() - 1), orig(static_cast<size_t>(nnz));
  std::vector<int> ari(static_cast<size_t>(nnz));
  for (int j = 0; j < n; ++j)
    for (int p = A.col_ptr[j]; p < A.col_ptr[j + 1]; ++p) {
      const int pi = S.iperm[A.row_ind[p]], pj = S.iperm[j];
      const int s = nx[std::max(pi, pj)]++;
      ari[s] = std::min(pi, pj);
      orig[s] = p;
    }
  S.a_map.assign(static_cast<size_t>(nnz), 0);
  std::vector<std::pair<int, int>> buf;
  for (int c = 0; c < n; ++c) {
    buf.clear();
    for (int s = acp[c]; s < acp[c + 1]; ++s) buf.emplace_back(ari[s], orig[s]);
    std::sort(buf.begin(), buf.end());
    for (int k = 0; k < static_cast<int>(buf.size()); ++k) {
      ari[acp[c] + k] = buf[k].first;
      S.a_map[buf[k].second] = acp[c] + k;
    }
  }
  // elimination tree + column counts by up-looking reach
  S.parent.assign(static_cast<size_t>(n), -1);
  std::vector<int> lnz(static_cast<size_t>(n), 0), flag(static_cast<size_t>(n), -1);
  for (int k = 0; k < n; ++k) {
    flag[k] = k;
    for (int p = acp[k]; p < acp[k + 1]; ++p) {
      int i = ari[p];
      if (i >= k) continue;
      while (flag[i] != k) {
        if (S.parent[i] == -1) S.parent[i] = k;
        lnz[i]++;
        flag[i] = k;
        i = S.parent[i];
      }
    }
  }
  S.lcol_ptr.assign(static_cast<size_t>(n) + 1, 0);
  for (int c = 0; c < n; ++c) S.lcol_ptr[c + 1] = S.lcol_ptr[c] + lnz[c];
  return S;
}

// ---------------------------------------------------------------------------
// Fundamental supernodes, front structures, maps and schedules.
std::vector<int> l_row_pattern(const LowerCsc& A, const Symbolic& S) {
  const int n = S.n;
  // permuted lower pattern by row: columns j < i of row i
  std::vector<int> rp(static_cast<size_t>(n) + 1, 0);
  for (int c = 0; c < n; ++c)
    for (int p = A.col_ptr[c]; p < A.col_ptr[c + 1]; ++p) {
      const int i = S.iperm[A.row_ind[p]], j = S.iperm[c];
      if (i != j) rp[std::max(i, j) + 1]++;
    }
  for (int i = 0; i < n; ++i) rp[i + 1] += rp[i];
  std::vector<int> rc(static_cast<size_t>(rp[n]));
  {
    std::vector<int> nx(rp.begin(), rp.end() - 1);
    for (int c = 0; c < n; ++c)
      for (int p = A.col_ptr[c]; p < A.col_ptr[c + 1]; ++p) {
        const int i = S.iperm[A.row_ind[p]], j = S.iperm[c];
        if (i != j) rc[nx[std::max(i, j)]++] = std::min(i, j);
      }
  }
  // row k's columns = its reach in the elimination tree (sparse.cpp:157-175)
  std::vector<int> out(static_cast<size_t>(S.lcol_ptr[n]));
  std::vector<int> fill(S.lcol_ptr.begin(), S.lcol_ptr.end() - 1), mark(static_cast<size_t>(n), -1);
  for (int k = 0; k < n; ++k) {
    mark[k] = k;
    for (int p = rp[k]; p < rp[k + 1]; ++p)
      for (int j = rc[p]; j >= 0 && mark[j] != k; j = S.parent[j]) {
        mark[j] = k;
        out[fill[j]++] = k;
      }
  }
  return out;
}

std::vector<int> tallest_child_last(const LowerCsc& A, const std::vector<int>& perm) {
  const Symbolic S0 = analyze_with_permutation(A, perm);
  const int n = S0.n;
  std::vector<int> height(static_cast<size_t>(n), 0);
  for (int j = 0; j < n; ++j)
    if (S0.parent[j] >= 0) height[S0.parent[j]] = std::max(height[S0.parent[j]], height[j] + 1);
  std::vector<std::vector<int>> kids(static_cast<size_t>(n));
  std::vector<int> roots, order;
  order.reserve(static_cast<size_t>(n));
  for (int j = 0; j < n; ++j) (S0.parent[j] >= 0 ? kids[S0.parent[j]] : roots).push_back(j);
  for (auto& v : kids)
    std::stable_sort(v.begin(), v.end(), [&](int a, int b) { return height[a] < height[b]; });
  std::vector<std::pair<int, int>> stack;
  for (int r : roots) {
    stack.push_back({r, 0});
    while (!stack.empty()) {
      auto& [v, i] = stack.back();
      if (i < static_cast<int>(kids[v].size())) {
        const int c = kids[v][i++];
        stack.push_back({c, 0});
      } else {
        order.push_back(v);
        stack.pop_back();
      }
    }
  }
  std::vector<int> np(static_cast<size_t>(n));
  for (int k = 0; k < n; ++k) np[k] = perm[order[k]];
  return np;
}

bool level_is_huge(int fmax, int nfronts) {
  static const int huge_min_f = [] {
    const char* e = std::getenv("NCL_HUGE_MIN_F");
    return e ? std::atoi(e) : kHugeMinF;
  }();
  static const int huge_max_n = [] {
    const char* e = std::getenv("NCL_HUGE_MAX_N");
    return e ? std::atoi(e) : kHugeMaxN;
  }();
  return fmax > kHugeFront || (fmax >= huge_min_f && nfronts <= huge_max_n);
}

// Orders extend-add entries (dst, src) into chunks of 32 with pairwise
// distinct destinations, entries of one destination kept in their given
// order (so the sums are deterministic); a chunk with fewer than 32
// destinations left is padded with -1.  Destinations with the most entries
// left go first, which keeps the chunk count at max(total / 32, deepest).
static void chunk_entries(const std::vector<std::pair<int, long long>>& ent, std::vector<long long>& out) {
  if (ent.empty()) return;
  std::vector<int> dsts;
  for (const auto& e : ent) dsts.push_back(e.first);
  std::sort(dsts.begin(), dsts.end());
  dsts.erase(std::unique(dsts.begin(), dsts.end()), dsts.end());
  std::vector<std::vector<long long>> q(dsts.size());
  for (const auto& e : ent)
    q[std::lower_bound(dsts.begin(), dsts.end(), e.first) - dsts.begin()].push_back(e.second);
  std::vector<size_t> head(dsts.size(), 0);
  std::vector<int> order(dsts.size());
  size_t left = ent.size();
  while (left > 0) {
    order.clear();
    for (size_t d = 0; d < dsts.size(); ++d)
      if (head[d] < q[d].size()) order.push_back(static_cast<int>(d));
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      return q[a].size() - head[a] > q[b].size() - head[b];
    });
    const size_t take = std::min<size_t>(order.size(), 32);
    for (size_t t = 0; t < take; ++t) {
      const int d = order[t];
      out.push_back(q[d][head[d]++] | (static_cast<long long>(dsts[d]) << 48));
      --left;
    }
    for (size_t t = take; t < 32; ++t) out.push_back(-1);
  }
}

Supernodal build_supernodal(const LowerCsc& A, const Symbolic& S, int schur_n0) {
  const int n = S.n;
  Supernodal T;
  T.n = n;
  std::vector<int> cnt(static_cast<size_t>(n)), nchild(static_cast<size_t>(n), 0);
  for (int j = 0; j < n; ++j) {
    cnt[j] = S.lcol_ptr[j + 1] - S.lcol_ptr[j];
    if (S.parent[j] >= 0) nchild[S.parent[j]]++;
    T.flops += static_cast<long long>(cnt[j]) * (cnt[j] + 2);
  }
  // supernodes: j+1 continues j iff parent[j] == j+1 and count(j) ==
  // count(j+1) + 1 (column j's pattern is exactly {j+1} + column j+1's)
  T.first.push_back(0);
  // Schur mode also relaxes them: column j joins its child j-1's supernode
  // whenever the explicit zeros that adds keep the dense front within 25 % of
  // the true nonzeros (column j-1's pattern minus j lies inside column j's, so
  // the front is still k + count(last)) -- up to as many zeros as nonzeros, at
  // most 96 pivots.  Block-arrowhead problems carry the
  // coupling rows through every block front, and chains of 4-pivot fronts
  // collapse into a few wide ones.  (Not in the default mode: the reference's
  // L pattern is read back from the fronts there.)
  // Relaxed supernodes: in Schur mode (see above); otherwise only while the
  // merged front still fits the warp tier (<= 32 rows) -- chains of tiny
  // fronts (ring power grids: 30k+ supernodes on one path) collapse into
  // fewer, larger warp-tier fronts at the price of explicit zeros.
  const bool schur_relax = schur_n0 > 0;
  long long sn_true = n > 0 ? cnt[0] + 1 : 0;  // true nonzeros of the open supernode
  for (int j = 1; j < n; ++j) {
    const int k = j - T.first.back();
    // exact nesting (no explicit zeros); other children of j may hang off the
    // supernode's interior columns -- their updates land in its front rows
    bool cont = S.parent[j - 1] == j && cnt[j - 1] == cnt[j] + 1 && k < 65535;
    if (!cont && S.parent[j - 1] == j && k < 96) {
      const long long f = k + 1 + cnt[j];                    // front with j joined
      const long long dense = (2 * f - k) * (k + 1) / 2;     // sum_{i<=k} (f - i)
      const long long truenz = sn_true + cnt[j] + 1;
      cont = dense - truenz <= truenz && (schur_relax || f <= kWarpFront);
    }
    if (cont) {
      sn_true += cnt[j] + 1;
    } else {
      T.first.push_back(j);
      sn_true = cnt[j] + 1;
    }
  }
  if (schur_n0 > 0 && schur_n0 <= n) {  // one supernode for the coupling columns
    while (!T.first.empty() && T.first.back() > n - schur_n0) T.first.pop_back();
    if (T.first.empty() || T.first.back() < n - schur_n0) T.first.push_back(n - schur_n0);
  }
  if (n > 0) T.first.push_back(n);
  T.nsn = n > 0 ? static_cast<int>(T.first.size()) - 1 : 0;
  if (schur_n0 > 0 && schur_n0 <= n) T.schur = T.nsn - 1;
  if (n == 0) T.first.assign(1, 0);
  const int nsn = T.nsn;
  std::vector<int> col2sn(static_cast<size_t>(n));
  for (int s = 0; s < nsn; ++s)
    for (int c = T.first[s]; c < T.first[s + 1]; ++c) col2sn[c] = s;
  T.sparent.assign(static_cast<size_t>(nsn), -1);
  T.f.assign(static_cast<size_t>(nsn), 0);
  for (int s = 0; s < nsn; ++s) {
    const int last = T.first[s + 1] - 1;
    const int p = S.parent[last];
    T.sparent[s] = p >= 0 ? col2sn[p] : -1;
    T.f[s] = (T.first[s + 1] - T.first[s]) + cnt[last];
  }
  // children lists (increasing)
  T.ch_ptr.assign(static_cast<size_t>(nsn) + 1, 0);
  for (int s = 0; s < nsn; ++s)
    if (T.sparent[s] >= 0) T.ch_ptr[T.sparent[s] + 1]++;
  for (int s = 0; s < nsn; ++s) T.ch_ptr[s + 1] += T.ch_ptr[s];
  T.ch.assign(static_cast<size_t>(T.ch_ptr[nsn]), 0);
  {
    std::vector<int> nx(T.ch_ptr.begin(), T.ch_ptr.end() - 1);
    for (int s = 0; s < nsn; ++s)
      if (T.sparent[s] >= 0) T.ch[nx[T.sparent[s]]++] = s;
  }
  // permuted lower pattern by column: (row, slot of A)
  std::vector<int> lcp(static_cast<size_t>(n) + 1, 0);
  for (int j = 0; j < n; ++j)
    for (int p = A.col_ptr[j]; p < A.col_ptr[j + 1]; ++p)
      lcp[std::min(S.iperm[A.row_ind[p]], S.iperm[j]) + 1]++;
  for (int c = 0; c < n; ++c) lcp[c + 1] += lcp[c];
  std::vector<int> lri(static_cast<size_t>(A.nnz())), lsl(static_cast<size_t>(A.nnz()));
  {
    std::vector<int> nx(lcp.begin(), lcp.end() - 1);
    for (int j = 0; j < n; ++j)
      for (int p = A.col_ptr[j]; p < A.col_ptr[j + 1]; ++p) {
        const int pi = S.iperm[A.row_ind[p]], pj = S.iperm[j];
        const int q = nx[std::min(pi, pj)]++;
        lri[q] = std::max(pi, pj);
        lsl[q] = p;
      }
  }
  // front rows: pivots, then union of A rows and children's update rows
  T.rows_ptr.assign(static_cast<size_t>(nsn) + 1, 0);
  std::vector<int> mark(static_cast<size_t>(n), -1), pos(static_cast<size_t>(n), -1);
  std::vector<int> below;
  T.asm_ptr.assign(static_cast<size_t>(nsn) + 1, 0);
  T.asm_cp.assign(static_cast<size_t>(n) + 1, 0);
  T.rel_ptr.assign(static_cast<size_t>(nsn) + 1, 0);
  for (int s = 0; s < nsn; ++s) {
    const int c0 = T.first[s], c1 = T.first[s + 1], k = c1 - c0;
    below.clear();
    for (int c = c0; c < c1; ++c)
      for (int q = lcp[c]; q < lcp[c + 1]; ++q) {
        const int r = lri[q];
        if (r >= c1 && mark[r] != s) {
          mark[r] = s;
          below.push_back(r);
        }
      }
    for (int q = T.ch_ptr[s]; q < T.ch_ptr[s + 1]; ++q) {
      const int c = T.ch[q];
      const int* cr = T.rows.data() + T.rows_ptr[c];
      const int kc = T.first[c + 1] - T.first[c];
      for (int i = kc; i < T.f[c]; ++i) {
        const int r = cr[i];
        if (r >= c1 && mark[r] != s) {
          mark[r] = s;
          below.push_back(r);
        }
      }
    }
    std::sort(below.begin(), below.end());
    if (k + static_cast<int>(below.size()) != T.f[s])
      throw std::logic_error("supernodal: front size disagrees with column counts");
    for (int c = c0; c < c1; ++c) T.rows.push_back(c);
    T.rows.insert(T.rows.end(), below.begin(), below.end());
    T.rows_ptr[s + 1] = static_cast<int>(T.rows.size());
    const int* rs = T.rows.data() + T.rows_ptr[s];
    for (int i = 0; i < T.f[s]; ++i) pos[rs[i]] = i;
    for (int c = c0; c < c1; ++c) {
      T.asm_cp[c] = static_cast<int>(T.asm_pos.size());
      for (int q = lcp[c]; q < lcp[c + 1]; ++q) {
        T.asm_pos.push_back(pos[lri[q]] | ((c - c0) << 16));
        T.asm_slot.push_back(lsl[q]);
      }
    }
    T.asm_ptr[s + 1] = static_cast<int>(T.asm_pos.size());
    for (int q = T.ch_ptr[s]; q < T.ch_ptr[s + 1]; ++q) {
      const int c = T.ch[q];
      const int* cr = T.rows.data() + T.rows_ptr[c];
      const int kc = T.first[c + 1] - T.first[c];
      // rel entries of child c are stored contiguously at rel_ptr[c]
      (void)cr;
      (void)kc;
    }
    T.max_f = std::max(T.max_f, T.f[s]);
  }
  T.asm_cp[n] = static_cast<int>(T.asm_pos.size());
  // rel maps (need final row lists of parents)
  for (int c = 0; c < nsn; ++c) {
    const int kc = T.first[c + 1] - T.first[c];
    T.rel_ptr[c + 1] = T.rel_ptr[c] + (T.f[c] - kc);
  }
  T.rel.assign(static_cast<size_t>(T.rel_ptr[nsn]), 0);
  for (int s = 0; s < nsn; ++s) {
    const int* rs = T.rows.data() + T.rows_ptr[s];
    for (int i = 0; i < T.f[s]; ++i) pos[rs[i]] = i;
    for (int q = T.ch_ptr[s]; q < T.ch_ptr[s + 1]; ++q) {
      const int c = T.ch[q];
      const int* cr = T.rows.data() + T.rows_ptr[c];
      const int kc = T.first[c + 1] - T.first[c];
      for (int i = kc; i < T.f[c]; ++i) T.rel[T.rel_ptr[c] + i - kc] = pos[cr[i]];
    }
  }
  // tiers: wide = front above the warp limit, closed upward
  T.wide.assign(static_cast<size_t>(nsn), 0);
  for (int s = 0; s < nsn; ++s) {
    if (T.f[s] > kWarpFront || s == T.schur) T.wide[s] = 1;
    if (T.wide[s] && T.sparent[s] >= 0) T.wide[T.sparent[s]] = 1;
  }
  // storage.  Warp tier: an f x k column-major L block in lval and a compact
  // (f-k)^2 update block in upd.  Wide tier: the whole f x f column-major
  // front lives in lval (its first k columns ARE the L block, leading
  // dimension wide_ld(f) = f rounded up to even) and the update block is the
  // trailing (f-k)^2 corner of it (u_ld = wide_ld(f)).
  T.l_off.assign(static_cast<size_t>(nsn) + 1, 0);
  T.u_off.assign(static_cast<size_t>(nsn), 0);
  T.u_ld.assign(static_cast<size_t>(nsn), 0);
  long long uoff = 0;
  for (int s = 0; s < nsn; ++s) {
    const int k = T.first[s + 1] - T.first[s];
    const int fu = T.f[s] - k;
    if (T.wide[s]) {
      const long long ld = wide_ld(T.f[s]);
      T.l_off[s + 1] = T.l_off[s] + ld * T.f[s];
      T.u_off[s] = T.l_off[s] + static_cast<long long>(k) * ld + k;
      T.u_ld[s] = static_cast<int>(ld);
      T.max_wide_f = std::max(T.max_wide_f, T.f[s]);
      T.wide_front_elems += static_cast<long long>(T.f[s]) * T.f[s];
    } else {
      T.l_off[s + 1] = T.l_off[s] + static_cast<long long>(T.f[s]) * k;
      T.u_off[s] = uoff;
      T.u_ld[s] = fu;
      uoff += static_cast<long long>(fu) * fu;
    }
    T.l_off[s + 1] = (T.l_off[s + 1] + 1) & ~1LL;  // every block 16-byte aligned
  }
  T.u_total = uoff;
  // heights (supernodal), heavy child = child of maximal height
  std::vector<int> height(static_cast<size_t>(nsn), 0);
  for (int s = 0; s < nsn; ++s)
    if (T.sparent[s] >= 0)
      height[T.sparent[s]] = std::max(height[T.sparent[s]], height[s] + 1);
  for (int s = 0; s < nsn; ++s) T.sn_height = std::max(T.sn_height, height[s] + 1);
  std::vector<int> heavy(static_cast<size_t>(nsn), -1);
  for (int s = 0; s < nsn; ++s) {
    int best = -1;
    for (int q = T.ch_ptr[s]; q < T.ch_ptr[s + 1]; ++q) {
      const int c = T.ch[q];
      if (T.wide[c]) continue;
      if (best < 0 || height[c] > height[best]) best = c;
    }
    heavy[s] = T.wide[s] ? -1 : best;
  }
  // warp-tier paths: tops are narrow nodes that are not the heavy child of a
  // narrow parent; a path runs from its top down the heavy children
  std::vector<int> depth(static_cast<size_t>(nsn), 0);
  for (int s = nsn - 1; s >= 0; --s)
    depth[s] = T.sparent[s] >= 0 ? depth[T.sparent[s]] + 1 : 0;
  std::vector<int> tops;
  for (int s = 0; s < nsn; ++s) {
    if (T.wide[s]) continue;
    const int p = T.sparent[s];
    if (p < 0 || T.wide[p] || heavy[p] != s) tops.push_back(s);
  }
  std::stable_sort(tops.begin(), tops.end(),
                   [&](int a, int b) { return depth[a] > depth[b]; });
  T.path_ptr.assign(1, 0);
  std::vector<int> tmp;
  for (int t : tops) {
    tmp.clear();
    for (int s = t; s >= 0; s = heavy[s]) tmp.push_back(s);
    std::reverse(tmp.begin(), tmp.end());  // bottom -> top
    T.path_nodes.insert(T.path_nodes.end(), tmp.begin(), tmp.end());
    T.path_ptr.push_back(static_cast<int>(T.path_nodes.size()));
  }
  // Long paths that no other warp-tier path waits on (top is a root or has a
  // wide parent) are handed out first: a chain-shaped tree's spine otherwise
  // starts only after every side path has been taken.  Deadlock-free: the
  // moved paths wait only on later paths, which never wait on them, and
  // there are far fewer of them (<= kFrontPaths) than resident warps.  The
  // backward solve keeps the reverse depth order (bwd_path).
  {
    const int np = static_cast<int>(T.path_ptr.size()) - 1;
    std::vector<int> cand;
    for (int p = 0; p < np; ++p) {
      const int top = T.path_nodes[T.path_ptr[p + 1] - 1];
      const int par = T.sparent[top];
      if ((par < 0 || T.wide[par]) && T.path_ptr[p + 1] - T.path_ptr[p] >= kFrontPathLen) cand.push_back(p);
    }
    std::stable_sort(cand.begin(), cand.end(), [&](int a, int b) {
      return T.path_ptr[a + 1] - T.path_ptr[a] > T.path_ptr[b + 1] - T.path_ptr[b];
    });
    if (cand.size() > static_cast<size_t>(kFrontPaths)) cand.resize(kFrontPaths);
    std::vector<int> order(cand.begin(), cand.end()), isfront(static_cast<size_t>(np), 0);
    for (int p : cand) isfront[p] = 1;
    for (int p = 0; p < np; ++p)
      if (!isfront[p]) order.push_back(p);
    std::vector<int> nptr(1, 0), nnodes, newidx(static_cast<size_t>(np));
    for (int i = 0; i < np; ++i) {
      const int p = order[i];
      newidx[p] = i;
      nnodes.insert(nnodes.end(), T.path_nodes.begin() + T.path_ptr[p], T.path_nodes.begin() + T.path_ptr[p + 1]);
      nptr.push_back(static_cast<int>(nnodes.size()));
    }
    T.path_ptr.swap(nptr);
    T.path_nodes.swap(nnodes);
    T.bwd_path.assign(static_cast<size_t>(np), 0);
    for (int j = 0; j < np; ++j) T.bwd_path[j] = newidx[np - 1 - j];
  }
  // light-child extend-add lists of the warp tier (ldl_kernels.cu)
  {
    std::vector<int> pred(static_cast<size_t>(nsn), -1);
    for (size_t pi = 0; pi + 1 < T.path_ptr.size(); ++pi)
      for (int q = T.path_ptr[pi] + 1; q < T.path_ptr[pi + 1]; ++q)
        pred[T.path_nodes[q]] = T.path_nodes[q - 1];
    T.lt_ptr.assign(static_cast<size_t>(nsn) + 1, 0);
    T.ls_ptr.assign(static_cast<size_t>(nsn) + 1, 0);
    std::vector<std::pair<int, long long>> et, es;
    for (int s = 0; s < nsn; ++s) {
      et.clear();
      es.clear();
      if (!T.wide[s]) {
        for (int q = T.ch_ptr[s]; q < T.ch_ptr[s + 1]; ++q) {
          const int c = T.ch[q];
          if (c == pred[s]) continue;
          const int fu = T.f[c] - (T.first[c + 1] - T.first[c]);
          const int* rl = T.rel.data() + T.rel_ptr[c];
          for (int j = 0; j < fu; ++j)
            for (int i = j; i < fu; ++i)
              et.emplace_back(rl[i] | (rl[j] << 5), T.u_off[c] + i + static_cast<long long>(j) * fu);
          for (int i = 0; i < fu; ++i) es.emplace_back(rl[i], T.rel_ptr[c] + i);
        }
      }
      chunk_entries(et, T.lt_ent);
      chunk_entries(es, T.ls_ent);
      T.lt_ptr[s + 1] = static_cast<int>(T.lt_ent.size());
      T.ls_ptr[s + 1] = static_cast<int>(T.ls_ent.size());
    }
  }
  // per-path-position records of the warp tier
  T.prec.assign(T.path_nodes.size() * 16, 0);
  T.poff.assign(T.path_nodes.size() * 2, 0);
  for (size_t q = 0; q < T.path_nodes.size(); ++q) {
    const int s = T.path_nodes[q];
    const int r[16] = {s, T.first[s], T.first[s + 1] - T.first[s], T.f[s],
                       T.ch_ptr[s], T.ch_ptr[s + 1], T.lt_ptr[s], T.lt_ptr[s + 1],
                       T.asm_ptr[s], T.asm_ptr[s + 1], T.rel_ptr[s], T.rows_ptr[s],
                       T.ls_ptr[s], T.ls_ptr[s + 1], T.sparent[s], 0};
    std::copy(r, r + 16, T.prec.begin() + 16 * q);
    T.poff[2 * q] = T.l_off[s];
    T.poff[2 * q + 1] = T.u_off[s];
  }
  // wide-tier levels by wide-height (children first)
  std::vector<int> wl(static_cast<size_t>(nsn), -1);
  int nlev = 0;
  for (int s = 0; s < nsn; ++s) {
    if (!T.wide[s]) continue;
    int l = 0;
    for (int q = T.ch_ptr[s]; q < T.ch_ptr[s + 1]; ++q) {
      const int c = T.ch[q];
      if (T.wide[c]) l = std::max(l, wl[c] + 1);
    }
    wl[s] = l;
    nlev = std::max(nlev, l + 1);
  }
  T.lvl_ptr.assign(static_cast<size_t>(nlev) + 1, 0);
  for (int s = 0; s < nsn; ++s)
    if (T.wide[s]) T.lvl_ptr[wl[s] + 1]++;
  for (int l = 0; l < nlev; ++l) T.lvl_ptr[l + 1] += T.lvl_ptr[l];
  T.lvl_nodes.assign(static_cast<size_t>(T.lvl_ptr[nlev]), 0);
  {
    std::vector<int> nx(T.lvl_ptr.begin(), T.lvl_ptr.end() - 1);
    for (int s = 0; s < nsn; ++s)
      if (T.wide[s]) T.lvl_nodes[nx[wl[s]]++] = s;
  }
  // column-wise extend-add lists of the wide fronts: front column J receives
  // child column j iff rel_c[j] == J; entries in child order so the sums are
  // accumulated in the same (deterministic) order as a child-by-child pass
  T.cc_off.assign(static_cast<size_t>(nsn), -1);
  T.cc_ptr.assign(1, 0);
  {
    std::vector<std::vector<std::array<int, 2>>> colv;
    auto push = [&](int c, int j) {
      const int fu = T.f[c] - (T.first[c + 1] - T.first[c]);
      const long long ld = T.u_ld[c];
      T.cc_ubase.push_back(T.u_off[c] + j * ld + j);
      T.cc_rbase.push_back(T.rel_ptr[c] + j);
      T.cc_cnt.push_back((fu - j) | (T.wide[c] ? (1 << 30) : 0));
    };
    for (int s = 0; s < nsn; ++s) {
      if (!T.wide[s]) continue;
      T.cc_off[s] = static_cast<int>(T.cc_ptr.size()) - 1;
      colv.assign(static_cast<size_t>(T.f[s]), {});
      for (int q = T.ch_ptr[s]; q < T.ch_ptr[s + 1]; ++q) {
        const int c = T.ch[q];
        const int fu = T.f[c] - (T.first[c + 1] - T.first[c]);
        for (int j = 0; j < fu; ++j) colv[T.rel[T.rel_ptr[c] + j]].push_back({c, j});
      }
      for (int J = 0; J < T.f[s]; ++J) {
        for (const auto& e : colv[J]) push(e[0], e[1]);
        T.cc_ptr.push_back(static_cast<int>(T.cc_cnt.size()));
      }
    }
  }
  // fronts with very many children (the Schur mode's coupling front: one
  // contribution per contingency block and column): their extend-add is
  // pre-summed over groups of contributions by a wide grid (ldl_kernels.cu
  // k_cc_partial / k_uv_partial) before the front's own kernel adds the
  // group sums in group order
  T.split_ng.assign(static_cast<size_t>(nsn), 0);
  T.split_off.assign(static_cast<size_t>(nsn), 0);
  T.usplit_ng.assign(static_cast<size_t>(nsn), 0);
  T.usplit_off.assign(static_cast<size_t>(nsn), 0);
  for (int s = 0; s < nsn; ++s) {
    if (!T.wide[s] || T.f[s] > kSplitMaxF) continue;
    int maxc = 0;
    for (int J = 0; J < T.f[s]; ++J)
      maxc = std::max(maxc, T.cc_ptr[T.cc_off[s] + J + 1] - T.cc_ptr[T.cc_off[s] + J]);
    if (maxc >= kSplitMin) {
      const int ng = std::min(kSplitMaxG, (maxc + kSplitPerGroup - 1) / kSplitPerGroup);
      T.split_ng[s] = ng;
      T.split_off[s] = T.split_total;
      T.split_total += static_cast<long long>(ng) * T.f[s] * T.f[s];
    }
    const int nch = T.ch_ptr[s + 1] - T.ch_ptr[s];
    if (nch >= kSplitMin) {
      const int ng = std::min(kSplitMaxG, (nch + kSplitPerGroup - 1) / kSplitPerGroup);
      T.usplit_ng[s] = ng;
      T.usplit_off[s] = T.usplit_total;
      T.usplit_total += static_cast<long long>(ng) * T.f[s];
    }
  }
  // huge-front launch schedule: per level, assembly tasks (front, kAsmCols
  // columns); per (level, panel) the fronts that factor that panel, their
  // TRSM row blocks and the 32x32 tiles of their trailing lower triangle
  T.asm_task_ptr.assign(1, 0);
  T.lp_ptr.assign(static_cast<size_t>(nlev) + 1, 0);
  T.pn_ptr.assign(1, 0);
  T.tl_ptr.assign(1, 0);
  T.tl64_ptr.assign(1, 0);
  T.ts_ptr.assign(1, 0);
  T.dg_ptr.assign(1, 0);
  for (int l = 0; l < nlev; ++l) {
    int maxp = 0, fmax = 0;
    for (int q = T.lvl_ptr[l]; q < T.lvl_ptr[l + 1]; ++q) fmax = std::max(fmax, T.f[T.lvl_nodes[q]]);
    const bool huge = level_is_huge(fmax, T.lvl_ptr[l + 1] - T.lvl_ptr[l]);
    for (int q = T.lvl_ptr[l]; q < T.lvl_ptr[l + 1] && huge; ++q) {
      const int s = T.lvl_nodes[q];
      const int f = T.f[s], k = s == T.schur ? 0 : T.first[s + 1] - T.first[s];
      for (int cb = 0; cb < f; cb += kAsmCols) T.asm_task.push_back({s, cb, 0, 0});
      maxp = std::max(maxp, (k + kWidePanel - 1) / kWidePanel);
    }
    // the tallest fronts' columns first (more rows per task; tasks are independent)
    std::stable_sort(T.asm_task.begin() + T.asm_task_ptr.back(), T.asm_task.end(),
                     [&](const std::array<int, 4>& a, const std::array<int, 4>& b) { return T.f[a[0]] > T.f[b[0]]; });
    T.asm_task_ptr.push_back(static_cast<int>(T.asm_task.size()));
    for (int p = 0; p < maxp; ++p) {
      for (int q = T.lvl_ptr[l]; q < T.lvl_ptr[l + 1]; ++q) {
        const int s = T.lvl_nodes[q];
        const int f = T.f[s], k = s == T.schur ? 0 : T.first[s + 1] - T.first[s];
        if (k <= p * kWidePanel) continue;
        const int p1 = std::min((p + 1) * kWidePanel, k);
        const int mt = f - p1;
        const int di = static_cast<int>(T.dg_nodes.size()) - T.dg_ptr.back();
        T.dg_nodes.push_back(s);
        const int nrb = std::max(1, (mt + kPanelRows - 1) / kPanelRows);  // >= 1: the diag
        for (int rb = 0; rb < nrb; ++rb) T.pn_tasks.push_back({s, rb, di, 0});
        const int nt = (mt + kUpdTile - 1) / kUpdTile;
        // the next panel's columns (lookahead strip) apart from the rest
        const bool more = p1 < k;
        for (int ti = 0; ti < nt; ++ti)
          for (int tj = 0; tj <= ti; ++tj)
            (more && tj == 0 ? T.tiles_s : T.tiles).push_back({s, p1 + ti * kUpdTile, p1 + tj * kUpdTile, p});
        {  // the rest region (columns from p1, or p1 + 32 when the next panel takes that strip) in 64x64 tiles
          const int c0 = p1 + (more ? kUpdTile : 0);
          for (int q0 = c0; q0 < f; q0 += 2 * kUpdTile)
            for (int r0 = q0; r0 < f; r0 += 2 * kUpdTile) T.tiles64.push_back({s, r0, q0, p});
        }
        T.wide_update_flops += 2LL * (p1 - p * kWidePanel) * mt * (mt + 1) / 2;
      }
      T.pn_ptr.push_back(static_cast<int>(T.pn_tasks.size()));
      T.tl_ptr.push_back(static_cast<int>(T.tiles.size()));
      T.tl64_ptr.push_back(static_cast<int>(T.tiles64.size()));
      T.ts_ptr.push_back(static_cast<int>(T.tiles_s.size()));
      T.dg_ptr.push_back(static_cast<int>(T.dg_nodes.size()));
      T.max_dg = std::max(T.max_dg, T.dg_ptr.back() - T.dg_ptr[T.dg_ptr.size() - 2]);
    }
    T.lp_ptr[l + 1] = T.lp_ptr[l] + maxp;
  }
  return T;
}

}  // namespace nclb

namespace nclb {

// Invariants of the warp-tier schedule (tests/test_warp_schedule.py).
std::string check_warp_schedule(const Supernodal& T) {
  const int nsn = T.nsn;
  const int np = static_cast<int>(T.path_ptr.size()) - 1;
  std::vector<int> path_of(static_cast<size_t>(nsn), -1), pos_of(static_cast<size_t>(nsn), -1);
  for (int p = 0; p < np; ++p)
    for (int q = T.path_ptr[p]; q < T.path_ptr[p + 1]; ++q) {
      const int s = T.path_nodes[q];
      if (s < 0 || s >= nsn || T.wide[s]) return "path holds a wide or invalid node";
      if (path_of[s] >= 0) return "node on two paths";
      path_of[s] = p;
      pos_of[s] = q;
      if (q > T.path_ptr[p] && T.sparent[T.path_nodes[q - 1]] != s) return "path step is not child -> parent";
    }
  for (int s = 0; s < nsn; ++s)
    if (!T.wide[s] && path_of[s] < 0) return "warp node on no path";
  // hand-out order: front paths first (tops without a warp-tier parent), the
  // others after every path they wait on
  int nfront = 0;
  while (nfront < np) {
    const int top = T.path_nodes[T.path_ptr[nfront + 1] - 1];
    const int par = T.sparent[top];
    if (T.path_ptr[nfront + 1] - T.path_ptr[nfront] < kFrontPathLen || !(par < 0 || T.wide[par])) break;
    ++nfront;
  }
  if (nfront > kFrontPaths) return "too many front paths";
  for (int p = 0; p < np; ++p)
    for (int q = T.path_ptr[p]; q < T.path_ptr[p + 1]; ++q) {
      const int s = T.path_nodes[q];
      const int pred = q > T.path_ptr[p] ? T.path_nodes[q - 1] : -1;
      for (int e = T.ch_ptr[s]; e < T.ch_ptr[s + 1]; ++e) {
        const int c = T.ch[e];
        if (c == pred) continue;
        const int pc = path_of[c];
        if (pc < 0 || T.path_nodes[T.path_ptr[pc + 1] - 1] != c) return "light child is not a path top";
        if (pc < nfront) return "a front path is some node's light child";
        if (p >= nfront && pc > p) return "path handed out before a light child's path";
      }
    }
  // backward order: a permutation, each path after the path of its top's parent
  if (static_cast<int>(T.bwd_path.size()) != np) return "bwd_path size";
  std::vector<int> bpos(static_cast<size_t>(np), -1);
  for (int j = 0; j < np; ++j) {
    const int p = T.bwd_path[j];
    if (p < 0 || p >= np || bpos[p] >= 0) return "bwd_path is not a permutation";
    bpos[p] = j;
  }
  for (int p = 0; p < np; ++p) {
    const int par = T.sparent[T.path_nodes[T.path_ptr[p + 1] - 1]];
    if (par >= 0 && !T.wide[par] && bpos[path_of[par]] > bpos[p]) return "bwd: child path before its parent's";
  }
  // light-child chunks: distinct destinations per chunk, per destination in
  // child order, exactly the light children's entries
  for (int s = 0; s < nsn; ++s) {
    for (int which = 0; which < 2; ++which) {
      const std::vector<int>& ptr = which ? T.ls_ptr : T.lt_ptr;
      const std::vector<long long>& ent = which ? T.ls_ent : T.lt_ent;
      const int b = ptr[s], e = ptr[s + 1];
      if ((e - b) % 32) return "chunk list not padded to 32";
      std::vector<std::pair<int, long long>> want;
      if (!T.wide[s]) {
        const int q = pos_of[s];
        const int pred = q > T.path_ptr[path_of[s]] ? T.path_nodes[q - 1] : -1;
        for (int k = T.ch_ptr[s]; k < T.ch_ptr[s + 1]; ++k) {
          const int c = T.ch[k];
          if (c == pred) continue;
          const int fu = T.f[c] - (T.first[c + 1] - T.first[c]);
          const int* rl = T.rel.data() + T.rel_ptr[c];
          if (which) {
            for (int i = 0; i < fu; ++i) want.emplace_back(rl[i], T.rel_ptr[c] + i);
          } else {
            for (int j = 0; j < fu; ++j)
              for (int i = j; i < fu; ++i)
                want.emplace_back(rl[i] | (rl[j] << 5), T.u_off[c] + i + static_cast<long long>(j) * fu);
          }
        }
      }
      std::vector<std::pair<int, long long>> got;
      for (int c0 = b; c0 < e; c0 += 32) {
        std::vector<int> seen;
        for (int t = c0; t < c0 + 32; ++t) {
          if (ent[t] < 0) continue;
          const int dst = static_cast<int>(ent[t] >> 48);
          if (std::find(seen.begin(), seen.end(), dst) != seen.end()) return "destination twice in a chunk";
          seen.push_back(dst);
          got.emplace_back(dst, ent[t] & ((1LL << 48) - 1));
        }
      }
      // per destination, the sources in the order the children contribute them
      auto by_dst = [](std::vector<std::pair<int, long long>> v) {
        std::stable_sort(v.begin(), v.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
        return v;
      };
      if (by_dst(got) != by_dst(want)) return "chunk entries differ from the light children's";
    }
  }
  // path-position records
  if (T.prec.size() != 16 * T.path_nodes.size() || T.poff.size() != 2 * T.path_nodes.size()) return "record sizes";
  for (size_t q = 0; q < T.path_nodes.size(); ++q) {
    const int s = T.path_nodes[q];
    const int* r = T.prec.data() + 16 * q;
    if (r[0] != s || r[1] != T.first[s] || r[2] != T.first[s + 1] - T.first[s] || r[3] != T.f[s] ||
        r[4] != T.ch_ptr[s] || r[5] != T.ch_ptr[s + 1] || r[6] != T.lt_ptr[s] || r[7] != T.lt_ptr[s + 1] ||
        r[8] != T.asm_ptr[s] || r[9] != T.asm_ptr[s + 1] || r[10] != T.rel_ptr[s] || r[11] != T.rows_ptr[s] ||
        r[12] != T.ls_ptr[s] || r[13] != T.ls_ptr[s + 1] || r[14] != T.sparent[s] ||
        T.poff[2 * q] != T.l_off[s] || T.poff[2 * q + 1] != T.u_off[s])
      return "path record mismatch";
  }
  return "";
}

}  // namespace nclb
