/*
 * ncl_oracle.c -- TEST INFRASTRUCTURE ONLY (see ncl_oracle.h).
 *
 * Plain-C restatement of the reference's per-Newton-step path:
 *   proj/src/sparse.cpp   (triplets, matvec, AMD call, analyze, factorize,
 *                          ldl_solve, solve_refined)
 *   Eigen AMDOrdering      (Eigen/src/OrderingMethods/Amd.h; external,
 *                          restated: see orc_amd_full_pattern)
 *   proj/src/kkt.cpp      (KktContext, refill, build_rhs, recover, solve,
 *                          recover_bound_duals, barrier_kkt_residual)
 *   proj/src/ipm.cpp      (fraction_to_boundary, solve_prepared input,
 *                          clip_duals)
 *   proj/src/solver.cpp   (outer schedule, init_multipliers)
 * Compiled with -O2 -ffp-contract=off so no FMA contraction happens (the
 * reference is built with -Wall -Wextra only, x86-64 default: SSE2, no FMA;
 * proj/src/CMakeLists.txt:13).
 */
#include "ncl_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define MAXI(a, b) ((a) > (b) ? (a) : (b))
#define MINI(a, b) ((a) < (b) ? (a) : (b))

static void* xcalloc(size_t n, size_t s) {
  void* p = calloc(n ? n : 1, s);
  if (!p) abort();
  return p;
}

/* ------------------------------------------------------------------------ */
/* sym_from_triplets: proj/src/sparse.cpp:33-68.  Upper entries mirrored,
 * sorted by (col,row), duplicates summed in sorted order.  The reference uses
 * std::sort (unstable) on (col,row) keys; equal keys are summed in an
 * unspecified order there.  We break ties by input position (a stable order);
 * every production call site in the reference has either zero values
 * (kkt.cpp:93) or unique keys (solver.cpp:55-79), where the two agree. */
typedef struct {
  int c, r, k;
  double v;
} trip_t;

static int trip_cmp(const void* a, const void* b) {
  const trip_t* x = (const trip_t*)a;
  const trip_t* y = (const trip_t*)b;
  if (x->c != y->c) return x->c < y->c ? -1 : 1;
  if (x->r != y->r) return x->r < y->r ? -1 : 1;
  return x->k < y->k ? -1 : (x->k > y->k);
}

int orc_sym_from_triplets(int n, int nt, const int* rows, const int* cols,
                          const double* vals, orc_csc* out) {
  trip_t* e = (trip_t*)xcalloc((size_t)nt, sizeof(trip_t));
  for (int k = 0; k < nt; ++k) {
    int i = rows[k], j = cols[k];
    if (i < 0 || i >= n || j < 0 || j >= n) {
      free(e);
      return -1;
    }
    if (i < j) {
      int t = i;
      i = j;
      j = t;
    }
    e[k].c = j;
    e[k].r = i;
    e[k].k = k;
    e[k].v = vals ? vals[k] : 0.0;
  }
  qsort(e, (size_t)nt, sizeof(trip_t), trip_cmp);
  out->n = n;
  out->col_ptr = (int*)xcalloc((size_t)n + 1, sizeof(int));
  out->row_ind = (int*)xcalloc((size_t)nt, sizeof(int));
  out->val = (double*)xcalloc((size_t)nt, sizeof(double));
  int nnz = 0;
  for (int k = 0; k < nt; ++k) {
    if (k > 0 && e[k].c == e[k - 1].c && e[k].r == e[k - 1].r) {
      out->val[nnz - 1] += e[k].v;
    } else {
      out->col_ptr[e[k].c + 1]++;
      out->row_ind[nnz] = e[k].r;
      out->val[nnz] = e[k].v;
      nnz++;
    }
  }
  for (int j = 0; j < n; ++j) out->col_ptr[j + 1] += out->col_ptr[j];
  out->nnz = nnz;
  free(e);
  return 0;
}

void orc_csc_free(orc_csc* A) {
  free(A->col_ptr);
  free(A->row_ind);
  free(A->val);
  memset(A, 0, sizeof(*A));
}

/* sym_matvec: sparse.cpp:70-79 (y += A x, lower storage) */
void orc_sym_matvec(const orc_csc* A, const double* x, double* y) {
  for (int j = 0; j < A->n; ++j)
    for (int p = A->col_ptr[j]; p < A->col_ptr[j + 1]; ++p) {
      const int i = A->row_ind[p];
      const double v = A->val[p];
      y[i] += v * x[j];
      if (i != j) y[j] += v * x[i];
    }
}

/* ------------------------------------------------------------------------ */
/* Eigen AMDOrdering<int> restated (Eigen/src/OrderingMethods/Amd.h,
 * "minimum_degree_ordering"; CSparse cs_amd lineage, Davis).  Differences from
 * CSparse that Eigen introduces and that this restatement keeps:
 *   - the input is the pattern of A^T + A WITH its diagonal (Eigen does not
 *     prune it), so initial degrees count the diagonal entry;
 *   - a node with degree 1 and a structural diagonal is empty (own root);
 *   - a node with degree > dense OR without a structural diagonal is
 *     absorbed into the dummy element n (ordered last).
 * Input: full symmetric pattern, CSC, rows sorted, diagonal present where
 * structural.  Output perm[k] = node eliminated k-th (k < n). */
static int amd_flip(int i) { return -i - 2; }

static int cs_wclear(int mark, int lemax, int* w, int n) {
  if (mark < 2 || (mark + lemax < 0)) {
    for (int k = 0; k < n; k++)
      if (w[k] != 0) w[k] = 1;
    mark = 2;
  }
  return mark;
}

static int cs_tdfs(int j, int k, int* head, const int* next, int* post,
                   int* stack) {
  int i, p, top = 0;
  stack[0] = j;
  while (top >= 0) {
    p = stack[top];
    i = head[p];
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

int orc_amd_full_pattern(int n, const int* Ap, const int* Ai, int* perm_out) {
  int d, dk, dext, lemax = 0, e, elenk, eln, i, j, k, k1, k2, k3, jlast, ln,
      dense, nzmax, mindeg = 0, nvi, nvj, nvk, mark, wnvi, ok, nel = 0, p, p1,
      p2, p3, p4, pj, pk, pk1, pk2, pn, q, t, h;
  if (n == 0) return 0;
  dense = MAXI(16, (int)(10 * sqrt((double)n)));
  dense = MINI(n - 2, dense);
  int cnz = Ap[n];
  t = cnz + cnz / 5 + 2 * n;
  int* Cp = (int*)xcalloc((size_t)n + 1, sizeof(int));
  int* Ci = (int*)xcalloc((size_t)t, sizeof(int));
  memcpy(Cp, Ap, sizeof(int) * ((size_t)n + 1));
  memcpy(Ci, Ai, sizeof(int) * (size_t)cnz);
  int* W = (int*)xcalloc(8 * ((size_t)n + 1), sizeof(int));
  int* P = (int*)xcalloc((size_t)n + 1, sizeof(int));
  int* len = W;
  int* nv = W + (n + 1);
  int* next = W + 2 * (n + 1);
  int* head = W + 3 * (n + 1);
  int* elen = W + 4 * (n + 1);
  int* degree = W + 5 * (n + 1);
  int* w = W + 6 * (n + 1);
  int* hhead = W + 7 * (n + 1);
  int* last = P; /* P used as workspace for last */

  for (k = 0; k < n; k++) len[k] = Cp[k + 1] - Cp[k];
  len[n] = 0;
  nzmax = t;
  for (i = 0; i <= n; i++) {
    head[i] = -1;
    last[i] = -1;
    next[i] = -1;
    hhead[i] = -1;
    nv[i] = 1;
    w[i] = 1;
    elen[i] = 0;
    degree[i] = len[i];
  }
  mark = cs_wclear(0, 0, w, n);

  for (i = 0; i < n; i++) {
    int has_diag = 0;
    for (p = Cp[i]; p < Cp[i + 1]; ++p)
      if (Ci[p] == i) {
        has_diag = 1;
        break;
      }
    d = degree[i];
    if (d == 1 && has_diag) {
      elen[i] = -2;
      nel++;
      Cp[i] = -1;
      w[i] = 0;
    } else if (d > dense || !has_diag) {
      nv[i] = 0;
      elen[i] = -1;
      nel++;
      Cp[i] = amd_flip(n);
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
    /* select node of minimum approximate degree */
    for (k = -1; mindeg < n && (k = head[mindeg]) == -1; mindeg++) {
    }
    if (next[k] != -1) last[next[k]] = -1;
    head[mindeg] = next[k];
    elenk = elen[k];
    nvk = nv[k];
    nel += nvk;

    /* garbage collection */
    if (elenk > 0 && cnz + mindeg >= nzmax) {
      for (j = 0; j < n; j++) {
        if ((p = Cp[j]) >= 0) {
          Cp[j] = Ci[p];
          Ci[p] = amd_flip(j);
        }
      }
      for (q = 0, p = 0; p < cnz;) {
        if ((j = amd_flip(Ci[p++])) >= 0) {
          Ci[q] = Cp[j];
          Cp[j] = q++;
          for (k3 = 0; k3 < len[j] - 1; k3++) Ci[q++] = Ci[p++];
        }
      }
      cnz = q;
    }

    /* construct new element */
    dk = 0;
    nv[k] = -nvk;
    p = Cp[k];
    pk1 = (elenk == 0) ? p : cnz;
    pk2 = pk1;
    for (k1 = 1; k1 <= elenk + 1; k1++) {
      if (k1 > elenk) {
        e = k;
        pj = p;
        ln = len[k] - elenk;
      } else {
        e = Ci[p++];
        pj = Cp[e];
        ln = len[e];
      }
      for (k2 = 1; k2 <= ln; k2++) {
        i = Ci[pj++];
        if ((nvi = nv[i]) <= 0) continue;
        dk += nvi;
        nv[i] = -nvi;
        Ci[pk2++] = i;
        if (next[i] != -1) last[next[i]] = last[i];
        if (last[i] != -1) {
          next[last[i]] = next[i];
        } else {
          head[degree[i]] = next[i];
        }
      }
      if (e != k) {
        Cp[e] = amd_flip(k);
        w[e] = 0;
      }
    }
    if (elenk != 0) cnz = pk2;
    degree[k] = dk;
    Cp[k] = pk1;
    len[k] = pk2 - pk1;
    elen[k] = -2;

    /* find set differences */
    mark = cs_wclear(mark, lemax, w, n);
    for (pk = pk1; pk < pk2; pk++) {
      i = Ci[pk];
      if ((eln = elen[i]) <= 0) continue;
      nvi = -nv[i];
      wnvi = mark - nvi;
      for (p = Cp[i]; p <= Cp[i] + eln - 1; p++) {
        e = Ci[p];
        if (w[e] >= mark) {
          w[e] -= nvi;
        } else if (w[e] != 0) {
          w[e] = degree[e] + wnvi;
        }
      }
    }

    /* degree update */
    for (pk = pk1; pk < pk2; pk++) {
      i = Ci[pk];
      p1 = Cp[i];
      p2 = p1 + elen[i] - 1;
      pn = p1;
      for (h = 0, d = 0, p = p1; p <= p2; p++) {
        e = Ci[p];
        if (w[e] != 0) {
          dext = w[e] - mark;
          if (dext > 0) {
            d += dext;
            Ci[pn++] = e;
            h += e;
          } else {
            Cp[e] = amd_flip(k);
            w[e] = 0;
          }
        }
      }
      elen[i] = pn - p1 + 1;
      p3 = pn;
      p4 = p1 + len[i];
      for (p = p2 + 1; p < p4; p++) {
        j = Ci[p];
        if ((nvj = nv[j]) <= 0) continue;
        d += nvj;
        Ci[pn++] = j;
        h += j;
      }
      if (d == 0) {
        Cp[i] = amd_flip(k);
        nvi = -nv[i];
        dk -= nvi;
        nvk += nvi;
        nel += nvi;
        nv[i] = 0;
        elen[i] = -1;
      } else {
        degree[i] = MINI(degree[i], d);
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
    lemax = MAXI(lemax, dk);
    mark = cs_wclear(mark + lemax, lemax, w, n);

    /* supernode detection */
    for (pk = pk1; pk < pk2; pk++) {
      i = Ci[pk];
      if (nv[i] >= 0) continue;
      h = last[i];
      i = hhead[h];
      hhead[h] = -1;
      for (; i != -1 && next[i] != -1; i = next[i], mark++) {
        ln = len[i];
        eln = elen[i];
        for (p = Cp[i] + 1; p <= Cp[i] + ln - 1; p++) w[Ci[p]] = mark;
        jlast = i;
        for (j = next[i]; j != -1;) {
          ok = (len[j] == ln) && (elen[j] == eln);
          for (p = Cp[j] + 1; ok && p <= Cp[j] + ln - 1; p++) {
            if (w[Ci[p]] != mark) ok = 0;
          }
          if (ok) {
            Cp[j] = amd_flip(i);
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

    /* finalize new element */
    for (p = pk1, pk = pk1; pk < pk2; pk++) {
      i = Ci[pk];
      if ((nvi = -nv[i]) <= 0) continue;
      nv[i] = nvi;
      d = degree[i] + dk - nvi;
      d = MINI(d, n - nel - nvi);
      if (head[d] != -1) last[head[d]] = i;
      next[i] = head[d];
      last[i] = -1;
      head[d] = i;
      mindeg = MINI(mindeg, d);
      degree[i] = d;
      Ci[p++] = i;
    }
    nv[k] = nvk;
    if ((len[k] = p - pk1) == 0) {
      Cp[k] = -1;
      w[k] = 0;
    }
    if (elenk != 0) cnz = p;
  }

  /* postordering */
  for (i = 0; i < n; i++) Cp[i] = amd_flip(Cp[i]);
  for (j = 0; j <= n; j++) head[j] = -1;
  for (j = n; j >= 0; j--) {
    if (nv[j] > 0) continue;
    next[j] = head[Cp[j]];
    head[Cp[j]] = j;
  }
  for (e = n; e >= 0; e--) {
    if (nv[e] <= 0) continue;
    if (Cp[e] != -1) {
      next[e] = head[Cp[e]];
      head[Cp[e]] = e;
    }
  }
  for (k = 0, i = 0; i <= n; i++) {
    if (Cp[i] == -1) k = cs_tdfs(i, k, head, next, P, w);
  }
  memcpy(perm_out, P, sizeof(int) * (size_t)n);
  free(Cp);
  free(Ci);
  free(W);
  free(P);
  return 0;
}

/* amd_order: sparse.cpp:81-100.  Full symmetric pattern (both triangles plus
 * the stored diagonal), compressed with sorted rows as Eigen's
 * setFromTriplets + makeCompressed produce, then ordering_helper_at_plus_a
 * (pattern of M^T + M == M here) and the minimum-degree ordering above. */
int orc_amd_order(const orc_csc* A, int* perm) {
  const int n = A->n;
  int* cnt = (int*)xcalloc((size_t)n + 1, sizeof(int));
  for (int j = 0; j < n; ++j)
    for (int p = A->col_ptr[j]; p < A->col_ptr[j + 1]; ++p) {
      const int i = A->row_ind[p];
      cnt[j]++;
      if (i != j) cnt[i]++;
    }
  int* Mp = (int*)xcalloc((size_t)n + 1, sizeof(int));
  for (int j = 0; j < n; ++j) Mp[j + 1] = Mp[j] + cnt[j];
  int* Mi = (int*)xcalloc((size_t)Mp[n], sizeof(int));
  int* nx = (int*)xcalloc((size_t)n + 1, sizeof(int));
  memcpy(nx, Mp, sizeof(int) * (size_t)n);
  /* rows sorted per column: column i first receives its mirrored rows r < i
   * (scanning source columns r ascending), then its own lower part. */
  for (int r = 0; r < n; ++r)
    for (int p = A->col_ptr[r]; p < A->col_ptr[r + 1]; ++p) {
      const int i = A->row_ind[p];
      if (i != r) Mi[nx[i]++] = r; /* column i gets row r (< i) */
    }
  for (int j = 0; j < n; ++j)
    for (int p = A->col_ptr[j]; p < A->col_ptr[j + 1]; ++p)
      Mi[nx[j]++] = A->row_ind[p];
  int rc = orc_amd_full_pattern(n, Mp, Mi, perm);
  free(cnt);
  free(Mp);
  free(Mi);
  free(nx);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* analyze_with_permutation: sparse.cpp:102-176 */
typedef struct {
  int r, o;
} pair_t;
static int pair_cmp(const void* a, const void* b) {
  const pair_t* x = (const pair_t*)a;
  const pair_t* y = (const pair_t*)b;
  if (x->r != y->r) return x->r < y->r ? -1 : 1;
  return x->o < y->o ? -1 : (x->o > y->o);
}

static int validate_lower_csc(const orc_csc* A) {
  if (A->n < 0) return -1;
  for (int j = 0; j < A->n; ++j) {
    if (A->col_ptr[j] > A->col_ptr[j + 1]) return -1;
    for (int p = A->col_ptr[j]; p < A->col_ptr[j + 1]; ++p) {
      if (A->row_ind[p] < j || A->row_ind[p] >= A->n) return -1;
      if (p > A->col_ptr[j] && A->row_ind[p] <= A->row_ind[p - 1]) return -1;
    }
  }
  return 0;
}

int orc_analyze_with_permutation(const orc_csc* A, const int* perm,
                                 orc_symbolic* S) {
  if (validate_lower_csc(A)) return -1;
  const int n = A->n;
  memset(S, 0, sizeof(*S));
  S->n = n;
  S->perm = (int*)xcalloc((size_t)n, sizeof(int));
  S->iperm = (int*)xcalloc((size_t)n, sizeof(int));
  for (int k = 0; k < n; ++k) S->iperm[k] = -1;
  for (int k = 0; k < n; ++k) {
    if (perm[k] < 0 || perm[k] >= n || S->iperm[perm[k]] != -1) {
      orc_symbolic_free(S);
      return -1;
    }
    S->perm[k] = perm[k];
    S->iperm[perm[k]] = k;
  }
  const int nnz = A->col_ptr[n];
  S->nnz = nnz;
  S->a_col_ptr = (int*)xcalloc((size_t)n + 1, sizeof(int));
  int* colcount = (int*)xcalloc((size_t)n, sizeof(int));
  for (int j = 0; j < n; ++j)
    for (int p = A->col_ptr[j]; p < A->col_ptr[j + 1]; ++p) {
      const int pi = S->iperm[A->row_ind[p]];
      const int pj = S->iperm[j];
      colcount[MAXI(pi, pj)]++;
    }
  for (int c = 0; c < n; ++c)
    S->a_col_ptr[c + 1] = S->a_col_ptr[c] + colcount[c];
  S->a_row_ind = (int*)xcalloc((size_t)nnz, sizeof(int));
  int* orig_of_slot = (int*)xcalloc((size_t)nnz, sizeof(int));
  int* next = (int*)xcalloc((size_t)n + 1, sizeof(int));
  memcpy(next, S->a_col_ptr, sizeof(int) * (size_t)n);
  for (int j = 0; j < n; ++j)
    for (int p = A->col_ptr[j]; p < A->col_ptr[j + 1]; ++p) {
      const int pi = S->iperm[A->row_ind[p]];
      const int pj = S->iperm[j];
      const int c = MAXI(pi, pj);
      const int slot = next[c]++;
      S->a_row_ind[slot] = MINI(pi, pj);
      orig_of_slot[slot] = p;
    }
  S->a_map = (int*)xcalloc((size_t)nnz, sizeof(int));
  pair_t* buf = (pair_t*)xcalloc((size_t)n + 1, sizeof(pair_t));
  for (int c = 0; c < n; ++c) {
    const int b = S->a_col_ptr[c], e = S->a_col_ptr[c + 1];
    for (int s = b; s < e; ++s) {
      buf[s - b].r = S->a_row_ind[s];
      buf[s - b].o = orig_of_slot[s];
    }
    qsort(buf, (size_t)(e - b), sizeof(pair_t), pair_cmp);
    for (int k = 0; k < e - b; ++k) {
      S->a_row_ind[b + k] = buf[k].r;
      S->a_map[buf[k].o] = b + k;
    }
  }
  /* etree + column counts (up-looking reach), sparse.cpp:157-175 */
  S->parent = (int*)xcalloc((size_t)n, sizeof(int));
  int* lnz = (int*)xcalloc((size_t)n, sizeof(int));
  int* flag = (int*)xcalloc((size_t)n, sizeof(int));
  for (int k = 0; k < n; ++k) {
    S->parent[k] = -1;
    flag[k] = -1;
  }
  for (int k = 0; k < n; ++k) {
    flag[k] = k;
    for (int p = S->a_col_ptr[k]; p < S->a_col_ptr[k + 1]; ++p) {
      int i = S->a_row_ind[p];
      if (i >= k) continue;
      while (flag[i] != k) {
        if (S->parent[i] == -1) S->parent[i] = k;
        lnz[i]++;
        flag[i] = k;
        i = S->parent[i];
      }
    }
  }
  S->lcol_ptr = (int*)xcalloc((size_t)n + 1, sizeof(int));
  for (int c = 0; c < n; ++c) S->lcol_ptr[c + 1] = S->lcol_ptr[c] + lnz[c];
  free(colcount);
  free(orig_of_slot);
  free(next);
  free(buf);
  free(lnz);
  free(flag);
  return 0;
}

int orc_analyze(const orc_csc* A, orc_symbolic* S) {
  int* perm = (int*)xcalloc((size_t)A->n, sizeof(int));
  orc_amd_order(A, perm);
  int rc = orc_analyze_with_permutation(A, perm, S);
  free(perm);
  return rc;
}

void orc_symbolic_free(orc_symbolic* S) {
  free(S->perm);
  free(S->iperm);
  free(S->parent);
  free(S->lcol_ptr);
  free(S->a_col_ptr);
  free(S->a_row_ind);
  free(S->a_map);
  memset(S, 0, sizeof(*S));
}

/* ------------------------------------------------------------------------ */
/* factorize: sparse.cpp:182-256 (up-looking LDL^T with static pivoting) */
int orc_factorize(const orc_symbolic* S, const orc_csc* A, double pivot_eps,
                  orc_factors* F) {
  const int n = S->n;
  if (A->n != n || A->col_ptr[n] != S->nnz) return -1;
  memset(F, 0, sizeof(*F));
  F->n = n;
  F->pivot_eps = pivot_eps;
  const int lnz = S->lcol_ptr[n];
  F->lcol_ptr = (int*)xcalloc((size_t)n + 1, sizeof(int));
  memcpy(F->lcol_ptr, S->lcol_ptr, sizeof(int) * ((size_t)n + 1));
  F->lrow_ind = (int*)xcalloc((size_t)lnz, sizeof(int));
  F->lval = (double*)xcalloc((size_t)lnz, sizeof(double));
  F->d = (double*)xcalloc((size_t)n, sizeof(double));

  double* ax = (double*)xcalloc((size_t)S->nnz, sizeof(double));
  for (int p = 0; p < A->col_ptr[n]; ++p) ax[S->a_map[p]] = A->val[p];
  double* y = (double*)xcalloc((size_t)n, sizeof(double));
  int* pattern = (int*)xcalloc((size_t)n, sizeof(int));
  int* stack = (int*)xcalloc((size_t)n, sizeof(int));
  int* flag = (int*)xcalloc((size_t)n, sizeof(int));
  int* lfill = (int*)xcalloc((size_t)n, sizeof(int));
  for (int k = 0; k < n; ++k) flag[k] = -1;
  int rc_ok = 1;
  for (int k = 0; k < n; ++k) {
    int top = n;
    flag[k] = k;
    double dk = 0.0;
    for (int p = S->a_col_ptr[k]; p < S->a_col_ptr[k + 1]; ++p) {
      int i = S->a_row_ind[p];
      if (i == k) {
        dk += ax[p];
        continue;
      }
      y[i] = ax[p];
      int len = 0;
      while (flag[i] != k) {
        stack[len++] = i;
        flag[i] = k;
        i = S->parent[i];
      }
      while (len > 0) pattern[--top] = stack[--len];
    }
    for (int p = top; p < n; ++p) {
      const int i = pattern[p];
      const double yi = y[i];
      y[i] = 0.0;
      const int q0 = F->lcol_ptr[i];
      const int q1 = q0 + lfill[i];
      for (int q = q0; q < q1; ++q) y[F->lrow_ind[q]] -= F->lval[q] * yi;
      const double lki = yi / F->d[i];
      dk -= lki * yi;
      F->lrow_ind[q1] = k;
      F->lval[q1] = lki;
      lfill[i]++;
    }
    if (fabs(dk) < pivot_eps) {
      dk = (dk >= 0.0) ? pivot_eps : -pivot_eps;
      F->perturbed++;
    }
    if (!isfinite(dk) || dk == 0.0) {
      rc_ok = 0;
      break;
    }
    F->d[k] = dk;
    if (dk > 0.0)
      F->n_pos++;
    else
      F->n_neg++;
  }
  if (rc_ok)
    for (int q = 0; q < lnz; ++q)
      if (!isfinite(F->lval[q])) {
        rc_ok = 0;
        break;
      }
  F->ok = rc_ok;
  free(ax);
  free(y);
  free(pattern);
  free(stack);
  free(flag);
  free(lfill);
  return 0;
}

void orc_factors_free(orc_factors* F) {
  free(F->lcol_ptr);
  free(F->lrow_ind);
  free(F->lval);
  free(F->d);
  memset(F, 0, sizeof(*F));
}

/* ldl_solve: sparse.cpp:258-276 */
void orc_ldl_solve(const orc_symbolic* S, const orc_factors* F,
                   const double* b, double* x) {
  const int n = S->n;
  double* w = (double*)xcalloc((size_t)n, sizeof(double));
  for (int k = 0; k < n; ++k) w[k] = b[S->perm[k]];
  for (int j = 0; j < n; ++j) {
    const double wj = w[j];
    for (int p = F->lcol_ptr[j]; p < F->lcol_ptr[j + 1]; ++p)
      w[F->lrow_ind[p]] -= F->lval[p] * wj;
  }
  for (int j = 0; j < n; ++j) w[j] /= F->d[j];
  for (int j = n - 1; j >= 0; --j) {
    double wj = w[j];
    for (int p = F->lcol_ptr[j]; p < F->lcol_ptr[j + 1]; ++p)
      wj -= F->lval[p] * w[F->lrow_ind[p]];
    w[j] = wj;
  }
  for (int k = 0; k < n; ++k) x[S->perm[k]] = w[k];
  free(w);
}

/* solve_refined: sparse.cpp:278-322 */
static double residual_into(const orc_csc* A, const double* b,
                            const double* x, double* r) {
  const int n = A->n;
  for (int i = 0; i < n; ++i) r[i] = -b[i];
  orc_sym_matvec(A, x, r);
  double nrm = 0.0;
  for (int i = 0; i < n; ++i) {
    r[i] = -r[i];
    nrm = fmax(nrm, fabs(r[i]));
  }
  return nrm;
}

int orc_solve_refined(const orc_symbolic* S, const orc_factors* F,
                      const orc_csc* A, const double* b, int max_ref,
                      double tol, double* xout, double* rel_residual,
                      int* converged) {
  const int n = A->n;
  double* x = (double*)xcalloc((size_t)n, sizeof(double));
  orc_ldl_solve(S, F, b, x);
  double bnorm = 0.0;
  for (int i = 0; i < n; ++i) bnorm = fmax(bnorm, fabs(b[i]));
  const double denom = (bnorm > 0.0) ? bnorm : 1.0;
  double* r = (double*)xcalloc((size_t)n, sizeof(double));
  double* dx = (double*)xcalloc((size_t)n, sizeof(double));
  double* xn = (double*)xcalloc((size_t)n, sizeof(double));
  double* rn = (double*)xcalloc((size_t)n, sizeof(double));
  double res = residual_into(A, b, x, r);
  double prev = res;
  int stagnant = 0, steps = 0;
  while (steps < max_ref && res > tol * denom) {
    orc_ldl_solve(S, F, r, dx);
    for (int i = 0; i < n; ++i) xn[i] = x[i] + dx[i];
    const double res_new = residual_into(A, b, xn, rn);
    if (!isfinite(res_new) || res_new >= res) break;
    double* t = x;
    x = xn;
    xn = t;
    t = r;
    r = rn;
    rn = t;
    steps++;
    stagnant = (res_new > 0.5 * prev) ? stagnant + 1 : 0;
    prev = res_new;
    res = res_new;
    if (stagnant >= 2) break;
  }
  memcpy(xout, x, sizeof(double) * (size_t)n);
  if (rel_residual) *rel_residual = res / denom;
  if (converged) *converged = res <= tol * denom;
  free(x);
  free(r);
  free(dx);
  free(xn);
  free(rn);
  return steps;
}

/* ------------------------------------------------------------------------ */
/* KktContext: kkt.cpp:41-314 */
struct orc_kkt {
  int form;
  orc_kkt_opts opt;
  int nt, ns, n, m_eq, m_ineq, m;
  int* jp_ptr;
  int* jp_idx;
  int hnnz, jnnz;
  orc_csc mat;
  orc_symbolic sym;
  int* h_slot;
  int* diag_slot;
  int* j_slot;
  int* slack_slot;
  int* rdiag_slot;
  int* ry_slot;
  int* ydiag_slot;
  int* pair_slot;
  int* pair_ptr;
  int npairs;
  orc_factors last;
  int have_last;
};

/* slot_of: kkt.cpp:31-37 (binary search; -1 where the reference throws) */
static int slot_of(const orc_csc* A, int i, int j) {
  int lo = A->col_ptr[j], hi = A->col_ptr[j + 1];
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (A->row_ind[mid] < i)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo == A->col_ptr[j + 1] || A->row_ind[lo] != i) return -1;
  return lo;
}

typedef struct {
  int *r, *c;
  int n, cap;
} tvec;
static void tadd(tvec* t, int i, int j) {
  if (t->n == t->cap) {
    t->cap = t->cap ? 2 * t->cap : 1024;
    t->r = (int*)realloc(t->r, sizeof(int) * (size_t)t->cap);
    t->c = (int*)realloc(t->c, sizeof(int) * (size_t)t->cap);
    if (!t->r || !t->c) abort();
  }
  t->r[t->n] = i;
  t->c[t->n] = j;
  t->n++;
}

orc_kkt* orc_kkt_create(int nt, const int* hp_ptr, const int* hp_idx, int m,
                        const int* jp_ptr, const int* jp_idx, int ns, int m_eq,
                        int form, const orc_kkt_opts* opt) {
  if (form < 0 || form > 2) return NULL;
  if (m - m_eq != ns) return NULL; /* kkt.cpp:52-53 */
  orc_kkt* K = (orc_kkt*)xcalloc(1, sizeof(orc_kkt));
  K->form = form;
  if (opt)
    K->opt = *opt;
  else {
    K->opt.pivot_eps = 1e-10;
    K->opt.max_refine = 10;
    K->opt.refine_tol = 1e-12;
    K->opt.delta_max = 1e40;
    K->opt.accept_tol = 1e-8;
  }
  K->nt = nt;
  K->ns = ns;
  K->n = nt + ns;
  K->m_eq = m_eq;
  K->m_ineq = m - m_eq;
  K->m = m;
  K->jnnz = jp_ptr[m];
  K->hnnz = hp_ptr[nt];
  K->jp_ptr = (int*)xcalloc((size_t)m + 1, sizeof(int));
  K->jp_idx = (int*)xcalloc((size_t)K->jnnz, sizeof(int));
  memcpy(K->jp_ptr, jp_ptr, sizeof(int) * ((size_t)m + 1));
  memcpy(K->jp_idx, jp_idx, sizeof(int) * (size_t)K->jnnz);
  const int n = K->n;
  int size = form == ORC_K2 ? n + 2 * m : (form == ORC_K2R ? n + m : nt);
  tvec t = {0};
  for (int j = 0; j < nt; ++j)
    for (int p = hp_ptr[j]; p < hp_ptr[j + 1]; ++p) tadd(&t, hp_idx[p], j);
  if (form == ORC_K1S) {
    for (int i = 0; i < nt; ++i) tadd(&t, i, i);
    for (int i = 0; i < m; ++i)
      for (int pa = jp_ptr[i]; pa < jp_ptr[i + 1]; ++pa)
        for (int pb = jp_ptr[i]; pb <= pa; ++pb)
          tadd(&t, jp_idx[pa], jp_idx[pb]);
  } else {
    for (int i = 0; i < n; ++i) tadd(&t, i, i);
    const int yb = (form == ORC_K2) ? n + m : n;
    for (int i = 0; i < m; ++i)
      for (int p = jp_ptr[i]; p < jp_ptr[i + 1]; ++p)
        tadd(&t, yb + i, jp_idx[p]);
    for (int k = 0; k < K->m_ineq; ++k) tadd(&t, yb + m_eq + k, nt + k);
    if (form == ORC_K2) {
      for (int i = 0; i < m; ++i) tadd(&t, n + i, n + i);
      for (int i = 0; i < m; ++i) tadd(&t, n + m + i, n + i);
    } else {
      for (int i = 0; i < m; ++i) tadd(&t, n + i, n + i);
    }
  }
  if (orc_sym_from_triplets(size, t.n, t.r, t.c, NULL, &K->mat)) {
    free(t.r);
    free(t.c);
    orc_kkt_destroy(K);
    return NULL;
  }
  free(t.r);
  free(t.c);
  orc_analyze(&K->mat, &K->sym);

  int bad = 0;
  K->h_slot = (int*)xcalloc((size_t)K->hnnz, sizeof(int));
  int q = 0;
  for (int j = 0; j < nt; ++j)
    for (int p = hp_ptr[j]; p < hp_ptr[j + 1]; ++p) {
      K->h_slot[q] = slot_of(&K->mat, hp_idx[p], j);
      bad |= K->h_slot[q++] < 0;
    }
  const int nd = (form == ORC_K1S) ? nt : n;
  K->diag_slot = (int*)xcalloc((size_t)nd, sizeof(int));
  for (int i = 0; i < nd; ++i) K->diag_slot[i] = slot_of(&K->mat, i, i);
  if (form == ORC_K1S) {
    K->pair_ptr = (int*)xcalloc((size_t)m + 1, sizeof(int));
    for (int i = 0; i < m; ++i) {
      const int v = jp_ptr[i + 1] - jp_ptr[i];
      K->pair_ptr[i + 1] = K->pair_ptr[i] + v * (v + 1) / 2;
    }
    K->npairs = K->pair_ptr[m];
    K->pair_slot = (int*)xcalloc((size_t)K->npairs, sizeof(int));
    q = 0;
    for (int i = 0; i < m; ++i)
      for (int pa = jp_ptr[i]; pa < jp_ptr[i + 1]; ++pa)
        for (int pb = jp_ptr[i]; pb <= pa; ++pb) {
          K->pair_slot[q] = slot_of(&K->mat, jp_idx[pa], jp_idx[pb]);
          bad |= K->pair_slot[q++] < 0;
        }
  } else {
    const int yb = (form == ORC_K2) ? n + m : n;
    K->j_slot = (int*)xcalloc((size_t)K->jnnz, sizeof(int));
    q = 0;
    for (int i = 0; i < m; ++i)
      for (int p = jp_ptr[i]; p < jp_ptr[i + 1]; ++p)
        K->j_slot[q++] = slot_of(&K->mat, yb + i, jp_idx[p]);
    K->slack_slot = (int*)xcalloc((size_t)K->m_ineq, sizeof(int));
    for (int k = 0; k < K->m_ineq; ++k)
      K->slack_slot[k] = slot_of(&K->mat, yb + m_eq + k, nt + k);
    if (form == ORC_K2) {
      K->rdiag_slot = (int*)xcalloc((size_t)m, sizeof(int));
      K->ry_slot = (int*)xcalloc((size_t)m, sizeof(int));
      for (int i = 0; i < m; ++i) {
        K->rdiag_slot[i] = slot_of(&K->mat, n + i, n + i);
        K->ry_slot[i] = slot_of(&K->mat, n + m + i, n + i);
      }
    } else {
      K->ydiag_slot = (int*)xcalloc((size_t)m, sizeof(int));
      for (int i = 0; i < m; ++i)
        K->ydiag_slot[i] = slot_of(&K->mat, n + i, n + i);
    }
  }
  if (bad) {
    orc_kkt_destroy(K);
    return NULL;
  }
  return K;
}

void orc_kkt_destroy(orc_kkt* K) {
  if (!K) return;
  free(K->jp_ptr);
  free(K->jp_idx);
  orc_csc_free(&K->mat);
  orc_symbolic_free(&K->sym);
  free(K->h_slot);
  free(K->diag_slot);
  free(K->j_slot);
  free(K->slack_slot);
  free(K->rdiag_slot);
  free(K->ry_slot);
  free(K->ydiag_slot);
  free(K->pair_slot);
  free(K->pair_ptr);
  if (K->have_last) orc_factors_free(&K->last);
  free(K);
}

int orc_kkt_system_size(const orc_kkt* K) { return K->mat.n; }
int orc_kkt_nnz(const orc_kkt* K) { return K->mat.nnz; }
int orc_kkt_num_pairs(const orc_kkt* K) { return K->npairs; }
const orc_symbolic* orc_kkt_symbolic(const orc_kkt* K) { return &K->sym; }
const orc_factors* orc_kkt_last_factors(const orc_kkt* K) {
  return K->have_last ? &K->last : NULL;
}

/* inertia_target: kkt.cpp:140-147 */
void orc_kkt_inertia_target(const orc_kkt* K, int* tgt) {
  tgt[2] = 0;
  if (K->form == ORC_K2) {
    tgt[0] = K->n + K->m;
    tgt[1] = K->m;
  } else if (K->form == ORC_K2R) {
    tgt[0] = K->n;
    tgt[1] = K->m;
  } else {
    tgt[0] = K->nt;
    tgt[1] = 0;
  }
}

void orc_kkt_matrix(const orc_kkt* K, int* col_ptr, int* row_ind,
                    double* val) {
  if (col_ptr)
    memcpy(col_ptr, K->mat.col_ptr, sizeof(int) * ((size_t)K->mat.n + 1));
  if (row_ind) memcpy(row_ind, K->mat.row_ind, sizeof(int) * (size_t)K->mat.nnz);
  if (val) memcpy(val, K->mat.val, sizeof(double) * (size_t)K->mat.nnz);
}

void orc_kkt_slots(const orc_kkt* K, int* h_slot, int* diag_slot,
                   int* pair_or_j_slot, int* slack_slot, int* ydiag_slot) {
  if (h_slot) memcpy(h_slot, K->h_slot, sizeof(int) * (size_t)K->hnnz);
  const int nd = (K->form == ORC_K1S) ? K->nt : K->n;
  if (diag_slot) memcpy(diag_slot, K->diag_slot, sizeof(int) * (size_t)nd);
  if (pair_or_j_slot) {
    if (K->form == ORC_K1S)
      memcpy(pair_or_j_slot, K->pair_slot, sizeof(int) * (size_t)K->npairs);
    else
      memcpy(pair_or_j_slot, K->j_slot, sizeof(int) * (size_t)K->jnnz);
  }
  if (slack_slot && K->slack_slot)
    memcpy(slack_slot, K->slack_slot, sizeof(int) * (size_t)K->m_ineq);
  if (ydiag_slot && K->ydiag_slot)
    memcpy(ydiag_slot, K->ydiag_slot, sizeof(int) * (size_t)K->m);
}

/* refill: kkt.cpp:149-186 */
void orc_kkt_refill(orc_kkt* K, const double* hv, const double* jv,
                    const double* sigma, double rho, double delta) {
  double* val = K->mat.val;
  memset(val, 0, sizeof(double) * (size_t)K->mat.nnz);
  const double rho_hat = rho + delta;
  for (int k = 0; k < K->hnnz; ++k) val[K->h_slot[k]] += hv[k];
  if (K->form == ORC_K1S) {
    for (int i = 0; i < K->nt; ++i) val[K->diag_slot[i]] += sigma[i] + delta;
    int q = 0;
    for (int i = 0; i < K->m; ++i) {
      double omega = 1.0;
      if (i >= K->m_eq) {
        const double ss = sigma[K->nt + (i - K->m_eq)] + delta;
        omega = ss / (ss + rho_hat);
      }
      const double w = rho_hat * omega;
      for (int pa = K->jp_ptr[i]; pa < K->jp_ptr[i + 1]; ++pa)
        for (int pb = K->jp_ptr[i]; pb <= pa; ++pb)
          val[K->pair_slot[q++]] += w * jv[pa] * jv[pb];
    }
  } else {
    for (int i = 0; i < K->n; ++i) val[K->diag_slot[i]] += sigma[i] + delta;
    for (int p = 0; p < K->jnnz; ++p) val[K->j_slot[p]] += jv[p];
    for (int k = 0; k < K->m_ineq; ++k) val[K->slack_slot[k]] += -1.0;
    if (K->form == ORC_K2) {
      for (int i = 0; i < K->m; ++i) {
        val[K->rdiag_slot[i]] += rho_hat;
        val[K->ry_slot[i]] += 1.0;
      }
    } else {
      for (int i = 0; i < K->m; ++i) val[K->ydiag_slot[i]] += -1.0 / rho_hat;
    }
  }
}

/* build_rhs: kkt.cpp:188-222 */
void orc_kkt_build_rhs(const orc_kkt* K, const double* jv, const double* sigma,
                       const double* rbar1, const double* rbar2,
                       const double* rbar3, double rho, double delta,
                       double* rhs) {
  const double rho_hat = rho + delta;
  const int n = K->n, m = K->m, nt = K->nt;
  if (K->form == ORC_K2) {
    for (int i = 0; i < n; ++i) rhs[i] = -rbar1[i];
    for (int i = 0; i < m; ++i) rhs[n + i] = -rbar2[i];
    for (int i = 0; i < m; ++i) rhs[n + m + i] = -rbar3[i];
  } else if (K->form == ORC_K2R) {
    for (int i = 0; i < n; ++i) rhs[i] = -rbar1[i];
    for (int i = 0; i < m; ++i) rhs[n + i] = -rbar3[i] + rbar2[i] / rho_hat;
  } else {
    double* v = (double*)xcalloc((size_t)m, sizeof(double));
    for (int i = 0; i < m; ++i) v[i] = rbar2[i] - rho_hat * rbar3[i];
    for (int i = 0; i < nt; ++i) rhs[i] = -rbar1[i];
    for (int i = 0; i < m; ++i)
      for (int p = K->jp_ptr[i]; p < K->jp_ptr[i + 1]; ++p)
        rhs[K->jp_idx[p]] += jv[p] * v[i];
    for (int k = 0; k < K->m_ineq; ++k) {
      const int row = K->m_eq + k;
      const double rs = -rbar1[nt + k] - v[row];
      const double pk = sigma[nt + k] + delta + rho_hat;
      const double w = rho_hat * rs / pk;
      for (int p = K->jp_ptr[row]; p < K->jp_ptr[row + 1]; ++p)
        rhs[K->jp_idx[p]] += jv[p] * w;
    }
    free(v);
  }
}

/* recover: kkt.cpp:224-264 */
static void kkt_recover(const orc_kkt* K, const double* jv,
                        const double* sigma, const double* rbar1,
                        const double* rbar2, const double* rbar3, double rho,
                        double delta, const double* sol, double* dx,
                        double* dr, double* dy) {
  const double rho_hat = rho + delta;
  const int n = K->n, m = K->m, nt = K->nt;
  if (K->form == ORC_K2) {
    for (int i = 0; i < n; ++i) dx[i] = sol[i];
    for (int i = 0; i < m; ++i) dr[i] = sol[n + i];
    for (int i = 0; i < m; ++i) dy[i] = -sol[n + m + i];
  } else if (K->form == ORC_K2R) {
    for (int i = 0; i < n; ++i) dx[i] = sol[i];
    for (int i = 0; i < m; ++i) dy[i] = -sol[n + i];
    for (int i = 0; i < m; ++i) dr[i] = (dy[i] - rbar2[i]) / rho_hat;
  } else {
    double* jdt = (double*)xcalloc((size_t)m, sizeof(double));
    for (int i = 0; i < m; ++i)
      for (int p = K->jp_ptr[i]; p < K->jp_ptr[i + 1]; ++p)
        jdt[i] += jv[p] * sol[K->jp_idx[p]];
    double* v = (double*)xcalloc((size_t)m, sizeof(double));
    for (int i = 0; i < m; ++i) v[i] = rbar2[i] - rho_hat * rbar3[i];
    for (int i = 0; i < nt; ++i) dx[i] = sol[i];
    for (int k = 0; k < K->m_ineq; ++k) {
      const int row = K->m_eq + k;
      const double rs = -rbar1[nt + k] - v[row];
      const double pk = sigma[nt + k] + delta + rho_hat;
      dx[nt + k] = (rho_hat * jdt[row] + rs) / pk;
    }
    for (int i = 0; i < m; ++i) {
      double jxdx = jdt[i];
      if (i >= K->m_eq) jxdx -= dx[nt + (i - K->m_eq)];
      dy[i] = v[i] - rho_hat * jxdx;
    }
    for (int i = 0; i < m; ++i) dr[i] = (dy[i] - rbar2[i]) / rho_hat;
    free(jdt);
    free(v);
  }
}

/* solve: kkt.cpp:266-314 */
int orc_kkt_solve(orc_kkt* K, const double* hv, const double* jv,
                  const double* sigma, const double* rbar1,
                  const double* rbar2, const double* rbar3, double rho,
                  double warm_delta, double* dx, double* dr, double* dy,
                  orc_kkt_stats* st) {
  memset(st, 0, sizeof(*st));
  int tgt[3];
  orc_kkt_inertia_target(K, tgt);
  double hmax = 0.0;
  for (int k = 0; k < K->hnnz; ++k) hmax = fmax(hmax, fabs(hv[k]));
  for (int i = 0; i < K->n; ++i) hmax = fmax(hmax, fabs(sigma[i]));
  const int N = K->mat.n;
  double* rhs = (double*)xcalloc((size_t)N, sizeof(double));
  double* sol = (double*)xcalloc((size_t)N, sizeof(double));
  double delta = 0.0;
  int first = 1;
  for (;;) {
    st->factor_attempts++;
    orc_kkt_refill(K, hv, jv, sigma, rho, delta);
    if (K->have_last) orc_factors_free(&K->last);
    orc_factorize(&K->sym, &K->mat, K->opt.pivot_eps, &K->last);
    K->have_last = 1;
    const orc_factors* F = &K->last;
    if (F->ok && F->n_pos == tgt[0] && F->n_neg == tgt[1] && F->n_zero == 0) {
      orc_kkt_build_rhs(K, jv, sigma, rbar1, rbar2, rbar3, rho, delta, rhs);
      double rel = 0.0;
      int conv = 0;
      const int steps =
          orc_solve_refined(&K->sym, F, &K->mat, rhs, K->opt.max_refine,
                            K->opt.refine_tol, sol, &rel, &conv);
      double bn = 0.0;
      for (int i = 0; i < N; ++i) bn = fmax(bn, fabs(rhs[i]));
      const double abs_res = rel * (bn > 0.0 ? bn : 1.0);
      const int accept =
          F->perturbed == 0 || abs_res <= K->opt.accept_tol * fmax(1.0, bn);
      if (accept) {
        st->delta = delta;
        st->refine_steps = steps;
        st->perturbed_pivots = F->perturbed;
        st->rel_residual = rel;
        kkt_recover(K, jv, sigma, rbar1, rbar2, rbar3, rho, delta, sol, dx,
                    dr, dy);
        int fin = 1;
        for (int i = 0; i < K->n; ++i) fin &= isfinite(dx[i]) != 0;
        for (int i = 0; i < K->m; ++i)
          fin &= (isfinite(dy[i]) != 0) & (isfinite(dr[i]) != 0);
        st->ok = fin;
        free(rhs);
        free(sol);
        return 0;
      }
    }
    if (first) {
      delta = warm_delta > 0.0 ? fmax(1e-20, warm_delta / 3.0)
                               : 1e-8 * fmax(1.0, hmax);
      first = 0;
    } else {
      delta *= 8.0;
    }
    if (delta > K->opt.delta_max) {
      st->ok = 0;
      free(rhs);
      free(sol);
      return 0;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* recover_bound_duals: kkt.cpp:316-328 */
void orc_recover_bound_duals(int n, const double* x, const double* lb,
                             const double* ub, const double* zl,
                             const double* zu, double mu, const double* dx,
                             double* dzl, double* dzu) {
  for (int i = 0; i < n; ++i) {
    dzl[i] = 0.0;
    dzu[i] = 0.0;
    if (isfinite(lb[i])) dzl[i] = -(zl[i] * dx[i] - mu) / (x[i] - lb[i]) - zl[i];
    if (isfinite(ub[i])) dzu[i] = (zu[i] * dx[i] + mu) / (ub[i] - x[i]) - zu[i];
  }
}

/* barrier_kkt_residual: kkt.cpp:341-366 (+ ResidualParts norms :330-339) */
void orc_barrier_kkt_residual(int nt, int ns, int m, const int* jp_ptr,
                              const int* jp_idx, const double* jval,
                              const double* grad_phi, const double* c,
                              const double* r, const double* y,
                              const double* yk, double rho, const double* x,
                              const double* lb, const double* ub,
                              const double* zl, const double* zu, double mu,
                              double* stat, double* mult, double* primal,
                              double* compl_l, double* compl_u, double* out5) {
  const int n = nt + ns, m_eq = m - ns;
  double* st = (double*)xcalloc((size_t)n, sizeof(double));
  for (int i = 0; i < n; ++i) st[i] = grad_phi[i] - zl[i] + zu[i];
  for (int i = 0; i < m; ++i)
    for (int p = jp_ptr[i]; p < jp_ptr[i + 1]; ++p)
      st[jp_idx[p]] -= jval[p] * y[i];
  for (int k = 0; k < ns; ++k) st[nt + k] += y[m_eq + k];
  double ns0 = 0, ns1 = 0, ns2 = 0, ns3 = 0, ns4 = 0;
  for (int i = 0; i < n; ++i) ns0 = fmax(ns0, fabs(st[i]));
  for (int i = 0; i < m; ++i) {
    const double mv = yk[i] + rho * r[i] - y[i];
    const double pv = c[i] + r[i];
    if (mult) mult[i] = mv;
    if (primal) primal[i] = pv;
    ns1 = fmax(ns1, fabs(mv));
    ns2 = fmax(ns2, fabs(pv));
  }
  for (int i = 0; i < n; ++i) {
    double cl = 0.0, cu = 0.0;
    if (isfinite(lb[i])) cl = zl[i] * (x[i] - lb[i]) - mu;
    if (isfinite(ub[i])) cu = zu[i] * (ub[i] - x[i]) - mu;
    if (compl_l) compl_l[i] = cl;
    if (compl_u) compl_u[i] = cu;
    ns3 = fmax(ns3, fabs(cl));
    ns4 = fmax(ns4, fabs(cu));
  }
  if (stat) memcpy(stat, st, sizeof(double) * (size_t)n);
  free(st);
  if (out5) {
    out5[0] = ns0;
    out5[1] = ns1;
    out5[2] = ns2;
    out5[3] = ns3;
    out5[4] = ns4;
  }
}

/* fraction_to_boundary / dual_fraction_to_boundary: ipm.cpp:124-141 */
double orc_fraction_to_boundary(int n, const double* x, const double* lb,
                                const double* ub, const double* dx,
                                double tau) {
  double a = 1.0;
  for (int i = 0; i < n; ++i) {
    if (dx[i] < 0.0 && isfinite(lb[i]))
      a = fmin(a, tau * (x[i] - lb[i]) / (-dx[i]));
    else if (dx[i] > 0.0 && isfinite(ub[i]))
      a = fmin(a, tau * (ub[i] - x[i]) / dx[i]);
  }
  return fmax(a, 0.0);
}

double orc_dual_fraction_to_boundary(int n, const double* z, const double* dz,
                                     double tau) {
  double a = 1.0;
  for (int i = 0; i < n; ++i)
    if (z[i] > 0.0 && dz[i] < 0.0) a = fmin(a, tau * z[i] / (-dz[i]));
  return fmax(a, 0.0);
}

/* clip_duals: ipm.cpp:232-249 */
static double clampd(double v, double lo, double hi) {
  return v < lo ? lo : (hi < v ? hi : v);
}
void orc_clip_duals(int n, const double* x, const double* lb,
                    const double* ub, double mu, double* zl, double* zu) {
  const double kap = 1e10;
  for (int i = 0; i < n; ++i) {
    if (isfinite(lb[i])) {
      const double gap = fmax(x[i] - lb[i], 1e-300);
      zl[i] = clampd(zl[i], mu / (kap * gap), kap * mu / gap);
    } else {
      zl[i] = 0.0;
    }
    if (isfinite(ub[i])) {
      const double gap = fmax(ub[i] - x[i], 1e-300);
      zu[i] = clampd(zu[i], mu / (kap * gap), kap * mu / gap);
    } else {
      zu[i] = 0.0;
    }
  }
}

/* solve_prepared KktInput formation: ipm.cpp:180-208 */
void orc_kkt_input(int nt, int ns, int m, const int* jp_ptr,
                   const int* jp_idx, const double* jval, const double* grad,
                   const double* c, const double* x, const double* lb,
                   const double* ub, const double* zl, const double* zu,
                   const double* r, const double* y, const double* yk,
                   double mu, double rho, double* sigma, double* rbar1,
                   double* rbar2, double* rbar3) {
  const int n = nt + ns, m_eq = m - ns;
  for (int i = 0; i < n; ++i) {
    sigma[i] = 0.0;
    rbar1[i] = grad[i];
  }
  for (int i = 0; i < n; ++i) {
    if (isfinite(lb[i])) {
      const double gl = x[i] - lb[i];
      sigma[i] += zl[i] / gl;
      rbar1[i] -= mu / gl;
    }
    if (isfinite(ub[i])) {
      const double gu = ub[i] - x[i];
      sigma[i] += zu[i] / gu;
      rbar1[i] += mu / gu;
    }
  }
  for (int i = 0; i < m; ++i)
    for (int p = jp_ptr[i]; p < jp_ptr[i + 1]; ++p)
      rbar1[jp_idx[p]] -= jval[p] * y[i];
  for (int k = 0; k < ns; ++k) rbar1[nt + k] += y[m_eq + k];
  for (int i = 0; i < m; ++i) {
    rbar2[i] = yk[i] + rho * r[i] - y[i];
    rbar3[i] = c[i] + r[i];
  }
}

/* outer schedule: solver.cpp:21-41 */
void orc_initial_outer_state(double mu0, double rho0, double rho_max,
                             double* s) {
  s[0] = mu0;
  s[1] = pow(mu0, 1.1);
  s[2] = 100.0 * pow(mu0, 1.05);
  s[3] = rho0;
  s[4] = rho_max;
}

int orc_outer_update(double* s, double rnorm) {
  if (rnorm <= s[1]) {
    const double mu_old = s[0];
    s[0] = fmax(fmin(pow(mu_old, 1.99), 0.2 * mu_old), 1e-14);
    s[1] = fmax(fmin(pow(s[0], 1.1), 0.1 * mu_old), 1e-12);
    s[2] = fmax(100.0 * pow(s[0], 1.05), 1e-12);
    return 1;
  }
  s[3] = fmin(s[4], 10.0 * s[3]);
  return 0;
}

/* init_multipliers: solver.cpp:43-91.  Same triplets as the reference's
 * all-pairs loop (nonzero dots only, ascending-column merge order), factored
 * with eps = 1e-14, unrefined solve, clip to +-1e3. */
void orc_init_multipliers(int m, int m_eq, const int* jp_ptr,
                          const int* jp_idx, const double* jv,
                          const double* g, double* y) {
  if (m == 0) return;
  tvec t = {0};
  int cap = 0;
  double* vals = NULL;
  for (int i = 0; i < m; ++i) {
    for (int j = 0; j <= i; ++j) {
      double dot = 0.0;
      int pa = jp_ptr[i], pb = jp_ptr[j];
      while (pa < jp_ptr[i + 1] && pb < jp_ptr[j + 1]) {
        if (jp_idx[pa] < jp_idx[pb])
          ++pa;
        else if (jp_idx[pa] > jp_idx[pb])
          ++pb;
        else
          dot += jv[pa++] * jv[pb++];
      }
      double v;
      int keep = 0;
      if (i == j) {
        if (i >= m_eq) dot += 1.0;
        v = dot + 1e-8;
        keep = 1;
      } else if (dot != 0.0) {
        v = dot;
        keep = 1;
      }
      if (keep) {
        tadd(&t, i, j);
        if (t.n > cap) {
          cap = t.cap;
          vals = (double*)realloc(vals, sizeof(double) * (size_t)cap);
          if (!vals) abort();
        }
        vals[t.n - 1] = v;
      }
    }
  }
  orc_csc A;
  orc_sym_from_triplets(m, t.n, t.r, t.c, vals, &A);
  orc_symbolic S;
  orc_analyze(&A, &S);
  orc_factors F;
  orc_factorize(&S, &A, 1e-14, &F);
  double* rhs = (double*)xcalloc((size_t)m, sizeof(double));
  for (int i = 0; i < m; ++i)
    for (int p = jp_ptr[i]; p < jp_ptr[i + 1]; ++p)
      rhs[i] += jv[p] * g[jp_idx[p]];
  orc_ldl_solve(&S, &F, rhs, y);
  for (int i = 0; i < m; ++i) y[i] = clampd(y[i], -1e3, 1e3);
  free(rhs);
  orc_factors_free(&F);
  orc_symbolic_free(&S);
  orc_csc_free(&A);
  free(t.r);
  free(t.c);
  free(vals);
}
