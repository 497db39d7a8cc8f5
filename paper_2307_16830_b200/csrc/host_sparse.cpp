// Host symbolic sparse linear algebra: condensation pattern, exact minimum
// degree ordering, symbolic Cholesky and the supernodal (multifrontal) front
// plan consumed by the CUDA factorisation in chol.cu.
//
// Reference semantics followed (bit-exact outputs):
//   coo_to_csc          csc.py:52-76        (col<<32|row keys, np.unique inverse)
//   symbolic_condense   kkt.py:243-283      (W, I, tril(A^T A) per Jacobian row)
//   amd_order           amd.py:18-54        (greedy MD, key (deg, deg0, index))
//   symbolic_cholesky   cholesky.py:94-144  (permute, etree 56-70, row
//                                            patterns 73-91, L CSC)
#include <omp.h>

#include <algorithm>
#include <memory>
#include <cmath>

#include <cstdlib>
#include <cstring>
#include <new>
#include <queue>
#include <tuple>

#include "internal.h"

namespace gn {

// Per-thread key histograms -> bucket pointers and per-(thread, key) start
// offsets (stable: thread chunks in order inside a key).  The totals and the
// offsets are parallel over keys; only the prefix over keys is serial.
static void merge_histograms(std::vector<std::vector<int64_t>> &hist, int64_t nkeys, int nt,
                             std::vector<int64_t> &ptr) {
  ptr.assign(nkeys + 1, 0);
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t c = 0; c < nkeys; ++c) {
    int64_t tot = 0;
    for (int t = 0; t < nt; ++t) tot += hist[t][c];
    ptr[c + 1] = tot;
  }
  for (int64_t c = 0; c < nkeys; ++c) ptr[c + 1] += ptr[c];
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t c = 0; c < nkeys; ++c) {
    int64_t run = ptr[c];
    for (int t = 0; t < nt; ++t) {
      const int64_t h = hist[t][c];
      hist[t][c] = run;
      run += h;
    }
  }
}

// (row, col) coordinates -> lower CSC with sorted unique rows per column, and
// the slot of every input coordinate (the np.unique(col<<32|row) inverse of
// csc.py:52-76).  Bucketed by column: O(nnz + sum_c u_c log u_c).
static void csc_from_coords(int64_t n, const std::vector<int32_t> &rows, const std::vector<int32_t> &cols,
                            std::vector<int64_t> &indptr, std::vector<int64_t> &indices,
                            std::vector<int64_t> &slot, std::vector<int32_t> *bucket_out = nullptr,
                            std::vector<int64_t> *bptr_out = nullptr) {
  const int64_t K = static_cast<int64_t>(rows.size());
  for (int64_t t = 0; t < K; ++t) GN_REQUIRE(cols[t] >= 0 && cols[t] < n, "column out of range");
  // bucket the coordinates by column: per-thread histograms over contiguous
  // input chunks keep the bucket order stable (deterministic)
  const int nt = std::max(1, std::min(omp_get_max_threads(), static_cast<int>(K / 65536 + 1)));
  std::vector<std::vector<int64_t>> hist(nt, std::vector<int64_t>(n + 1, 0));
  auto chunk = [&](int t) { return std::make_pair(K * t / nt, K * (t + 1) / nt); };
#pragma omp parallel for num_threads(nt) schedule(static, 1)
  for (int t = 0; t < nt; ++t) {
    auto [lo, hi] = chunk(t);
    for (int64_t q = lo; q < hi; ++q) hist[t][cols[q]]++;
  }
  std::vector<int64_t> bptr;
  merge_histograms(hist, n, nt, bptr);
  std::vector<int32_t> bucket(K);
#pragma omp parallel for num_threads(nt) schedule(static, 1)
  for (int t = 0; t < nt; ++t) {
    auto [lo, hi] = chunk(t);
    for (int64_t q = lo; q < hi; ++q) bucket[hist[t][cols[q]]++] = static_cast<int32_t>(q);
  }
  // per column: sorted unique rows (count pass, prefix, fill pass)
  std::vector<int64_t> ucount(n, 0);
  indptr.assign(n + 1, 0);
  slot.resize(K);
  std::vector<int32_t> urows(K);   // unique rows, at the column's bucket offset
#pragma omp parallel num_threads(nt)
  {
    std::vector<int64_t> mark(n, -1);
#pragma omp for schedule(dynamic, 512)
    for (int64_t c = 0; c < n; ++c) {
      int64_t u = bptr[c];
      for (int64_t q = bptr[c]; q < bptr[c + 1]; ++q) {
        const int32_t r = rows[bucket[q]];
        if (mark[r] != c) {
          mark[r] = c;
          urows[u++] = r;
        }
      }
      std::sort(urows.begin() + bptr[c], urows.begin() + u);
      ucount[c] = u - bptr[c];
    }
  }
  for (int64_t c = 0; c < n; ++c) indptr[c + 1] = indptr[c] + ucount[c];
  indices.resize(indptr[n]);
#pragma omp parallel num_threads(nt)
  {
    std::vector<int64_t> pos(n, 0);
#pragma omp for schedule(dynamic, 512)
    for (int64_t c = 0; c < n; ++c) {
      const int64_t base = indptr[c];
      for (int64_t u = 0; u < ucount[c]; ++u) {
        const int32_t r = urows[bptr[c] + u];
        indices[base + u] = r;
        pos[r] = base + u;
      }
      for (int64_t q = bptr[c]; q < bptr[c + 1]; ++q) slot[bucket[q]] = pos[rows[bucket[q]]];
    }
  }
  if (bucket_out) *bucket_out = std::move(bucket);
  if (bptr_out) *bptr_out = std::move(bptr);
}

// Stable parallel bucketing: items 0..N-1 with key(i) in [0, nkeys) ->
// ptr (nkeys+1) and dest(i), the item's slot, ascending i inside a key.
// Per-thread histograms over contiguous item chunks keep the order stable.
template <class KeyFn, class PlaceFn>
static void par_bucket(int64_t nkeys, int64_t N, KeyFn key, PlaceFn place, std::vector<int64_t> &ptr) {
  const int nt = std::max(1, std::min(omp_get_max_threads(), static_cast<int>(N / 65536 + 1)));
  std::vector<std::vector<int64_t>> hist(nt);
  auto chunk = [&](int t) { return std::make_pair(N * t / nt, N * (t + 1) / nt); };
#pragma omp parallel for num_threads(nt) schedule(static, 1)
  for (int t = 0; t < nt; ++t) {
    hist[t].assign(nkeys, 0);
    auto [lo, hi] = chunk(t);
    for (int64_t i = lo; i < hi; ++i) hist[t][key(i)]++;
  }
  merge_histograms(hist, nkeys, nt, ptr);
#pragma omp parallel for num_threads(nt) schedule(static, 1)
  for (int t = 0; t < nt; ++t) {
    auto [lo, hi] = chunk(t);
    for (int64_t i = lo; i < hi; ++i) place(i, hist[t][key(i)]++);
  }
}

static inline uint64_t ckey(int64_t row, int64_t col) {
  return (static_cast<uint64_t>(col) << 32) | static_cast<uint64_t>(row);
}

// product q of segment g: local index -> (la, lb) with lb <= la, in
// np.tril_indices order (row-major lower triangle)
void Condense::product(int64_t q, int64_t g, int64_t &row, int64_t &s1, int64_t &s2) const {
  const int64_t local = q - seg_poff[g];
  int64_t la = static_cast<int64_t>((std::sqrt(8.0 * static_cast<double>(local) + 1.0) - 1.0) * 0.5);
  while ((la + 1) * (la + 2) / 2 <= local) ++la;
  while (la * (la + 1) / 2 > local) --la;
  const int64_t lb = local - la * (la + 1) / 2;
  row = seg_row[g];
  s1 = seg[g] + la;
  s2 = seg[g] + lb;
}

int64_t Condense::product_segment(int64_t q) const {
  return static_cast<int64_t>(std::upper_bound(seg_poff.begin(), seg_poff.end(), q) - seg_poff.begin()) - 1;
}

// Condensed pattern K = tril(W + I + A^T A) straight from the factors, one
// column at a time (a symbolic sparse product, no coordinate list): column c
// collects its W rows, the diagonal, and for every Jacobian row r holding c
// the entries of r at or after c.  A second pass over the same column writes
// the sorted rows, the slot of each W/diagonal/product coordinate and the
// column's slice of the assembly plan -- the products grouped by K slot in
// ascending product index (kkt.py:243-283 summation order), which is the
// order a column visits them: Jacobian rows ascending, then la ascending.
// Columns are independent, so both passes are parallel over columns.
static void condense(Condense &C, int64_t n, int64_t nh, const int64_t *hr, const int64_t *hc,
                     int64_t nj, const int64_t *jr, const int64_t *jc) {
  PhaseTimer tm_total("condense.total");
  C.n = n;
  C.nnz_h = nh;
  C.nnz_j = nj;
  GN_REQUIRE(n < (int64_t(1) << 31) && nh < (int64_t(1) << 31) && nj < (int64_t(1) << 31),
             "too many variables or nonzeros for 32-bit indices");
  int bad = 0;
#pragma omp parallel for reduction(| : bad)
  for (int64_t t = 0; t < nj; ++t)
    bad |= !(jc[t] >= 0 && jc[t] < n &&
             (t == 0 || jr[t] > jr[t - 1] || (jr[t] == jr[t - 1] && jc[t] > jc[t - 1])));
  GN_REQUIRE(!bad, "Jacobian coordinates must be sorted row-major, unique and in range");
#pragma omp parallel for reduction(| : bad)
  for (int64_t t = 0; t < nh; ++t) bad |= !(hc[t] <= hr[t] && hr[t] >= 0 && hr[t] < n && hc[t] >= 0);
  GN_REQUIRE(!bad, "Hessian entry out of range or above the diagonal");
  // Jacobian row segments and their product offsets (np.tril_indices order)
  // (parallel: segment starts, a blocked prefix count, then the placement)
  uvec<int32_t> pseg(nj);
  int64_t nseg = 0;
  {
    const int nt = std::max(1, std::min(omp_get_max_threads(), static_cast<int>(nj / 65536 + 1)));
    std::vector<int64_t> cnt(nt + 1, 0);
#pragma omp parallel num_threads(nt)
    {
      const int t = omp_get_thread_num();
      const int64_t lo = nj * t / nt, hi = nj * (t + 1) / nt;
      int64_t c = 0;
      for (int64_t e = lo; e < hi; ++e) c += (e == 0 || jr[e] != jr[e - 1]);
      cnt[t + 1] = c;
#pragma omp barrier
#pragma omp single
      for (int q = 0; q < nt; ++q) cnt[q + 1] += cnt[q];
      int64_t g = cnt[t] - 1;
      for (int64_t e = lo; e < hi; ++e) {
        g += (e == 0 || jr[e] != jr[e - 1]);
        pseg[e] = static_cast<int32_t>(g);
      }
    }
    nseg = cnt[nt];
  }
  C.seg.resize(nseg + 1);
  C.seg_row.resize(nseg + 1);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < nj; ++e)
    if (e == 0 || jr[e] != jr[e - 1]) {
      C.seg[pseg[e]] = e;
      C.seg_row[pseg[e]] = jr[e];
    }
  C.seg[nseg] = nj;
  C.seg_row[nseg] = -1;
  C.seg_poff.assign(nseg + 1, 0);
  for (int64_t g = 0; g < nseg; ++g) {
    const int64_t k = C.seg[g + 1] - C.seg[g];
    C.seg_poff[g + 1] = C.seg_poff[g] + k * (k + 1) / 2;
  }
  const int64_t np = C.seg_poff[nseg];
  C.np = np;
  GN_REQUIRE(np < (int64_t(1) << 31), "too many A^T A products for 32-bit offsets");
  PhaseTimer tm_all("condense");
  // Jacobian entries by column (ascending entry, hence ascending row) and
  // W entries by column (input order)
  PhaseTimer tm_b("condense.buckets");
  std::vector<int64_t> &aptr = C.a_colptr, hptr;
  uvec<int32_t> &alist = C.a_colent;
  uvec<int32_t> hlist(nh);
  alist.resize(nj);
  par_bucket(n, nj, [&](int64_t p) { return jc[p]; },
             [&](int64_t p, int64_t d) { alist[d] = static_cast<int32_t>(p); }, aptr);
  par_bucket(n, nh, [&](int64_t t) { return hc[t]; },
             [&](int64_t t, int64_t d) { hlist[d] = static_cast<int32_t>(t); }, hptr);
  tm_b.~PhaseTimer();
  new (&tm_b) PhaseTimer("condense.pass1");
  // pass 1: unique rows and products per column
  std::vector<int64_t> ucount(n), pcount(n);
#pragma omp parallel
  {
    std::vector<int32_t> mark(n, -1);
#pragma omp for schedule(dynamic, 512)
    for (int64_t c = 0; c < n; ++c) {
      int64_t u = 1, prods = 0;
      mark[c] = static_cast<int32_t>(c);
      for (int64_t k = hptr[c]; k < hptr[c + 1]; ++k) {
        const int64_t r = hr[hlist[k]];
        if (mark[r] != c) mark[r] = static_cast<int32_t>(c), ++u;
      }
      for (int64_t k = aptr[c]; k < aptr[c + 1]; ++k) {
        const int64_t p = alist[k], en = C.seg[pseg[p] + 1];
        prods += en - p;
        for (int64_t e = p; e < en; ++e)
          if (mark[jc[e]] != c) mark[jc[e]] = static_cast<int32_t>(c), ++u;
      }
      ucount[c] = u;
      pcount[c] = prods;
    }
  }
  tm_b.~PhaseTimer();
  new (&tm_b) PhaseTimer("condense.alloc");
  C.indptr.assign(n + 1, 0);
  std::vector<int64_t> pptr(n + 1, 0);
  for (int64_t c = 0; c < n; ++c) {
    C.indptr[c + 1] = C.indptr[c] + ucount[c];
    pptr[c + 1] = pptr[c] + pcount[c];
  }
  const int64_t nk = C.indptr[n], base = nh + n;
  C.indices.resize(nk);
  C.slot.resize(base + np);
  C.k_ptr.resize(nk + 1);
  C.k_row.resize(np);
  C.k_s1.resize(np);
  C.k_s2.resize(np);
  tm_b.~PhaseTimer();
  new (&tm_b) PhaseTimer("condense.pass2");
  // pass 2: sorted rows, slots, assembly plan
#pragma omp parallel
  {
    std::vector<int32_t> mark(n, -1);
    std::vector<int64_t> pos(n, 0);
    std::vector<int32_t> fill;
#pragma omp for schedule(dynamic, 512)
    for (int64_t c = 0; c < n; ++c) {
      const int64_t s0 = C.indptr[c];
      int64_t u = s0;
      mark[c] = static_cast<int32_t>(c);
      C.indices[u++] = c;
      for (int64_t k = hptr[c]; k < hptr[c + 1]; ++k) {
        const int64_t r = hr[hlist[k]];
        if (mark[r] != c) mark[r] = static_cast<int32_t>(c), C.indices[u++] = r;
      }
      for (int64_t k = aptr[c]; k < aptr[c + 1]; ++k) {
        const int64_t p = alist[k], en = C.seg[pseg[p] + 1];
        for (int64_t e = p; e < en; ++e)
          if (mark[jc[e]] != c) mark[jc[e]] = static_cast<int32_t>(c), C.indices[u++] = jc[e];
      }
      std::sort(C.indices.begin() + s0, C.indices.begin() + u);
      for (int64_t t = s0; t < u; ++t) pos[C.indices[t]] = t;
      for (int64_t k = hptr[c]; k < hptr[c + 1]; ++k) C.slot[hlist[k]] = pos[hr[hlist[k]]];
      C.slot[nh + c] = pos[c];
      // products of the column per slot, then their plan entries
      fill.assign(u - s0, 0);
      for (int64_t k = aptr[c]; k < aptr[c + 1]; ++k) {
        const int64_t p = alist[k], en = C.seg[pseg[p] + 1];
        for (int64_t e = p; e < en; ++e) fill[pos[jc[e]] - s0]++;
      }
      int32_t run = static_cast<int32_t>(pptr[c]);
      for (int64_t t = s0; t < u; ++t) {
        const int32_t h = fill[t - s0];
        C.k_ptr[t] = run;
        fill[t - s0] = run;
        run += h;
      }
      for (int64_t k = aptr[c]; k < aptr[c + 1]; ++k) {
        const int64_t p = alist[k], g = pseg[p], st = C.seg[g], en = C.seg[g + 1];
        const int64_t lb = p - st, qb = C.seg_poff[g] + lb;
        for (int64_t e = p; e < en; ++e) {
          const int64_t la = e - st, s = pos[jc[e]];
          C.slot[base + qb + la * (la + 1) / 2] = s;
          const int32_t d = fill[s - s0]++;
          C.k_row[d] = static_cast<int32_t>(C.seg_row[g]);
          C.k_s1[d] = static_cast<int32_t>(e);
          C.k_s2[d] = static_cast<int32_t>(p);
        }
      }
    }
  }
  C.k_ptr[nk] = static_cast<int32_t>(np);
  C.plan_built = true;
}

// the plan is built with the pattern (kept for callers of the old split)
void Condense::ensure_assembly_plan() {}

// ------------------------------------------------------------ ordering
// Explicit elimination graph exactly as the reference builds it: eliminating
// v turns its neighbourhood nb into a clique, adj[u] = adj[u] - {v} + nb - {u}
// for u in nb, degree[u] = |adj[u]|.  Adjacency lists are unsorted; set
// union uses two stamp arrays, so one elimination costs
// sum_{u in nb} (|adj[u]| + |nb|) cheap operations.  Selection uses a heap
// keyed (degree, initial degree, index) with lazy deletion, which is the
// reference's strict-< scan order.
static void min_degree(int64_t n, const int64_t *indptr, const int64_t *indices, int64_t *perm) {
  std::vector<std::vector<int32_t>> adj(n);
  {
    std::vector<int32_t> cnt(n, 0);
    for (int64_t j = 0; j < n; ++j)
      for (int64_t p = indptr[j]; p < indptr[j + 1]; ++p)
        if (indices[p] != j) cnt[indices[p]]++, cnt[j]++;
    for (int64_t v = 0; v < n; ++v) adj[v].reserve(cnt[v]);
    for (int64_t j = 0; j < n; ++j)
      for (int64_t p = indptr[j]; p < indptr[j + 1]; ++p) {
        const int64_t i = indices[p];
        if (i != j) {
          adj[i].push_back(static_cast<int32_t>(j));
          adj[j].push_back(static_cast<int32_t>(i));
        }
      }
    // duplicate coordinates are not expected in a CSC pattern, but keep set
    // semantics if they occur
    std::vector<int64_t> seen(n, -1);
    for (int64_t v = 0; v < n; ++v) {
      auto &a = adj[v];
      size_t w = 0;
      for (int32_t x : a)
        if (seen[x] != v) seen[x] = v, a[w++] = x;
      a.resize(w);
    }
  }
  std::vector<int64_t> deg(n), deg0(n);
  std::vector<char> alive(n, 1);
  using Key = std::tuple<int64_t, int64_t, int64_t>;
  std::vector<Key> hv;
  hv.reserve(static_cast<size_t>(n) * 4);
  std::priority_queue<Key, std::vector<Key>, std::greater<Key>> heap(std::greater<Key>(), std::move(hv));
  for (int64_t v = 0; v < n; ++v) {
    deg[v] = deg0[v] = static_cast<int64_t>(adj[v].size());
    heap.emplace(deg[v], deg0[v], v);
  }
  std::vector<int64_t> in_nb(n, -1);    // == k: member of the current pivot's nb
  std::vector<int64_t> in_adj(n, -1);   // == stamp: member of adj[u] (current u)
  int64_t stamp = 0;
  for (int64_t k = 0; k < n; ++k) {
    int64_t v;
    for (;;) {
      auto [d, d0, u] = heap.top();
      heap.pop();
      if (alive[u] && d == deg[u]) {
        v = u;
        break;
      }
    }
    perm[k] = v;
    alive[v] = 0;
    std::vector<int32_t> nb;
    nb.swap(adj[v]);
    const int64_t dnb = static_cast<int64_t>(nb.size());
    for (int32_t x : nb) in_nb[x] = k;
    for (int32_t u : nb) {
      auto &au = adj[u];
      ++stamp;
      size_t w = 0;
      int64_t present = 0;
      for (int32_t x : au) {
        if (x == v) continue;
        au[w++] = x;
        if (in_nb[x] == k) {
          ++present;
          in_adj[x] = stamp;
        }
      }
      au.resize(w);
      if (present < dnb - 1)   // nb - {u} not yet contained: append the missing
        for (int32_t x : nb)
          if (x != u && in_adj[x] != stamp) au.push_back(x);
    }
    for (int32_t u : nb) {
      const int64_t nd = static_cast<int64_t>(adj[u].size());
      if (nd != deg[u]) {
        deg[u] = nd;
        heap.emplace(nd, deg0[u], u);
      }
    }
  }
}

// ------------------------------------------------------ symbolic Cholesky
static void symbolic(Symbolic &S, int64_t n, const int64_t *indptr, const int64_t *indices,
                     const int64_t *perm) {
  PhaseTimer tm("symbolic");
  S.n = n;
  int64_t nnz = indptr[n];
  S.nnz_a = nnz;
  S.perm.assign(perm, perm + n);
  std::vector<int64_t> pinv(n, -1);
  for (int64_t k = 0; k < n; ++k) {
    GN_REQUIRE(perm[k] >= 0 && perm[k] < n && pinv[perm[k]] == -1, "ordering is not a permutation");
    pinv[perm[k]] = k;
  }
  PhaseTimer tm_perm("symbolic.permute+sort");
  uvec<int64_t> prow(nnz), pcol(nnz);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t j = 0; j < n; ++j)
    for (int64_t p = indptr[j]; p < indptr[j + 1]; ++p) {
      int64_t a = pinv[indices[p]], b = pinv[j];
      prow[p] = std::max(a, b);
      pcol[p] = std::min(a, b);
    }
  // order by (prow, pcol): bucket by prow, then sort each row by pcol (the
  // pairs are unique, so this is the reference's stable lexicographic order)
  uvec<int64_t> o2(nnz);
  par_bucket(n, nnz, [&](int64_t p) { return prow[p]; }, [&](int64_t p, int64_t d) { o2[d] = p; },
             S.a_rowptr);
  S.a_rowcol.resize(nnz);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t r = 0; r < n; ++r) {
    std::sort(o2.begin() + S.a_rowptr[r], o2.begin() + S.a_rowptr[r + 1],
              [&](int64_t x, int64_t y) { return pcol[x] < pcol[y]; });
    for (int64_t t = S.a_rowptr[r]; t < S.a_rowptr[r + 1]; ++t) S.a_rowcol[t] = pcol[o2[t]];
  }
  S.a_srcslot = std::move(o2);
  tm_perm.~PhaseTimer();
  new (&tm_perm) PhaseTimer("symbolic.etree");
  // elimination tree (cholesky.py:56-70)
  S.parent.assign(n, -1);
  std::vector<int64_t> anc(n, -1);
  for (int64_t k = 0; k < n; ++k)
    for (int64_t t = S.a_rowptr[k]; t < S.a_rowptr[k + 1]; ++t) {
      int64_t i = S.a_rowcol[t];
      while (anc[i] != -1 && anc[i] != k) {
        int64_t nx = anc[i];
        anc[i] = k;
        i = nx;
      }
      if (anc[i] == -1 && i != k) {
        anc[i] = k;
        S.parent[i] = k;
      }
    }
  tm_perm.~PhaseTimer();
  new (&tm_perm) PhaseTimer("symbolic.row_patterns");
  // row patterns (cholesky.py:73-91): etree reach of every row, rows in
  // parallel (count pass, prefix, fill + sort pass)
  S.row_ptr.assign(n + 1, 0);
  {
    std::vector<int64_t> rc(n, 0);
#pragma omp parallel
    {
      std::vector<int64_t> mark(n, -1);
#pragma omp for schedule(dynamic, 1024)
      for (int64_t k = 0; k < n; ++k) {
        int64_t c = 0;
        mark[k] = k;
        for (int64_t t = S.a_rowptr[k]; t < S.a_rowptr[k + 1]; ++t)
          for (int64_t i = S.a_rowcol[t]; i != -1 && mark[i] != k; i = S.parent[i]) {
            mark[i] = k;
            ++c;
          }
        rc[k] = c;
      }
    }
    for (int64_t k = 0; k < n; ++k) S.row_ptr[k + 1] = S.row_ptr[k] + rc[k];
    S.row_cols.resize(S.row_ptr[n]);   // etree-reach order; sorted on export
#pragma omp parallel
    {
      std::vector<int64_t> mark(n, -1);
#pragma omp for schedule(dynamic, 1024)
      for (int64_t k = 0; k < n; ++k) {
        int64_t o = S.row_ptr[k];
        mark[k] = k;
        for (int64_t t = S.a_rowptr[k]; t < S.a_rowptr[k + 1]; ++t)
          for (int64_t i = S.a_rowcol[t]; i != -1 && mark[i] != k; i = S.parent[i]) {
            mark[i] = k;
            S.row_cols[o++] = i;
          }
      }
    }
  }
  tm_perm.~PhaseTimer();
  new (&tm_perm) PhaseTimer("symbolic.col_counts");
  // column counts of L (diagonal + row-pattern entries per column); the row
  // indices themselves are only built for exports (ensure_l_csc)
  {
    const int nt = omp_get_max_threads();
    std::vector<std::vector<int32_t>> h(nt);
    const int64_t nrc = S.row_ptr[n];
#pragma omp parallel num_threads(nt)
    {
      std::vector<int32_t> &mine = h[omp_get_thread_num()];
      mine.assign(n, 0);
#pragma omp for schedule(static)
      for (int64_t t = 0; t < nrc; ++t) mine[S.row_cols[t]]++;
    }
    S.l_colptr.assign(n + 1, 0);
    std::vector<int64_t> cnt(n);
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j) {
      int64_t c = 1;
      for (int t = 0; t < nt; ++t) c += h[t][j];
      cnt[j] = c;
    }
    for (int64_t j = 0; j < n; ++j) S.l_colptr[j + 1] = S.l_colptr[j] + cnt[j];
    S.nnz_l = S.l_colptr[n];
  }
}

// L in CSC, diagonal first, rows increasing (cholesky.py:118-131): a stable
// bucketing of the row-pattern entries by column.  Export only.
void Symbolic::ensure_l_csc() {
  std::lock_guard<std::mutex> g(lazy_mu);
  if (static_cast<int64_t>(l_rowidx.size()) == nnz_l) return;
  const int64_t nrc = row_ptr[n];
  std::vector<int32_t> rowof(nrc);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t k = 0; k < n; ++k)
    for (int64_t t = row_ptr[k]; t < row_ptr[k + 1]; ++t) rowof[t] = static_cast<int32_t>(k);
  std::vector<int64_t> cptr;
  l_rowidx.assign(nrc + n, 0);
  par_bucket(n, nrc, [&](int64_t t) { return row_cols[t]; },
             [&](int64_t t, int64_t d) { l_rowidx[d + row_cols[t] + 1] = rowof[t]; }, cptr);
  for (int64_t j = 0; j < n; ++j) l_rowidx[l_colptr[j]] = j;
}

// reference L slot -> offset in the front storage.  Export only.
void Symbolic::ensure_l_export() {
  ensure_l_csc();
  std::lock_guard<std::mutex> g(lazy_mu);
  if (static_cast<int64_t>(l_export.size()) == nnz_l) return;
  l_export.assign(nnz_l, 0);
  int missing = 0;
#pragma omp parallel reduction(| : missing)
  {
    std::vector<int32_t> pos(n, -1);
#pragma omp for schedule(dynamic, 64)
    for (int64_t J = 0; J < nf; ++J) {
      const int64_t r0 = f_rows_off[J], r1 = f_rows_off[J + 1], sJ = front_ld(f_nrows[J]);
      for (int64_t q = r0; q < r1; ++q) pos[f_rows[q]] = static_cast<int32_t>(q - r0);
      for (int64_t j = f_first[J]; j < f_first[J] + f_ncols[J]; ++j) {
        const int64_t base = f_off[J] + (j - f_first[J]) * sJ;
        for (int64_t p = l_colptr[j]; p < l_colptr[j + 1]; ++p) {
          const int32_t v = pos[l_rowidx[p]];
          missing |= v < 0;
          l_export[p] = base + (v < 0 ? 0 : v);
        }
      }
      for (int64_t q = r0; q < r1; ++q) pos[f_rows[q]] = -1;
    }
  }
  GN_REQUIRE(!missing, "row missing from front structure");
}

// ------------------------------------------------------------ front plan
// Supernodes are maximal runs j, j+1, ... with parent[j] == j+1 (contiguous in
// the reference elimination order, so the reference's pivot sequence is kept),
// relaxed: a column joins the running supernode when the explicit zeros stay
// below a width-dependent fraction (CHOLMOD-style amalgamation rule).
static void front_plan(Symbolic &S) {
  PhaseTimer tm("front_plan");
  const int64_t n = S.n;
  std::vector<int64_t> cc(n);
  for (int64_t j = 0; j < n; ++j) cc[j] = S.l_colptr[j + 1] - S.l_colptr[j];
  std::vector<int32_t> snode_of(n);
  S.f_first.clear();
  S.f_ncols.clear();
  int64_t f = 0;
  int64_t true_nnz = cc[0];
  for (int64_t j = 1; j <= n; ++j) {
    bool join = false;
    if (j < n && S.parent[j - 1] == j) {
      int64_t w = j - f + 1;               // width if column j joins
      int64_t s = w + cc[j] - 1;           // front rows: [f..j] + struct(j)
      int64_t dense = w * s - w * (w - 1) / 2;
      int64_t tn = true_nnz + cc[j];
      double zfrac = static_cast<double>(dense - tn) / static_cast<double>(dense);
      if (cc[j - 1] == cc[j] + 1) join = true;  // fundamental: no new zeros
      else if (w <= 4) join = true;
      else if (w <= 16 && zfrac < 0.5) join = true;
      else if (w <= 48 && zfrac < 0.1) join = true;
      else if (zfrac < 0.05) join = true;
    }
    if (join) {
      true_nnz += cc[j];
      continue;
    }
    S.f_first.push_back(static_cast<int32_t>(f));
    S.f_ncols.push_back(static_cast<int32_t>(j - f));
    if (j < n) {
      f = j;
      true_nnz = cc[j];
    }
  }
  const int64_t nf = static_cast<int64_t>(S.f_first.size());
  S.nf = nf;
  for (int64_t J = 0; J < nf; ++J)
    for (int64_t c = S.f_first[J]; c < S.f_first[J] + S.f_ncols[J]; ++c) snode_of[c] = static_cast<int32_t>(J);
  // rows, sizes, offsets.  Front rows = its columns, then the structure of
  // its last column below the diagonal: the row-pattern entries (k, l) with
  // l a last column, bucketed by front in ascending k.
  S.f_nrows.resize(nf);
  S.f_parent.assign(nf, -1);
  S.f_rows_off.assign(nf + 1, 0);
  S.f_off.assign(nf + 1, 0);
  S.f_voff.assign(nf + 1, 0);
  S.max_front = S.max_cols = 0;
  S.flops = 0;
  std::vector<int32_t> last_of(n, -1);
  for (int64_t J = 0; J < nf; ++J) {
    int64_t first = S.f_first[J], w = S.f_ncols[J], l = first + w - 1;
    last_of[l] = static_cast<int32_t>(J);
    int64_t s = w + cc[l] - 1;
    S.f_nrows[J] = static_cast<int32_t>(s);
    S.f_rows_off[J + 1] = S.f_rows_off[J] + s;
    S.f_off[J + 1] = S.f_off[J] + s * front_ld(s);   // even ld: 16-byte aligned columns
    S.f_voff[J + 1] = S.f_voff[J] + s;
    S.max_front = std::max(S.max_front, s);
    S.max_cols = std::max(S.max_cols, w);
    if (S.parent[l] != -1) S.f_parent[J] = snode_of[S.parent[l]];
    for (int64_t c = 0; c < w; ++c) S.flops += (s - c - 1) * (s - c - 1) + 2 * (s - c);
  }
  {
    PhaseTimer tm_rows("front_plan.rows");
    const int64_t nrc = S.row_ptr[n];
    uvec<int32_t> rowof(nrc);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t k = 0; k < n; ++k)
      for (int64_t t = S.row_ptr[k]; t < S.row_ptr[k + 1]; ++t) rowof[t] = static_cast<int32_t>(k);
    std::vector<int64_t> sptr;
    S.f_rows.resize(S.f_rows_off[nf]);             // every entry written below
    uvec<int32_t> srow(S.f_rows_off[nf]);          // >= the struct entries
    par_bucket(nf + 1, nrc,
               [&](int64_t t) { const int32_t J = last_of[S.row_cols[t]]; return J >= 0 ? J : nf; },
               [&](int64_t t, int64_t d) {
                 if (last_of[S.row_cols[t]] >= 0) srow[d] = rowof[t];
               },
               sptr);
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t J = 0; J < nf; ++J) {
      const int64_t o = S.f_rows_off[J], w = S.f_ncols[J];
      GN_REQUIRE(sptr[J + 1] - sptr[J] == S.f_nrows[J] - w, "front structure mismatch");
      for (int64_t c = 0; c < w; ++c) S.f_rows[o + c] = static_cast<int32_t>(S.f_first[J] + c);
      for (int64_t q = sptr[J]; q < sptr[J + 1]; ++q) S.f_rows[o + w + (q - sptr[J])] = srow[q];
    }
  }
  S.dinv_off = S.f_off[nf];                // 1 / L[k][k] per column, after the fronts
  S.front_doubles = S.f_off[nf] + n;
  S.xp_off = S.f_voff[nf];
  S.vec_doubles = S.f_voff[nf] + n;
  // children CSR (increasing child index)
  S.f_child_ptr.assign(nf + 1, 0);
  for (int64_t J = 0; J < nf; ++J)
    if (S.f_parent[J] >= 0) S.f_child_ptr[S.f_parent[J] + 1]++;
  for (int64_t J = 0; J < nf; ++J) S.f_child_ptr[J + 1] += S.f_child_ptr[J];
  S.f_child.assign(S.f_child_ptr[nf], 0);
  {
    std::vector<int32_t> fl(S.f_child_ptr.begin(), S.f_child_ptr.end() - 1);
    for (int64_t J = 0; J < nf; ++J)
      if (S.f_parent[J] >= 0) S.f_child[fl[S.f_parent[J]]++] = static_cast<int32_t>(J);
  }
  PhaseTimer tm_maps("front_plan.maps");
  // A entries grouped by front (ascending row inside a front)
  const int64_t na = S.a_rowptr[n];
  uvec<int32_t> arow(na);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t k = 0; k < n; ++k)
    for (int64_t t = S.a_rowptr[k]; t < S.a_rowptr[k + 1]; ++t) arow[t] = static_cast<int32_t>(k);
  uvec<int64_t> a_t(na);
  par_bucket(nf, na, [&](int64_t t) { return snode_of[S.a_rowcol[t]]; },
             [&](int64_t t, int64_t d) { a_t[d] = t; }, S.f_a_ptr);
  const std::vector<int64_t> &per = S.f_a_ptr;
  // relmap offsets (child update rows, in child order)
  S.f_relmap_off.assign(nf + 1, 0);
  for (int64_t C = 0; C < nf; ++C) {
    const int64_t w = S.f_ncols[C], sC = S.f_nrows[C];
    if (S.f_parent[C] < 0) GN_REQUIRE(sC == w, "root front with an update block");
    S.f_relmap_off[C + 1] = S.f_relmap_off[C] + (S.f_parent[C] >= 0 ? sC - w : 0);
  }
  S.relmap.resize(S.f_relmap_off[nf]);   // every entry written below
  S.a_kslot.resize(na);
  S.a_fpos.resize(na);
  // local row positions through a dense per-thread position map filled per
  // front (O(1) lookups); every front writes disjoint ranges (its own A
  // entries, its columns of L, its children's relmaps)
  int missing = 0;
#pragma omp parallel reduction(| : missing)
  {
    std::vector<int32_t> pos(n, -1);
#pragma omp for schedule(dynamic, 64)
    for (int64_t J = 0; J < nf; ++J) {
      const int64_t r0 = S.f_rows_off[J], r1 = S.f_rows_off[J + 1];
      for (int64_t q = r0; q < r1; ++q) pos[S.f_rows[q]] = static_cast<int32_t>(q - r0);
      const int64_t sJ = front_ld(S.f_nrows[J]);
      auto local = [&](int64_t row) -> int64_t {
        const int32_t v = pos[row];
        missing |= v < 0;
        return v < 0 ? 0 : v;
      };
      for (int32_t e = S.f_child_ptr[J]; e < S.f_child_ptr[J + 1]; ++e) {   // children's relmaps
        const int64_t C = S.f_child[e], w = S.f_ncols[C], sC = S.f_nrows[C];
        int64_t o = S.f_relmap_off[C];
        for (int64_t i = w; i < sC; ++i)
          S.relmap[o++] = static_cast<int32_t>(local(S.f_rows[S.f_rows_off[C] + i]));
      }
      for (int64_t q = per[J]; q < per[J + 1]; ++q) {   // A scatter
        const int64_t t = a_t[q], j = S.a_rowcol[t];
        S.a_kslot[q] = S.a_srcslot[t];
        S.a_fpos[q] = S.f_off[J] + (j - S.f_first[J]) * sJ + local(arow[t]);
      }
      for (int64_t q = r0; q < r1; ++q) pos[S.f_rows[q]] = -1;
    }
  }
  GN_REQUIRE(!missing, "row missing from front structure");
  // levels (leaves 0) and task order
  S.level.assign(nf, 0);
  int64_t maxl = 0;
  for (int64_t J = 0; J < nf; ++J) {  // children precede parents in index order
    for (int32_t t = S.f_child_ptr[J]; t < S.f_child_ptr[J + 1]; ++t)
      S.level[J] = std::max(S.level[J], S.level[S.f_child[t]] + 1);
    maxl = std::max<int64_t>(maxl, S.level[J]);
  }
  S.n_levels = nf ? maxl + 1 : 0;
  // warp tasks: fronts of <= kWarpFrontRows rows whose whole subtree is small
  // (children precede parents in index order, so one pass suffices)
  std::vector<char> small(nf, 0);
  for (int64_t J = 0; J < nf; ++J) {
    bool ok = S.f_nrows[J] <= kWarpFrontRows;
    for (int32_t t = S.f_child_ptr[J]; ok && t < S.f_child_ptr[J + 1]; ++t) ok = small[S.f_child[t]];
    small[J] = ok;
  }
  // task order: small fronts by level, then the other fronts by level
  S.order.resize(nf);
  S.nf_small = 0;
  {
    std::vector<int64_t> lc(2 * S.n_levels + 1, 0);
    auto bucket = [&](int64_t J) { return (small[J] ? 0 : S.n_levels) + S.level[J]; };
    for (int64_t J = 0; J < nf; ++J) lc[bucket(J) + 1]++, S.nf_small += small[J];
    for (int64_t l = 0; l < 2 * S.n_levels; ++l) lc[l + 1] += lc[l];
    // level boundaries of the small part (warp kernels run level by level)
    S.small_lptr.assign(S.n_levels + 1, 0);
    for (int64_t l = 0; l < S.n_levels; ++l) S.small_lptr[l + 1] = static_cast<int32_t>(lc[l + 1]);
    while (S.small_lptr.size() > 1 && S.small_lptr[S.small_lptr.size() - 2] == S.small_lptr.back())
      S.small_lptr.pop_back();
    for (int64_t J = 0; J < nf; ++J) S.order[lc[bucket(J)]++] = static_cast<int32_t>(J);
  }
  // top fronts: the highest complete levels of the large part holding at
  // most kTopFronts fronts, all of them tall (the cluster kernel's share)
  S.nf_top = 0;
  const char *e_tf = std::getenv("GN_TOP_FRONTS"), *e_tr = std::getenv("GN_TOP_MIN_ROWS");
  const int64_t top_fronts = e_tf ? std::atoll(e_tf) : kTopFronts;
  const int64_t top_min_rows = e_tr ? std::atoll(e_tr) : kTopMinRows;
  {
    int64_t k = nf, lev = -1;
    while (k > S.nf_small) {
      const int64_t l = S.level[S.order[k - 1]];
      int64_t b = k;
      while (b > S.nf_small && S.level[S.order[b - 1]] == l) --b;
      bool tall = true;
      for (int64_t q = b; q < k; ++q) tall = tall && S.f_nrows[S.order[q]] >= top_min_rows;
      if (!tall || nf - b > top_fronts) break;
      k = b;
      lev = l;
    }
    S.nf_top = lev >= 0 ? nf - k : 0;
  }
}

}  // namespace gn

using namespace gn;

extern "C" int gn_condense_create(int64_t n, int64_t nh, const int64_t *hr, const int64_t *hc,
                                  int64_t nj, const int64_t *jr, const int64_t *jc,
                                  gn_condense **out) {
  return guarded([&] {
    auto *C = new gn_condense();
    try {
      condense(*C, n, nh, hr, hc, nj, jr, jc);
    } catch (...) {
      delete C;
      throw;
    }
    *out = C;
  });
}

extern "C" int gn_condense_info(const gn_condense *C, int64_t *nnz_k, int64_t *np) {
  return guarded([&] {
    if (nnz_k) *nnz_k = static_cast<int64_t>(C->indices.size());
    if (np) *np = C->np;
  });
}

template <class T, class A>
static void copy_out(T *dst, const std::vector<T, A> &v) {
  if (dst && !v.empty()) std::memcpy(dst, v.data(), sizeof(T) * v.size());
}

extern "C" int gn_condense_export(const gn_condense *C, int64_t *indptr, int64_t *indices,
                                  int64_t *w_map, int64_t *diag_map, int64_t *ata_map,
                                  int64_t *ata_row, int64_t *ata_s1, int64_t *ata_s2) {
  return guarded([&] {
    copy_out(indptr, C->indptr);
    copy_out(indices, C->indices);
    const int64_t nh = C->nnz_h, n = C->n, np = C->np;
    if (w_map) std::memcpy(w_map, C->slot.data(), sizeof(int64_t) * nh);
    if (diag_map) std::memcpy(diag_map, C->slot.data() + nh, sizeof(int64_t) * n);
    if (ata_map) std::memcpy(ata_map, C->slot.data() + nh + n, sizeof(int64_t) * np);
    if (ata_row || ata_s1 || ata_s2) {
      const int64_t nseg = static_cast<int64_t>(C->seg.size()) - 1;
#pragma omp parallel for schedule(dynamic, 256)
      for (int64_t g = 0; g < nseg; ++g)
        for (int64_t q = C->seg_poff[g]; q < C->seg_poff[g + 1]; ++q) {
          int64_t row, s1, s2;
          C->product(q, g, row, s1, s2);
          if (ata_row) ata_row[q] = row;
          if (ata_s1) ata_s1[q] = s1;
          if (ata_s2) ata_s2[q] = s2;
        }
    }
  });
}

extern "C" void gn_condense_destroy(gn_condense *C) { delete C; }

extern "C" int gn_coo_to_csc(int64_t n, int64_t nnz, const int64_t *rows, const int64_t *cols,
                             int64_t *nnz_out, int64_t *indptr_out, int64_t *indices_out,
                             int64_t *slot_out) {
  return guarded([&] {
    GN_REQUIRE(n < (int64_t(1) << 31), "matrix too large for 32-bit indices");
    std::vector<int32_t> r32(nnz), c32(nnz);
    for (int64_t t = 0; t < nnz; ++t) {
      GN_REQUIRE(rows[t] >= 0 && rows[t] < n && cols[t] >= 0 && cols[t] < n, "index out of range");
      GN_REQUIRE(cols[t] <= rows[t], "entry above the diagonal");
      r32[t] = static_cast<int32_t>(rows[t]);
      c32[t] = static_cast<int32_t>(cols[t]);
    }
    std::vector<int64_t> indptr, indices, slot;
    csc_from_coords(n, r32, c32, indptr, indices, slot);
    if (nnz_out) *nnz_out = static_cast<int64_t>(indices.size());
    copy_out(indptr_out, indptr);
    copy_out(indices_out, indices);
    copy_out(slot_out, slot);
  });
}

extern "C" int gn_min_degree(int64_t n, const int64_t *indptr, const int64_t *indices, int64_t *perm) {
  return guarded([&] { min_degree(n, indptr, indices, perm); });
}

extern "C" int gn_symbolic_create(int64_t n, const int64_t *indptr, const int64_t *indices,
                                  const int64_t *perm, gn_symbolic **out) {
  return guarded([&] {
    GN_REQUIRE(n < (int64_t(1) << 31), "matrix too large for 32-bit device indices");
    auto *S = new gn_symbolic();
    try {
      symbolic(*S, n, indptr, indices, perm);
      if (n > 0) front_plan(*S);
    } catch (...) {
      delete S;
      throw;
    }
    *out = S;
  });
}

// The whole host analysis of one sparsity pattern in one call (condensed
// pattern, minimum degree unless `perm` is given, symbolic factor, front
// plan): a caller running it on a worker thread holds no interpreter lock
// in between.  `perm_out` (n) receives the ordering used.
extern "C" int gn_analyze(int64_t n, int64_t nh, const int64_t *hr, const int64_t *hc, int64_t nj,
                          const int64_t *jr, const int64_t *jc, const int64_t *perm, int64_t *perm_out,
                          gn_condense **cs_out, gn_symbolic **sym_out) {
  return guarded([&] {
    GN_REQUIRE(n < (int64_t(1) << 31), "matrix too large for 32-bit device indices");
    std::unique_ptr<gn_condense> C(new gn_condense());
    condense(*C, n, nh, hr, hc, nj, jr, jc);
    if (perm) {
      std::memcpy(perm_out, perm, sizeof(int64_t) * n);
    } else {
      PhaseTimer tm("min_degree");
      min_degree(n, C->indptr.data(), C->indices.data(), perm_out);
    }
    std::unique_ptr<gn_symbolic> S(new gn_symbolic());
    symbolic(*S, n, C->indptr.data(), C->indices.data(), perm_out);
    if (n > 0) front_plan(*S);
    *cs_out = C.release();
    *sym_out = S.release();
  });
}

extern "C" int gn_symbolic_info(const gn_symbolic *S, gn_symbolic_info_t *info) {
  return guarded([&] {
    info->n = S->n;
    info->nnz_a = S->nnz_a;
    info->nnz_l = S->nnz_l;
    info->n_fronts = S->nf;
    info->front_doubles = S->front_doubles;
    info->vec_doubles = S->vec_doubles;
    info->max_front = S->max_front;
    info->max_cols = S->max_cols;
    info->n_levels = S->n_levels;
    info->flops = S->flops;
  });
}

extern "C" int gn_symbolic_export(const gn_symbolic *S, int64_t *parent, int64_t *a_rowptr,
                                  int64_t *a_rowcol, int64_t *a_srcslot, int64_t *row_ptr,
                                  int64_t *row_cols, int64_t *l_colptr, int64_t *l_rowidx) {
  return guarded([&] {
    copy_out(parent, S->parent);
    copy_out(a_rowptr, S->a_rowptr);
    copy_out(a_rowcol, S->a_rowcol);
    copy_out(a_srcslot, S->a_srcslot);
    copy_out(row_ptr, S->row_ptr);
    if (row_cols) {   // the reference's sorted row patterns
      copy_out(row_cols, S->row_cols);
      const int64_t n = S->n;
#pragma omp parallel for schedule(dynamic, 1024)
      for (int64_t k = 0; k < n; ++k) std::sort(row_cols + S->row_ptr[k], row_cols + S->row_ptr[k + 1]);
    }
    copy_out(l_colptr, S->l_colptr);
    if (l_rowidx) {
      const_cast<Symbolic *>(static_cast<const Symbolic *>(S))->ensure_l_csc();
      copy_out(l_rowidx, S->l_rowidx);
    }
  });
}

extern "C" int gn_symbolic_fronts(const gn_symbolic *S, int32_t *first, int32_t *ncols, int32_t *nrows,
                                  int32_t *parent, int32_t *order, int64_t *nf_small) {
  return guarded([&] {
    copy_out(first, S->f_first);
    copy_out(ncols, S->f_ncols);
    copy_out(nrows, S->f_nrows);
    copy_out(parent, S->f_parent);
    copy_out(order, S->order);
    if (nf_small) *nf_small = S->nf_small;
  });
}

extern "C" void gn_symbolic_destroy(gn_symbolic *S) { delete S; }
