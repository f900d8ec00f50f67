// host.cpp — the two steps either side of the GPU hot path, on the host (SURVEY.md §8(a)
// "off path, reported separately"):
//
//   dim0_union_find   §5.2.5: Kruskal / union-find over the edges in
//                     filtration order.  Elder rule under §5.1.4: every vertex has diameter
//                     0, so a LARGER vertex id is OLDER; a component is named by its max id
//                     and on a merging edge the component with the smaller name dies,
//                     giving the pair (that vertex, edge) (reading A26).
//
//   residual_reduce   the submatrix reduction of the non-apparent, non-cleared columns in
//                     coboundary order with the implicit coboundary (§5.2.8): cofacets are
//                     generated from cidx and the rank matrix (Alg 14), the working column is
//                     a heap with Z/2 cancellation, pivot = the OLDEST cofacet (smallest
//                     diameter, then largest cidx: the lowest row of the coboundary matrix).
//                     Modes: reduction matrix V (§5.2.9, Ripser's default) or oblivious
//                     (Alg 12; Lemma 5.2.10).  Emergent shortcut (§5.2.11).
//                     Pivot lookup = this dimension's residual pairs (hash map, layer 1 of
//                     Fig 5.10) then the apparent pairs, RECOMPUTED instead of stored
//                     (layer 2): row t is claimed by an apparent column f iff f, the youngest
//                     facet of t, has t as its lex-greatest equal-diameter cofacet.  Every
//                     apparent row counts as claimed even if f lies to the right: f's row has
//                     only zeros to the left of f (Def 5.3.4), so no column left of f can
//                     ever have its pivot there.
#include <algorithm>
#include <cstring>
#include <cmath>
#include <cstdint>
#include <queue>
#include <unordered_map>
#include <vector>

#include "vr_internal.h"

#define VR_RINF_H 0xFFFFFFFFu

namespace vr {

// ------------------------------------------------------------------ dimension 0
void dim0_union_find(int64_t n, const uint64_t* edges_sorted, uint64_t m, int kbits, HostPairs& out,
                     std::vector<uint64_t>& deaths_sorted) {
  const uint64_t N = (uint64_t)n * (uint64_t)(n - 1) / 2;
  const uint64_t kmask = kbits >= 64 ? ~0ull : ((1ull << kbits) - 1);
  std::vector<int32_t> parent((size_t)n), name((size_t)n);
  for (int64_t i = 0; i < n; ++i) parent[(size_t)i] = (int32_t)i, name[(size_t)i] = (int32_t)i;
  auto find = [&](int32_t x) {
    while (parent[(size_t)x] != x) {
      parent[(size_t)x] = parent[(size_t)parent[(size_t)x]];
      x = parent[(size_t)x];
    }
    return x;
  };
  int64_t comps = n;
  deaths_sorted.clear();
  for (uint64_t e = 0; e < m && comps > 1; ++e) {
    const uint64_t key = edges_sorted[e];
    const uint64_t k = N - 1 - (key & kmask);  // lower-distance index == edge cidx
    uint32_t fb = (uint32_t)(key >> kbits);
    float diam;
    std::memcpy(&diam, &fb, sizeof diam);
    int64_t i = (int64_t)std::floor((1.0 + std::sqrt(1.0 + 8.0 * (double)k)) / 2.0);
    while (i * (i - 1) / 2 > (int64_t)k) --i;
    while ((i + 1) * i / 2 <= (int64_t)k) ++i;
    const int64_t j = (int64_t)k - i * (i - 1) / 2;
    int32_t ri = find((int32_t)i), rj = find((int32_t)j);
    if (ri == rj) continue;
    // the younger component (smaller oldest-vertex id) dies at this edge
    int32_t young = name[(size_t)ri] < name[(size_t)rj] ? ri : rj;
    int32_t old = young == ri ? rj : ri;
    out.push(0.0f, diam, (uint64_t)name[(size_t)young], k);
    deaths_sorted.push_back(k);
    parent[(size_t)young] = old;
    --comps;
  }
  for (int64_t i = 0; i < n; ++i)
    if (find((int32_t)i) == (int32_t)i) out.push(0.0f, INFINITY, (uint64_t)name[(size_t)i], UINT64_MAX);
  std::sort(deaths_sorted.begin(), deaths_sorted.end());
}

// ------------------------------------------------------------------ residual reduction
namespace {

struct Entry {
  uint32_t r;     // diameter rank
  uint64_t cidx;
  bool operator==(const Entry& o) const { return r == o.r && cidx == o.cidx; }
};
// priority_queue top = the pivot: smallest rank, then largest cidx
struct PivotLess {
  bool operator()(const Entry& a, const Entry& b) const { return a.r > b.r || (a.r == b.r && a.cidx < b.cidx); }
};
using Heap = std::priority_queue<Entry, std::vector<Entry>, PivotLess>;

struct Ctx {
  const HostMatrix& M;
  int d;  // column dimension
  std::unordered_map<uint64_t, int64_t> apparent_memo;  // row cidx -> partner column cidx or -1
  Ctx(const HostMatrix& m, int dd) : M(m), d(dd) {}

  void decode(uint64_t cidx, int k /*vertices*/, int* v) const {
    int64_t hi = M.n;
    for (int p = 0; p < k; ++p) {
      const int kk = k - p;
      int64_t lo = kk - 1, h = hi - 1;
      while (lo < h) {
        int64_t mid = (lo + h + 1) >> 1;
        if (M.C(mid, kk) <= cidx) lo = mid; else h = mid - 1;
      }
      v[p] = (int)lo;
      cidx -= M.C(lo, kk);
      hi = lo;
    }
  }
  // coboundary of the d-simplex s in lex-decreasing order (Alg 14, reading A2), with ranks
  template <class F>
  void cofacets(const int* s, uint64_t cidx, uint32_t rs, F&& emit) const {
    uint64_t below = cidx, above = 0;
    int k = d + 1, j = 0;
    for (int64_t v = M.n - 1; v >= 0; --v) {
      while (j <= d && v == s[j]) {
        below -= M.C(s[j], k);
        above += M.C(s[j], k + 1);
        --k; ++j; --v;
      }
      if (v < 0) break;
      uint32_t r = rs;
      const uint32_t* row = &M.rank[(size_t)v * (size_t)M.n];
      for (int q = 0; q <= d; ++q) r = std::max(r, row[s[q]]);
      if (r == VR_RINF_H) continue;
      if (!emit(Entry{r, above + M.C(v, k + 1) + below})) return;
    }
  }
  // first v (descending) not in S (K vertices) with max_{w in S} R[v][w] <= r, or -1
  int64_t first_equal_cofacet_vertex(const int* S, int K, uint32_t r) const {
    for (int64_t v = M.n - 1; v >= 0; --v) {
      const uint32_t* row = &M.rank[(size_t)v * (size_t)M.n];
      bool ok = true;
      for (int q = 0; q < K && ok; ++q) ok = (v != S[q]) && row[S[q]] <= r;
      if (ok) return v;
    }
    return -1;
  }
  // Is row t (a (d+1)-simplex of rank rt) the apparent cofacet of some column f?  Returns f.
  int64_t apparent_partner(uint64_t tcidx, uint32_t rt) {
    auto it = apparent_memo.find(tcidx);
    if (it != apparent_memo.end()) return it->second;
    int t[16];
    decode(tcidx, d + 2, t);
    int64_t res = -1;
    // youngest facet: the first in Alg 16 order (drop t[0], t[1], ...) with diameter rt
    for (int j = 0; j < d + 2 && res < 0; ++j) {
      int f[16], m = 0;
      uint32_t df = 0;
      for (int q = 0; q < d + 2; ++q)
        if (q != j) f[m++] = t[q];
      for (int a = 0; a < m; ++a)
        for (int b = a + 1; b < m; ++b) df = std::max(df, M.R(f[a], f[b]));
      if (df != rt) continue;
      if (first_equal_cofacet_vertex(f, d + 1, rt) == t[j]) {
        uint64_t c = 0;
        for (int p = 0; p < m; ++p) c += M.C(f[p], m - p);
        res = (int64_t)c;
      }
      break;  // only the youngest facet can be the apparent partner
    }
    apparent_memo.emplace(tcidx, res);
    return res;
  }
  uint32_t diam_rank(const int* s) const {
    uint32_t r = 0;
    for (int a = 0; a <= d; ++a)
      for (int b = a + 1; b <= d; ++b) r = std::max(r, M.R(s[a], s[b]));
    return r;
  }
};

bool pop_pivot(Heap& h, Entry& out) {
  while (!h.empty()) {
    Entry e = h.top();
    h.pop();
    if (!h.empty() && h.top() == e) {
      h.pop();
      continue;
    }
    out = e;
    return true;
  }
  return false;
}
bool get_pivot(Heap& h, Entry& out) {
  if (!pop_pivot(h, out)) return false;
  h.push(out);
  return true;
}

}  // namespace

void residual_reduce(const HostMatrix& M, int d, uint32_t maxr, int cbits, const uint64_t* keys, uint64_t nkeys, int mode,
                     HostPairs& out, std::vector<uint64_t>& deaths_sorted, ResidualStats& st) {
  Ctx cx(M, d);
  const uint64_t cmask = cbits >= 64 ? ~0ull : ((1ull << cbits) - 1);
  struct Col {
    uint64_t cidx;
    uint32_t r;
    std::vector<Entry> V;  // reduction column (simplices whose coboundaries sum to R_j), incl. itself
  };
  std::vector<Col> cols;
  std::unordered_map<uint64_t, int64_t> pivot_col;  // row cidx -> index into cols
  deaths_sorted.clear();
  int s[16], f[16];

  for (uint64_t c = 0; c < nkeys; ++c) {
    const uint64_t key = keys[c];
    const uint32_t rs = maxr - (uint32_t)(key >> cbits);
    const uint64_t sc = key & cmask;
    cx.decode(sc, d + 1, s);

    auto claimed = [&](const Entry& e, int64_t& col, int64_t& app) {
      auto it = pivot_col.find(e.cidx);
      if (it != pivot_col.end()) { col = it->second; app = -1; return true; }
      int64_t a = cx.apparent_partner(e.cidx, e.r);
      if (a >= 0) { col = -1; app = a; return true; }
      return false;
    };

    Heap W;
    std::vector<Entry> work_v;  // reduction column under construction (Z/2, cancelled at the end)
    work_v.push_back(Entry{rs, sc});
    // initial coboundary with the emergent check on the first equal-diameter cofacet
    bool check = true, emergent = false;
    Entry piv{0, 0};
    cx.cofacets(s, sc, rs, [&](const Entry& e) {
      if (check && e.r == rs) {
        int64_t col, app;
        if (!claimed(e, col, app)) { piv = e; emergent = true; return false; }
        check = false;
      }
      W.push(e);
      return true;
    });
    bool have = emergent;
    if (!emergent) have = get_pivot(W, piv);
    if (emergent) ++st.emergent;
    while (have && !emergent) {
      int64_t col, app;
      if (!claimed(piv, col, app)) break;
      ++st.additions;
      auto add_simplex = [&](uint64_t cidx, uint32_t r) {
        cx.decode(cidx, d + 1, f);
        cx.cofacets(f, cidx, r, [&](const Entry& e) { W.push(e); return true; });
      };
      if (col >= 0) {
        const Col& K = cols[(size_t)col];
        if (mode == 0) {
          for (const Entry& e : K.V) { add_simplex(e.cidx, e.r); work_v.push_back(e); }
        } else {
          add_simplex(K.cidx, K.r);
        }
      } else {
        int fv[16];
        cx.decode((uint64_t)app, d + 1, fv);
        const uint32_t fr = cx.diam_rank(fv);
        add_simplex((uint64_t)app, fr);
        if (mode == 0) work_v.push_back(Entry{fr, (uint64_t)app});
      }
      have = get_pivot(W, piv);
    }
    const float birth = M.value[rs];
    if (have) {
      const float death = M.value[piv.r];
      out.push(birth, death, sc, piv.cidx);
      deaths_sorted.push_back(piv.cidx);
      Col K{sc, rs, {}};
      if (mode == 0 && !emergent) {
        // Z/2-cancel the reduction column
        std::sort(work_v.begin(), work_v.end(), [](const Entry& a, const Entry& b) { return a.cidx < b.cidx; });
        for (size_t i = 0; i < work_v.size();) {
          size_t j = i;
          while (j < work_v.size() && work_v[j].cidx == work_v[i].cidx) ++j;
          if ((j - i) & 1) K.V.push_back(work_v[i]);
          i = j;
        }
      } else {
        K.V.push_back(Entry{rs, sc});
      }
      pivot_col.emplace(piv.cidx, (int64_t)cols.size());
      cols.push_back(std::move(K));
    } else {
      out.push(birth, INFINITY, sc, UINT64_MAX);  // zero column: essential class
    }
  }
  std::sort(deaths_sorted.begin(), deaths_sorted.end());
}

}  // namespace vr
