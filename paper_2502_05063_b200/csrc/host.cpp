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
#if defined(__x86_64__)
#include <immintrin.h>
#endif
#include <atomic>
#include <thread>
#include <functional>
#include <chrono>
#include <cstdio>
#include <cstdlib>
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

// Dense scan of first_equal_cofacet_vertex, 8 vertices per step (AVX2): the first v
// (descending) with max_q rows[q][v] <= r, skipping members of S.
#if defined(__x86_64__)
__attribute__((target("avx2"))) int64_t first_equal_dense_avx2(const uint32_t* const* rows, const int* S, int K, uint32_t r,
                                                              int64_t n) {
  const __m256i vr = _mm256_set1_epi32((int)(r ^ 0x80000000u));
  const __m256i flip = _mm256_set1_epi32((int)0x80000000u);
  int64_t v = n;
  while (v >= 8) {
    const int64_t b = v - 8;  // lanes b .. b+7
    __m256i m = _mm256_loadu_si256((const __m256i*)(rows[0] + b));
    for (int q = 1; q < K; ++q) m = _mm256_max_epu32(m, _mm256_loadu_si256((const __m256i*)(rows[q] + b)));
    // m <= r (unsigned): !(m > r), signed compare after flipping the sign bit
    const __m256i gt = _mm256_cmpgt_epi32(_mm256_xor_si256(m, flip), vr);
    unsigned ok = ~(unsigned)_mm256_movemask_ps(_mm256_castsi256_ps(gt)) & 0xFFu;
    while (ok) {
      const int lane = 31 - __builtin_clz(ok);  // highest vertex first
      const int64_t c = b + lane;
      bool member = false;
      for (int q = 0; q < K; ++q) member = member || S[q] == c;
      if (!member) return c;
      ok &= ~(1u << lane);
    }
    v = b;
  }
  for (int64_t c = v - 1; c >= 0; --c) {
    bool ok = true;
    for (int q = 0; q < K && ok; ++q) ok = (c != S[q]) && rows[q][c] <= r;
    if (ok) return c;
  }
  return -1;
}
const bool g_host_avx2 = __builtin_cpu_supports("avx2");
// out[i] = max(rs, max_q rows[q][lo + i]), i = 0..7
__attribute__((target("avx2"))) void block_max8_avx2(const uint32_t* const* rows, int K, int64_t lo, uint32_t rs,
                                                     uint32_t* out) {
  __m256i m = _mm256_set1_epi32((int)rs);
  for (int q = 0; q < K; ++q) m = _mm256_max_epu32(m, _mm256_loadu_si256((const __m256i*)(rows[q] + lo)));
  _mm256_store_si256((__m256i*)out, m);
}
#endif

struct Ctx {
  const HostMatrix& M;
  int d;  // column dimension
  int64_t apparent_checks = 0;  // apparent_partner evaluations (the callers memoize)
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
  // coboundary of the d-simplex s in lex-decreasing order (Alg 14, reading A2), with ranks.
  // The rank matrix is symmetric, so R[v][s_q] is read as the contiguous row R[s_q][.].
  // With a threshold-graph adjacency only the neighbours of the vertex of s with the
  // fewest neighbours are visited (a cofacet under the threshold needs v adjacent to all
  // of s), in the same descending order; the cofacet index is then computed in closed
  // form: with j vertices of s above v, cidx(s ∪ {v}) = A_j + C(v, d+2-j) + B_j.
  template <class F>
  void cofacets(const int* s, uint64_t cidx, uint32_t rs, F&& emit) const {
    const uint32_t* rows[16];
    for (int q = 0; q <= d; ++q) rows[q] = &M.rank[(size_t)s[q] * (size_t)M.n];
    if (!M.adj_off.empty()) {
      uint64_t A[17], B[17];
      A[0] = 0;
      for (int j = 0; j <= d; ++j) A[j + 1] = A[j] + M.C(s[j], d + 2 - j);
      B[d + 1] = 0;
      for (int j = d; j >= 0; --j) B[j] = B[j + 1] + M.C(s[j], d + 1 - j);
      int anchor = s[0];
      uint32_t best = ~0u;
      for (int q = 0; q <= d; ++q) {
        const uint32_t dg = M.adj_off[(size_t)s[q] + 1] - M.adj_off[(size_t)s[q]];
        if (dg < best) { best = dg; anchor = s[q]; }
      }
      const uint16_t* L = M.adj.data() + M.adj_off[(size_t)anchor];
      int j = 0;  // vertices of s above v
      for (uint32_t k = 0; k < best; ++k) {
        const int v = L[k];
        while (j <= d && s[j] > v) ++j;
        if (j <= d && s[j] == v) continue;
        uint32_t r = rs;
        for (int q = 0; q <= d; ++q) r = std::max(r, rows[q][v]);
        if (r == VR_RINF_H) continue;
        if (!emit(Entry{r, A[j] + M.C(v, d + 2 - j) + B[j]})) return;
      }
      return;
    }
    // blocks of 8 vertices: the rank maxima of a block in one vector pass, then the
    // (sequential) cofacet-index bookkeeping and the emits
    uint64_t below = cidx, above = 0;
    int k = d + 1, j = 0;
    alignas(32) uint32_t rb[8];
    for (int64_t v = M.n - 1; v >= 0;) {
      const int64_t lo = v >= 7 ? v - 7 : 0;
#if defined(__x86_64__)
      if (g_host_avx2 && v - lo == 7) block_max8_avx2(rows, d + 1, lo, rs, rb);
      else
#endif
        for (int64_t u = lo; u <= v; ++u) {
          uint32_t r = rs;
          for (int q = 0; q <= d; ++q) r = std::max(r, rows[q][u]);
          rb[u - lo] = r;
        }
      for (int64_t u = v; u >= lo; --u) {
        if (j <= d && u == s[j]) {  // a vertex of s: one more vertex above the next cofacets
          below -= M.C(s[j], k);
          above += M.C(s[j], k + 1);
          --k;
          ++j;
          continue;
        }
        const uint32_t r = rb[u - lo];
        if (r == VR_RINF_H) continue;
        if (!emit(Entry{r, above + M.C(u, k + 1) + below})) return;
      }
      v = lo - 1;
    }
  }
  // first v (descending) not in S (K vertices) with max_{w in S} R[w][v] <= r, or -1
  int64_t first_equal_cofacet_vertex(const int* S, int K, uint32_t r) const {
    const uint32_t* rows[16];
    for (int q = 0; q < K; ++q) rows[q] = &M.rank[(size_t)S[q] * (size_t)M.n];
    if (!M.adj_off.empty()) {
      int anchor = S[0];
      uint32_t best = ~0u;
      for (int q = 0; q < K; ++q) {
        const uint32_t dg = M.adj_off[(size_t)S[q] + 1] - M.adj_off[(size_t)S[q]];
        if (dg < best) { best = dg; anchor = S[q]; }
      }
      const uint16_t* L = M.adj.data() + M.adj_off[(size_t)anchor];
      for (uint32_t k = 0; k < best; ++k) {
        const int v = L[k];
        bool ok = true;
        for (int q = 0; q < K && ok; ++q) ok = (v != S[q]) && rows[q][v] <= r;
        if (ok) return v;
      }
      return -1;
    }
#if defined(__x86_64__)
    if (g_host_avx2) return first_equal_dense_avx2(rows, S, K, r, M.n);
#endif
    for (int64_t v = M.n - 1; v >= 0; --v) {
      bool ok = true;
      for (int q = 0; q < K && ok; ++q) ok = (v != S[q]) && rows[q][v] <= r;
      if (ok) return v;
    }
    return -1;
  }
  // Is row t (a (d+1)-simplex of rank rt) the apparent cofacet of some column f?  Returns f.
  int64_t apparent_partner(uint64_t tcidx, uint32_t rt) {
    ++apparent_checks;
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
    return res;
  }
  uint32_t diam_rank(const int* s) const {
    uint32_t r = 0;
    for (int a = 0; a <= d; ++a)
      for (int b = a + 1; b <= d; ++b) r = std::max(r, M.R(s[a], s[b]));
    return r;
  }
};

// Open-addressing hash map uint64 -> int64 (linear probing; key ~0 = empty).
struct U64Map {
  std::vector<uint64_t> k;
  std::vector<int64_t> v;
  size_t n = 0, mask = 0;
  explicit U64Map(size_t cap = 1024) { rehash(cap); }
  static uint64_t h(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
  }
  void rehash(size_t cap) {
    size_t c = 16;
    while (c < cap * 2) c <<= 1;
    std::vector<uint64_t> ok = std::move(k);
    std::vector<int64_t> ov = std::move(v);
    k.assign(c, ~0ull);
    v.assign(c, 0);
    mask = c - 1;
    n = 0;
    for (size_t i = 0; i < ok.size(); ++i)
      if (ok[i] != ~0ull) put(ok[i], ov[i]);
  }
  bool get(uint64_t key, int64_t& out) const {
    for (size_t i = h(key) & mask;; i = (i + 1) & mask) {
      if (k[i] == key) { out = v[i]; return true; }
      if (k[i] == ~0ull) return false;
    }
  }
  void put(uint64_t key, int64_t val) {
    if ((n + 1) * 2 > k.size()) rehash(k.size());
    for (size_t i = h(key) & mask;; i = (i + 1) & mask) {
      if (k[i] == key) { v[i] = val; return; }
      if (k[i] == ~0ull) { k[i] = key; v[i] = val; ++n; return; }
    }
  }
};

template <class K> inline int bitlen(K x);
template <> inline int bitlen<uint64_t>(uint64_t x) { return x ? 64 - __builtin_clzll(x) : 0; }
template <> inline int bitlen<unsigned __int128>(unsigned __int128 x) {
  const uint64_t hi = (uint64_t)(x >> 64), lo = (uint64_t)x;
  return hi ? 128 - __builtin_clzll(hi) : (lo ? 64 - __builtin_clzll(lo) : 0);
}

// Monotone radix heap over packed (rank, ~cidx) row keys, with Z/2 cancellation, for the
// reduction-matrix mode.  Valid because the pivot of the working column never decreases
// in row order: each added column R_k = sum of the coboundaries of V_k has the current
// pivot as its minimum, so whatever it pushes below the pivot occurs an even number of
// times and cancels — such pushes are dropped, which keeps every key >= `last`.
template <class K>
struct RadixHeap {
  static constexpr int NB = (int)sizeof(K) * 8 + 1;
  std::vector<K> b[NB];
  K last = 0;
  size_t sz = 0;
  int cb;
  K mask;
  RadixHeap(uint32_t, int cbits) : cb(cbits), mask(cbits >= (int)sizeof(K) * 8 ? ~(K)0 : (((K)1 << cbits) - 1)) {}
  void push(uint32_t r, uint64_t c) {
    const K x = ((K)r << cb) | (mask - (K)c);
    if (x < last) return;  // below the pivot: cancels within the added column
    b[bitlen<K>(x ^ last)].push_back(x);
    ++sz;
  }
  void clear() {
    for (auto& v : b) v.clear();
    last = 0;
    sz = 0;
  }
  bool settle() {
    if (sz == 0) return false;
    if (!b[0].empty()) return true;
    int i = 1;
    while (b[i].empty()) ++i;
    K m = b[i][0];
    for (K x : b[i]) m = x < m ? x : m;
    last = m;
    for (K x : b[i]) b[bitlen<K>(x ^ last)].push_back(x);
    b[i].clear();
    return true;
  }
  bool pivot(uint32_t& r, uint64_t& c) {
    while (settle()) {
      const size_t n0 = b[0].size();
      if (n0 & 1) {
        if (n0 > 1) { b[0].resize(1); sz -= n0 - 1; }
        r = (uint32_t)(last >> cb);
        c = (uint64_t)(mask - (last & mask));
        return true;
      }
      sz -= n0;
      b[0].clear();
    }
    return false;
  }
};

// Binary heap over packed (rank, ~cidx) keys for the oblivious mode (Alg 12 adds raw
// coboundaries D_k, whose entries can lie below the current pivot: not monotone).
template <class K>
struct BinHeap {
  std::vector<K> h;
  int cb;
  K mask;
  BinHeap(uint32_t, int cbits) : cb(cbits), mask(cbits >= (int)sizeof(K) * 8 ? ~(K)0 : (((K)1 << cbits) - 1)) {}
  void push(uint32_t r, uint64_t c) {
    h.push_back(((K)r << cb) | (mask - (K)c));
    std::push_heap(h.begin(), h.end(), std::greater<K>());
  }
  void clear() { h.clear(); }
  bool pivot(uint32_t& r, uint64_t& c) {
    while (!h.empty()) {
      K m = h.front();
      std::pop_heap(h.begin(), h.end(), std::greater<K>());
      h.pop_back();
      if (!h.empty() && h.front() == m) {
        std::pop_heap(h.begin(), h.end(), std::greater<K>());
        h.pop_back();
        continue;
      }
      h.push_back(m);
      std::push_heap(h.begin(), h.end(), std::greater<K>());
      r = (uint32_t)(m >> cb);
      c = (uint64_t)(mask - (m & mask));
      return true;
    }
    return false;
  }
};

template <class HeapT>
void residual_reduce_t(const HostMatrix& M, int d, uint32_t maxr, int cbits, const uint64_t* keys, uint64_t nkeys,
                       int mode, HeapT& W, HostPairs& out, std::vector<uint64_t>& deaths_sorted, ResidualStats& st) {
  Ctx cx(M, d);
  const uint64_t cmask = cbits >= 64 ? ~0ull : ((1ull << cbits) - 1);
  auto colkey = [&](uint32_t r, uint64_t c) -> uint64_t { return ((uint64_t)(maxr - r) << cbits) | c; };
  // stored reduction columns V_k (column keys), pool-allocated
  std::vector<uint64_t> vpool;
  std::vector<std::pair<uint64_t, uint32_t>> vcol;  // (offset, length) per residual column with a pivot
  U64Map pivot_col((size_t)nkeys + 16);             // row cidx -> index into vcol
  U64Map app_memo(1024);                            // row cidx -> apparent partner cidx or -1
  std::vector<uint64_t> work_v;
  deaths_sorted.clear();
  int s[16], f[16];

  auto apparent_of = [&](const Entry& e) -> int64_t {
    int64_t a;
    if (app_memo.get(e.cidx, a)) return a;
    a = cx.apparent_partner(e.cidx, e.r);
    app_memo.put(e.cidx, a);
    return a;
  };
  auto push_coboundary = [&](uint64_t cidx, uint32_t r) {
    ++st.coboundaries;
    cx.decode(cidx, d + 1, f);
    cx.cofacets(f, cidx, r, [&](const Entry& e) { W.push(e.r, e.cidx); return true; });
  };

  for (uint64_t c = 0; c < nkeys; ++c) {
    const uint64_t key = keys[c];
    const uint32_t rs = maxr - (uint32_t)(key >> cbits);
    const uint64_t sc = key & cmask;
    cx.decode(sc, d + 1, s);
    W.clear();
    work_v.clear();
    work_v.push_back(key);
    // initial coboundary; emergent check on the first equal-diameter cofacet (§5.2.11)
    bool check = true, emergent = false;
    Entry first{0, 0};
    cx.cofacets(s, sc, rs, [&](const Entry& e) {
      if (check && e.r == rs) {
        int64_t col;
        if (!pivot_col.get(e.cidx, col) && apparent_of(e) < 0) { first = e; emergent = true; return false; }
        check = false;
      }
      W.push(e.r, e.cidx);
      return true;
    });
    const float birth = M.value[rs];
    if (emergent) {
      ++st.emergent;
      out.push(birth, M.value[first.r], sc, first.cidx);
      deaths_sorted.push_back(first.cidx);
      pivot_col.put(first.cidx, (int64_t)vcol.size());
      vcol.push_back({vpool.size(), 1});
      vpool.push_back(key);
      continue;
    }
    Entry pe{0, 0};
    bool have = W.pivot(pe.r, pe.cidx);
    while (have) {
      int64_t col;
      if (pivot_col.get(pe.cidx, col)) {
        const auto& vc = vcol[(size_t)col];
        if (mode == 0) {
          for (uint32_t q = 0; q < vc.second; ++q) {
            const uint64_t vk = vpool[vc.first + q];
            push_coboundary(vk & cmask, maxr - (uint32_t)(vk >> cbits));
            work_v.push_back(vk);
          }
        } else {
          const uint64_t vk = vpool[vc.first];  // the column's own simplex (first entry)
          push_coboundary(vk & cmask, maxr - (uint32_t)(vk >> cbits));
        }
      } else {
        const int64_t a = apparent_of(pe);
        if (a < 0) break;  // unclaimed pivot
        int fv[16];
        cx.decode((uint64_t)a, d + 1, fv);
        const uint32_t fr = cx.diam_rank(fv);
        push_coboundary((uint64_t)a, fr);
        if (mode == 0) work_v.push_back(colkey(fr, (uint64_t)a));
      }
      ++st.additions;
      have = W.pivot(pe.r, pe.cidx);
    }
    if (have) {
      out.push(birth, M.value[pe.r], sc, pe.cidx);
      deaths_sorted.push_back(pe.cidx);
      pivot_col.put(pe.cidx, (int64_t)vcol.size());
      const size_t off = vpool.size();
      if (mode == 0 && work_v.size() > 1) {
        // Z/2-cancel the reduction column; keep the column's own simplex first
        std::sort(work_v.begin() + 1, work_v.end());
        vpool.push_back(key);
        for (size_t i = 1; i < work_v.size();) {
          size_t j = i;
          while (j < work_v.size() && work_v[j] == work_v[i]) ++j;
          if (((j - i) & 1) && work_v[i] != key) vpool.push_back(work_v[i]);
          i = j;
        }
      } else {
        vpool.push_back(key);
      }
      vcol.push_back({off, (uint32_t)(vpool.size() - off)});
    } else {
      out.push(birth, INFINITY, sc, UINT64_MAX);  // zero column: essential class
    }
  }
  std::sort(deaths_sorted.begin(), deaths_sorted.end());
  st.apparent_checks += cx.apparent_checks;
}

// ------------------------------------------------------------------ parallel (speculative)
// Reduction-matrix mode on T threads with IN-ORDER COMMIT.  Threads take columns in
// coboundary order and reduce them concurrently against the pivots committed so far
// (every addition of an earlier column with the same pivot is a step the standard
// algorithm, Alg 11, could take).  A column may only claim its final pivot when every
// earlier column has committed: it waits for its turn, re-checks the pivot against the
// now complete table of earlier pivots, keeps reducing if needed, then commits.  The
// committed pivots are therefore exactly the sequential algorithm's.
struct ConcPivotMap {  // insert-only, one writer at a time (the committing column)
  std::vector<std::atomic<uint64_t>> k;
  std::vector<int64_t> v;
  size_t mask;
  explicit ConcPivotMap(size_t cap) {
    size_t c = 16;
    while (c < cap * 2) c <<= 1;
    k = std::vector<std::atomic<uint64_t>>(c);
    for (auto& x : k) x.store(~0ull, std::memory_order_relaxed);
    v.assign(c, -1);
    mask = c - 1;
  }
  bool get(uint64_t key, int64_t& out) const {
    for (size_t i = U64Map::h(key) & mask;; i = (i + 1) & mask) {
      const uint64_t x = k[i].load(std::memory_order_acquire);
      if (x == key) { out = v[i]; return true; }
      if (x == ~0ull) return false;
    }
  }
  void put(uint64_t key, int64_t val) {
    for (size_t i = U64Map::h(key) & mask;; i = (i + 1) & mask) {
      if (k[i].load(std::memory_order_relaxed) == ~0ull) {
        v[i] = val;
        k[i].store(key, std::memory_order_release);
        return;
      }
    }
  }
};

template <class K>
void residual_reduce_par(const HostMatrix& M, int d, uint32_t maxr, int cbits, const uint64_t* keys, uint64_t nkeys, int cb,
                         int nthreads, HostPairs& out, std::vector<uint64_t>& deaths_sorted, ResidualStats& stats) {
  const uint64_t cmask = cbits >= 64 ? ~0ull : ((1ull << cbits) - 1);
  struct ColOut {
    uint32_t death_r = 0;
    uint64_t death_cidx = UINT64_MAX;  // UINT64_MAX: essential
    bool emergent = false;
    int64_t adds = 0, cobs = 0;
  };
  std::vector<ColOut> res((size_t)nkeys);
  std::vector<std::vector<uint64_t>> vcols((size_t)nkeys);
  ConcPivotMap pivots((size_t)nkeys + 16);
  std::atomic<uint64_t> next_commit{0}, next_col{0};

  auto worker = [&]() {
    Ctx cx(M, d);
    U64Map app_memo(1024);
    RadixHeap<K> W(maxr, cb);
    std::vector<uint64_t> work_v;
    int s[16], f[16];
    auto apparent_of = [&](const Entry& e) -> int64_t {
      int64_t a;
      if (app_memo.get(e.cidx, a)) return a;
      a = cx.apparent_partner(e.cidx, e.r);
      app_memo.put(e.cidx, a);
      return a;
    };
    auto wait_turn = [&](uint64_t j) {
      int spins = 0;
      while (next_commit.load(std::memory_order_acquire) != j) {
        if (++spins > 64) std::this_thread::yield();
      }
    };
    for (;;) {
      const uint64_t j = next_col.fetch_add(1, std::memory_order_relaxed);
      if (j >= nkeys) break;
      ColOut& R = res[(size_t)j];
      const uint64_t key = keys[j];
      const uint32_t rs = maxr - (uint32_t)(key >> cbits);
      const uint64_t sc = key & cmask;
      cx.decode(sc, d + 1, s);
      W.clear();
      work_v.clear();
      work_v.push_back(key);
      auto push_coboundary = [&](uint64_t cidx, uint32_t r) {
        ++R.cobs;
        cx.decode(cidx, d + 1, f);
        cx.cofacets(f, cidx, r, [&](const Entry& e) { W.push(e.r, e.cidx); return true; });
      };
      // initial coboundary with the emergent check (§5.2.11), speculative
      bool check = true, emergent = false;
      Entry first{0, 0};
      cx.cofacets(s, sc, rs, [&](const Entry& e) {
        if (check && e.r == rs) {
          int64_t col;
          if (!pivots.get(e.cidx, col) && apparent_of(e) < 0) { first = e; emergent = true; return false; }
          check = false;
        }
        W.push(e.r, e.cidx);
        return true;
      });
      if (emergent) {
        wait_turn(j);
        int64_t col;
        if (!pivots.get(first.cidx, col)) {
          R.emergent = true;
          R.death_r = first.r;
          R.death_cidx = first.cidx;
          vcols[(size_t)j].assign(1, key);
          pivots.put(first.cidx, (int64_t)j);
          next_commit.store(j + 1, std::memory_order_release);
          continue;
        }
        // an earlier column took that row meanwhile: reduce normally (we hold the turn)
        W.clear();
        cx.cofacets(s, sc, rs, [&](const Entry& e) { W.push(e.r, e.cidx); return true; });
      }
      Entry pe{0, 0};
      bool have = W.pivot(pe.r, pe.cidx);
      bool my_turn = emergent;
      for (;;) {
        while (have) {
          int64_t col;
          if (pivots.get(pe.cidx, col)) {
            for (const uint64_t vk : vcols[(size_t)col]) {
              push_coboundary(vk & cmask, maxr - (uint32_t)(vk >> cbits));
              work_v.push_back(vk);
            }
          } else {
            const int64_t a = apparent_of(pe);
            if (a < 0) break;
            int fv[16];
            cx.decode((uint64_t)a, d + 1, fv);
            const uint32_t fr = cx.diam_rank(fv);
            push_coboundary((uint64_t)a, fr);
            work_v.push_back(((uint64_t)(maxr - fr) << cbits) | (uint64_t)a);
          }
          ++R.adds;
          have = W.pivot(pe.r, pe.cidx);
        }
        if (my_turn) break;
        wait_turn(j);  // every earlier column has committed: the pivot table is final for us
        my_turn = true;
        int64_t col;
        if (have && pivots.get(pe.cidx, col)) continue;
        if (have && apparent_of(pe) >= 0) continue;
        break;
      }
      if (have) {
        R.death_r = pe.r;
        R.death_cidx = pe.cidx;
        auto& V = vcols[(size_t)j];
        V.clear();
        V.push_back(key);
        if (work_v.size() > 1) {
          std::sort(work_v.begin() + 1, work_v.end());
          for (size_t i = 1; i < work_v.size();) {
            size_t q = i;
            while (q < work_v.size() && work_v[q] == work_v[i]) ++q;
            if (((q - i) & 1) && work_v[i] != key) V.push_back(work_v[i]);
            i = q;
          }
        }
        pivots.put(pe.cidx, (int64_t)j);
      }
      next_commit.store(j + 1, std::memory_order_release);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < nthreads; ++t) pool.emplace_back(worker);
  for (auto& th : pool) th.join();

  deaths_sorted.clear();
  for (uint64_t j = 0; j < nkeys; ++j) {
    const ColOut& R = res[(size_t)j];
    const uint32_t rs = maxr - (uint32_t)(keys[j] >> cbits);
    const uint64_t sc = keys[j] & cmask;
    stats.additions += R.adds;
    stats.coboundaries += R.cobs;
    stats.emergent += R.emergent;
    if (R.death_cidx != UINT64_MAX) {
      out.push(M.value[rs], M.value[R.death_r], sc, R.death_cidx);
      deaths_sorted.push_back(R.death_cidx);
    } else {
      out.push(M.value[rs], INFINITY, sc, UINT64_MAX);
    }
  }
  std::sort(deaths_sorted.begin(), deaths_sorted.end());
}

}  // namespace

void residual_reduce(const HostMatrix& M, int d, uint32_t maxr, int cbits, const uint64_t* keys, uint64_t nkeys, int mode,
                     HostPairs& out, std::vector<uint64_t>& deaths_sorted, ResidualStats& st) {
  // row keys pack (rank, ~cofacet cidx): 64 bits when they fit, else 128
  const uint64_t cof = M.C(M.n, d + 2);
  int cb = 1;
  while (cb < 64 && (cof >> cb) != 0) ++cb;
  int rb = 1;
  while (rb < 32 && (maxr >> rb) != 0) ++rb;
  using u128 = unsigned __int128;
  int nthreads = (int)std::min<unsigned>(16u, std::max(1u, std::thread::hardware_concurrency()));
  if (const char* e = std::getenv("VR_RESIDUAL_THREADS")) nthreads = std::max(1, std::atoi(e));
  if (mode == 0 && nthreads > 1 && nkeys >= 64) {
    if (rb + cb <= 64) residual_reduce_par<uint64_t>(M, d, maxr, cbits, keys, nkeys, cb, nthreads, out, deaths_sorted, st);
    else residual_reduce_par<u128>(M, d, maxr, cbits, keys, nkeys, cb, nthreads, out, deaths_sorted, st);
    return;
  }
  if (rb + cb <= 64) {
    if (mode == 0) {
      RadixHeap<uint64_t> W(maxr, cb);
      residual_reduce_t(M, d, maxr, cbits, keys, nkeys, mode, W, out, deaths_sorted, st);
    } else {
      BinHeap<uint64_t> W(maxr, cb);
      residual_reduce_t(M, d, maxr, cbits, keys, nkeys, mode, W, out, deaths_sorted, st);
    }
  } else {
    if (mode == 0) {
      RadixHeap<u128> W(maxr, cb);
      residual_reduce_t(M, d, maxr, cbits, keys, nkeys, mode, W, out, deaths_sorted, st);
    } else {
      BinHeap<u128> W(maxr, cb);
      residual_reduce_t(M, d, maxr, cbits, keys, nkeys, mode, W, out, deaths_sorted, st);
    }
  }
}

}  // namespace vr
