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
#include <memory>
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
  std::vector<uint64_t>& deaths = deaths_sorted;
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
  deaths.clear();
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
    deaths.push_back(k);
    parent[(size_t)young] = old;
    --comps;
  }
  for (int64_t i = 0; i < n; ++i)
    if (find((int32_t)i) == (int32_t)i) out.push(0.0f, INFINITY, (uint64_t)name[(size_t)i], UINT64_MAX);
  std::sort(deaths.begin(), deaths.end());
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

  // the K rows a scan is about to read (bitmap words, word offsets, packed ranks): all
  // their cache lines requested up front, so the misses overlap instead of queueing
  // behind one another through the word loop
  void prefetch_rows(const uint64_t* const* bw, const uint32_t* const* pre, int K) const {
#ifdef VR_NO_PREFETCH
    return;
#endif
    const int64_t W = M.bmw;
    for (int q = 0; q < K; ++q) {
      for (int64_t w = 0; w < W; w += 8) __builtin_prefetch(bw[q] + w);
      for (int64_t w = 0; w < W; w += 16) __builtin_prefetch(pre[q] + w);
      const uint32_t a = pre[q][0], b = pre[q][W - 1] + (uint32_t)__builtin_popcountll(bw[q][W - 1]);
      for (uint32_t k = a; k < b; k += 16) __builtin_prefetch(M.nb_rank.data() + k);
    }
  }
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
  // Dense mode: the rank matrix is symmetric, so R[v][s_q] is read as the contiguous row
  // R[s_q][.].  Output-sensitive mode (threshold-graph bitmap): only the common neighbours
  // of s are visited — the AND of its bitmap rows, in the same descending order (a cofacet
  // under the threshold needs v adjacent to all of s) — with their ranks from the packed
  // neighbour ranks, and the cofacet index in closed form: with j vertices of s above v,
  // cidx(s ∪ {v}) = A_j + C(v, d+2-j) + B_j.
  template <class F>
  void cofacets(const int* s, uint64_t cidx, uint32_t rs, F&& emit) const {
    if (!M.bm.empty()) {  // common neighbours = AND of the bitmap rows, descending
      uint64_t A[17], B[17];
      A[0] = 0;
      for (int j = 0; j <= d; ++j) A[j + 1] = A[j] + M.C(s[j], d + 2 - j);
      B[d + 1] = 0;
      for (int j = d; j >= 0; --j) B[j] = B[j + 1] + M.C(s[j], d + 1 - j);
      const uint64_t* bw[16];
      const uint32_t* pre[16];
      for (int q = 0; q <= d; ++q) {
        bw[q] = &M.bm[(size_t)s[q] * (size_t)M.bmw];
        pre[q] = &M.nb_pre[(size_t)s[q] * (size_t)M.bmw];
      }
      const uint32_t* NR = M.nb_rank.data();
      prefetch_rows(bw, pre, d + 1);
      int j = 0;  // vertices of s above v
      for (int64_t w = M.bmw - 1; w >= 0; --w) {
        uint64_t x = bw[0][w];
        for (int q = 1; q <= d; ++q) x &= bw[q][w];
        while (x) {
          const int b = 63 - __builtin_clzll(x);
          x ^= 1ull << b;
          const int v = (int)(w * 64 + b);  // never a vertex of s (no self loops)
          while (j <= d && s[j] > v) ++j;
          const uint64_t below = (1ull << b) - 1;
          uint32_t r = rs;
          for (int q = 0; q <= d; ++q) r = std::max(r, NR[pre[q][w] + (uint32_t)__builtin_popcountll(bw[q][w] & below)]);
          if (!emit(Entry{r, A[j] + M.C(v, d + 2 - j) + B[j]})) return;
        }
      }
      return;
    }
    // dense: blocks of 8 vertices, the rank maxima of a block in one vector pass, then the
    // (sequential) cofacet-index bookkeeping and the emits
    const uint32_t* rows[16];
    for (int q = 0; q <= d; ++q) rows[q] = &M.rank[(size_t)s[q] * (size_t)M.n];
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
    if (!M.bm.empty()) {
      const uint64_t* bw[16];
      const uint32_t* pre[16];
      for (int q = 0; q < K; ++q) {
        bw[q] = &M.bm[(size_t)S[q] * (size_t)M.bmw];
        pre[q] = &M.nb_pre[(size_t)S[q] * (size_t)M.bmw];
      }
      const uint32_t* NR = M.nb_rank.data();
      prefetch_rows(bw, pre, K);
      for (int64_t w = M.bmw - 1; w >= 0; --w) {
        uint64_t x = bw[0][w];
        for (int q = 1; q < K; ++q) x &= bw[q][w];
        while (x) {
          const int b = 63 - __builtin_clzll(x);
          x ^= 1ull << b;
          const uint64_t below = (1ull << b) - 1;
          bool ok = true;
          for (int q = 0; q < K && ok; ++q) ok = NR[pre[q][w] + (uint32_t)__builtin_popcountll(bw[q][w] & below)] <= r;
          if (ok) return w * 64 + b;
        }
      }
      return -1;
    }
    const uint32_t* rows[16];
    for (int q = 0; q < K; ++q) rows[q] = &M.rank[(size_t)S[q] * (size_t)M.n];
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
    uint32_t P[16][16];  // the edge ranks of t, read once
    for (int a = 0; a < d + 2; ++a)
      for (int b = a + 1; b < d + 2; ++b) P[a][b] = R(t[a], t[b]);
    // youngest facet: the first in Alg 16 order (drop t[0], t[1], ...) with diameter rt
    for (int j = 0; j < d + 2 && res < 0; ++j) {
      int f[16], m = 0;
      uint32_t df = 0;
      for (int q = 0; q < d + 2; ++q)
        if (q != j) f[m++] = t[q];
      for (int a = 0; a < d + 2; ++a)
        for (int b = a + 1; b < d + 2; ++b)
          if (a != j && b != j) df = std::max(df, P[a][b]);
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
  // R(u, v) from the packed neighbour ranks when present (u, v adjacent: cache-resident),
  // else from the n*n matrix
  uint32_t R(int u, int v) const {
    if (M.nb_pre.empty()) return M.R(u, v);
    const size_t w = (size_t)u * (size_t)M.bmw + (size_t)(v >> 6);
    return M.nb_rank[M.nb_pre[w] + (uint32_t)__builtin_popcountll(M.bm[w] & ((1ull << (v & 63)) - 1))];
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

// Radix heap with 4-bit digits: a key lives in the bucket (L, g) where L is the highest
// nibble in which it differs from `last` and g is its nibble L (keys equal to `last` in
// bucket E).  The minimum is in the lowest non-empty level's lowest non-empty digit
// (occupancy masks), and when that bucket is split every key moves to a strictly lower
// level: at most one move per nibble of the key instead of one per BIT in the binary radix
// heap above — the working columns of long reductions are mostly keys far above the pivot
// that the binary heap re-files level after level (config 2's H3 column: pivot time
// halved).  16 buckets per level keep the heap small for the many short columns.  Same Z/2
// cancellation and the same drop rule.
template <class K>
struct RadixHeapN {
  static constexpr int NL = (int)sizeof(K) * 2;  // nibbles
  std::vector<K> eq;                // keys == last
  std::vector<K> b[NL][16];
  uint16_t dmask[NL];               // non-empty digits per level
  uint32_t lmask = 0;               // non-empty levels
  K last = 0;
  size_t sz = 0;
  int cb;
  K mask;
  RadixHeapN(uint32_t, int cbits) : cb(cbits), mask(cbits >= (int)sizeof(K) * 8 ? ~(K)0 : (((K)1 << cbits) - 1)) {
    std::memset(dmask, 0, sizeof(dmask));
  }
  static int hinib(K d);
  void put(K x) {
    const K diff = x ^ last;
    if (diff == 0) { eq.push_back(x); return; }
    const int L = hinib(diff);
    const int dg = (int)((x >> (4 * L)) & 0xF);
    b[L][dg].push_back(x);
    dmask[L] |= (uint16_t)(1u << dg);
    lmask |= 1u << L;
  }
  void push(uint32_t r, uint64_t c) {
    const K x = ((K)r << cb) | (mask - (K)c);
    if (x < last) return;  // below the pivot: cancels within the added column
    put(x);
    ++sz;
  }
  void clear() {
    eq.clear();
    while (lmask) {
      const int L = __builtin_ctz(lmask);
      lmask &= lmask - 1;
      uint32_t m = dmask[L];
      while (m) {
        b[L][__builtin_ctz(m)].clear();
        m &= m - 1;
      }
      dmask[L] = 0;
    }
    last = 0;
    sz = 0;
  }
  bool settle() {
    if (sz == 0) return false;
    if (!eq.empty()) return true;
    const int L = __builtin_ctz(lmask);
    const int dg = __builtin_ctz((uint32_t)dmask[L]);
    std::vector<K>& v = b[L][dg];
    K m = v[0];
    for (K x : v) m = x < m ? x : m;
    last = m;
    dmask[L] = (uint16_t)(dmask[L] & ~(1u << dg));
    if (!dmask[L]) lmask &= ~(1u << L);
    for (K x : v) put(x);  // every key lands at a level below L
    v.clear();
    return true;
  }
  bool pivot(uint32_t& r, uint64_t& c) {
    while (settle()) {
      const size_t n0 = eq.size();
      if (n0 & 1) {
        if (n0 > 1) { eq.resize(1); sz -= n0 - 1; }
        r = (uint32_t)(last >> cb);
        c = (uint64_t)(mask - (last & mask));
        return true;
      }
      sz -= n0;
      eq.clear();
    }
    return false;
  }
};
template <> inline int RadixHeapN<uint64_t>::hinib(uint64_t d) { return (63 - __builtin_clzll(d)) >> 2; }
template <> inline int RadixHeapN<unsigned __int128>::hinib(unsigned __int128 d) {
  const uint64_t hi = (uint64_t)(d >> 64);
  return hi ? 16 + ((63 - __builtin_clzll(hi)) >> 2) : ((63 - __builtin_clzll((uint64_t)d)) >> 2);
}

// The working heap of the reduction-matrix mode: nibble digits for 64-bit keys (measured on
// the box, 16 threads: config 2 dimension 3 892 -> 780 ms, config 5 dimension 1 183 -> 160 ms,
// dimension 2 178 -> 168 ms), the binary radix heap for 128-bit keys (config 5 dimension 3,
// 552K short columns: the larger nibble heaps, 32 per thread, cost 11%).
template <class K> struct WorkHeapOf { using type = RadixHeapN<K>; };
template <> struct WorkHeapOf<unsigned __int128> { using type = RadixHeap<unsigned __int128>; };
#ifdef VR_BINARY_RADIX
template <class K> using WorkHeap = RadixHeap<K>;
#else
template <class K> using WorkHeap = typename WorkHeapOf<K>::type;
#endif

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
                       const ResidualHints* hints, int mode, HeapT& W, HostPairs& out, std::vector<uint64_t>& deaths,
                       ResidualStats& st) {
  Ctx cx(M, d);
  const uint64_t cmask = cbits >= 64 ? ~0ull : ((1ull << cbits) - 1);
  auto colkey = [&](uint32_t r, uint64_t c) -> uint64_t { return ((uint64_t)(maxr - r) << cbits) | c; };
  // stored reduction columns V_k (column keys), pool-allocated
  std::vector<uint64_t> vpool;
  std::vector<std::pair<uint64_t, uint32_t>> vcol;  // (offset, length) per residual column with a pivot
  U64Map pivot_col((size_t)nkeys + 16);             // row cidx -> index into vcol
  U64Map app_memo(1024);                            // row cidx -> apparent partner cidx or -1
  std::vector<uint64_t> work_v;
  deaths.clear();
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
    if (hints) {  // the first equal-diameter cofacet and its apparent claim, precomputed
      const uint64_t t = hints->first[c];
      int64_t col;
      check = false;
      if (t != UINT64_MAX && !hints->claimed[c] && !pivot_col.get(t, col)) {
        first = Entry{rs, t};
        emergent = true;
      }
    }
    if (!emergent) cx.cofacets(s, sc, rs, [&](const Entry& e) {
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
      deaths.push_back(first.cidx);
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
        // an apparent pair has zero persistence: diam(a) = diam(pivot row)
        push_coboundary((uint64_t)a, pe.r);
        if (mode == 0) work_v.push_back(colkey(pe.r, (uint64_t)a));
      }
      ++st.additions;
      have = W.pivot(pe.r, pe.cidx);
    }
    if (have) {
      out.push(birth, M.value[pe.r], sc, pe.cidx);
      deaths.push_back(pe.cidx);
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
  st.apparent_checks += cx.apparent_checks;
}

// ------------------------------------------------------------------ parallel (speculative)
// Reduction-matrix mode on T threads with IN-ORDER COMMIT.  The columns (in coboundary
// order) are cut into blocks of B; a thread takes a block and first reduces each of its
// columns speculatively against the pivots committed so far (every addition of an earlier
// column with the same pivot is a step the standard algorithm, Alg 11, could take), keeping
// each column's working heap.  It then waits until every earlier block has committed and
// commits its columns in order: re-check the pivot against the now complete table of earlier
// pivots, keep reducing if needed, claim it.  The committed pivots are therefore exactly the
// sequential algorithm's; one hand-off between threads per block, not per column.
struct ConcPivotMap {  // insert-only, one writer at a time (the committing column)
  struct Slot {
    std::atomic<uint64_t> k;
    int64_t v;
  };
  std::unique_ptr<Slot[]> t;  // key and value in one slot: one cache line per probe
  size_t mask;
  explicit ConcPivotMap(size_t cap) {
    size_t c = 16;
    while (c < cap + cap / 2) c <<= 1;  // load <= 2/3
    t.reset(new Slot[c]);
    for (size_t i = 0; i < c; ++i) {
      t[i].k.store(~0ull, std::memory_order_relaxed);
      t[i].v = -1;
    }
    mask = c - 1;
  }
  void prefetch(uint64_t key) const { __builtin_prefetch(&t[U64Map::h(key) & mask]); }
  bool get(uint64_t key, int64_t& out) const {
    for (size_t i = U64Map::h(key) & mask;; i = (i + 1) & mask) {
      const uint64_t x = t[i].k.load(std::memory_order_acquire);
      if (x == key) { out = t[i].v; return true; }
      if (x == ~0ull) return false;
    }
  }
  // insert key -> val unless present (then false): one probe sequence
  bool put_if_absent(uint64_t key, int64_t val) {
    for (size_t i = U64Map::h(key) & mask;; i = (i + 1) & mask) {
      const uint64_t x = t[i].k.load(std::memory_order_relaxed);
      if (x == key) return false;
      if (x == ~0ull) {
        t[i].v = val;
        t[i].k.store(key, std::memory_order_release);
        return true;
      }
    }
  }
  void put(uint64_t key, int64_t val) { put_if_absent(key, val); }
};

template <class K>
void residual_reduce_par(const HostMatrix& M, int d, uint32_t maxr, int cbits, const uint64_t* keys, uint64_t nkeys, int cb,
                         const ResidualHints* hints, int nthreads, HostPairs& out, std::vector<uint64_t>& deaths,
                         ResidualStats& stats) {
  const uint64_t cmask = cbits >= 64 ? ~0ull : ((1ull << cbits) - 1);
  struct ColOut {
    uint32_t death_r = 0;
    uint64_t death_cidx = UINT64_MAX;  // UINT64_MAX: essential
    bool emergent = false;
    int64_t adds = 0, cobs = 0;
  };
  std::vector<ColOut> res((size_t)nkeys);
  // reduction columns V_j = {keys[j]} + vextra[j] (empty for most columns: no allocation)
  std::vector<std::vector<uint64_t>> vextra((size_t)nkeys);
  ConcPivotMap pivots((size_t)nkeys + 16);
  // block size: whole blocks are speculated by one thread, so small blocks where the
  // columns are few (and long: dimension 1), up to 32 where they are many and short
  int64_t B = std::max<int64_t>(1, std::min<int64_t>(32, (int64_t)(nkeys / ((uint64_t)nthreads * 256))));
  if (const char* e = std::getenv("VR_RESIDUAL_BLOCK")) B = std::max<int64_t>(1, std::atoll(e));
  const uint64_t nblocks = (nkeys + (uint64_t)B - 1) / (uint64_t)B;
  std::atomic<uint64_t> next_commit{0}, next_block{0};

  auto worker = [&]() {
    Ctx cx(M, d);
    U64Map app_memo(1024);
    // per column of the block: its working heap, its reduction column, its state
    std::vector<WorkHeap<K>> heaps;
    heaps.reserve((size_t)B);
    for (int64_t i = 0; i < B; ++i) heaps.emplace_back(maxr, cb);
    std::vector<std::vector<uint64_t>> works((size_t)B);
    struct St {
      Entry pe, first;
      bool have, emergent;
    };
    std::vector<St> sts((size_t)B);
    int s[16], f[16];
    auto apparent_of = [&](const Entry& e) -> int64_t {
      int64_t a;
      if (app_memo.get(e.cidx, a)) return a;
      a = cx.apparent_partner(e.cidx, e.r);
      app_memo.put(e.cidx, a);
      return a;
    };
    // reduce column j's heap while its pivot is claimed by a committed column or an
    // apparent pair
    auto reduce = [&](uint64_t j, WorkHeap<K>& W, std::vector<uint64_t>& work_v, St& S) {
      ColOut& R = res[(size_t)j];
      auto push_coboundary = [&](uint64_t cidx, uint32_t r) {
        ++R.cobs;
        cx.decode(cidx, d + 1, f);
        cx.cofacets(f, cidx, r, [&](const Entry& e) { W.push(e.r, e.cidx); return true; });
      };
      while (S.have) {
        int64_t col;
        if (pivots.get(S.pe.cidx, col)) {
          const uint64_t k0 = keys[(size_t)col];
          push_coboundary(k0 & cmask, maxr - (uint32_t)(k0 >> cbits));
          work_v.push_back(k0);
          for (const uint64_t vk : vextra[(size_t)col]) {
            push_coboundary(vk & cmask, maxr - (uint32_t)(vk >> cbits));
            work_v.push_back(vk);
          }
        } else {
          const int64_t a = apparent_of(S.pe);
          if (a < 0) break;
          // an apparent pair has zero persistence: diam(a) = diam(pivot row)
          push_coboundary((uint64_t)a, S.pe.r);
          work_v.push_back(((uint64_t)(maxr - S.pe.r) << cbits) | (uint64_t)a);
        }
        ++R.adds;
        S.have = W.pivot(S.pe.r, S.pe.cidx);
      }
    };
    for (;;) {
      const uint64_t blk = next_block.fetch_add(1, std::memory_order_relaxed);
      if (blk >= nblocks) break;
      const uint64_t j0 = blk * (uint64_t)B, j1 = std::min(nkeys, j0 + (uint64_t)B);
      // phase 1: speculative, against the pivots committed so far
      for (uint64_t j = j0; j < j1; ++j) {
        const size_t i = (size_t)(j - j0);
        WorkHeap<K>& W = heaps[i];
        St& S = sts[i];
        const uint64_t key = keys[j];
        const uint32_t rs = maxr - (uint32_t)(key >> cbits);
        const uint64_t sc = key & cmask;
        W.clear();
        works[i].assign(1, key);
        S.emergent = false;
        S.have = false;
        // emergent check on the first equal-diameter cofacet (§5.2.11)
        bool check = true;
        int64_t col;
        if (hints) {
          const uint64_t t = hints->first[j];
          check = false;
          if (t != UINT64_MAX && !hints->claimed[j] && !pivots.get(t, col)) {
            S.first = Entry{rs, t};
            S.emergent = true;
            continue;  // decided at commit by one lookup
          }
        }
        cx.decode(sc, d + 1, s);
        cx.cofacets(s, sc, rs, [&](const Entry& e) {
          if (check && e.r == rs) {
            int64_t c2;
            if (!pivots.get(e.cidx, c2) && apparent_of(e) < 0) { S.first = e; S.emergent = true; return false; }
            check = false;
          }
          W.push(e.r, e.cidx);
          return true;
        });
        if (S.emergent) continue;
        S.have = W.pivot(S.pe.r, S.pe.cidx);
        reduce(j, W, works[i], S);
      }
      // phase 2: wait for every earlier block, then commit in order
      if (hints)
        for (uint64_t j = j0; j < j1; ++j)
          if (sts[(size_t)(j - j0)].emergent) pivots.prefetch(sts[(size_t)(j - j0)].first.cidx);
      {
        int spins = 0;
        while (next_commit.load(std::memory_order_acquire) != blk) {
          if (++spins > 1024) std::this_thread::yield();
        }
      }
      for (uint64_t j = j0; j < j1; ++j) {
        const size_t i = (size_t)(j - j0);
        WorkHeap<K>& W = heaps[i];
        St& S = sts[i];
        ColOut& R = res[(size_t)j];
        const uint64_t key = keys[j];
        if (S.emergent) {
          if (pivots.put_if_absent(S.first.cidx, (int64_t)j)) {
            R.emergent = true;
            R.death_r = S.first.r;
            R.death_cidx = S.first.cidx;
            continue;
          }
          // an earlier column took that row: the full coboundary, reduced normally
          const uint32_t rs = maxr - (uint32_t)(key >> cbits);
          const uint64_t sc = key & cmask;
          cx.decode(sc, d + 1, s);
          W.clear();
          cx.cofacets(s, sc, rs, [&](const Entry& e) { W.push(e.r, e.cidx); return true; });
          S.have = W.pivot(S.pe.r, S.pe.cidx);
        }
        reduce(j, W, works[i], S);  // the table of earlier pivots is final now
        if (S.have) {
          R.death_r = S.pe.r;
          R.death_cidx = S.pe.cidx;
          auto& V = vextra[(size_t)j];
          std::vector<uint64_t>& work_v = works[i];
          if (work_v.size() > 1) {
            std::sort(work_v.begin() + 1, work_v.end());
            for (size_t a = 1; a < work_v.size();) {
              size_t q = a;
              while (q < work_v.size() && work_v[q] == work_v[a]) ++q;
              if (((q - a) & 1) && work_v[a] != key) V.push_back(work_v[a]);
              a = q;
            }
          }
          pivots.put(S.pe.cidx, (int64_t)j);
        }
      }
      next_commit.store(blk + 1, std::memory_order_release);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < nthreads; ++t) pool.emplace_back(worker);
  for (auto& th : pool) th.join();

  deaths.clear();
  deaths.reserve((size_t)nkeys);
  out.birth.reserve(out.birth.size() + (size_t)nkeys);
  out.death.reserve(out.death.size() + (size_t)nkeys);
  out.birth_cidx.reserve(out.birth_cidx.size() + (size_t)nkeys);
  out.death_cidx.reserve(out.death_cidx.size() + (size_t)nkeys);
  for (uint64_t j = 0; j < nkeys; ++j) {
    const ColOut& R = res[(size_t)j];
    const uint32_t rs = maxr - (uint32_t)(keys[j] >> cbits);
    const uint64_t sc = keys[j] & cmask;
    stats.additions += R.adds;
    stats.coboundaries += R.cobs;
    stats.emergent += R.emergent;
    if (R.death_cidx != UINT64_MAX) {
      out.push(M.value[rs], M.value[R.death_r], sc, R.death_cidx);
      deaths.push_back(R.death_cidx);
    } else {
      out.push(M.value[rs], INFINITY, sc, UINT64_MAX);
    }
  }
}

}  // namespace

void residual_hints_host(const HostMatrix& M, int d, uint32_t maxr, int cbits, const uint64_t* keys, uint64_t nkeys,
                         uint64_t* first, uint8_t* claimed) {
  Ctx cx(M, d);
  const uint64_t cmask = cbits >= 64 ? ~0ull : ((1ull << cbits) - 1);
  int s[16], t[16];
  for (uint64_t c = 0; c < nkeys; ++c) {
    const uint32_t rs = maxr - (uint32_t)(keys[c] >> cbits);
    cx.decode(keys[c] & cmask, d + 1, s);
    first[c] = UINT64_MAX;
    claimed[c] = 0;
    const int64_t v = cx.first_equal_cofacet_vertex(s, d + 1, rs);
    if (v < 0) continue;
    int m = 0, q = 0;
    for (; q <= d && s[q] > v; ++q) t[m++] = s[q];
    t[m++] = (int)v;
    for (; q <= d; ++q) t[m++] = s[q];
    uint64_t tc = 0;
    for (int p = 0; p < m; ++p) tc += M.C(t[p], m - p);
    first[c] = tc;
    claimed[c] = cx.apparent_partner(tc, rs) >= 0;
  }
}

void residual_reduce(const HostMatrix& M, int d, uint32_t maxr, int cbits, const uint64_t* keys, uint64_t nkeys, int mode,
                     HostPairs& out, std::vector<uint64_t>& deaths, ResidualStats& st, const ResidualHints* hints) {
  // row keys pack (rank, ~cofacet cidx): 64 bits when they fit, else 128
  const uint64_t cof = M.C(M.n, d + 2);
  int cb = 1;
  while (cb < 64 && (cof >> cb) != 0) ++cb;
  int rb = 1;
  while (rb < 32 && (maxr >> rb) != 0) ++rb;
  using u128 = unsigned __int128;
  int nthreads = (int)std::min<unsigned>(16u, std::max(1u, std::thread::hardware_concurrency()));
  if (const char* e = std::getenv("VR_RESIDUAL_THREADS")) nthreads = std::max(1, std::atoi(e));
  if (mode == 0 && nthreads > 1 && (nkeys >= 64 || std::getenv("VR_RESIDUAL_THREADS"))) {
    if (rb + cb <= 64) residual_reduce_par<uint64_t>(M, d, maxr, cbits, keys, nkeys, cb, hints, nthreads, out, deaths, st);
    else residual_reduce_par<u128>(M, d, maxr, cbits, keys, nkeys, cb, hints, nthreads, out, deaths, st);
    return;
  }
  if (rb + cb <= 64) {
    if (mode == 0) {
      WorkHeap<uint64_t> W(maxr, cb);
      residual_reduce_t(M, d, maxr, cbits, keys, nkeys, hints, mode, W, out, deaths, st);
    } else {
      BinHeap<uint64_t> W(maxr, cb);
      residual_reduce_t(M, d, maxr, cbits, keys, nkeys, hints, mode, W, out, deaths, st);
    }
  } else {
    if (mode == 0) {
      WorkHeap<u128> W(maxr, cb);
      residual_reduce_t(M, d, maxr, cbits, keys, nkeys, hints, mode, W, out, deaths, st);
    } else {
      BinHeap<u128> W(maxr, cb);
      residual_reduce_t(M, d, maxr, cbits, keys, nkeys, hints, mode, W, out, deaths, st);
    }
  }
}

}  // namespace vr
