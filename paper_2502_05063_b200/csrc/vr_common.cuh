// vr_common.cuh — device-side building blocks shared by the libvr kernels.
//
// Data layout in HBM:
//   rank   : uint32 n x n, row-major, symmetric.  rank[i*n+j] = position of the first
//            occurrence of d(i,j) in the ascending sort of all n(n-1)/2 distances, if
//            d(i,j) <= t, else RINF.  Ranks preserve order and equality of the fp32
//            distances exactly, so every diameter comparison of the method (Eq 5.3, the
//            "diam(t) = diam(s)" tests of Lemma 5.3.6) is an exact integer comparison, and
//            a rank maps back to the fp32 distance bit-exactly (sorted[rank]).
//   binom  : uint64 [k][v], k in [0, kmax], v in [0, n]: C(v, k) (Eq 5.6).
//   keys   : uint64 column key = ((maxr - rank(diam)) << cbits) | cidx, so that ascending
//            key order is coboundary order: diameter descending, cidx ascending
//            (Fig 5.2 caption).
#pragma once
#include <cassert>
#include <cstdint>
#include <cuda_runtime.h>

// Bounds checks of shared-memory lists, output slots and table probes: compiled in by the
// checked build (build.py --checks -> libvr_checks.so, -DVR_CHECKS), which the GPU tests can
// run (VR_LIB=...libvr_checks.so) in place of compute-sanitizer (closed on this pool).
#ifdef VR_CHECKS
#define VR_ASSERT(c) assert(c)
#else
#define VR_ASSERT(c) ((void)0)
#endif

#include "vr_types.h"

#define VR_RINF 0xFFFFFFFFu

namespace vr {

struct Tables {
  const uint32_t* __restrict__ rank;  // n*n
  const uint64_t* __restrict__ binom; // (kmax+1)*(n+1)
  int32_t n;
  int32_t kmax;
};

__device__ __forceinline__ uint64_t binom(const Tables& T, int v, int k) {
  return __ldg(T.binom + (size_t)k * (size_t)(T.n + 1) + (size_t)v);
}

// (32-bit index arithmetic: n <= 65535 keeps i*n + j below 2^32)
__device__ __forceinline__ uint32_t rank_at(const Tables& T, int i, int j) {
  return __ldg(T.rank + ((uint32_t)i * (uint32_t)T.n + (uint32_t)j));
}

// Largest v in [k-1, hi-1] with C(v, k) <= x  (C(., k) is non-decreasing; C(k-1, k) = 0).
// This is the per-vertex search of the combinatorial number system (A31): a float
// estimate v ~ (k! x)^(1/k) + (k-1)/2 (C(v,k) ~ (v-(k-1)/2)^k / k!), then exact integer
// steps on the binomial table — one or two table reads instead of a binary search.
__device__ __forceinline__ int cns_find(const Tables& T, uint64_t x, int k, int hi) {
  int g;
  if (k == 1) {
    g = x < (uint64_t)hi ? (int)x : hi - 1;
  } else {
    float kf = 1.f;
    for (int i = 2; i <= k; ++i) kf *= (float)i;
    const float est = (k == 2) ? sqrtf(2.f * (float)x) + 0.5f : __powf(kf * (float)x, 1.f / (float)k) + 0.5f * (float)(k - 1);
    g = (int)est;
    g = g < k - 1 ? k - 1 : (g > hi - 1 ? hi - 1 : g);
  }
  while (g > k - 1 && binom(T, g, k) > x) --g;
  while (g + 1 < hi && binom(T, g + 1, k) <= x) ++g;
  return g;
}

// Eq 5.6 decode: cidx of a dim-d simplex -> vertices s[0] > s[1] > ... > s[d].
template <int D>
__device__ __forceinline__ void cns_decode(const Tables& T, uint64_t cidx, int (&s)[D + 1]) {
  int hi = T.n;
#pragma unroll
  for (int p = 0; p <= D; ++p) {
    const int k = D + 1 - p;
    int v = cns_find(T, cidx, k, hi);
    s[p] = v;
    cidx -= binom(T, v, k);
    hi = v;
  }
}

// Eq 5.6 encode of vertices in decreasing order.
template <int K>
__device__ __forceinline__ uint64_t cns_encode(const Tables& T, const int (&s)[K]) {
  uint64_t c = 0;
#pragma unroll
  for (int p = 0; p < K; ++p) c += binom(T, s[p], K - p);
  return c;
}

// cidx of the cofacet s ∪ {v} (v not in s) — Eq 5.6 on the merged decreasing tuple.
template <int D>
__device__ __forceinline__ uint64_t cofacet_cidx(const Tables& T, const int (&s)[D + 1], int v) {
  uint64_t c = 0;
  int pos = 0;  // position in the merged tuple (0 = largest)
  bool placed = false;
#pragma unroll
  for (int p = 0; p <= D; ++p) {
    if (!placed && v > s[p]) { c += binom(T, v, D + 2 - pos); ++pos; placed = true; }
    c += binom(T, s[p], D + 2 - pos);
    ++pos;
  }
  if (!placed) c += binom(T, v, 1);
  return c;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Warp-aggregated append (§5.5.3 "warp-based filtering": one atomic per warp, ballot
// within the warp).  Every lane of the warp must call it.  Returns the slot or ~0 if
// the lane does not append.  Order within a warp step is lane order.
__device__ __forceinline__ unsigned long long warp_append(bool pred, unsigned long long* counter) {
  const uint32_t m = __ballot_sync(0xffffffffu, pred);
  if (!m) return ~0ull;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(counter, (unsigned long long)__popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  return pred ? base + (unsigned long long)__popc(m & lanemask_lt()) : ~0ull;
}

__device__ __forceinline__ bool sorted_contains(const uint64_t* __restrict__ a, int64_t n, uint64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < x) lo = mid + 1; else hi = mid;
  }
  return lo < n && __ldg(a + lo) == x;
}

__device__ __forceinline__ uint32_t umax(uint32_t a, uint32_t b) { return a > b ? a : b; }

__device__ __forceinline__ bool bit_test(const uint32_t* __restrict__ bm, uint64_t i) {
  return (__ldg(bm + (i >> 5)) >> (i & 31)) & 1u;
}
__device__ __forceinline__ void bit_set(uint32_t* bm, uint64_t i) { atomicOr(bm + (i >> 5), 1u << (i & 31)); }
// open-addressing set of 64-bit keys (~0 = empty slot, linear probing); the caller sizes the
// table to at least twice the keys it can receive
__device__ __forceinline__ uint64_t hash_slot(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}
__device__ __forceinline__ void hash_put(uint64_t* t, uint64_t mask, uint64_t k) {
  VR_ASSERT(k != ~0ull);
#ifdef VR_CHECKS
  uint64_t probes = 0;
#endif
  for (uint64_t i = hash_slot(k) & mask;; i = (i + 1) & mask) {
#ifdef VR_CHECKS
    assert(++probes <= mask + 1);  // (a full table would loop forever)
#endif
    const unsigned long long prev = atomicCAS((unsigned long long*)(t + i), ~0ull, (unsigned long long)k);
    if (prev == ~0ull || prev == k) return;
  }
}
__device__ __forceinline__ bool hash_has(const uint64_t* t, uint64_t mask, uint64_t k) {
  for (uint64_t i = hash_slot(k) & mask;; i = (i + 1) & mask) {
    const uint64_t x = __ldcg(t + i);
    if (x == k) return true;
    if (x == ~0ull) return false;
  }
}

// The clearing set of a dimension (output-sensitive mode): the cidx of its columns that are
// pivots (deaths) of the dimension below, in the open-addressing table above, fronted by a
// blocked Bloom filter — one 32-bit word per key with 3 bits set — that answers most of the
// (mostly negative) membership probes from a few MB that stay in L2.
__device__ __forceinline__ void bloom_of(const ClearSet& c, uint64_t h, uint32_t& word, uint32_t& bits) {
  word = (uint32_t)(((uint64_t)(uint32_t)(h >> 32) * (uint64_t)c.bloom_words) >> 32);
  bits = (1u << (h & 31)) | (1u << ((h >> 5) & 31)) | (1u << ((h >> 10) & 31));
}
__device__ __forceinline__ void set_put(const ClearSet& c, uint64_t k) {
  uint32_t w, b;
  bloom_of(c, hash_slot(k), w, b);
  atomicOr(c.bloom + w, b);
  hash_put(c.table, c.mask, k);
}
__device__ __forceinline__ bool set_has(const ClearSet& c, uint64_t k) {
  uint32_t w, b;
  bloom_of(c, hash_slot(k), w, b);
  if ((__ldcg(c.bloom + w) & b) != b) return false;
  return hash_has(c.table, c.mask, k);
}

template <int D>
__device__ __forceinline__ uint4 pack_vertices(const int (&s)[D + 1]) {
  uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
  for (int i = 0; i <= D; ++i) w[i >> 1] |= (uint32_t)s[i] << ((i & 1) * 16);
  return make_uint4(w[0], w[1], w[2], w[3]);
}
template <int D>
__device__ __forceinline__ void unpack_vertices(uint4 p, int (&s)[D + 1]) {
  const uint32_t w[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
  for (int i = 0; i <= D; ++i) s[i] = (int)((w[i >> 1] >> ((i & 1) * 16)) & 0xFFFFu);
}

}  // namespace vr
