// residual_prep.cu — device-side preparation of the host residual reduction (SURVEY.md §8(a)
// "off path": the residual columns' reduction, §5.2.8-5.2.11), so that the host does only
// what is sequential by nature.
//
//   k_neighbour_ranks : the threshold graph's edge ranks packed per row, in ascending
//                       neighbour order, plus per (row, 64-bit bitmap word) the index of the
//                       word's first neighbour.  The host then reads R(u, v) for adjacent
//                       u, v as nb_rank[nb_pre[u, v/64] + popc(bits of the word below v)] —
//                       a few MB that stay in the host caches — and never copies the n x n
//                       rank matrix (64 MB at n = 4096).  Output-sensitive mode only.
//
//   k_residual_hints  : per residual column σ (sorted keys), the first equal-diameter
//                       cofacet t = the lex-greatest cofacet with diam(t) = diam(σ) (the
//                       first entry of σ's coboundary in the order of P:4757 with diam(σ);
//                       none if every cofacet is longer), and whether t is the apparent
//                       cofacet of some column f (Def 5.3.4: f = the youngest facet of t
//                       with diam(f) = diam(t), Lemma 5.3.6, and t is f's first equal-
//                       diameter cofacet).  The host's emergent-pair test (§5.2.11,
//                       P:4874-4888) is then one pivot-table lookup: σ is emergent iff t
//                       exists, is not apparent-claimed, and no earlier residual column has
//                       pivot t.  One warp per column; the same scans as the host's
//                       first_equal_cofacet_vertex (bitmap AND in sparse mode, a descending
//                       sweep of the rank rows in dense mode — the diagonal is RINF, so the
//                       simplex's own vertices never pass).
#include <cstdint>
#include <cuda_runtime.h>

#include "vr_common.cuh"
#include "vr_internal.h"

namespace vr {

constexpr int RP_THREADS = 256;

// One warp per row v.  bm: n rows of nw 32-bit words (nw a multiple of 2); the 64-bit word
// w of row v is words 2w, 2w+1.  The row's segment of nb_rank is allocated with one atomic
// (rows land in any order; nb_pre holds absolute indices).
__global__ void __launch_bounds__(RP_THREADS) k_neighbour_ranks(const uint32_t* __restrict__ rank, int n,
                                                                const uint32_t* __restrict__ bm, int nw,
                                                                const uint32_t* __restrict__ deg,
                                                                uint32_t* __restrict__ counter,
                                                                uint32_t* __restrict__ nb_pre,
                                                                uint32_t* __restrict__ nb_rank) {
  const int lane = threadIdx.x & 31;
  const int v = (int)(((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (v >= n) return;
  const int bmw = nw / 2;
  uint32_t base = 0;
  if (lane == 0) base = atomicAdd(counter, __ldg(deg + v));
  base = __shfl_sync(0xffffffffu, base, 0);
  const uint32_t* row = bm + (size_t)v * (size_t)nw;
  const uint32_t* rrow = rank + (size_t)v * (size_t)n;
  for (int w0 = 0; w0 < bmw; w0 += 32) {
    const int w = w0 + lane;
    uint64_t x = 0;
    if (w < bmw) x = (uint64_t)__ldg(row + 2 * w) | ((uint64_t)__ldg(row + 2 * w + 1) << 32);
    const uint32_t c = (uint32_t)__popcll(x);
    uint32_t incl = c;  // warp inclusive scan of the words' counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    uint32_t pos = base + incl - c;
    if (w < bmw) nb_pre[(size_t)v * (size_t)bmw + (size_t)w] = pos;
    while (x) {
      const int b = __ffsll((long long)x) - 1;
      x &= x - 1;
      nb_rank[pos++] = __ldg(rrow + 64 * w + b);
    }
    base += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// First v (descending) adjacent to every vertex of S with max_q R[S_q][v] <= r, or -1;
// every lane returns it.
template <int K>
__device__ __forceinline__ int warp_first_equal(const Tables& T, const uint32_t* __restrict__ bm, int nw,
                                                const int (&S)[K], uint32_t r) {
  const int lane = threadIdx.x & 31;
  if (bm) {
    for (int k0 = nw - 1; k0 >= 0; k0 -= 32) {
      const int k = k0 - lane;
      uint32_t m = 0;
      if (k >= 0) {
        m = ~0u;
#pragma unroll
        for (int q = 0; q < K; ++q) m &= __ldg(bm + (size_t)S[q] * (size_t)nw + k);
      }
      int hit = -1;
      while (m) {
        const int b = 31 - __clz(m);
        m ^= 1u << b;
        const int v = 32 * k + b;
        bool ok = true;
#pragma unroll
        for (int q = 0; q < K; ++q) ok = ok && rank_at(T, S[q], v) <= r;
        if (ok) { hit = v; break; }
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, hit >= 0);
      if (bal) return __shfl_sync(0xffffffffu, hit, __ffs(bal) - 1);  // lowest lane = highest word
    }
    return -1;
  }
  for (int v0 = T.n - 1; v0 >= 0; v0 -= 32) {
    const int v = v0 - lane;
    bool ok = v >= 0;
#pragma unroll
    for (int q = 0; q < K; ++q) ok = ok && rank_at(T, S[q], v) <= r;  // R[v][v] = RINF
    const uint32_t bal = __ballot_sync(0xffffffffu, ok);
    if (bal) return v0 - (__ffs(bal) - 1);
  }
  return -1;
}

template <int D>
__global__ void __launch_bounds__(RP_THREADS) k_residual_hints(Tables T, const uint32_t* __restrict__ bm, int nw,
                                                               const uint64_t* __restrict__ keys, uint64_t nkeys,
                                                               uint32_t maxr, int cbits, uint64_t* __restrict__ first,
                                                               uint8_t* __restrict__ claimed) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t cmask = cbits >= 64 ? ~0ull : ((1ull << cbits) - 1);
  for (uint64_t c = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < nkeys; c += warps) {
    const uint64_t key = __ldg(keys + c);
    const uint32_t rs = maxr - (uint32_t)(key >> cbits);
    int s[D + 1];
    cns_decode<D>(T, key & cmask, s);
    const int v = warp_first_equal<D + 1>(T, bm, nw, s, rs);
    uint64_t tc = ~0ull;
    uint8_t cl = 0;
    if (v >= 0) {
      tc = cofacet_cidx<D>(T, s, v);
      int t[D + 2];
      {
        int m = 0, q = 0;
        while (q <= D && s[q] > v) t[m++] = s[q++];
        t[m++] = v;
        while (q <= D) t[m++] = s[q++];
      }
      // youngest facet of t with diameter diam(t) = rs (drop t[0], t[1], ...)
      for (int j = 0; j < D + 2; ++j) {
        uint32_t df = 0;
        for (int a = 0; a < D + 2; ++a)
          for (int b = a + 1; b < D + 2; ++b)
            if (a != j && b != j) df = umax(df, rank_at(T, t[a], t[b]));
        if (df != rs) continue;
        int f[D + 1];
        int m = 0;
        for (int q = 0; q < D + 2; ++q)
          if (q != j) f[m++] = t[q];
        cl = warp_first_equal<D + 1>(T, bm, nw, f, rs) == t[j];
        break;  // only the youngest facet can be t's apparent partner
      }
    }
    if (lane == 0) {
      first[c] = tc;
      claimed[c] = cl;
    }
  }
}

void launch_neighbour_ranks(const uint32_t* rank, int n, const uint32_t* bm, int nw, const uint32_t* deg,
                            uint32_t* counter, uint32_t* nb_pre, uint32_t* nb_rank, cudaStream_t st, int64_t* launches) {
  if (n <= 0) return;
  cudaMemsetAsync(counter, 0, 4, st);
  const unsigned blocks = (unsigned)(((uint64_t)n * 32 + RP_THREADS - 1) / RP_THREADS);
  k_neighbour_ranks<<<blocks, RP_THREADS, 0, st>>>(rank, n, bm, nw, deg, counter, nb_pre, nb_rank);
  if (launches) *launches += 1;
}

void launch_residual_hints(const uint32_t* rank, const uint64_t* binom, int n, int kmax, int d, const uint32_t* bm,
                           int nw, const uint64_t* keys, uint64_t nkeys, uint32_t maxr, int cbits, uint64_t* first,
                           uint8_t* claimed, cudaStream_t st, int64_t* launches) {
  if (nkeys == 0) return;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms <= 0) sms = 148;
  const Tables T{rank, binom, n, kmax};
  const uint64_t want = (nkeys * 32 + RP_THREADS - 1) / RP_THREADS;
  const unsigned blocks = (unsigned)(want < (uint64_t)sms * 8 ? want : (uint64_t)sms * 8);
  switch (d) {
#define RP_CASE(DD) \
  case DD: k_residual_hints<DD><<<blocks, RP_THREADS, 0, st>>>(T, bm, nw, keys, nkeys, maxr, cbits, first, claimed); break;
    RP_CASE(1) RP_CASE(2) RP_CASE(3) RP_CASE(4) RP_CASE(5) RP_CASE(6)
#undef RP_CASE
    default: return;
  }
  if (launches) *launches += 1;
}

}  // namespace vr
