// sparse.cu — the output-sensitive ("sparse") hot path for thresholds far below the
// enclosing radius (config 5: t = 1.4, ~2.8% of the edges), SURVEY.md §8(a) a1/a5
// "output-sensitive" and §8(f) NEXT-2; §5.3.12-5.3.13 (sparse 1-skeleton, Alg 15)
// and P:5967 (Ripser++ switched o3 to its sparse mode).
//
// Threshold graph G_t as a bitmap: bit w of row v is set iff v != w and d(v, w) <= t
// (R[v][w] != RINF); nw = ceil(n/32) words per row, 512 B per row at n = 4096 (2 MiB in
// all: L2-resident, rows read coalesced).  A "row" of dimension d is a (d-1)-simplex
// σ = (u_d > ... > u_1) with diam <= t (a survivor of dimension d-1, written by that
// dimension's kernel; the vertices themselves for d = 1).  Every d-simplex with diam <= t
// is produced exactly once, as σ ∪ {w} with w = its smallest vertex:
//
//   C(σ) = N(u_1) ∩ ... ∩ N(u_d)    (AND of the d bitmap rows)
//   the d-simplices of row σ        = { σ ∪ {w} : w ∈ C(σ), w < u_1 }
//
// — the AND is exactly the threshold test of Eq 5.3 for the new edges (σ itself is under
// t), so no rank is gathered for a candidate that does not survive (reading A33: Alg 15's
// goto structure is not followed literally; this is the same set by neighbourhood
// intersection, §5.3.12-13).  The apparent test (Lemma 5.3.6 condition 1) needs the
// lex-greatest cofacet s ∪ {v} with diam = diam(s); such a v is adjacent to every vertex of
// s (reading A32), so it lies in C(σ) ∩ N(w).  The warp lists C(σ) in descending order in
// shared memory, once per row, with m(v) = max_i R[u_i][v] (the prefix part of the new
// edges' maximum); each survivor lane then walks that list — one broadcast shared load
// per step, and one rank gather R[w][v] only where m(v) <= diam(s).  Condition 2 (no
// lex-smaller facet of the cofacet with the same diameter) follows as in hotpath.cu.
//
// The scan covers all of C(σ), so a column leaves this kernel decided (apparent, cleared or
// residual) — except in the recompute mode (no clearing set: sharded runs), where the
// non-apparent ones go to k_resolve_sparse for the clearing decision by recomputation.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "vr_common.cuh"
#include "vr_internal.h"

namespace vr {

constexpr int SP_THREADS = 256;
constexpr int SP_WARPS = SP_THREADS / 32;
constexpr int SP_LCAP = 256;  // C(σ) entries listed per warp at a time (longer lists: segments)

// ------------------------------------------------------------------ threshold-graph bitmap
// one warp per vertex v: word k of row v from the 32 coalesced ranks R[v][32k .. 32k+31];
// also deg(v) and deg_below(v) = #{w < v adjacent to v} (the row bound's per-vertex term)
__global__ void k_bitmap(const uint32_t* __restrict__ rank, int n, int nw, uint32_t* __restrict__ bm,
                         uint32_t* __restrict__ deg, uint32_t* __restrict__ deg_below) {
  const int lane = threadIdx.x & 31;
  const int v = (int)(((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (v >= n) return;
  const uint32_t* row = rank + (size_t)v * (size_t)n;
  uint32_t* out = bm + (size_t)v * (size_t)nw;
  uint32_t c = 0, cb = 0, mine = 0;
  for (int k = 0; k < nw; ++k) {
    const int w = 32 * k + lane;
    const bool e = w < n && __ldg(row + w) != VR_RINF;  // R[v][v] = RINF: no self loop
    const uint32_t x = __ballot_sync(0xffffffffu, e);
    if ((k & 31) == lane) mine = x;
    if ((k & 31) == 31 || k == nw - 1) {
      const int k0 = k & ~31;
      if (k0 + lane <= k) out[k0 + lane] = mine;
    }
    c += e;
    cb += e && w < v;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  cb = __reduce_add_sync(0xffffffffu, cb);
  if (lane == 0) {
    deg[v] = c;
    deg_below[v] = cb;
  }
}

// ------------------------------------------------------------------ bitmap lists
// The set bits of AND_{i<K} bm[x_i] over the words k <= *word, in descending vertex order,
// appended to list[0..cap) (the word *word itself masked by *top_mask).  Rows are padded to
// a multiple of 4 words, so a round reads one 16-byte quad of words per lane and row
// (lane l takes quad `(*word >> 2) - l`: 128 words = 4096 vertices per round, coalesced),
// and a warp prefix sum of the popcounts places each lane's bits.  Stops before the first
// quad that does not fit (cap >= 128 keeps one quad always fitting).  Returns the entries
// written; *word = the next word to list (-1 when done), *top_mask = its mask (all ones).
// *above (if given) counts the entries >= `split` (the survivors are the entries < split).
template <int K>
__device__ __forceinline__ int bm_list(const SparseRows& S, const int (&x)[K], int& word, uint32_t& top_mask,
                                       uint16_t* __restrict__ list, int cap, int split, int* above) {
  const int lane = threadIdx.x & 31;
  int fill = 0, nab = 0;
  while (word >= 0) {
    const int q = (word >> 2) - lane;
    uint32_t wv[4] = {0, 0, 0, 0};  // words 4q .. 4q+3
    if (q >= 0) {
      wv[0] = wv[1] = wv[2] = wv[3] = 0xffffffffu;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const uint4 t = __ldg(reinterpret_cast<const uint4*>(S.bm + (size_t)x[i] * (size_t)S.nw) + q);
        wv[0] &= t.x; wv[1] &= t.y; wv[2] &= t.z; wv[3] &= t.w;
      }
      if (lane == 0) {  // the first quad: drop the words above `word`, mask `word`
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int k = 4 * q + j;
          wv[j] = k > word ? 0u : (k == word ? (wv[j] & top_mask) : wv[j]);
        }
      }
    }
    const int c = __popc(wv[0]) + __popc(wv[1]) + __popc(wv[2]) + __popc(wv[3]);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const bool fits = fill + incl <= cap;  // monotone in the lane: a prefix of the lanes fits
    const int nfit = __popc(__ballot_sync(0xffffffffu, fits));
    int ab = 0;
    if (fits && c) {
      int pos = fill + incl - c;
      VR_ASSERT(fill + incl <= cap);
#pragma unroll
      for (int j = 3; j >= 0; --j) {
        uint32_t bits = wv[j];
        const int base = 32 * (4 * q + j);
        if (above) {
          const int r = split - base;  // bits >= r are >= split
          ab += r <= 0 ? __popc(bits) : (r >= 32 ? 0 : __popc(bits >> r));
        }
        while (bits) {
          const int b = 31 - __clz(bits);
          list[pos++] = (uint16_t)(base + b);
          bits &= ~(1u << b);
        }
      }
    }
    if (above) nab += __reduce_add_sync(0xffffffffu, (unsigned)ab);
    const int added = nfit ? __shfl_sync(0xffffffffu, incl, nfit - 1) : 0;
    fill += added;
    if (nfit) {
      word = 4 * ((word >> 2) - nfit) + 3;  // the top word of the first quad left (< 0: done)
      top_mask = 0xffffffffu;
    }
    if (nfit < 32) break;
  }
  __syncwarp();
  if (above) *above = nab;
  return fill;
}

// ------------------------------------------------------------------ phase 1 (+ decision)
// per-warp counters in 32 bits (registers are the kernel's limit), flushed into the 64-bit
// device counters before any can overflow (maybe_flush after every row)
struct Acc {
  uint32_t surv = 0, app = 0, scan = 0, clr = 0, next_bound = 0;  // next_bound: per lane
  uint32_t cand = 0;  // rank reads of the candidate examination (list maxima, C(σ) compaction)
};

// Lemma 5.3.6 condition 1 over a lane's list cl[0..fill) (descending; ml = m(v), the
// prefix part of the new edges' maximum; rw = the lane's rank-matrix row R[w][.]): the first
// v with v != w and max(m(v), R[w][v]) <= rs.  Four candidates per round: their rank
// gathers (only where m(v) <= rs) are in flight together, so a lane's scan of L candidates
// costs ~L/4 dependent L2 round trips.  `examined` counts the candidates up to the hit, as a
// one-at-a-time scan would.
__device__ __forceinline__ void scan4(const uint16_t* cl, const uint32_t* ml, int fill, const uint32_t* rw, int w,
                                      uint32_t rs, bool& active, int& hitv, int& examined) {
  for (int k = 0; __any_sync(0xffffffffu, active); k += 4) {
    if (!active) continue;
    int v[4];
    uint32_t r[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[i] = -1;
      r[i] = VR_RINF;
      if (k + i < fill) {
        v[i] = cl[k + i];
        if (v[i] != w && ml[k + i] <= rs) r[i] = __ldg(rw + v[i]);
      }
    }
    int h = -1;
#pragma unroll
    for (int i = 3; i >= 0; --i)
      if (r[i] <= rs) h = i;
    if (h >= 0) {
      hitv = v[h];
      examined += h + 1;
      active = false;
    } else {
      examined += (fill - k < 4 ? fill - k : 4);
      if (k + 4 >= fill) active = false;
    }
  }
}

// Lemma 5.3.6 condition 1 over one list segment: the first v of cv[0..fill) (descending)
// with v != w and max(m(v), R[w][v]) <= rs; all lanes step together (broadcast shared
// loads), a rank is gathered only where m(v) <= rs.  Clears `active` on a hit.
__device__ __forceinline__ int scan_list(const Tables& T, const uint16_t* cv, const uint32_t* cm, int fill, int w,
                                         uint32_t rs, bool& active, int& examined) {
  int hitv = -1;
  for (int k = 0; k < fill; k += 2) {
    {
      const int v = cv[k];
      const uint32_t m = cm[k];
      examined += active;
      if (active && v != w && m <= rs && rank_at(T, w, v) <= rs) {
        hitv = v;
        active = false;
      }
    }
    if (k + 1 < fill) {
      const int v = cv[k + 1];
      const uint32_t m = cm[k + 1];
      examined += active;
      if (active && v != w && m <= rs && rank_at(T, w, v) <= rs) {
        hitv = v;
        active = false;
      }
    }
    if (!__any_sync(0xffffffffu, active)) break;
  }
  return hitv;
}

// Entry of a batch of survivors s = σ ∪ {w} (one per valid lane): the survivor count, the
// row of a later dimension (rows_out), the next dimension's bound term deg_below(w), and the
// clearing test (the dimension-(d-1) pivots, Lemma 4.2.3).  Returns `cleared`.
template <int D>
__device__ __forceinline__ bool survivor_head(const HotBuffers& B, const SparseRows& S, const int (&s)[D + 1], bool valid,
                                              int nb, uint64_t cidx, Acc& acc) {
  acc.surv += (uint32_t)nb;
  if (S.rows_out) {
    const unsigned long long slot = warp_append(valid, S.rows_out_count);
    if (valid && slot < S.rows_out_cap) S.rows_out[slot] = pack_vertices<D>(s);
  }
  if (valid) acc.next_bound += __ldg(S.deg_below + s[D]);
  bool cleared = false;
  if (valid) {
    if (B.clr) cleared = bit_test(B.clr, cidx);
    else if (B.clr_set.table) cleared = set_has(B.clr_set, cidx);
  }
  acc.clr += __popc(__ballot_sync(0xffffffffu, cleared));
  return cleared;
}

// Exit of a batch: Lemma 5.3.6 condition 2 for the lanes with a hit (no facet of
// t = s ∪ {hitv} lex-smaller than s — one without a vertex x > hitv — has diam(t) = diam(s)),
// then the outputs: apparent -> counted + its cofacet into the next dimension's clearing
// set; non-apparent -> residual list (or the recompute queue).
template <int D>
__device__ __forceinline__ void survivor_tail(const Tables& T, const DimParams& p, const HotBuffers& B, const int (&u)[D + 1],
                                              uint32_t pm_up, const uint32_t (&pm_ex)[D + 1], const int (&s)[D + 1], int w,
                                              uint32_t rs, uint64_t cidx, bool valid, bool cleared, int hitv, int examined,
                                              Acc& acc) {
  acc.scan += __reduce_add_sync(0xffffffffu, (unsigned)examined);
  bool app = false;
  if (hitv >= 0) {
    app = true;
    uint32_t a[D + 1], b[D + 1];
    uint32_t bup = 0;
#pragma unroll
    for (int i = 1; i <= D; ++i) {
      a[i] = rank_at(T, u[i], w);
      b[i] = rank_at(T, hitv, u[i]);
      bup = umax(bup, b[i]);
    }
    const uint32_t b0 = rank_at(T, hitv, w);
    if (w > hitv && umax(pm_up, bup) == rs) app = false;
#pragma unroll
    for (int j = 1; j <= D; ++j) {
      if (u[j] > hitv) {
        uint32_t m = umax(pm_ex[j], b0);
#pragma unroll
        for (int i = 1; i <= D; ++i)
          if (i != j) m = umax(m, umax(a[i], b[i]));
        if (m == rs) app = false;
      }
    }
  }
  acc.app += __popc(__ballot_sync(0xffffffffu, app));
  if (app && (B.clr_next || B.clr_next_set.table || B.app_pairs)) {
    const uint64_t tc = cofacet_cidx<D>(T, s, hitv);
    if (B.clr_next) bit_set(B.clr_next, tc);
    if (B.clr_next_set.table) set_put(B.clr_next_set, tc);
    if (B.exp_list) {  // sharded: the other ranks' sets receive it too (exchange A)
      const unsigned long long slot = atomicAdd(&B.ctr->exported, 1ull);
      if (slot < B.exp_cap) B.exp_list[slot] = tc;
    }
    if (B.app_pairs) {
      const unsigned long long slot = atomicAdd(&B.ctr->app_pairs, 1ull);
      if (slot < B.app_cap) {
        B.app_pairs[2 * slot] = cidx;
        B.app_pairs[2 * slot + 1] = tc;
      }
    }
  }
  const bool clrmode = B.clr || B.clr_set.table;  // clearing decided here (else in k_resolve_sparse)
  const bool nonapp = valid && !cleared && !app;
  const bool to_resid = clrmode && nonapp;
  const bool to_queue = !clrmode && nonapp;
  const uint64_t key = ((uint64_t)(p.maxr - rs) << p.cbits) | cidx;
  const unsigned long long rslot = warp_append(to_resid, &B.ctr->residual);
  if (to_resid && rslot < B.rcap) B.resid[rslot] = key;
  const unsigned long long qslot = warp_append(to_queue, &B.ctr->queued);
  if (to_queue && qslot < B.qcap) {
    B.qkey[qslot] = key;
    B.qvert[qslot] = pack_vertices<D>(s);
  }
}

// The survivors of a row σ = (u_D > ... > u_1) whose C(σ) list is complete in cv/cm (m(v) =
// max_i R[u_i][v]): they are its tail cv[first_w..fill) (the entries < u_1), 32 per batch.
template <int D>
__device__ __forceinline__ void row_from_list(const Tables& T, const DimParams& p, const HotBuffers& B, const SparseRows& S,
                                              const int (&u)[D + 1], uint32_t pm_up, const uint32_t (&pm_ex)[D + 1],
                                              uint64_t cbase, const uint16_t* cv, const uint32_t* cm, int fill, int first_w,
                                              Acc& acc) {
  const int lane = threadIdx.x & 31;
  for (int s0 = first_w; s0 < fill; s0 += 32) {
    const int nb = fill - s0 < 32 ? fill - s0 : 32;
    const bool valid = lane < nb;
    const int w = valid ? (int)cv[s0 + lane] : 0;
    const uint32_t rs = valid ? umax(pm_up, cm[s0 + lane]) : 0;
    int s[D + 1];  // s[0] > ... > s[D] = w
#pragma unroll
    for (int i = 0; i < D; ++i) s[i] = u[D - i];
    s[D] = w;
    const uint64_t cidx = cbase + (uint64_t)w;
    const bool cleared = survivor_head<D>(B, S, s, valid, nb, cidx, acc);
    bool active = valid && !cleared;
    int examined = 0, hitv = -1;
    scan4(cv, cm, fill, T.rank + (uint32_t)w * (uint32_t)T.n, w, rs, active, hitv, examined);
    survivor_tail<D>(T, p, B, u, pm_up, pm_ex, s, w, rs, cidx, valid, cleared, hitv, examined, acc);
  }
}

// prefix pair maxima of σ: pm_up over all pairs, pm_ex[j] over the pairs avoiding u_j
template <int D>
__device__ __forceinline__ void pair_maxima(const Tables& T, const int (&u)[D + 1], int from, uint32_t& pm_up,
                                            uint32_t (&pm_ex)[D + 1]) {
  pm_up = 0;
#pragma unroll
  for (int j = 0; j <= D; ++j) pm_ex[j] = 0;
#pragma unroll
  for (int a = 1; a <= D; ++a)
#pragma unroll
    for (int b = a + 1; b <= D; ++b) {
      if (a < from) continue;
      const uint32_t rr = rank_at(T, u[a], u[b]);
      pm_up = umax(pm_up, rr);
#pragma unroll
      for (int j = 1; j <= D; ++j)
        if (j != a && j != b) pm_ex[j] = umax(pm_ex[j], rr);
    }
}

// m(v) = max_{i >= from} R[u_i][v] for the list entries, into cm
template <int D>
__device__ __forceinline__ void list_maxima(const Tables& T, const int (&u)[D + 1], int from, const uint16_t* cv,
                                            uint32_t* cm, int fill) {
  const int lane = threadIdx.x & 31;
  for (int j = lane; j < fill; j += 32) {
    const int v = cv[j];
    uint32_t m = 0;
#pragma unroll
    for (int i = 1; i <= D; ++i)
      if (i >= from) m = umax(m, rank_at(T, u[i], v));
    cm[j] = m;
  }
  __syncwarp();
}

// One row σ = (u_D > ... > u_1), any list length: C(σ) in segments of SP_LCAP entries from
// the top (the buffer keeps the segment it holds across survivor batches), the survivors
// listed from the bitmap words below u_1 in batches.  Buffers: cv/cm (SP_LCAP), sw (128).
template <int D>
__device__ void row_general(const Tables& T, const DimParams& p, const HotBuffers& B, const SparseRows& S, const int (&u)[D + 1],
                            uint16_t* cv, uint32_t* cm, uint16_t* sw, Acc& acc) {
  const int lane = threadIdx.x & 31;
  const int u1 = u[1];
  if (u1 == 0) return;
  int x[D];
#pragma unroll
  for (int i = 0; i < D; ++i) x[i] = u[i + 1];
  uint32_t pm_up;
  uint32_t pm_ex[D + 1];
  pair_maxima<D>(T, u, 1, pm_up, pm_ex);
  uint64_t cbase = 0;
#pragma unroll
  for (int i = 1; i <= D; ++i) cbase += binom(T, u[i], i + 1);
  const int top_word = (T.n - 1) >> 5;
  const uint32_t top_word_mask = (T.n & 31) ? ((1u << (T.n & 31)) - 1) : 0xffffffffu;
  int c_word = top_word;
  uint32_t c_mask = top_word_mask;
  int nabove = 0;
  int c_fill = bm_list<D>(S, x, c_word, c_mask, cv, SP_LCAP, u1, &nabove);
  list_maxima<D>(T, u, 1, cv, cm, c_fill);
  acc.cand += (uint32_t)(c_fill * D);
  if (c_word < 0) {  // the whole list fits: the survivors are its tail
    row_from_list<D>(T, p, B, S, u, pm_up, pm_ex, cbase, cv, cm, c_fill, nabove, acc);
    return;
  }
  int c_seg = 0;  // the segment held in cv/cm; c_word / c_mask continue after it
  int s_word = (u1 - 1) >> 5;
  uint32_t s_mask = (u1 & 31) ? ((1u << (u1 & 31)) - 1) : 0xffffffffu;
  int s_fill = 0, s_pos = 0;
  while (true) {
    if (s_pos == s_fill) {
      if (s_word < 0) break;
      s_fill = bm_list<D>(S, x, s_word, s_mask, sw, 128, 0, nullptr);
      s_pos = 0;
      if (s_fill == 0) break;
    }
    const int nb = s_fill - s_pos < 32 ? s_fill - s_pos : 32;
    const bool valid = lane < nb;
    int w = 0;
    uint32_t rs = 0;
    if (valid) {
      w = sw[s_pos + lane];
      uint32_t m = 0;
#pragma unroll
      for (int i = 1; i <= D; ++i) m = umax(m, rank_at(T, u[i], w));
      rs = umax(pm_up, m);
    }
    s_pos += nb;
    int s[D + 1];
#pragma unroll
    for (int i = 0; i < D; ++i) s[i] = u[D - i];
    s[D] = w;
    const uint64_t cidx = cbase + (uint64_t)w;
    const bool cleared = survivor_head<D>(B, S, s, valid, nb, cidx, acc);
    bool active = valid && !cleared;
    int hitv = -1, examined = 0;
    int seg = 0;
    while (__any_sync(0xffffffffu, active)) {
      if (c_seg != seg) {  // (re)build segment `seg`
        if (seg == 0) {
          c_word = top_word;
          c_mask = top_word_mask;
        }
        c_fill = bm_list<D>(S, x, c_word, c_mask, cv, SP_LCAP, 0, nullptr);
        list_maxima<D>(T, u, 1, cv, cm, c_fill);
        acc.cand += (uint32_t)(c_fill * D);
        c_seg = seg;
      }
      const int h = scan_list(T, cv, cm, c_fill, w, rs, active, examined);
      if (h >= 0) hitv = h;
      if (c_word < 0) break;  // this was the last segment
      ++seg;
    }
    survivor_tail<D>(T, p, B, u, pm_up, pm_ex, s, w, rs, cidx, valid, cleared, hitv, examined, acc);
  }
}

// rows handed out by a shared counter, `grab` per atomic; the shard's rows are every
// shard_world-th row
__device__ __forceinline__ bool next_rows(const DimParams& p, const HotBuffers& B, uint64_t nrows, uint64_t& g0,
                                          uint64_t& gend) {
  const int lane = threadIdx.x & 31;
  unsigned long long g = 0;
  if (lane == 0) g = atomicAdd(&B.ctr->row_next, (unsigned long long)p.grab);
  g = __shfl_sync(0xffffffffu, g, 0);
  if (g >= nrows) return false;
  g0 = g;
  gend = g + (uint64_t)p.grab < nrows ? g + (uint64_t)p.grab : nrows;
  return true;
}

template <int K>
__device__ __forceinline__ void unpack_row(const uint4* rows, uint64_t r, int (&t)[K]) {
  const uint4 pk = rows[r];
  const uint32_t w4[4] = {pk.x, pk.y, pk.z, pk.w};
#pragma unroll
  for (int i = 0; i < K; ++i) t[i] = (int)((w4[i >> 1] >> ((i & 1) * 16)) & 0xFFFFu);
}

__device__ __forceinline__ void flush_acc(const HotBuffers& B, Acc& acc) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    if (acc.surv) atomicAdd(&B.ctr->survivors, (unsigned long long)acc.surv);
    if (acc.app) atomicAdd(&B.ctr->apparent1, (unsigned long long)acc.app);
    if (acc.scan) atomicAdd(&B.ctr->scanned, (unsigned long long)acc.scan);
    if (acc.clr) atomicAdd(&B.ctr->cleared, (unsigned long long)acc.clr);
    if (acc.cand) atomicAdd(&B.ctr->cand_reads, (unsigned long long)acc.cand);
  }
  unsigned long long nbsum = acc.next_bound;  // per lane
#pragma unroll
  for (int o = 16; o; o >>= 1) nbsum += __shfl_xor_sync(0xffffffffu, nbsum, o);
  if (lane == 0 && nbsum) atomicAdd(&B.ctr->next_bound, nbsum);
  acc = Acc{};
}
// flushes when a counter passes 2^30 (a row adds far less)
__device__ __forceinline__ void maybe_flush(const HotBuffers& B, Acc& acc) {
  const uint32_t big = acc.surv | acc.app | acc.scan | acc.clr | acc.cand;
  if (__any_sync(0xffffffffu, (big | acc.next_bound) >= (1u << 30))) flush_acc(B, acc);
}

// Single level: a row is a (D-1)-simplex σ (a survivor of dimension D-1; the vertices for
// D = 1), extended by w ∈ C(σ), w < u_1.
template <int D>
__global__ void __launch_bounds__(SP_THREADS, 4) k_enum_sparse(Tables T, DimParams p, HotBuffers B, SparseRows S) {
  __shared__ uint16_t s_cv[SP_WARPS][SP_LCAP];
  __shared__ uint32_t s_cm[SP_WARPS][SP_LCAP];
  __shared__ uint16_t s_w[SP_WARPS][128];
  const int wi = threadIdx.x >> 5;
  Acc acc;
  const uint64_t W = (uint64_t)p.shard_world;
  const uint64_t all = p.row_end - p.row_begin;
  const uint64_t nrows = all > (uint64_t)p.shard_rank ? (all - (uint64_t)p.shard_rank + W - 1) / W : 0;
  uint64_t g0, gend;
  while (next_rows(p, B, nrows, g0, gend)) {
    for (uint64_t g = g0; g < gend; ++g) {
      // vertex rows from the top down: a vertex's rows grow with its index (its neighbours
      // below it), so the largest go first (no long tail at the end of the launch)
      const uint64_t gg = S.rows_in == nullptr ? nrows - 1 - g : g;
      const uint64_t r = p.row_begin + gg * W + (uint64_t)p.shard_rank;
      int u[D + 1];  // u[1] < ... < u[D] (u[0] unused)
      u[0] = 0;
      if (S.rows_in == nullptr) {
        u[1] = (int)r;
      } else {
        int t[D];
        unpack_row<D>(S.rows_in, r, t);
#pragma unroll
        for (int i = 1; i <= D; ++i) u[i] = t[D - i];
      }
      row_general<D>(T, p, B, S, u, s_cv[wi], s_cm[wi], s_w[wi], acc);
      maybe_flush(B, acc);
    }
  }
  flush_acc(B, acc);
}

// Two levels (D >= 2): a row is a (D-2)-simplex τ = (u_D > ... > u_2) (a survivor of
// dimension D-2; the vertices for D = 2).  C(τ) is listed once, with m_τ(v) = max_{i>=2}
// R[u_i][v]; each x ∈ C(τ), x < u_2 — a (D-1)-simplex σ = τ ∪ {x} — then gets its own
// C(σ) = { v ∈ C(τ) : R[x][v] != RINF } with m_σ(v) = max(m_τ(v), R[x][v]): ONE rank gather
// per list entry instead of the AND of D bitmap rows and D gathers.  The σ lists are packed
// side by side in shared memory so that one batch of 32 lanes takes the survivors of
// several σ (≈ 10 each at config 5, dimension 3): the survivor tests, scans and outputs run
// with full warps.  τ lists longer than SP_LCAP fall back to row_general per σ.
constexpr int SP_PCAP = 512;  // packed C(σ) entries per warp
constexpr int SP_MAXG = 16;   // σ per group

// one warp's shared memory: every array addressed from one base register
template <int D>
struct alignas(16) Sp2Smem {
  uint32_t tm[SP_LCAP];          // m_τ
  uint32_t cm[SP_PCAP];          // m_σ, packed
  uint32_t gpm[SP_MAXG][D + 1];  // per σ of the group: [0] pm_up, [j] pm_ex[j]
  uint16_t tv[SP_LCAP];          // C(τ)
  uint16_t cv[SP_PCAP];          // C(σ) lists, packed
  uint16_t sw[128];              // (fallback path)
  int16_t gx[SP_MAXG], goff[SP_MAXG], gfill[SP_MAXG], gfw[SP_MAXG], gslot[SP_MAXG + 1];
};

template <int D, int MINB>
__global__ void __launch_bounds__(SP_THREADS, MINB) k_enum_sparse2(Tables T, DimParams p, HotBuffers B, SparseRows S) {
  __shared__ Sp2Smem<D> smem[SP_WARPS];
  const int lane = threadIdx.x & 31;
  Sp2Smem<D>& M = smem[threadIdx.x >> 5];
  uint16_t* tv = M.tv;
  uint32_t* tm = M.tm;
  uint16_t* cv = M.cv;
  uint32_t* cm = M.cm;
  Acc acc;
  const uint64_t W = (uint64_t)p.shard_world;
  const uint64_t all = p.row_end - p.row_begin;
  const uint64_t nrows = all > (uint64_t)p.shard_rank ? (all - (uint64_t)p.shard_rank + W - 1) / W : 0;
  const int top_word = (T.n - 1) >> 5;
  const uint32_t top_word_mask = (T.n & 31) ? ((1u << (T.n & 31)) - 1) : 0xffffffffu;
  // work item g = (row g / slices, slice g % slices): slice k takes every slices-th x
  // (few rows with long lists, e.g. D = 2 with vertex rows, are split over warps)
  const uint32_t NS = (uint32_t)p.slices;  // (rows x slices < 2^32: checked by the launcher / caller)
  uint64_t g0, gend;
  while (next_rows(p, B, nrows * NS, g0, gend)) {
    for (uint32_t gi = (uint32_t)g0; gi < (uint32_t)gend; ++gi) {
      const uint32_t g = gi / NS;
      const int slice = (int)(gi - g * NS);
      const uint64_t gg = S.rows_in == nullptr ? nrows - 1 - (uint64_t)g : (uint64_t)g;  // (largest vertex rows first)
      const uint64_t r = p.row_begin + gg * W + (uint64_t)p.shard_rank;
      int u[D + 1];
      u[0] = u[1] = 0;
      if (S.rows_in == nullptr) {  // D = 2: τ is a vertex
        u[2] = (int)r;
      } else {
        int t[D - 1];
        unpack_row<D - 1>(S.rows_in, r, t);
#pragma unroll
        for (int i = 2; i <= D; ++i) u[i] = t[D - i];
      }
      const int u2 = u[2];
      if (u2 < 2) continue;  // no x < u_2 with a w < x
      int xt[D - 1];
#pragma unroll
      for (int i = 0; i < D - 1; ++i) xt[i] = u[i + 2];
      int word = top_word;
      uint32_t mask = top_word_mask;
      int nab = 0;
      const int tfill = bm_list<D - 1>(S, xt, word, mask, tv, SP_LCAP, u2, &nab);
      if (word >= 0) {  // C(τ) longer than the list: every σ on the general path
        int s_word = (u2 - 1) >> 5;
        uint32_t s_mask = (u2 & 31) ? ((1u << (u2 & 31)) - 1) : 0xffffffffu;
        int base = 0;  // list index of tv[0] among the x's
        while (s_word >= 0) {
          const int nx = bm_list<D - 1>(S, xt, s_word, s_mask, tv, SP_LCAP, 0, nullptr);
          for (int ix = 0; ix < nx; ++ix) {
            if ((base + ix) % (int)p.slices != slice) continue;
            u[1] = tv[ix];
            row_general<D>(T, p, B, S, u, cv, cm, M.sw, acc);
            maybe_flush(B, acc);
          }
          base += nx;
          __syncwarp();
        }
        continue;
      }
      list_maxima<D>(T, u, 2, tv, tm, tfill);
      acc.cand += (uint32_t)(tfill * (D - 1));
      // τ's pair maxima and cidx part
      uint32_t pt_up;
      uint32_t pt_ex[D + 1];
      pair_maxima<D>(T, u, 2, pt_up, pt_ex);
      uint32_t pt_ex_l = 0;  // lane j (2..D): pt_ex[j]
#pragma unroll
      for (int j = 2; j <= D; ++j)
        if (lane == j) pt_ex_l = pt_ex[j];
      uint64_t cb_t = 0;
#pragma unroll
      for (int i = 2; i <= D; ++i) cb_t += binom(T, u[i], i + 1);
      int ix = nab + slice;  // the next σ (x = tv[ix], descending)
      // a σ listed but left out of the previous group (its survivors did not fit) waits in
      // the group tables at index `carry` with its list at g_off[carry]; it moves to the
      // front of the next group
      int carry = -1;
      while (true) {
        // ---- a group: σ lists packed in cv/cm, their survivors slot after slot
        int ng = 0, poff = 0, slots = 0;
        if (carry >= 0) {
          const int c_off = M.goff[carry], c_fill = M.gfill[carry];
          for (int j0 = 0; j0 < c_fill; j0 += 32) {  // move down (sources above destinations)
            const int j = j0 + lane;
            uint16_t v = 0;
            uint32_t m = 0;
            if (j < c_fill) { v = cv[c_off + j]; m = cm[c_off + j]; }
            __syncwarp();
            if (j < c_fill) { cv[j] = v; cm[j] = m; }
            __syncwarp();
          }
          if (lane == 0) {
            M.gx[0] = M.gx[carry];
            M.goff[0] = 0;
            M.gfill[0] = (int16_t)c_fill;
            M.gfw[0] = M.gfw[carry];
            M.gslot[0] = 0;
          }
          if (lane <= D) M.gpm[0][lane] = M.gpm[carry][lane];
          __syncwarp();
          ng = 1;
          poff = c_fill;
          slots = c_fill - M.gfw[0];
          carry = -1;
        }
        while (ix < tfill && ng < SP_MAXG && poff + tfill <= SP_PCAP && slots < 32) {
          const int x = tv[ix];
          const int xi = ix;  // x's position in C(τ)
          ix += (int)p.slices;
          if (x == 0) continue;
          // C(σ): the entries of C(τ) adjacent to x, order kept (ballot compaction); the
          // rank gathers of two 32-entry rounds are issued together
          const uint32_t* rx_row = T.rank + (uint32_t)x * (uint32_t)T.n;
          uint32_t axl = 0;  // σ's new edges (x, u_i), lane i-2 holds one
          if (lane < D - 1) axl = __ldg(rx_row + u[2 + lane]);
          int fill = 0, first_w = 0;
          for (int j0 = 0; j0 < tfill; j0 += 64) {
            const int ja = j0 + lane, jb = j0 + 32 + lane;
            int va = 0, vb = 0;
            uint32_t ra = VR_RINF, rb = VR_RINF;
            if (ja < tfill) va = tv[ja];
            if (jb < tfill) vb = tv[jb];
            if (ja < tfill) ra = __ldg(rx_row + va);  // RINF: not adjacent (or v = x)
            if (jb < tfill) rb = __ldg(rx_row + vb);
            const bool ka = ra != VR_RINF, kb = rb != VR_RINF;
            const uint32_t kma = __ballot_sync(0xffffffffu, ka);
            const uint32_t kmb = __ballot_sync(0xffffffffu, kb);
            const int na = __popc(kma);
            VR_ASSERT(poff + fill + na + __popc(kmb) <= SP_PCAP);
            if (ka) {
              const int pos = poff + fill + __popc(kma & lanemask_lt());
              cv[pos] = (uint16_t)va;
              cm[pos] = umax(tm[ja], ra);
            }
            if (kb) {
              const int pos = poff + fill + na + __popc(kmb & lanemask_lt());
              cv[pos] = (uint16_t)vb;
              cm[pos] = umax(tm[jb], rb);
            }
            // the kept entries above x are those before x's own position ix (tv descends)
            const int ra_n = xi - j0, rb_n = xi - j0 - 32;  // entries of this round before x
            first_w += __popc(kma & (ra_n >= 32 ? 0xffffffffu : (ra_n <= 0 ? 0u : ((1u << ra_n) - 1)))) +
                       __popc(kmb & (rb_n >= 32 ? 0xffffffffu : (rb_n <= 0 ? 0u : ((1u << rb_n) - 1))));
            fill += na + __popc(kmb);
          }
          acc.cand += (uint32_t)tfill;  // one rank read R[x][v] per entry of C(τ)
          const int ns = fill - first_w;
          if (ns <= 0) continue;  // no d-simplex in this σ's row
          // σ's pair maxima from τ's and the D-1 new edges: [0] pm_up, [1] avoiding x (τ's),
          // [j] avoiding u_j
          if (lane <= D) {
            uint32_t mine = lane == 1 ? pt_up : (lane == 0 ? pt_up : pt_ex_l);
#pragma unroll
            for (int i = 2; i <= D; ++i) {
              const uint32_t ai = __shfl_sync(0x0000ffffu & ((1u << (D + 1)) - 1), axl, i - 2);
              if (lane == 0 || (lane >= 2 && lane != i)) mine = umax(mine, ai);
            }
            M.gpm[ng][lane] = mine;
          }
          VR_ASSERT(ng < SP_MAXG);
          if (lane == 0) {
            M.gx[ng] = (int16_t)x;
            M.goff[ng] = (int16_t)poff;
            M.gfill[ng] = (int16_t)fill;
            M.gfw[ng] = (int16_t)first_w;
            M.gslot[ng] = (int16_t)slots;
          }
          __syncwarp();
          if (slots > 0 && slots + ns > 32) {  // does not fit: first of the next group
            carry = ng;
            break;
          }
          ++ng;
          poff += fill;
          slots += ns;
        }
        if (ng == 0) break;
        if (lane == 0) M.gslot[ng] = (int16_t)slots;
        __syncwarp();
        // ---- the group's survivors, 32 slots per batch (several batches only for one σ
        // with more than 32 survivors)
        for (int b0 = 0; b0 < slots; b0 += 32) {
          const int t = b0 + lane;
          const bool valid = t < slots;
          int q = 0;
          while (q + 1 < ng && M.gslot[q + 1] <= t) ++q;
          const int off = M.goff[q], qfill = M.gfill[q];
          const int li = M.gfw[q] + (t - M.gslot[q]);
          VR_ASSERT(!valid || (li < qfill && off + qfill <= SP_PCAP));
          u[1] = M.gx[q];
          uint32_t pm_ex[D + 1];
          pm_ex[0] = 0;
#pragma unroll
          for (int j = 1; j <= D; ++j) pm_ex[j] = M.gpm[q][j];
          const uint32_t pm_up = M.gpm[q][0];
          int w = 0;
          uint32_t rs = 0;
          if (valid) {
            w = cv[off + li];
            rs = umax(pm_up, cm[off + li]);
          }
          int s[D + 1];
#pragma unroll
          for (int i = 0; i < D; ++i) s[i] = u[D - i];
          s[D] = w;
          const uint64_t cidx = cb_t + binom(T, u[1], 2) + (uint64_t)w;
          const int nb = slots - b0 < 32 ? slots - b0 : 32;
          const bool cleared = survivor_head<D>(B, S, s, valid, nb, cidx, acc);
          bool active = valid && !cleared;
          int examined = 0, hitv = -1;
          // Lemma 5.3.6 condition 1 over the lane's own C(σ) (descending)
          const uint16_t* cl = cv + off;
          const uint32_t* ml = cm + off;
          const uint32_t* rw = T.rank + (uint32_t)w * (uint32_t)T.n;
          scan4(cl, ml, qfill, rw, w, rs, active, hitv, examined);
          survivor_tail<D>(T, p, B, u, pm_up, pm_ex, s, w, rs, cidx, valid, cleared, hitv, examined, acc);
        }
        __syncwarp();
      }
      __syncwarp();
      maybe_flush(B, acc);
    }
  }
  flush_acc(B, acc);
}

// ------------------------------------------------------------------ phase 2 (recompute mode)
// First v (descending) in AND_{w in S} N(w) with max_{w in S} R[w][v] <= r, or -1: 32 words
// per step (one per lane), each lane tests its word's bits from the top, the lowest lane
// with a hit holds the lex-greatest one.
template <int K>
__device__ __forceinline__ int coop_scan_bm(const Tables& T, const SparseRows& SR, const int (&S)[K], uint32_t r,
                                            unsigned long long& scan_acc) {
  const int lane = threadIdx.x & 31;
  for (int word = SR.nw - 1; word >= 0; word -= 32) {
    const int k = word - lane;
    uint32_t bits = 0;
    if (k >= 0) {
      bits = 0xffffffffu;
#pragma unroll
      for (int i = 0; i < K; ++i) bits &= __ldg(SR.bm + (size_t)S[i] * (size_t)SR.nw + (size_t)k);
    }
    int hit = -1;
    unsigned examined = 0;
    while (bits) {
      const int b = 31 - __clz(bits);
      const int v = 32 * k + b;
      ++examined;
      uint32_t rt = 0;
#pragma unroll
      for (int i = 0; i < K; ++i) rt = umax(rt, rank_at(T, S[i], v));
      if (rt <= r) { hit = v; break; }
      bits &= ~(1u << b);
    }
    scan_acc += (unsigned long long)__reduce_add_sync(0xffffffffu, examined);
    const uint32_t m = __ballot_sync(0xffffffffu, hit >= 0);
    if (m) return __shfl_sync(0xffffffffu, hit, __ffs(m) - 1);
  }
  return -1;
}

// One warp per queued (non-apparent) column: clearing by recomputation — a binary search in
// the residual deaths of dimension d-1, or "s is the apparent cofacet of its youngest facet"
// (reading R1).  The apparent test was completed by k_enum_sparse.
template <int D>
__global__ void __launch_bounds__(SP_THREADS) k_resolve_sparse(Tables T, DimParams p, HotBuffers B, SparseRows SR, uint64_t qn) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t cmask = p.cbits >= 64 ? ~0ull : ((1ull << p.cbits) - 1);
  unsigned long long clr_acc = 0, scan_acc = 0;
  for (uint64_t e = warp; e < qn; e += nwarps) {
    const uint64_t key = __ldg(B.qkey + e);
    const uint32_t rs = p.maxr - (uint32_t)(key >> p.cbits);
    const uint64_t cidx = key & cmask;
    int s[D + 1];
    unpack_vertices<D>(B.qvert[e], s);
    bool cleared = sorted_contains(B.deaths, B.ndeaths, cidx);
    if (D >= 2 && !cleared) {
      uint32_t ex[D + 1];
#pragma unroll
      for (int j = 0; j <= D; ++j) ex[j] = 0;
#pragma unroll
      for (int a = 0; a <= D; ++a)
#pragma unroll
        for (int b = a + 1; b <= D; ++b) {
          const uint32_t r = rank_at(T, s[a], s[b]);
#pragma unroll
          for (int j = 0; j <= D; ++j)
            if (j != a && j != b) ex[j] = umax(ex[j], r);
        }
      // the youngest facet: the first (lex-ascending: drop the largest vertex first) with
      // the column's diameter
      int js = -1;
#pragma unroll
      for (int j = 0; j <= D; ++j)
        if (js < 0 && ex[j] == rs) js = j;
      if (js >= 0) {
        int f[D];
        int w = 0;
#pragma unroll
        for (int j = 0; j <= D; ++j) {
          const int x = s[j];
          if (j == js) w = x;
          else f[j < js ? j : j - 1] = x;
        }
        cleared = coop_scan_bm<D>(T, SR, f, rs, scan_acc) == w;
      }
    }
    if (cleared) {
      ++clr_acc;
      continue;
    }
    if (lane == 0) {
      const unsigned long long slot = atomicAdd(&B.ctr->residual, 1ull);
      if (slot < B.rcap) B.resid[slot] = key;
    }
  }
  if (lane == 0) {
    if (clr_acc) atomicAdd(&B.ctr->cleared, clr_acc);
    if (scan_acc) atomicAdd(&B.ctr->scanned2, scan_acc);
  }
}

__global__ void k_set_put(const uint64_t* __restrict__ list, int64_t m, ClearSet c) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = __ldg(list + i);
    if (k != ~0ull) set_put(c, k);  // ~0: the padding of a gathered list
  }
}

// ------------------------------------------------------------------ launchers
static int sp_sms() {
  int dev = 0, s = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
  return s > 0 ? s : 148;
}

// ------------------------------------------------------------------ row order (two-level, d >= 3)
// The work of a row τ grows with its smallest vertex u_2 (the σ = τ ∪ {x} take x < u_2), so
// the rows are handed out by u_2 descending — largest first, no long tail at the end of the
// launch (the vertex rows of d = 2 are taken top-down for the same reason).  Keys
// ((0xFFFF - u_2) << 32 | row) radix-sorted on bits 32..47, then the rows gathered.
template <int K>
__global__ void k_row_keys(const uint4* __restrict__ rows, uint64_t n, uint64_t* __restrict__ keys) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    int t[K];
    unpack_row<K>(rows, i, t);
    keys[i] = ((uint64_t)(0xFFFFu - (uint32_t)t[K - 1]) << 32) | i;
  }
}
__global__ void k_row_gather(const uint4* __restrict__ rows, const uint64_t* __restrict__ keys, uint64_t n,
                             uint4* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = rows[keys[i] & 0xFFFFFFFFull];
}
size_t order_rows_temp_bytes(uint64_t n) { return radix_sort_temp_bytes((size_t)n); }
void launch_order_rows(int k, const uint4* rows, uint64_t n, uint64_t* keys, uint64_t* alt, void* temp, uint4* out,
                       cudaStream_t st, int64_t* launches) {
  if (n == 0) return;
  const unsigned bl = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)sp_sms() * 8);
  switch (k) {
    case 2: k_row_keys<2><<<bl, 256, 0, st>>>(rows, n, keys); break;
    case 3: k_row_keys<3><<<bl, 256, 0, st>>>(rows, n, keys); break;
    case 4: k_row_keys<4><<<bl, 256, 0, st>>>(rows, n, keys); break;
    case 5: k_row_keys<5><<<bl, 256, 0, st>>>(rows, n, keys); break;
    default: k_row_keys<6><<<bl, 256, 0, st>>>(rows, n, keys); break;
  }
  const uint64_t* sorted = radix_sort_u64(keys, alt, (size_t)n, 32, 48, temp, st, launches);
  k_row_gather<<<bl, 256, 0, st>>>(rows, sorted, n, out);
  if (launches) *launches += 2;
}


void launch_threshold_bitmap(const uint32_t* rank, int n, int nw, uint32_t* bm, uint32_t* deg, uint32_t* deg_below,
                             cudaStream_t st, int64_t* launches) {
  const unsigned blocks = (unsigned)(((uint64_t)n * 32 + SP_THREADS - 1) / SP_THREADS);
  k_bitmap<<<blocks, SP_THREADS, 0, st>>>(rank, n, nw, bm, deg, deg_below);
  *launches += 1;
}

template <int D>
static void enum_sparse_d(const DimParams& p, const Tables& T, const HotBuffers& B, const SparseRows& S, bool two,
                          cudaStream_t st) {
  const uint64_t rows = p.row_end - p.row_begin;
  const uint64_t cap = (uint64_t)sp_sms() * 4;  // 4 CTAs of 8 warps per SM
  uint64_t blocks = (rows * 32 + SP_THREADS - 1) / SP_THREADS;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  DimParams q = p;
  // rows per atomic grab: 4 when every warp gets dozens of rows (one shared counter), else 1
  q.grab = rows >= cap * SP_WARPS * 64 ? 4 : 1;
  if constexpr (D >= 2) {
    if (two) {
      // slices per row so that there are >= 8 work items per resident warp
      const uint64_t slots = cap * SP_WARPS;
      uint64_t sl = rows ? (8 * slots + rows - 1) / rows : 1;
      q.slices = (int)(sl < 1 ? 1 : (sl > 16 ? 16 : sl));
      blocks = (rows * (uint64_t)q.slices * 32 + SP_THREADS - 1) / SP_THREADS;
      if (blocks > cap) blocks = cap;
      if (blocks < 1) blocks = 1;
      q.grab = rows * (uint64_t)q.slices >= cap * SP_WARPS * 64 ? 4 : 1;
      if (rows * (uint64_t)q.slices >= (1ull << 32)) q.slices = 1;  // (32-bit work-item indices; rows < 2^32
                                                                     // is checked by the caller)
      // (tuning: VR_SP_MINB = resident CTAs per SM the registers are budgeted for)
      static const int minb = std::getenv("VR_SP_MINB") ? std::atoi(std::getenv("VR_SP_MINB")) : 4;
      const unsigned bl = (unsigned)std::min<uint64_t>(blocks * (uint64_t)std::max(minb, 4) / 4, (uint64_t)sp_sms() * minb);
      if (minb == 3) k_enum_sparse2<D, 3><<<bl, SP_THREADS, 0, st>>>(T, q, B, S);
      else if (minb == 5) k_enum_sparse2<D, 5><<<bl, SP_THREADS, 0, st>>>(T, q, B, S);
      else if (minb == 6) k_enum_sparse2<D, 6><<<bl, SP_THREADS, 0, st>>>(T, q, B, S);
      else k_enum_sparse2<D, 4><<<(unsigned)blocks, SP_THREADS, 0, st>>>(T, q, B, S);
      return;
    }
  }
  k_enum_sparse<D><<<(unsigned)blocks, SP_THREADS, 0, st>>>(T, q, B, S);
}

template <int D>
static void resolve_sparse_d(const DimParams& p, const Tables& T, const HotBuffers& B, const SparseRows& S, uint64_t qn,
                             cudaStream_t st) {
  uint64_t blocks = (qn * 32 + SP_THREADS - 1) / SP_THREADS;
  const uint64_t cap = (uint64_t)sp_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  k_resolve_sparse<D><<<(unsigned)blocks, SP_THREADS, 0, st>>>(T, p, B, S, qn);
}

void launch_enumerate_sparse(const DimParams& p, const uint32_t* rank, const uint64_t* binom, int kmax, const HotBuffers& B,
                             const SparseRows& S, bool two_level, cudaStream_t st, int64_t* launches) {
  Tables T{rank, binom, (int32_t)p.n, kmax};
  switch (p.d) {
    case 1: enum_sparse_d<1>(p, T, B, S, false, st); break;
    case 2: enum_sparse_d<2>(p, T, B, S, two_level, st); break;
    case 3: enum_sparse_d<3>(p, T, B, S, two_level, st); break;
    case 4: enum_sparse_d<4>(p, T, B, S, two_level, st); break;
    case 5: enum_sparse_d<5>(p, T, B, S, two_level, st); break;
    case 6: enum_sparse_d<6>(p, T, B, S, two_level, st); break;
    default: return;
  }
  *launches += 1;
}

void launch_resolve_sparse(const DimParams& p, const uint32_t* rank, const uint64_t* binom, int kmax, const HotBuffers& B,
                           const SparseRows& S, uint64_t qn, cudaStream_t st, int64_t* launches) {
  if (qn == 0) return;
  Tables T{rank, binom, (int32_t)p.n, kmax};
  switch (p.d) {
    case 1: resolve_sparse_d<1>(p, T, B, S, qn, st); break;
    case 2: resolve_sparse_d<2>(p, T, B, S, qn, st); break;
    case 3: resolve_sparse_d<3>(p, T, B, S, qn, st); break;
    case 4: resolve_sparse_d<4>(p, T, B, S, qn, st); break;
    case 5: resolve_sparse_d<5>(p, T, B, S, qn, st); break;
    case 6: resolve_sparse_d<6>(p, T, B, S, qn, st); break;
    default: return;
  }
  *launches += 1;
}

void launch_set_put(const uint64_t* list, int64_t m, const ClearSet& c, cudaStream_t st, int64_t* launches) {
  if (m <= 0 || !c.table) return;
  const int64_t blocks = std::min<int64_t>((m + 255) / 256, (int64_t)sp_sms() * 8);
  k_set_put<<<(unsigned)blocks, 256, 0, st>>>(list, m, c);
  if (launches) *launches += 1;
}

}  // namespace vr
