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
#include <cuda_runtime.h>

#include "vr_common.cuh"
#include "vr_internal.h"

namespace vr {

constexpr int SP_THREADS = 256;
constexpr int SP_WARPS = SP_THREADS / 32;
constexpr int SP_LCAP = 128;  // C(σ) entries listed per warp at a time (longer lists: segments)

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

// sum over rows of deg_below(u_1): a bound on the d-simplices the rows can produce
__global__ void k_row_bound(const uint4* __restrict__ rows, uint64_t nrows, int dprev, const uint32_t* __restrict__ deg_below,
                            unsigned long long* __restrict__ out) {
  unsigned long long acc = 0;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 p = rows[r];
    const uint32_t w[4] = {p.x, p.y, p.z, p.w};
    const int u1 = (int)((w[dprev >> 1] >> ((dprev & 1) * 16)) & 0xFFFFu);  // smallest vertex s[dprev]
    acc += deg_below[u1];
  }
  acc = __reduce_add_sync(0xffffffffu, (unsigned)acc);  // per-warp partial fits 32 bits
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// ------------------------------------------------------------------ bitmap lists
// The set bits of AND_{i<K} bm[x_i] (words k <= word, descending vertex order, the top word
// masked by top_mask) appended to list[0..cap): 32 words per round, one per lane (lane l
// takes word `word - l`), a warp prefix sum of the popcounts places each lane's bits.  Stops
// before the first word that does not fit.  Returns the entries written; *word = the next
// word to list (-1 when done), *top_mask = the mask for that word (all ones).
template <int K>
__device__ __forceinline__ int bm_list(const SparseRows& S, const int (&x)[K], int& word, uint32_t& top_mask,
                                       uint16_t* __restrict__ list, int cap) {
  const int lane = threadIdx.x & 31;
  int fill = 0;
  while (word >= 0) {
    const int k = word - lane;
    uint32_t bits = 0;
    if (k >= 0) {
      bits = lane == 0 ? top_mask : 0xffffffffu;
#pragma unroll
      for (int i = 0; i < K; ++i) bits &= __ldg(S.bm + (size_t)x[i] * (size_t)S.nw + (size_t)k);
    }
    const int c = __popc(bits);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const bool fits = fill + incl <= cap;  // monotone in the lane: a prefix of the lanes fits
    const uint32_t fm = __ballot_sync(0xffffffffu, fits);
    const int nfit = __popc(fm);
    if (fits) {
      int pos = fill + incl - c;
      while (bits) {
        const int b = 31 - __clz(bits);
        list[pos++] = (uint16_t)(32 * k + b);
        bits &= ~(1u << b);
      }
    }
    const int added = nfit ? __shfl_sync(0xffffffffu, incl, nfit - 1) : 0;
    fill += added;
    word -= nfit;
    top_mask = nfit ? 0xffffffffu : top_mask;
    if (nfit < 32) break;
  }
  __syncwarp();
  return fill;
}

// ------------------------------------------------------------------ phase 1 (+ decision)
template <int D>
__global__ void __launch_bounds__(SP_THREADS, 4) k_enum_sparse(Tables T, DimParams p, HotBuffers B, SparseRows S) {
  __shared__ uint16_t s_cv[SP_WARPS][SP_LCAP];  // C(σ), descending (one segment)
  __shared__ uint32_t s_cm[SP_WARPS][SP_LCAP];  // m(v) = max_i R[u_i][v]
  __shared__ uint16_t s_w[SP_WARPS][32];        // a batch of survivors w < u_1
  const int lane = threadIdx.x & 31;
  const int wi = threadIdx.x >> 5;
  uint16_t* cv = s_cv[wi];
  uint32_t* cm = s_cm[wi];
  uint16_t* sw = s_w[wi];
  unsigned long long surv_acc = 0, app_acc = 0, scan_acc = 0, clr_acc = 0;
  const bool clrmode = B.clr || B.clr_hash;  // clearing decided here (else in k_resolve_sparse)
  const uint64_t W = (uint64_t)p.shard_world;
  const uint64_t all = p.row_end - p.row_begin;
  const uint64_t nrows = all > (uint64_t)p.shard_rank ? (all - (uint64_t)p.shard_rank + W - 1) / W : 0;  // this shard's rows
  while (true) {
    unsigned long long g = 0;
    if (lane == 0) g = atomicAdd(&B.ctr->row_next, 1ull);
    g = __shfl_sync(0xffffffffu, g, 0);
    if (g >= nrows) break;
    const uint64_t r = p.row_begin + g * W + (uint64_t)p.shard_rank;
    int u[D + 1];  // u[1] < ... < u[D] (u[0] unused)
    if (S.rows_in == nullptr) {  // dimension 1: the rows are the vertices
      u[1] = (int)r;
    } else {                    // the (D-1)-simplex t[0] > ... > t[D-1]: u_i = t[D-i]
      int t[D];
      const uint4 pk = S.rows_in[r];
      const uint32_t w4[4] = {pk.x, pk.y, pk.z, pk.w};
#pragma unroll
      for (int i = 0; i < D; ++i) t[i] = (int)((w4[i >> 1] >> ((i & 1) * 16)) & 0xFFFFu);
#pragma unroll
      for (int i = 1; i <= D; ++i) u[i] = t[D - i];
    }
    u[0] = 0;
    const int u1 = u[1];
    if (u1 == 0) continue;
    int x[D];  // the row's vertices (bitmap rows to AND)
#pragma unroll
    for (int i = 0; i < D; ++i) x[i] = u[i + 1];
    // prefix pair maxima: pm_up over all pairs of σ, pm_ex[j] over the pairs avoiding u_j
    uint32_t pm_up = 0;
    uint32_t pm_ex[D + 1];
#pragma unroll
    for (int j = 0; j <= D; ++j) pm_ex[j] = 0;
#pragma unroll
    for (int a = 1; a <= D; ++a)
#pragma unroll
      for (int b = a + 1; b <= D; ++b) {
        const uint32_t rr = rank_at(T, u[a], u[b]);
        pm_up = umax(pm_up, rr);
#pragma unroll
        for (int j = 1; j <= D; ++j)
          if (j != a && j != b) pm_ex[j] = umax(pm_ex[j], rr);
      }
    uint64_t cbase = 0;
#pragma unroll
    for (int i = 1; i <= D; ++i) cbase += binom(T, u[i], i + 1);
    // C(σ) in segments of SP_LCAP entries from the top; the buffer keeps the segment it
    // holds (c_seg) across survivor batches, and c_word / c_mask continue after it
    int c_word = 0, c_fill = 0, c_seg = -1;
    uint32_t c_mask = 0;
    // survivors w < u_1 in batches of 32
    int s_word = (u1 - 1) >> 5;
    uint32_t s_mask = (u1 & 31) ? ((1u << (u1 & 31)) - 1) : 0xffffffffu;
    while (s_word >= 0) {
      const int nb = bm_list<D>(S, x, s_word, s_mask, sw, 32);
      if (nb == 0) break;
      const bool valid = lane < nb;
      const int w = valid ? (int)sw[lane] : 0;
      uint32_t a[D + 1];
      uint32_t rs = pm_up;
#pragma unroll
      for (int i = 1; i <= D; ++i) {
        a[i] = valid ? rank_at(T, u[i], w) : 0;
        rs = umax(rs, a[i]);
      }
      surv_acc += (unsigned long long)nb;
      int s[D + 1];  // s[0] > ... > s[D] = w
#pragma unroll
      for (int i = 0; i < D; ++i) s[i] = u[D - i];
      s[D] = w;
      if (S.rows_out) {  // every survivor is a prefix row of dimension d+1
        const unsigned long long slot = warp_append(valid, S.rows_out_count);
        if (valid && slot < S.rows_out_cap) S.rows_out[slot] = pack_vertices<D>(s);
      }
      const uint64_t cidx = cbase + (uint64_t)w;
      bool cleared = false;
      if (valid) {
        if (B.clr) cleared = bit_test(B.clr, cidx);
        else if (B.clr_hash) cleared = hash_has(B.clr_hash, B.clr_hash_mask, cidx);
      }
      clr_acc += __popc(__ballot_sync(0xffffffffu, cleared));
      bool active = valid && !cleared;
      int hitv = -1, examined = 0;
      // Lemma 5.3.6 condition 1: the first v of C(σ) (descending) with v != w and
      // max(m(v), R[w][v]) <= diam(s)
      int seg = 0;
      while (__any_sync(0xffffffffu, active)) {
        if (c_seg != seg) {  // (re)build segment `seg` of C(σ)
          if (seg == 0) {
            c_word = S.nw - 1;
            c_mask = (T.n & 31) ? ((1u << (T.n & 31)) - 1) : 0xffffffffu;
          }
          c_fill = bm_list<D>(S, x, c_word, c_mask, cv, SP_LCAP);
          for (int j = lane; j < c_fill; j += 32) {
            const int v = cv[j];
            uint32_t m = 0;
#pragma unroll
            for (int i = 1; i <= D; ++i) m = umax(m, rank_at(T, u[i], v));
            cm[j] = m;
          }
          __syncwarp();
          c_seg = seg;
        }
        for (int k = 0; k < c_fill; k += 2) {
          {
            const int v = cv[k];
            const uint32_t m = cm[k];
            examined += active;
            if (active && v != w && m <= rs && rank_at(T, w, v) <= rs) {
              hitv = v;
              active = false;
            }
          }
          if (k + 1 < c_fill) {
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
        if (c_word < 0) break;  // this was the last segment
        ++seg;
      }
      active = false;
      scan_acc += (unsigned long long)__reduce_add_sync(0xffffffffu, (unsigned)examined);
      // condition 2: no facet of t = s ∪ {hitv} lex-smaller than s (one without a vertex
      // x > hitv) has diam(t) = diam(s)
      bool app = false;
      if (hitv >= 0) {
        app = true;
        uint32_t b[D + 1];
        uint32_t bup = 0;
#pragma unroll
        for (int i = 1; i <= D; ++i) {
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
      app_acc += __popc(__ballot_sync(0xffffffffu, app));
      if (app && (B.clr_next || B.clr_next_hash || B.app_pairs)) {
        const uint64_t tc = cofacet_cidx<D>(T, s, hitv);
        if (B.clr_next) bit_set(B.clr_next, tc);
        if (B.clr_next_hash) hash_put(B.clr_next_hash, B.clr_next_hash_mask, tc);
        if (B.app_pairs) {
          const unsigned long long slot = atomicAdd(&B.ctr->app_pairs, 1ull);
          if (slot < B.app_cap) {
            B.app_pairs[2 * slot] = cidx;
            B.app_pairs[2 * slot + 1] = tc;
          }
        }
      }
      const bool nonapp = valid && !cleared && !app;
      const bool to_resid = clrmode && nonapp;
      const bool to_queue = !clrmode && nonapp;  // clearing decided by k_resolve_sparse
      const uint64_t key = ((uint64_t)(p.maxr - rs) << p.cbits) | cidx;
      const unsigned long long rslot = warp_append(to_resid, &B.ctr->residual);
      if (to_resid && rslot < B.rcap) B.resid[rslot] = key;
      const unsigned long long qslot = warp_append(to_queue, &B.ctr->queued);
      if (to_queue && qslot < B.qcap) {
        B.qkey[qslot] = key;
        B.qvert[qslot] = pack_vertices<D>(s);
      }
    }
  }
  if (lane == 0) {
    if (surv_acc) atomicAdd(&B.ctr->survivors, surv_acc);
    if (app_acc) atomicAdd(&B.ctr->apparent1, app_acc);
    if (scan_acc) atomicAdd(&B.ctr->scanned, scan_acc);
    if (clr_acc) atomicAdd(&B.ctr->cleared, clr_acc);
  }
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

__global__ void k_hash_put(const uint64_t* __restrict__ list, int64_t m, uint64_t* __restrict__ t, uint64_t mask) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    hash_put(t, mask, __ldg(list + i));
}

// ------------------------------------------------------------------ launchers
static int sp_sms() {
  int dev = 0, s = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
  return s > 0 ? s : 148;
}

void launch_threshold_bitmap(const uint32_t* rank, int n, uint32_t* bm, uint32_t* deg, uint32_t* deg_below, cudaStream_t st,
                             int64_t* launches) {
  const int nw = (n + 31) / 32;
  const unsigned blocks = (unsigned)(((uint64_t)n * 32 + SP_THREADS - 1) / SP_THREADS);
  k_bitmap<<<blocks, SP_THREADS, 0, st>>>(rank, n, nw, bm, deg, deg_below);
  *launches += 1;
}

void launch_row_bound(const uint4* rows, uint64_t nrows, int dprev, const uint32_t* deg_below, unsigned long long* out,
                      cudaStream_t st, int64_t* launches) {
  if (!nrows) return;
  const uint64_t blocks = std::min<uint64_t>((nrows + 255) / 256, (uint64_t)sp_sms() * 8);
  k_row_bound<<<(unsigned)blocks, 256, 0, st>>>(rows, nrows, dprev, deg_below, out);
  *launches += 1;
}

template <int D>
static void enum_sparse_d(const DimParams& p, const Tables& T, const HotBuffers& B, const SparseRows& S, cudaStream_t st) {
  const uint64_t rows = p.row_end - p.row_begin;
  uint64_t blocks = (rows * 32 + SP_THREADS - 1) / SP_THREADS;
  const uint64_t cap = (uint64_t)sp_sms() * 4;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  k_enum_sparse<D><<<(unsigned)blocks, SP_THREADS, 0, st>>>(T, p, B, S);
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
                             const SparseRows& S, cudaStream_t st, int64_t* launches) {
  Tables T{rank, binom, (int32_t)p.n, kmax};
  switch (p.d) {
    case 1: enum_sparse_d<1>(p, T, B, S, st); break;
    case 2: enum_sparse_d<2>(p, T, B, S, st); break;
    case 3: enum_sparse_d<3>(p, T, B, S, st); break;
    case 4: enum_sparse_d<4>(p, T, B, S, st); break;
    case 5: enum_sparse_d<5>(p, T, B, S, st); break;
    case 6: enum_sparse_d<6>(p, T, B, S, st); break;
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

void launch_hash_put(const uint64_t* list, int64_t m, uint64_t* table, uint64_t mask, cudaStream_t st, int64_t* launches) {
  if (m <= 0) return;
  const int64_t blocks = std::min<int64_t>((m + 255) / 256, (int64_t)sp_sms() * 8);
  k_hash_put<<<(unsigned)blocks, 256, 0, st>>>(list, m, table, mask);
  if (launches) *launches += 1;
}

}  // namespace vr
