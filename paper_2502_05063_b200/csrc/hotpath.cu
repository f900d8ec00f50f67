// hotpath.cu — the per-dimension GPU hot path.
//
// Paper order (Fig 5.3(b), Alg 17/18, Alg 13): filter+clear all C(n,d+1) columns ->
// sort ALL survivors -> apparent test per sorted column -> partition.  The apparent test
// of Lemma 5.3.6 depends only on the column itself and the distance matrix (Cor 5.3.7,
// "we may generate the cofacets of simplex s and facets of cofacet t of s
// independently"), not on the column's position in the sorted order; and apparent
// columns are never cleared (Prop 5.3.9 argument).  So this design runs the
// apparent test INSIDE the enumeration, and only the few columns that are not apparent
// travel further:
//
//   k_enumerate<D>  (a1 + a2 + a5 phase 1 + a3)
//       one warp per "row" = a fixed upper-vertex prefix (u_D > ... > u_1); the 32 lanes
//       take consecutive v_0 < u_1, so the d-simplices of a row have consecutive cidx
//       (Eq 5.6) and every rank read R[u_i][v_0] is a coalesced row segment.  Per lane:
//       diameter rank = max pairwise rank, threshold (diam <= t, inclusive, Eq 5.3),
//       clearing (one bit of the dimension's clearing bitmap — the deaths of dimension
//       d-1, Lemma 4.2.3), then Lemma 5.3.6 over the cofacet vertices v = n-1, n-2, ...
//       (lex-decreasing cofacets, Alg 14) for at most `steps` vertices.  The prefix part
//       of every new-edge maximum, max_i R[u_i][v], is precomputed once per row for a
//       32-vertex window, one value per lane, and broadcast with __shfl_sync, so a scan
//       step costs one coalesced load R[v][v_0] per warp.  Condition 2 (no lex-smaller
//       facet of t with the same diameter) is evaluated once per chunk after the scan.
//       Apparent columns are counted and mark their cofacet in the next dimension's
//       clearing bitmap; non-apparent ones go straight to the residual list; columns
//       whose equal-diameter cofacet lies beyond the window go to the phase-2 queue with
//       their vertices (warp-aggregated appends, §5.5.3).
//
//   k_resolve<D>    (a5 phase 2 + a6)
//       one warp per queued column, resuming the Lemma 5.3.6 scan where phase 1 stopped,
//       32 cofacet vertices per step (ballot; the lowest set lane = the lex-greatest
//       equal-diameter cofacet).  Fallback when a clearing bitmap would be too large:
//       phase 1 queues every non-proven column and phase 2 decides clearing by
//       recomputation (the column is the apparent cofacet of its youngest facet) plus a
//       binary search in the dimension-(d-1) residual deaths.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>
#include <cuda_runtime.h>

#include "vr_common.cuh"
#include "vr_internal.h"

namespace vr {

constexpr int HP_THREADS = 256;
constexpr int64_t kWinMaxN = 544;  // shared-memory window up to n*144 B = 78 KB (3 CTAs/SM)

// ------------------------------------------------------------------ phase 1: enumerate
// Row-invariant parts of the upper prefix U = {u_D > ... > u_2}, reused by consecutive rows
// that differ only in u_1 (colex-consecutive rows): pair maxima over U (all, and avoiding
// each u_j), the cidx part sum_{i>=2} C(u_i, i+1), and the window maximum over U.
template <int D>
struct UpperCache {
  int key[D + 2];
  bool valid = false;
  uint32_t pmU, pmU_ex[D + 1], mupU;
  uint64_t cU;
};

template <int D>
__device__ __forceinline__ void process_row(const Tables& T, const DimParams& p, const HotBuffers& B, const int (&u)[D + 2],
                                            UpperCache<D>& uc, const uint32_t* __restrict__ Wt, uint32_t* __restrict__ mw,
                                            unsigned long long& surv_acc, unsigned long long& app_acc,
                                            unsigned long long& scan_acc, unsigned long long& clr_acc) {
  const int lane = threadIdx.x & 31;
  const int n = T.n;
  const int v1 = u[1];
  if (v1 == 0) return;  // no v_0 < v_1
  const uint32_t* __restrict__ rowu[D + 1];
#pragma unroll
  for (int i = 1; i <= D; ++i) rowu[i] = T.rank + (size_t)u[i] * (size_t)n;
  bool same = uc.valid;
#pragma unroll
  for (int i = 2; i <= D; ++i) same = same && uc.key[i] == u[i];
  if (!same) {
    uc.valid = true;
    uc.pmU = 0;
    uc.cU = 0;
#pragma unroll
    for (int j = 0; j <= D; ++j) uc.pmU_ex[j] = 0;
#pragma unroll
    for (int i = 2; i <= D; ++i) {
      uc.key[i] = u[i];
      uc.cU += binom(T, u[i], i + 1);
    }
#pragma unroll
    for (int a = 2; a <= D; ++a)
#pragma unroll
      for (int b = a + 1; b <= D; ++b) {
        const uint32_t r = __ldg(rowu[a] + u[b]);
        uc.pmU = umax(uc.pmU, r);
#pragma unroll
        for (int j = 2; j <= D; ++j)
          if (j != a && j != b) uc.pmU_ex[j] = umax(uc.pmU_ex[j], r);
      }
    const int v = n - 1 - lane;
    uint32_t m = v >= 0 ? 0u : VR_RINF;
    if (v >= 0) {
#pragma unroll
      for (int i = 2; i <= D; ++i) m = umax(m, __ldg(rowu[i] + v));  // R[u_i][u_i] = RINF
    }
    uc.mupU = m;
  }
  if (uc.pmU == VR_RINF) return;  // every simplex of the row is over the threshold
  // prefix pair maxima: pm_up over all prefix pairs, pm_ex[j] over pairs avoiding u[j]
  uint32_t r1[D + 1];
  uint32_t pm_up = uc.pmU;
#pragma unroll
  for (int b = 2; b <= D; ++b) {
    r1[b] = __ldg(rowu[1] + u[b]);
    pm_up = umax(pm_up, r1[b]);
  }
  if (pm_up == VR_RINF) return;
  uint32_t pm_ex[D + 1];
  pm_ex[0] = 0;
  pm_ex[1] = uc.pmU;
#pragma unroll
  for (int j = 2; j <= D; ++j) {
    uint32_t m = uc.pmU_ex[j];
#pragma unroll
    for (int b = 2; b <= D; ++b)
      if (b != j) m = umax(m, r1[b]);
    pm_ex[j] = m;
  }
  const uint64_t cbase = uc.cU + binom(T, u[1], 2);
  // window of the first 32 cofacet vertices v = n-1-lane: mup = max_i R[u_i][v]
  // (RINF for a prefix vertex, so the warp skips it)
  const int vw = n - 1 - lane;
  const uint32_t mup0 = vw >= 0 ? umax(uc.mupU, __ldg(rowu[1] + vw)) : VR_RINF;
  if (Wt) {  // the row's window maxima in shared memory, read 4 at a time by every lane
    __syncwarp();
    mw[lane] = mup0;
    __syncwarp();
  }
  const int steps = p.steps < n ? p.steps : n;
  const uint32_t* __restrict__ rowtop = T.rank + (size_t)(n - 1) * (size_t)n;  // row of v = n-1

  for (int base = 0; base < v1; base += 32) {
    const int v0 = base + lane;
    const bool valid = v0 < v1;
    uint32_t a[D + 1];
    uint32_t rs = pm_up;
#pragma unroll
    for (int i = 1; i <= D; ++i) {
      a[i] = valid ? __ldg(rowu[i] + v0) : VR_RINF;
      rs = umax(rs, a[i]);
    }
    const bool surv = valid && rs != VR_RINF;  // diam(s) <= t (Eq 5.3, Alg 17 line 3)
    const uint32_t msurv = __ballot_sync(0xffffffffu, surv);
    if (!msurv) continue;
    surv_acc += surv;  // lane-local counts, reduced once per warp at the end
    const uint64_t cidx = cbase + (uint64_t)v0;
    bool cleared = false;
    if (B.clr && surv) cleared = bit_test(B.clr, cidx);  // a death of dimension d-1
    clr_acc += cleared;
    bool active = surv && !cleared;
    bool nohit = false;  // resolved in-kernel: no equal-diameter cofacet at all
    int hitv = -1;
    int examined = 0;  // cofacet vertices this lane examined
    // Lemma 5.3.6 condition 1, lane-parallel: the first v with every new edge <= diam(s)
    const uint32_t* __restrict__ pv = rowtop + v0;  // &R[v][v0], v = n-1-j
    if (p.variant == 0) {
      // one vote per vertex; vertices no active lane can hit are skipped without loads
      for (int j = 0; j < steps; ++j, pv -= n) {
        const uint32_t mact = __ballot_sync(0xffffffffu, active);
        if (!mact) break;
        const int v = n - 1 - j;
        uint32_t m;
        if (j < 32) {
          m = __shfl_sync(0xffffffffu, mup0, j);
        } else {
          m = 0;
#pragma unroll
          for (int i = 1; i <= D; ++i) m = (v == u[i]) ? VR_RINF : umax(m, __ldg(rowu[i] + v));
        }
        examined += active;
        if (!__any_sync(0xffffffffu, active && m <= rs)) continue;
        if (active && v != v0 && m <= rs && umax(m, __ldg(pv)) <= rs) {
          hitv = v;
          active = false;
        }
      }
    } else {
      // one vote per 4 vertices.  Inside the 32-vertex window the prefix part m comes from
      // mup0 and the new-edge rank R[v][v0] from the rank matrix; with the shared-memory
      // window (p.win) both come 4 steps at a time: m4 = mw[j..j+3] (a broadcast) and
      // r4 = Wt[v0][j..j+3] (the transposed window row of v0), so a step is a max, a
      // compare and a select.  Otherwise m is shuffled from mup0 and R[v][v0] loaded
      // (unconditionally: row v, column v0 < n — in range, coalesced over the warp).
      const size_t nn = (size_t)n;
      const int wsteps4 = (steps < 32 ? steps : 32) & ~3;
      int j = 0;
      bool any_active = true;
      if (Wt) {
        const uint32_t* wrow = Wt + (size_t)(v0 < n ? v0 : n - 1) * 36;
        int hitj = -1;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          const int jj = 4 * g;
          if (jj >= wsteps4) break;
          const uint4 m4 = *reinterpret_cast<const uint4*>(mw + jj);
          const uint4 r4 = *reinterpret_cast<const uint4*>(wrow + jj);
          bool h;
          h = active & (umax(m4.x, r4.x) <= rs); hitj = h ? jj + 0 : hitj; active = active & !h;
          h = active & (umax(m4.y, r4.y) <= rs); hitj = h ? jj + 1 : hitj; active = active & !h;
          h = active & (umax(m4.z, r4.z) <= rs); hitj = h ? jj + 2 : hitj; active = active & !h;
          h = active & (umax(m4.w, r4.w) <= rs); hitj = h ? jj + 3 : hitj; active = active & !h;
          j = jj + 4;
          if (!__any_sync(0xffffffffu, active)) { any_active = false; break; }
        }
        if (hitj >= 0) hitv = n - 1 - hitj;
        pv -= (size_t)j * nn;
      } else {
        for (; j < wsteps4; j += 4, pv -= 4 * nn) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int v = n - 1 - (j + q);
            const uint32_t m = __shfl_sync(0xffffffffu, mup0, j + q);
            const uint32_t r = __ldg(pv - (size_t)q * nn);
            const bool hit = active & (umax(m, r) <= rs);  // v = v0: R[v0][v0] = RINF
            hitv = hit ? v : hitv;
            active = active & !hit;
          }
          if (!__any_sync(0xffffffffu, active)) { any_active = false; break; }
        }
      }
      if (any_active) {  // the rest of the budget, one vertex at a time (steps > 32 or n < 32)
        for (; j < steps; ++j, pv -= nn) {
          const int v = n - 1 - j;
          uint32_t m;
          if (j < 32) {
            m = __shfl_sync(0xffffffffu, mup0, j & 31);
          } else {
            m = 0;
#pragma unroll
            for (int i = 1; i <= D; ++i) m = (v == u[i]) ? VR_RINF : umax(m, __ldg(rowu[i] + v));
          }
          if (active && m <= rs && v != v0 && umax(m, __ldg(pv)) <= rs) {
            hitv = v;
            active = false;
          }
          if (!__any_sync(0xffffffffu, active)) break;
        }
      }
      // vertices this lane examined: up to its hit, or the whole budget
      examined = hitv >= 0 ? n - hitv : (active ? steps : 0);
    }
    if (p.variant == 2 && B.clr) {
      // columns still unresolved after the short lock-step scan: the whole warp resolves
      // them one at a time, 32 cofacet vertices per step (phase 2 folded into phase 1 —
      // no queue, no divergence tail)
      uint32_t mrem = __ballot_sync(0xffffffffu, active);
      while (mrem) {
        const int src = __ffs(mrem) - 1;
        mrem &= mrem - 1;
        const int v0s = __shfl_sync(0xffffffffu, v0, src);
        const uint32_t rss = __shfl_sync(0xffffffffu, rs, src);
        const uint32_t* __restrict__ rowv0 = T.rank + (size_t)v0s * (size_t)n;
        int hv = -1;
        for (int base = steps; base < n; base += 32) {
          const int j = base + lane;
          const int v = n - 1 - j;
          const uint32_t msh = __shfl_sync(0xffffffffu, mup0, j & 31);  // every lane takes part
          uint32_t m = VR_RINF;
          if (j < 32) {
            m = msh;
          } else if (v >= 0) {
            m = 0;
#pragma unroll
            for (int i = 1; i <= D; ++i) m = (v == u[i]) ? VR_RINF : umax(m, __ldg(rowu[i] + v));
          }
          const bool hit = v >= 0 && v != v0s && m <= rss && umax(m, __ldg(rowv0 + (v >= 0 ? v : 0))) <= rss;
          const uint32_t bal = __ballot_sync(0xffffffffu, hit);
          if (bal) {
            hv = n - 1 - (base + __ffs(bal) - 1);
            break;
          }
        }
        if (lane == src) {
          hitv = hv;
          active = false;
          examined = hv >= 0 ? n - hv : n;
          if (hv < 0) nohit = true;
        }
      }
    }
    scan_acc += (unsigned)examined;
    // condition 2 for lanes that found t = s ∪ {hitv}: no facet t \ {w}, w > hitv (the
    // lex-smaller facets), with diam = diam(s)
    // (a hit above every vertex of s has no lex-smaller facet to test: apparent at once)
    bool app = hitv >= 0;
    if (hitv >= 0 && hitv < u[D]) {
      uint32_t b[D + 1];
      uint32_t bup = 0;
      const int jh = n - 1 - hitv;
      uint32_t b0;
      if (Wt && jh < 32) {  // R[u_i][hitv] = Wt[u_i][jh], R[hitv][v0] = Wt[v0][jh]
#pragma unroll
        for (int i = 1; i <= D; ++i) {
          b[i] = Wt[(size_t)u[i] * 36 + jh];
          bup = umax(bup, b[i]);
        }
        b0 = Wt[(size_t)v0 * 36 + jh];
      } else {
#pragma unroll
        for (int i = 1; i <= D; ++i) {
          b[i] = __ldg(rowu[i] + hitv);
          bup = umax(bup, b[i]);
        }
        b0 = __ldg(rowtop - (size_t)jh * (size_t)n + v0);
      }
      if (v0 > hitv && umax(pm_up, bup) == rs) app = false;
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
    app_acc += app;
    if (app && (B.clr_next || B.app_pairs)) {
      int s[D + 1];
#pragma unroll
      for (int i = 0; i < D; ++i) s[i] = u[D - i];
      s[D] = v0;
      const uint64_t tc = cofacet_cidx<D>(T, s, hitv);
      if (B.clr_next) bit_set(B.clr_next, tc);
      if (B.app_pairs) {
        const unsigned long long slot = atomicAdd(&B.ctr->app_pairs, 1ull);
        if (slot < B.app_cap) {
          B.app_pairs[2 * slot] = cidx;
          B.app_pairs[2 * slot + 1] = tc;
        }
      }
    }
    const uint64_t key = ((uint64_t)(p.maxr - rs) << p.cbits) | cidx;
    // not apparent and not cleared: a residual column (bitmap mode only — without a
    // bitmap clearing is decided in phase 2)
    const bool to_resid = B.clr && ((hitv >= 0 && !app) || nohit);
    const bool to_queue = active || (!B.clr && hitv >= 0 && !app);
    if (__any_sync(0xffffffffu, to_resid | to_queue)) {  // rare: skip the appends' collectives
      const unsigned long long rslot = warp_append(to_resid, &B.ctr->residual);
      if (to_resid && rslot < B.rcap) B.resid[rslot] = key;
      const unsigned long long qslot = warp_append(to_queue, &B.ctr->queued);
      if (to_queue && qslot < B.qcap) {
        int s[D + 1];
#pragma unroll
        for (int i = 0; i < D; ++i) s[i] = u[D - i];
        s[D] = v0;
        B.qkey[qslot] = key;
        B.qvert[qslot] = pack_vertices<D>(s);
      }
    }
  }
}

template <int D>
__global__ void __launch_bounds__(HP_THREADS) k_enumerate(Tables T, DimParams p, HotBuffers B) {
  const int GRAB = p.grab;
  const int lane = threadIdx.x & 31;
  // shared-memory scan window (p.win): Wt[v][j] = R[n-1-j][v] for the 32 highest vertices
  // (row stride 36 words: 16-byte aligned uint4 reads, conflict-free over 8-lane phases),
  // then one 32-word row-maximum buffer per warp
  extern __shared__ __align__(16) uint32_t hp_smem[];
  uint32_t* Wt = nullptr;
  uint32_t* mw = nullptr;
  if (p.win) {
    const int n = T.n;
    for (int idx = threadIdx.x; idx < 32 * n; idx += blockDim.x) {
      const int jj = idx / n, v = idx - jj * n;  // coalesced over v
      const int row = n - 1 - jj;
      hp_smem[(size_t)v * 36 + jj] = row >= 0 ? __ldg(T.rank + (size_t)row * (size_t)n + v) : VR_RINF;
    }
    __syncthreads();
    Wt = hp_smem;
    mw = hp_smem + (size_t)n * 36 + (size_t)(threadIdx.x >> 5) * 32;
  }
  unsigned long long surv_acc = 0, app_acc = 0, scan_acc = 0, clr_acc = 0;
  // Rows are handed out from the LAST row down: the work of a row grows with its
  // smallest prefix vertex u_1 (row length), which grows with the row index, so the
  // small rows form the tail of the schedule.
  const uint64_t W = (uint64_t)p.shard_world;
  const uint64_t all = p.row_end - p.row_begin;
  const uint64_t nrows = all > (uint64_t)p.shard_rank ? (all - (uint64_t)p.shard_rank + W - 1) / W : 0;  // this shard's rows
  UpperCache<D> uc;  // kept across grabs: a warp's next grab often shares the upper prefix
  while (true) {
    unsigned long long g0 = 0;
    if (lane == 0) g0 = atomicAdd(&B.ctr->row_next, (unsigned long long)GRAB);
    g0 = __shfl_sync(0xffffffffu, g0, 0);
    if (g0 >= nrows) break;
    // process rows rtop, rtop-1, ... (GRAB is 1 when sharded)
    const uint64_t rtop = p.row_end - 1 - (g0 * W + (uint64_t)p.shard_rank);
    const uint64_t cnt = (g0 + GRAB <= nrows) ? (uint64_t)GRAB : nrows - g0;
    // decode prefix row rtop (colex rank of {u_D > ... > u_1}: r = sum_i C(u_i, i))
    int u[D + 2];
    {
      uint64_t x = rtop;
      int hi = T.n;
#pragma unroll
      for (int i = D; i >= 1; --i) {
        const int vv = cns_find(T, x, i, hi);
        u[i] = vv;
        x -= binom(T, vv, i);
        hi = vv;
      }
      u[0] = 0;
      u[D + 1] = T.n;
    }
    for (uint64_t k = 0; k < cnt; ++k) {
      if (k > 0) {  // colex predecessor of the prefix
        bool done = false;
        int top = 0;
#pragma unroll
        for (int i = 1; i <= D; ++i) {
          if (!done && u[i] > i - 1) { u[i] -= 1; top = i; done = true; }
        }
#pragma unroll
        for (int j = D; j >= 1; --j)
          if (j < top) u[j] = u[top] - (top - j);
      }
      process_row<D>(T, p, B, u, uc, Wt, mw, surv_acc, app_acc, scan_acc, clr_acc);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    surv_acc += __shfl_xor_sync(0xffffffffu, surv_acc, o);
    app_acc += __shfl_xor_sync(0xffffffffu, app_acc, o);
    scan_acc += __shfl_xor_sync(0xffffffffu, scan_acc, o);
    clr_acc += __shfl_xor_sync(0xffffffffu, clr_acc, o);
  }
  if (lane == 0) {
    if (surv_acc) atomicAdd(&B.ctr->survivors, surv_acc);
    if (app_acc) atomicAdd(&B.ctr->apparent1, app_acc);
    if (scan_acc) atomicAdd(&B.ctr->scanned, scan_acc);
    if (clr_acc) atomicAdd(&B.ctr->cleared, clr_acc);
  }
}

// ------------------------------------------------------------------ phase 1, flattened
// Dense dimensions with the shared-memory window: the candidates of a "super-row" (all
// d-simplices sharing the upper vertices u_D > ... > u_2) are the pairs (u_1, v_0),
// v_0 < u_1 < u_2, numbered i = C(u_1, 2) + v_0 — so cidx = sum_{i>=2} C(u_i, i+1) + i —
// and cut into chunks of `chunk` consecutive i (1024, or fewer — down to 128 — when the
// dimension has too few candidates to give every SM ~24 warps).  A warp takes one chunk per grab (largest
// super-rows first) and its 32 lanes take consecutive i, across row boundaries: no ragged
// row tails, and the per-row setup (prefix maxima, window, cidx base) becomes per-chunk.
// Per lane the row-dependent parts (R[u_1][u_b], R[u_1][v] in the window) are read for the
// lane's own u_1 (mostly shared by the warp).  Same tests and outputs as process_row.
constexpr int FL_CHUNK = 1024;  // largest chunk (VR_FL_CHUNK overrides, for tuning runs)

template <int D>
__global__ void __launch_bounds__(HP_THREADS, 4) k_enumerate_flat(Tables T, DimParams p, HotBuffers B,
                                                               const uint32_t* __restrict__ chunk_start, uint32_t nsuper,
                                                               uint32_t nchunks, int chunk) {
  const int lane = threadIdx.x & 31;
  const int n = T.n;
  extern __shared__ __align__(16) uint32_t hp_smem[];
  for (int idx = threadIdx.x; idx < 32 * n; idx += blockDim.x) {
    const int jj = idx / n, v = idx - jj * n;
    const int row = n - 1 - jj;
    hp_smem[(size_t)v * 36 + jj] = row >= 0 ? __ldg(T.rank + (size_t)row * (size_t)n + v) : VR_RINF;
  }
  __syncthreads();
  const uint32_t* Wt = hp_smem;
  uint32_t* mw = hp_smem + (size_t)n * 36 + (size_t)(threadIdx.x >> 5) * 32;  // window max over u_2..u_D
  // per-lane counters, reduced once at the end (no warp collective per iteration)
  uint32_t surv_c = 0, app_c = 0, clr_c = 0;
  unsigned long long scan_c = 0;
  const int steps = p.steps < n ? p.steps : n;
  const int wsteps4 = (steps < 32 ? steps : 32) & ~3;
  // shards: chunk c belongs to rank (nchunks-1-c) mod world (the chunks partition the
  // candidates, as the rows do for the row kernel)
  const uint64_t SW = (uint64_t)p.shard_world, SR = (uint64_t)p.shard_rank;
  const uint64_t mine = nchunks > SR ? ((uint64_t)nchunks - SR + SW - 1) / SW : 0;
  while (true) {
    unsigned long long g0 = 0;
    if (lane == 0) g0 = atomicAdd(&B.ctr->row_next, 1ull);
    g0 = __shfl_sync(0xffffffffu, g0, 0);
    if (g0 >= mine) break;
    const uint32_t c = nchunks - 1 - (uint32_t)(g0 * SW + SR);
    // super-row of chunk c: the last t with chunk_start[t] <= c
    uint32_t lo = 0, hi = nsuper - 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (__ldg(chunk_start + mid) <= c) lo = mid; else hi = mid - 1;
    }
    const uint32_t t = lo;
    int u[D + 2];
    uint64_t cU = 0;
    int u2 = n;
    {
      uint64_t x = t;
      int h = n;
#pragma unroll
      for (int i = D; i >= 2; --i) {
        const int vv = cns_find(T, x, i - 1, h);
        u[i] = vv;
        x -= binom(T, vv, i - 1);
        cU += binom(T, vv, i + 1);
        h = vv;
      }
      if (D >= 2) u2 = u[2];
    }
    const uint64_t cnt_sr = (uint64_t)u2 * (uint64_t)(u2 - 1) / 2;
    const uint64_t i0 = (uint64_t)(c - __ldg(chunk_start + t)) * (uint64_t)chunk;
    const uint64_t iend = (i0 + (uint64_t)chunk < cnt_sr) ? i0 + (uint64_t)chunk : cnt_sr;
    // upper-prefix parts: pair maxima over u_2..u_D (all / avoiding u_j), window maxima
    uint32_t pmU = 0, pmU_ex[D + 1];
#pragma unroll
    for (int j = 0; j <= D; ++j) pmU_ex[j] = 0;
#pragma unroll
    for (int a = 2; a <= D; ++a)
#pragma unroll
      for (int b = a + 1; b <= D; ++b) {
        const uint32_t r = rank_at(T, u[a], u[b]);
        pmU = umax(pmU, r);
#pragma unroll
        for (int j = 2; j <= D; ++j)
          if (j != a && j != b) pmU_ex[j] = umax(pmU_ex[j], r);
      }
    {
      const int v = n - 1 - lane;
      uint32_t m = v >= 0 ? 0u : VR_RINF;
#pragma unroll
      for (int q = 2; q <= D; ++q) m = v >= 0 ? umax(m, Wt[(size_t)u[q] * 36 + lane]) : m;  // R[u_q][v]
      __syncwarp();
      mw[lane] = m;
      __syncwarp();
    }
    if (pmU == VR_RINF) continue;  // every simplex of the super-row is over the threshold
    // (u_1, v_0) of i = C(u_1, 2) + v_0: decoded once per chunk (i < C(n,2) < 2^31), then
    // advanced by 32 per iteration (v_0 += 32, carried into u_1)
    int cu1, cv0;
    {
      const uint32_t ii = (uint32_t)(i0 + (uint64_t)lane);
      int x = (int)((1.0f + sqrtf(1.0f + 8.0f * (float)ii)) * 0.5f);
      while ((uint32_t)x * (uint32_t)(x - 1) / 2 > ii) --x;
      while ((uint32_t)(x + 1) * (uint32_t)x / 2 <= ii) ++x;
      cu1 = x;
      cv0 = (int)(ii - (uint32_t)x * (uint32_t)(x - 1) / 2);
    }
    // n <= kWinMaxN here: every rank-matrix offset fits 32 bits, and the rows of the
    // chunk-invariant vertices u_2..u_D are fixed for the whole chunk
    const uint32_t* __restrict__ rk = T.rank;
    uint32_t oq[D + 1];  // row offsets of u_2..u_D
#pragma unroll
    for (int q = 2; q <= D; ++q) oq[q] = (uint32_t)u[q] * (uint32_t)n;
    const uint32_t len = (uint32_t)(iend - i0);
    const uint64_t c0 = cU + i0;  // cidx of the chunk's first candidate
    // clearing-bitmap words of the chunk: bit c0 + il = bit (cb + il) of clrw
    const uint32_t* __restrict__ clrw = B.clr ? B.clr + (c0 >> 5) : nullptr;
    const uint32_t cb = (uint32_t)(c0 & 31);
    uint32_t scan_chunk = 0;
    int r1_u1 = -1;
    uint32_t r1[D + 1], r1_pm = 0;
    for (uint32_t off = 0; off < len; off += 32) {
      const uint32_t il = off + (uint32_t)lane;
      const bool valid = il < len;
      if (off != 0) {
        cv0 += 32;
        while (cv0 >= cu1) { cv0 -= cu1; ++cu1; }
      }
      const int u1 = valid ? cu1 : 1, v0 = valid ? cv0 : 0;
      u[1] = u1;
      const uint32_t o1 = (uint32_t)u1 * (uint32_t)n;
      uint32_t a[D + 1];
      if (u1 != r1_u1) {  // R[u_1][u_b] only when the lane's u_1 moved on
        r1_u1 = u1;
        r1_pm = pmU;
#pragma unroll
        for (int b = 2; b <= D; ++b) {
          r1[b] = __ldg(rk + (o1 + (uint32_t)u[b]));
          r1_pm = umax(r1_pm, r1[b]);
        }
      }
      const uint32_t pm_up = r1_pm;
      uint32_t rs = pm_up;
      a[1] = valid ? __ldg(rk + (o1 + (uint32_t)v0)) : VR_RINF;
      rs = umax(rs, a[1]);
#pragma unroll
      for (int q = 2; q <= D; ++q) {
        a[q] = valid ? __ldg(rk + (oq[q] + (uint32_t)v0)) : VR_RINF;
        rs = umax(rs, a[q]);
      }
      const bool surv = valid && rs != VR_RINF;
      const uint32_t msurv = __ballot_sync(0xffffffffu, surv);
      if (!msurv) continue;
      surv_c += surv;
      const uint64_t cidx = c0 + il;
      bool cleared = false;
      if (clrw && surv) {
        const uint32_t bo = cb + il;
        cleared = (__ldg(clrw + (bo >> 5)) >> (bo & 31)) & 1u;
      }
      clr_c += cleared;
      bool active = surv && !cleared;
      int hitv = -1;
      // scan: m_j = max(upper window mw[j], R[u_1][v_j] = Wt[u_1][j]), R[v_j][v_0] = Wt[v_0][j]
      const uint32_t* wrow0 = Wt + (size_t)v0 * 36;
      const uint32_t* wrow1 = Wt + (size_t)u1 * 36;
      int j = 0;
      bool any_active = true;
      {
        int hitj = -1;
#pragma unroll
        for (int gq = 0; gq < 8; ++gq) {
          const int jj = 4 * gq;
          if (jj >= wsteps4) break;
          const uint4 mu = *reinterpret_cast<const uint4*>(mw + jj);
          const uint4 m1 = *reinterpret_cast<const uint4*>(wrow1 + jj);
          const uint4 r4 = *reinterpret_cast<const uint4*>(wrow0 + jj);
          bool h;
          h = active & (umax(umax(mu.x, m1.x), r4.x) <= rs); hitj = h ? jj + 0 : hitj; active = active & !h;
          h = active & (umax(umax(mu.y, m1.y), r4.y) <= rs); hitj = h ? jj + 1 : hitj; active = active & !h;
          h = active & (umax(umax(mu.z, m1.z), r4.z) <= rs); hitj = h ? jj + 2 : hitj; active = active & !h;
          h = active & (umax(umax(mu.w, m1.w), r4.w) <= rs); hitj = h ? jj + 3 : hitj; active = active & !h;
          j = jj + 4;
          if (!__any_sync(0xffffffffu, active)) { any_active = false; break; }
        }
        if (hitj >= 0) hitv = n - 1 - hitj;
      }
      if (any_active) {  // beyond the window (steps > 32, or n % 4 leftovers)
        for (; j < steps; ++j) {
          const int v = n - 1 - j;
          uint32_t m = 0;
#pragma unroll
          for (int q = 1; q <= D; ++q) m = umax(m, __ldg(rk + ((q == 1 ? o1 : oq[q]) + (uint32_t)v)));
          if (active && m <= rs && umax(m, __ldg(rk + ((uint32_t)v * (uint32_t)n + (uint32_t)v0))) <= rs) {
            hitv = v;
            active = false;
          }
          if (!__any_sync(0xffffffffu, active)) break;
        }
      }
      const int examined = hitv >= 0 ? n - hitv : (active ? steps : 0);
      scan_chunk += (unsigned)examined;
      // condition 2 (as in process_row)
      bool app = hitv >= 0;
      if (hitv >= 0 && hitv < u[D]) {  // else no vertex of s above the hit: apparent
        uint32_t pm_ex[D + 1];
        pm_ex[0] = 0;
        pm_ex[1] = pmU;
#pragma unroll
        for (int jx = 2; jx <= D; ++jx) {
          uint32_t m = pmU_ex[jx];
#pragma unroll
          for (int b = 2; b <= D; ++b)
            if (b != jx) m = umax(m, r1[b]);
          pm_ex[jx] = m;
        }
        uint32_t bb[D + 1];
        uint32_t bup = 0;
        const int jh = n - 1 - hitv;
        uint32_t b0;
        if (jh < 32) {
#pragma unroll
          for (int q = 1; q <= D; ++q) {
            bb[q] = Wt[(size_t)u[q] * 36 + jh];
            bup = umax(bup, bb[q]);
          }
          b0 = Wt[(size_t)v0 * 36 + jh];
        } else {
#pragma unroll
          for (int q = 1; q <= D; ++q) {
            bb[q] = rank_at(T, u[q], hitv);
            bup = umax(bup, bb[q]);
          }
          b0 = rank_at(T, hitv, v0);
        }
        if (v0 > hitv && umax(pm_up, bup) == rs) app = false;
#pragma unroll
        for (int jx = 1; jx <= D; ++jx) {
          if (u[jx] > hitv) {
            uint32_t m = umax(pm_ex[jx], b0);
#pragma unroll
            for (int q = 1; q <= D; ++q)
              if (q != jx) m = umax(m, umax(a[q], bb[q]));
            if (m == rs) app = false;
          }
        }
      }
      app_c += app;
      if (app && (B.clr_next || B.app_pairs)) {
        int sv[D + 1];
#pragma unroll
        for (int q = 0; q < D; ++q) sv[q] = u[D - q];
        sv[D] = v0;
        const uint64_t tc = cofacet_cidx<D>(T, sv, hitv);
        if (B.clr_next) bit_set(B.clr_next, tc);
        if (B.app_pairs) {
          const unsigned long long slot = atomicAdd(&B.ctr->app_pairs, 1ull);
          if (slot < B.app_cap) {
            B.app_pairs[2 * slot] = cidx;
            B.app_pairs[2 * slot + 1] = tc;
          }
        }
      }
      const bool to_resid = B.clr && hitv >= 0 && !app;
      const bool to_queue = active || (!B.clr && hitv >= 0 && !app);
      if (__any_sync(0xffffffffu, to_resid | to_queue)) {  // rare: skip the appends' collectives
        const uint64_t key = ((uint64_t)(p.maxr - rs) << p.cbits) | cidx;
        const unsigned long long rslot = warp_append(to_resid, &B.ctr->residual);
        if (to_resid && rslot < B.rcap) B.resid[rslot] = key;
        const unsigned long long qslot = warp_append(to_queue, &B.ctr->queued);
        if (to_queue && qslot < B.qcap) {
          int sv[D + 1];
#pragma unroll
          for (int q = 0; q < D; ++q) sv[q] = u[D - q];
          sv[D] = v0;
          B.qkey[qslot] = key;
          B.qvert[qslot] = pack_vertices<D>(sv);
        }
      }
    }
    scan_c += scan_chunk;
  }
  const unsigned long long surv_acc = __reduce_add_sync(0xffffffffu, surv_c);
  const unsigned long long app_acc = __reduce_add_sync(0xffffffffu, app_c);
  const unsigned long long clr_acc = __reduce_add_sync(0xffffffffu, clr_c);
  unsigned long long scan_acc = scan_c;
#pragma unroll
  for (int o = 16; o; o >>= 1) scan_acc += __shfl_xor_sync(0xffffffffu, scan_acc, o);
  if (lane == 0) {
    if (surv_acc) atomicAdd(&B.ctr->survivors, surv_acc);
    if (app_acc) atomicAdd(&B.ctr->apparent1, app_acc);
    if (scan_acc) atomicAdd(&B.ctr->scanned, scan_acc);
    if (clr_acc) atomicAdd(&B.ctr->cleared, clr_acc);
  }
}

// ------------------------------------------------------------------ phase 2: resolve
// First v <= start (descending) not in S with max_{w in S} R[w][v] <= r, or -1.
// Lanes take v = base - lane: each load R[w][v] is a coalesced row segment.
template <int K>
__device__ __forceinline__ int coop_scan(const Tables& T, const int (&S)[K], uint32_t r, int start,
                                         unsigned long long& scan_acc) {
  const int lane = threadIdx.x & 31;
  for (int base = start; base >= 0; base -= 32) {
    scan_acc += (unsigned long long)(base + 1 < 32 ? base + 1 : 32);
    const int v = base - lane;
    bool ok = v >= 0;
    uint32_t rt = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (ok) {
        if (v == S[k]) ok = false;
        else rt = umax(rt, rank_at(T, S[k], v));
      }
    }
    const uint32_t m = __ballot_sync(0xffffffffu, ok && rt <= r);
    if (m) return base - (__ffs(m) - 1);
  }
  return -1;
}

template <int D>
__global__ void __launch_bounds__(HP_THREADS) k_resolve(Tables T, DimParams p, HotBuffers B, uint64_t qn) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t cmask = p.cbits >= 64 ? ~0ull : ((1ull << p.cbits) - 1);
  const int start = T.n - 1 - p.steps;  // phase 1 examined v = n-1 .. n-steps
  unsigned long long app_acc = 0, clr_acc = 0, scan_acc = 0;
  for (uint64_t e = warp; e < qn; e += nwarps) {
    const uint64_t key = __ldg(B.qkey + e);
    const uint32_t rs = p.maxr - (uint32_t)(key >> p.cbits);
    const uint64_t cidx = key & cmask;
    int s[D + 1];
    unpack_vertices<D>(B.qvert[e], s);
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
    // Lemma 5.3.6 condition 1 (without a bitmap, columns phase 1 already found
    // non-apparent are queued too and simply re-find their hit from the top)
    const int v = coop_scan<D + 1>(T, s, rs, B.clr ? start : T.n - 1, scan_acc);
    bool app = false;
    if (v >= 0) {
      // condition 2: no facet t \ {w}, w > v, with diam = diam(s); lane j checks w = s[j]
      bool bad = false;
      if (lane <= D) {
        const int j = lane;
        int w = 0;
        uint32_t m = 0;
#pragma unroll
        for (int q = 0; q <= D; ++q)
          if (q == j) { w = s[q]; m = ex[q]; }
        if (w > v) {
#pragma unroll
          for (int i = 0; i <= D; ++i)
            if (i != j) m = umax(m, rank_at(T, v, s[i]));
          bad = (m == rs);
        }
      }
      app = !__any_sync(0xffffffffu, bad);
    }
    if (app) {
      ++app_acc;
      if (lane == 0 && (B.clr_next || B.app_pairs)) {
        const uint64_t tc = cofacet_cidx<D>(T, s, v);
        if (B.clr_next) bit_set(B.clr_next, tc);
        if (B.app_pairs) {
          const unsigned long long slot = atomicAdd(&B.ctr->app_pairs, 1ull);
          if (slot < B.app_cap) {
            B.app_pairs[2 * slot] = cidx;
            B.app_pairs[2 * slot + 1] = tc;
          }
        }
      }
      continue;
    }
    if (!B.clr) {
      // clearing by recomputation (§5.2.3, Lemma 4.2.3): s is cleared iff it is the death
      // of a pair of dimension d-1 — a residual pair (sorted list) or an apparent pair:
      // s is the apparent cofacet of its youngest facet f (the first facet in Alg 16 order
      // — removing s[0], s[1], ... — with diam(f) = diam(s)) iff the lex-greatest
      // equal-diameter cofacet of f is s itself.
      bool cleared = sorted_contains(B.deaths, B.ndeaths, cidx);
      if (D >= 2 && !cleared) {
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
          cleared = coop_scan<D>(T, f, rs, T.n - 1, scan_acc) == w;
        }
      }
      if (cleared) {
        ++clr_acc;
        continue;
      }
    }
    if (lane == 0) {
      const unsigned long long slot = atomicAdd(&B.ctr->residual, 1ull);
      if (slot < B.rcap) B.resid[slot] = key;
    }
  }
  if (lane == 0) {
    if (app_acc) atomicAdd(&B.ctr->apparent2, app_acc);
    if (clr_acc) atomicAdd(&B.ctr->cleared, clr_acc);
    if (scan_acc) atomicAdd(&B.ctr->scanned2, scan_acc);
  }
}

__global__ void k_set_bits(const uint64_t* __restrict__ list, int64_t m, uint32_t* __restrict__ bm) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    bit_set(bm, __ldg(list + i));
}

// ------------------------------------------------------------------ launchers
static int sm_count() {
  static const char tag = 0;
  return device_memo(&tag, [] {
    int dev = 0, s = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
    return s > 0 ? s : 148;
  });
}

static uint64_t binom_u64(uint64_t v, int k) {
  if ((uint64_t)k > v) return 0;
  unsigned __int128 c = 1;
  for (int i = 1; i <= k; ++i) c = c * (unsigned __int128)(v - (uint64_t)k + (uint64_t)i) / (unsigned __int128)i;
  return (uint64_t)c;
}
static bool getenv_flag(const char* name) { return std::getenv(name) != nullptr; }

// Chunk table of k_enumerate_flat for (n, D): chunk_start[t] = chunks of the super-rows
// before t (super-rows in colex order of u_D > ... > u_2; one super-row when D = 1).  It
// depends only on (n, D), so it is built once per process on the host and kept on the
// device (like the binomial table).
struct FlatTable {
  uint32_t* d_start = nullptr;
  uint32_t nsuper = 0, nchunks = 0;
  int chunk = FL_CHUNK;
};
static const FlatTable* flat_table(int64_t n, int D) {
  static std::mutex mu;
  static std::map<std::pair<int64_t, int>, FlatTable> cache;
  std::lock_guard<std::mutex> g(mu);
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_pair(n * 64 + dev, D);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second.d_start ? &it->second : nullptr;
  FlatTable ft;
  const uint64_t ns = D >= 2 ? binom_u64((uint64_t)n, D - 1) : 1;
  if (ns == 0 || ns > (4u << 20)) { cache[key] = ft; return nullptr; }
  std::vector<uint32_t> start((size_t)ns);
  uint64_t acc = 0;
  // chunk size: 1024, or smaller (multiple of 32, >= 128) so that the dimension's
  // candidates C(n, D+1) still give ~24 warps per SM
  {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t total = binom_u64((uint64_t)n, D + 1);
    uint64_t wps = 24;  // target warps per SM (VR_FL_WARPS overrides, for tuning runs)
    if (const char* e = std::getenv("VR_FL_WARPS")) wps = std::max<uint64_t>(1, (uint64_t)std::atoll(e));
    uint64_t c = total / ((uint64_t)sms * wps);
    c = (c + 31) / 32 * 32;
    uint64_t cap = FL_CHUNK;
    if (const char* e = std::getenv("VR_FL_CHUNK")) cap = std::max<uint64_t>(128, (uint64_t)std::atoll(e) / 32 * 32);
    ft.chunk = (int)std::max<uint64_t>(128, std::min<uint64_t>(cap, c));
  }
  const uint64_t CH = (uint64_t)ft.chunk;
  // walk the (D-1)-subsets in colex order; u_2 = the smallest element
  std::vector<int> sub((size_t)std::max(D - 1, 0));
  for (int k = 0; k < D - 1; ++k) sub[(size_t)k] = k;  // ascending: sub[0] = u_2
  for (uint64_t t = 0; t < ns; ++t) {
    start[(size_t)t] = (uint32_t)acc;
    const uint64_t u2 = D >= 2 ? (uint64_t)sub[0] : (uint64_t)n;
    const uint64_t cnt = u2 * (u2 >= 1 ? u2 - 1 : 0) / 2;
    acc += (cnt + CH - 1) / CH;
    if (acc >= (1ull << 31)) { cache[key] = ft; return nullptr; }
    // colex successor
    for (int k = 0; k < D - 1; ++k) {
      if (k + 1 < D - 1 && sub[(size_t)k] + 1 == sub[(size_t)k + 1]) { sub[(size_t)k] = k; continue; }
      ++sub[(size_t)k];
      break;
    }
  }
  if (cudaMalloc(&ft.d_start, (size_t)ns * 4) != cudaSuccess) { cudaGetLastError(); cache[key] = FlatTable{}; return nullptr; }
  cudaMemcpy(ft.d_start, start.data(), (size_t)ns * 4, cudaMemcpyHostToDevice);
  ft.nsuper = (uint32_t)ns;
  ft.nchunks = (uint32_t)acc;
  cache[key] = ft;
  return &cache[key];
}

template <int D>
static int enumerate_d(const DimParams& p, const Tables& T, const HotBuffers& B, cudaStream_t st) {
  const uint64_t rows = p.row_end - p.row_begin;
  const uint64_t warps_needed = (rows + (uint64_t)p.grab - 1) / (uint64_t)p.grab;
  uint64_t blocks = (warps_needed * 32 + HP_THREADS - 1) / HP_THREADS;
  const uint64_t cap = (uint64_t)sm_count() * 8;  // 8 resident CTAs of 256 threads per SM
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  DimParams q = p;
  size_t smem = 0;
  if (q.variant == 1 && q.n >= 32 && q.n <= kWinMaxN) {
    q.win = 1;
    smem = (size_t)q.n * 36 * 4 + (HP_THREADS / 32) * 32 * 4;
    device_memo((const void*)k_enumerate<D>, [] {  // per instantiation and device
      return (int)cudaFuncSetAttribute(k_enumerate<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(kWinMaxN * 36 * 4 + 1024));
    });
  } else {
    q.win = 0;
  }
  // flattened chunks from d = 2 on (measured: equal on c2, -8% on c4a), and from d = 1 when
  // n >= 128 (one super-row of n long rows: -3.5% on c4a, -0.3% on c2; +2.5% on c1, n = 64,
  // where the row kernel stays); VR_FLAT_MIN_D overrides
  static const int flat_min_env = std::getenv("VR_FLAT_MIN_D") ? std::atoi(std::getenv("VR_FLAT_MIN_D")) : -1;
  const int flat_min_d = flat_min_env >= 0 ? flat_min_env : (q.n >= 128 ? 1 : 2);
  if (D >= flat_min_d && q.win && q.variant == 1 && q.row_begin == 0 &&
      q.row_end == binom_u64((uint64_t)q.n, D) && !getenv_flag("VR_NO_FLAT")) {
    const FlatTable* ft = flat_table(q.n, D);
    if (ft) {
      device_memo((const void*)k_enumerate_flat<D>, [] {
        return (int)cudaFuncSetAttribute(k_enumerate_flat<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(kWinMaxN * 36 * 4 + 1024));
      });
      const uint64_t warps = (ft->nchunks + (uint64_t)q.shard_world - 1) / (uint64_t)q.shard_world;
      uint64_t fb = (warps * 32 + HP_THREADS - 1) / HP_THREADS;
      if (fb > cap) fb = cap;
      if (fb < 1) fb = 1;
      k_enumerate_flat<D><<<(unsigned)fb, HP_THREADS, smem, st>>>(T, q, B, ft->d_start, ft->nsuper, ft->nchunks, ft->chunk);
      return VR_KERNEL_FLAT | VR_KERNEL_SMEM_WINDOW;
    }
  }
  k_enumerate<D><<<(unsigned)blocks, HP_THREADS, smem, st>>>(T, q, B);
  return VR_KERNEL_ROW | (q.win ? VR_KERNEL_SMEM_WINDOW : 0);
}

template <int D>
static void resolve_d(const DimParams& p, const Tables& T, const HotBuffers& B, uint64_t qn, cudaStream_t st) {
  uint64_t blocks = (qn * 32 + HP_THREADS - 1) / HP_THREADS;
  const uint64_t cap = (uint64_t)sm_count() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  k_resolve<D><<<(unsigned)blocks, HP_THREADS, 0, st>>>(T, p, B, qn);
}

int launch_enumerate(const DimParams& p, const uint32_t* rank, const uint64_t* binom, int kmax, const HotBuffers& B,
                     cudaStream_t st, int64_t* launches) {
  Tables T{rank, binom, (int32_t)p.n, kmax};
  int k = 0;
  switch (p.d) {
    case 1: k = enumerate_d<1>(p, T, B, st); break;
    case 2: k = enumerate_d<2>(p, T, B, st); break;
    case 3: k = enumerate_d<3>(p, T, B, st); break;
    case 4: k = enumerate_d<4>(p, T, B, st); break;
    case 5: k = enumerate_d<5>(p, T, B, st); break;
    case 6: k = enumerate_d<6>(p, T, B, st); break;
    default: return 0;
  }
  *launches += 1;
  return k;
}

void launch_resolve(const DimParams& p, const uint32_t* rank, const uint64_t* binom, int kmax, const HotBuffers& B,
                    uint64_t qn, cudaStream_t st, int64_t* launches) {
  if (qn == 0) return;
  Tables T{rank, binom, (int32_t)p.n, kmax};
  switch (p.d) {
    case 1: resolve_d<1>(p, T, B, qn, st); break;
    case 2: resolve_d<2>(p, T, B, qn, st); break;
    case 3: resolve_d<3>(p, T, B, qn, st); break;
    case 4: resolve_d<4>(p, T, B, qn, st); break;
    case 5: resolve_d<5>(p, T, B, qn, st); break;
    case 6: resolve_d<6>(p, T, B, qn, st); break;
    default: return;
  }
  *launches += 1;
}

void launch_set_bits(const uint64_t* list, int64_t m, uint32_t* bm, cudaStream_t st, int64_t* launches) {
  if (m <= 0) return;
  const int64_t blocks = std::min<int64_t>((m + 255) / 256, (int64_t)sm_count() * 8);
  k_set_bits<<<(unsigned)blocks, 256, 0, st>>>(list, m, bm);
  *launches += 1;
}

}  // namespace vr
