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
//   k_enumerate<D>  (a1 + a5 phase 1 + a3)
//       one warp per "row" = a fixed upper-vertex prefix (v_D > ... > v_1); the 32 lanes
//       take consecutive v_0, so the d-simplices of a row have consecutive cidx (Eq 5.6)
//       and every distance read R[v_i][v_0] is a coalesced row segment.  Per lane:
//       diameter rank = max pairwise rank, threshold (diam <= t, inclusive), then the
//       Lemma 5.3.6 scan over cofacet vertices v = n-1, n-2, ... (lex-decreasing
//       cofacets, Alg 14) for at most `steps` candidates, all lanes in lock-step on the
//       same v (broadcast loads of R[v][v_i], one coalesced load of R[v][v_0]).  Lanes
//       proven apparent are counted; every other survivor is appended (warp-aggregated,
//       §5.5.3) to the queue.
//
//   k_resolve<D>    (a5 phase 2 + a2 + a6)
//       one warp per queued column: the full Lemma 5.3.6 test with the 32 lanes testing
//       32 cofacet vertices per step (ballot, the lowest set lane = the lex-greatest
//       equal-diameter cofacet); then clearing for non-apparent columns (the column is a
//       death of dimension d-1: in the sorted residual-death list, or the apparent
//       cofacet of its youngest facet, recomputed); survivors are the residual columns.
#include <cstdint>
#include <cuda_runtime.h>

#include "vr_common.cuh"
#include "vr_internal.h"

namespace vr {

constexpr int HP_THREADS = 256;

__device__ __forceinline__ uint32_t umax(uint32_t a, uint32_t b) { return a > b ? a : b; }

// ------------------------------------------------------------------ phase 1: enumerate
template <int D>
__device__ __forceinline__ void process_row(const Tables& T, const DimParams& p, const int (&u)[D + 2], uint64_t* queue,
                                            uint64_t qcap, DimCounters* ctr, uint64_t* app_pairs, uint64_t app_cap,
                                            unsigned long long& surv_acc, unsigned long long& app_acc,
                                            unsigned long long& scan_acc) {
  const int lane = threadIdx.x & 31;
  const int n = T.n;
  const int v1 = u[1];
  if (v1 == 0) return;  // no v_0 < v_1
  // prefix pair maxima: pm_up over all prefix pairs, pm_ex[j] over pairs avoiding u[j]
  uint32_t pm_up = 0;
  uint32_t pm_ex[D + 1];
#pragma unroll
  for (int j = 0; j <= D; ++j) pm_ex[j] = 0;
#pragma unroll
  for (int a = 1; a <= D; ++a)
#pragma unroll
    for (int b = a + 1; b <= D; ++b) {
      const uint32_t r = rank_at(T, u[a], u[b]);
      pm_up = umax(pm_up, r);
#pragma unroll
      for (int j = 1; j <= D; ++j)
        if (j != a && j != b) pm_ex[j] = umax(pm_ex[j], r);
    }
  if (pm_up == VR_RINF) return;  // every simplex of the row is over the threshold
  uint64_t cbase = 0;
#pragma unroll
  for (int i = 1; i <= D; ++i) cbase += binom(T, u[i], i + 1);

  for (int base = 0; base < v1; base += 32) {
    const int v0 = base + lane;
    const bool valid = v0 < v1;
    uint32_t a[D + 1];
    uint32_t rs = pm_up;
#pragma unroll
    for (int i = 1; i <= D; ++i) {
      a[i] = valid ? rank_at(T, u[i], v0) : VR_RINF;
      rs = umax(rs, a[i]);
    }
    const bool surv = valid && rs != VR_RINF;  // diam(s) <= t (Eq 5.3, Alg 17 line 3)
    const uint32_t msurv = __ballot_sync(0xffffffffu, surv);
    if (!msurv) continue;
    surv_acc += __popc(msurv);
    // diameter of s \ {w} for each vertex w of s
    uint32_t ex[D + 1];
    ex[0] = pm_up;  // w = v_0
#pragma unroll
    for (int j = 1; j <= D; ++j) {
      uint32_t m = pm_ex[j];
#pragma unroll
      for (int i = 1; i <= D; ++i)
        if (i != j) m = umax(m, a[i]);
      ex[j] = m;
    }
    // Lemma 5.3.6, lane-parallel, at most p.steps cofacet vertices
    int state = surv ? 0 : 3;  // 0 scanning, 1 apparent, 2 not apparent, 3 idle
    int hitv = -1;
    int v = n - 1;
    for (int step = 0; step < p.steps; ++step) {
      const uint32_t mact = __ballot_sync(0xffffffffu, state == 0);
      if (!mact) break;
      bool up = true;
      while (up) {  // skip the prefix vertices (warp-uniform)
        up = false;
#pragma unroll
        for (int i = 1; i <= D; ++i) up |= (v == u[i]);
        if (up) --v;
      }
      if (v < 0) break;
      scan_acc += __popc(mact);
      uint32_t b[D + 1];
      uint32_t bup = 0;
#pragma unroll
      for (int i = 1; i <= D; ++i) {
        b[i] = rank_at(T, v, u[i]);
        bup = umax(bup, b[i]);
      }
      const uint32_t b0 = (state == 0) ? rank_at(T, v, v0) : VR_RINF;
      // t = s ∪ {v} has diam(t) = diam(s) iff every new edge is <= diam(s)
      if (state == 0 && v != v0 && umax(bup, b0) <= rs) {
        // condition 2: no facet t \ {w}, w > v (smaller cidx), with diam = diam(s)
        bool app = true;
        if (v0 > v && umax(ex[0], bup) == rs) app = false;
#pragma unroll
        for (int j = 1; j <= D; ++j) {
          if (u[j] > v) {
            uint32_t m = umax(ex[j], b0);
#pragma unroll
            for (int i = 1; i <= D; ++i)
              if (i != j) m = umax(m, b[i]);
            if (m == rs) app = false;
          }
        }
        state = app ? 1 : 2;
        hitv = v;
      }
      --v;
    }
    const uint32_t mapp = __ballot_sync(0xffffffffu, state == 1);
    app_acc += __popc(mapp);
    if (app_pairs) {
      unsigned long long slot = warp_append(state == 1, &ctr->app_pairs);
      if (state == 1 && slot < app_cap) {
        int s[D + 1];
#pragma unroll
        for (int i = 0; i < D; ++i) s[i] = u[D - i];
        s[D] = v0;
        app_pairs[2 * slot] = cbase + (uint64_t)v0;
        app_pairs[2 * slot + 1] = cofacet_cidx<D>(T, s, hitv);
      }
    }
    const bool q = surv && state != 1;
    const unsigned long long slot = warp_append(q, &ctr->queued);
    if (q && slot < qcap) queue[slot] = ((uint64_t)(p.maxr - rs) << p.cbits) | (cbase + (uint64_t)v0);
  }
}

template <int D>
__global__ void __launch_bounds__(HP_THREADS) k_enumerate(Tables T, DimParams p, uint64_t* __restrict__ queue, uint64_t qcap,
                                                          DimCounters* __restrict__ ctr, uint64_t* __restrict__ app_pairs,
                                                          uint64_t app_cap) {
  constexpr int GRAB = 4;
  const int lane = threadIdx.x & 31;
  unsigned long long surv_acc = 0, app_acc = 0, scan_acc = 0;
  while (true) {
    unsigned long long r0 = 0;
    if (lane == 0) r0 = atomicAdd(&ctr->row_next, (unsigned long long)GRAB);
    r0 = __shfl_sync(0xffffffffu, r0, 0) + p.row_begin;
    if (r0 >= p.row_end) break;
    const uint64_t rend = (r0 + GRAB < p.row_end) ? r0 + GRAB : p.row_end;
    // decode prefix row r0 (colex rank of {u_D > ... > u_1}: r = sum_i C(u_i, i))
    int u[D + 2];
    {
      uint64_t x = r0;
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
    for (uint64_t r = r0; r < rend; ++r) {
      if (r > r0) {  // colex successor of the prefix
        bool carry = true;
#pragma unroll
        for (int i = 1; i <= D; ++i) {
          if (carry) {
            if (i == D || u[i] + 1 < u[i + 1]) { u[i] += 1; carry = false; }
            else u[i] = i - 1;
          }
        }
      }
      process_row<D>(T, p, u, queue, qcap, ctr, app_pairs, app_cap, surv_acc, app_acc, scan_acc);
    }
  }
  if (lane == 0) {
    if (surv_acc) atomicAdd(&ctr->survivors, surv_acc);
    if (app_acc) atomicAdd(&ctr->apparent1, app_acc);
    if (scan_acc) atomicAdd(&ctr->scanned, scan_acc);
  }
}

// ------------------------------------------------------------------ phase 2: resolve
// First v (descending from n-1) not in S with max_{w in S} R[w][v] <= r, or -1.
// Lanes take v = base - lane: each load R[w][v] is a coalesced row segment.
template <int K>
__device__ __forceinline__ int coop_scan(const Tables& T, const int (&S)[K], uint32_t r, unsigned long long& scan_acc) {
  const int lane = threadIdx.x & 31;
  for (int base = T.n - 1; base >= 0; base -= 32) {
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
__global__ void __launch_bounds__(HP_THREADS) k_resolve(Tables T, DimParams p, const uint64_t* __restrict__ queue, uint64_t qn,
                                                        const uint64_t* __restrict__ deaths, int64_t ndeaths,
                                                        uint64_t* __restrict__ resid, uint64_t rcap,
                                                        DimCounters* __restrict__ ctr, uint64_t* __restrict__ app_pairs,
                                                        uint64_t app_cap) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t cmask = p.cbits >= 64 ? ~0ull : ((1ull << p.cbits) - 1);
  unsigned long long app_acc = 0, clr_acc = 0, scan_acc = 0;
  for (uint64_t e = warp; e < qn; e += nwarps) {
    const uint64_t key = __ldg(queue + e);
    const uint32_t rs = p.maxr - (uint32_t)(key >> p.cbits);
    const uint64_t cidx = key & cmask;
    int s[D + 1];
    cns_decode<D>(T, cidx, s);
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
    // Lemma 5.3.6 condition 1: the lex-greatest cofacet with diam(t) = diam(s)
    const int v = coop_scan<D + 1>(T, s, rs, scan_acc);
    bool app = false;
    if (v >= 0) {
      // condition 2: no facet t \ {w}, w > v, with diam = diam(s)
      app = true;
#pragma unroll
      for (int j = 0; j <= D; ++j) {
        if (s[j] > v) {
          uint32_t m = ex[j];
#pragma unroll
          for (int i = 0; i <= D; ++i)
            if (i != j) m = umax(m, rank_at(T, v, s[i]));
          if (m == rs) app = false;
        }
      }
    }
    if (app) {
      ++app_acc;
      if (app_pairs && lane == 0) {
        unsigned long long slot = atomicAdd(&ctr->app_pairs, 1ull);
        if (slot < app_cap) {
          app_pairs[2 * slot] = cidx;
          app_pairs[2 * slot + 1] = cofacet_cidx<D>(T, s, v);
        }
      }
      continue;
    }
    // clearing (§5.2.3, Lemma 4.2.3): s is cleared iff it is the death of a pair of
    // dimension d-1 — a residual pair (sorted list) or an apparent pair, recomputed:
    // s is the apparent cofacet of its youngest facet f (the first facet in Alg 16
    // order — removing s[0], s[1], ... — with diam(f) = diam(s)) iff the lex-greatest
    // equal-diameter cofacet of f is s itself.
    bool cleared = sorted_contains(deaths, ndeaths, cidx);
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
          int x = s[j];
          if (j == js) w = x;
          else f[j < js ? j : j - 1] = x;
        }
        cleared = coop_scan<D>(T, f, rs, scan_acc) == w;
      }
    }
    if (cleared) {
      ++clr_acc;
      continue;
    }
    if (lane == 0) {
      const unsigned long long slot = atomicAdd(&ctr->residual, 1ull);
      if (slot < rcap) resid[slot] = key;
    }
  }
  if (lane == 0) {
    if (app_acc) atomicAdd(&ctr->apparent2, app_acc);
    if (clr_acc) atomicAdd(&ctr->cleared, clr_acc);
    if (scan_acc) atomicAdd(&ctr->scanned2, scan_acc);
  }
}

// ------------------------------------------------------------------ launchers
static int g_sms = 0;
static int sm_count() {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}

template <int D>
static void enumerate_d(const DimParams& p, const Tables& T, uint64_t* queue, uint64_t qcap, DimCounters* ctr,
                        uint64_t* app_pairs, uint64_t app_cap, cudaStream_t st) {
  const uint64_t rows = p.row_end - p.row_begin;
  const uint64_t warps_needed = (rows + 3) / 4;
  uint64_t blocks = (warps_needed * 32 + HP_THREADS - 1) / HP_THREADS;
  const uint64_t cap = (uint64_t)sm_count() * 8;  // 8 resident CTAs of 256 threads per SM
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  k_enumerate<D><<<(unsigned)blocks, HP_THREADS, 0, st>>>(T, p, queue, qcap, ctr, app_pairs, app_cap);
}

template <int D>
static void resolve_d(const DimParams& p, const Tables& T, const uint64_t* queue, uint64_t qn, const uint64_t* deaths,
                      int64_t ndeaths, uint64_t* resid, uint64_t rcap, DimCounters* ctr, uint64_t* app_pairs,
                      uint64_t app_cap, cudaStream_t st) {
  uint64_t blocks = (qn * 32 + HP_THREADS - 1) / HP_THREADS;
  const uint64_t cap = (uint64_t)sm_count() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  k_resolve<D><<<(unsigned)blocks, HP_THREADS, 0, st>>>(T, p, queue, qn, deaths, ndeaths, resid, rcap, ctr, app_pairs,
                                                         app_cap);
}

void launch_enumerate(const DimParams& p, const uint32_t* rank, const uint64_t* binom, int kmax, uint64_t* queue,
                      uint64_t qcap, DimCounters* ctr, uint64_t* app_pairs, uint64_t app_cap, cudaStream_t st,
                      int64_t* launches) {
  Tables T{rank, binom, (int32_t)p.n, kmax};
  switch (p.d) {
    case 1: enumerate_d<1>(p, T, queue, qcap, ctr, app_pairs, app_cap, st); break;
    case 2: enumerate_d<2>(p, T, queue, qcap, ctr, app_pairs, app_cap, st); break;
    case 3: enumerate_d<3>(p, T, queue, qcap, ctr, app_pairs, app_cap, st); break;
    case 4: enumerate_d<4>(p, T, queue, qcap, ctr, app_pairs, app_cap, st); break;
    case 5: enumerate_d<5>(p, T, queue, qcap, ctr, app_pairs, app_cap, st); break;
    case 6: enumerate_d<6>(p, T, queue, qcap, ctr, app_pairs, app_cap, st); break;
    default: return;
  }
  *launches += 1;
}

void launch_resolve(const DimParams& p, const uint32_t* rank, const uint64_t* binom, int kmax, const uint64_t* queue,
                    uint64_t qn, const uint64_t* deaths, int64_t ndeaths, uint64_t* resid, uint64_t rcap,
                    DimCounters* ctr, uint64_t* app_pairs, uint64_t app_cap, cudaStream_t st, int64_t* launches) {
  if (qn == 0) return;
  Tables T{rank, binom, (int32_t)p.n, kmax};
  switch (p.d) {
    case 1: resolve_d<1>(p, T, queue, qn, deaths, ndeaths, resid, rcap, ctr, app_pairs, app_cap, st); break;
    case 2: resolve_d<2>(p, T, queue, qn, deaths, ndeaths, resid, rcap, ctr, app_pairs, app_cap, st); break;
    case 3: resolve_d<3>(p, T, queue, qn, deaths, ndeaths, resid, rcap, ctr, app_pairs, app_cap, st); break;
    case 4: resolve_d<4>(p, T, queue, qn, deaths, ndeaths, resid, rcap, ctr, app_pairs, app_cap, st); break;
    case 5: resolve_d<5>(p, T, queue, qn, deaths, ndeaths, resid, rcap, ctr, app_pairs, app_cap, st); break;
    case 6: resolve_d<6>(p, T, queue, qn, deaths, ndeaths, resid, rcap, ctr, app_pairs, app_cap, st); break;
    default: return;
  }
  *launches += 1;
}

}  // namespace vr
