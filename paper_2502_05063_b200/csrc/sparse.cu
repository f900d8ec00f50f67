// sparse.cu — the output-sensitive ("sparse") hot path for thresholds far below the
// enclosing radius (config 5: t = 1.4, ~2.8% of the edges), SURVEY.md §8(a) a1 "output-
// sensitive" and §8(f) NEXT-2; §5.3.12-5.3.13 (sparse 1-skeleton, Alg 15) and
// P:5967 (Ripser++ switched o3 to its sparse mode).
//
// Threshold graph G_t: vertex v's neighbours w (R[v][w] != RINF, w != v), stored in CSR
// with every list sorted DEScending.  Every d-simplex is produced exactly once as
// (u_D > ... > u_1) ∪ {v_0} where the prefix is a (d-1)-simplex with diam <= t (a
// survivor of dimension d-1, written by that dimension's kernel) and v_0 < u_1 is a
// neighbour of u_1 (reading A33: Alg 15's goto structure is not followed literally; this
// is the same candidate set by neighbour-list intersection).  The Lemma 5.3.6 scans only
// visit neighbours of u_1, in descending order: a cofacet s ∪ {v} with diam = diam(s) <= t
// needs v adjacent to every vertex of s (reading A32), so the first hit among them is the
// lex-greatest equal-diameter cofacet.  The per-lane logic is otherwise k_enumerate /
// k_resolve's (hotpath.cu).
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "vr_common.cuh"
#include "vr_internal.h"

namespace vr {

constexpr int SP_THREADS = 256;

// ------------------------------------------------------------------ adjacency (warp per row)
__global__ void k_adj_count(const uint32_t* __restrict__ rank, int n, uint32_t* __restrict__ deg,
                            uint32_t* __restrict__ deg_below) {
  const int lane = threadIdx.x & 31;
  const int v = (int)(((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (v >= n) return;
  const uint32_t* row = rank + (size_t)v * (size_t)n;
  uint32_t c = 0, cb = 0;
  for (int w = lane; w < n; w += 32) {
    const bool e = (w != v) && __ldg(row + w) != VR_RINF;
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

__global__ void k_adj_fill(const uint32_t* __restrict__ rank, int n, const uint32_t* __restrict__ off,
                           uint16_t* __restrict__ adj) {
  const int lane = threadIdx.x & 31;
  const int v = (int)(((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (v >= n) return;
  const uint32_t* row = rank + (size_t)v * (size_t)n;
  uint32_t pos = off[v];
  for (int base = n - 1; base >= 0; base -= 32) {  // descending neighbour order
    const int w = base - lane;
    const bool e = w >= 0 && w != v && __ldg(row + w) != VR_RINF;
    const uint32_t m = __ballot_sync(0xffffffffu, e);
    if (e) adj[pos + __popc(m & lanemask_lt())] = (uint16_t)w;
    pos += __popc(m);
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

// ------------------------------------------------------------------ phase 1
template <int D>
__device__ __forceinline__ void sparse_row(const Tables& T, const DimParams& p, const HotBuffers& B, const SparseRows& S,
                                           const int (&u)[D + 2], unsigned long long& surv_acc, unsigned long long& app_acc,
                                           unsigned long long& scan_acc, unsigned long long& clr_acc) {
  const int lane = threadIdx.x & 31;
  const int u1 = u[1];
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
  if (pm_up == VR_RINF) return;
  uint64_t cbase = 0;
#pragma unroll
  for (int i = 1; i <= D; ++i) cbase += binom(T, u[i], i + 1);
  const uint16_t* __restrict__ L = S.adj + __ldg(S.adj_off + u1);
  const int deg = (int)(__ldg(S.adj_off + u1 + 1) - __ldg(S.adj_off + u1));
  // first neighbour below u_1 (L is descending): after the deg - deg_below(u_1) above it
  int k0 = 0;
  if (S.deg_below) {
    k0 = deg - (int)__ldg(S.deg_below + u1);
  } else {
    int lo = 0, hi = deg;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((int)__ldg(L + mid) > u1) lo = mid + 1; else hi = mid;
    }
    k0 = lo;
  }
  if (k0 >= deg) return;
  // window: lane j holds neighbour L[j] and max_i R[u_i][L[j]] (RINF for a prefix vertex)
  int vwin = -1;
  uint32_t mwin = VR_RINF;
  if (lane < deg) {
    vwin = (int)__ldg(L + lane);
    uint32_t m = 0;
#pragma unroll
    for (int i = 1; i <= D; ++i) m = (vwin == u[i]) ? VR_RINF : umax(m, rank_at(T, u[i], vwin));
    mwin = m;
  }
  const int steps = p.steps < deg ? p.steps : deg;

  for (int base = k0; base < deg; base += 32) {
    const int idx = base + lane;
    const bool valid = idx < deg;
    const int v0 = valid ? (int)__ldg(L + idx) : 0;
    uint32_t a[D + 1];
    uint32_t rs = pm_up;
#pragma unroll
    for (int i = 1; i <= D; ++i) {
      a[i] = valid ? rank_at(T, u[i], v0) : VR_RINF;
      rs = umax(rs, a[i]);
    }
    const bool surv = valid && rs != VR_RINF;
    const uint32_t msurv = __ballot_sync(0xffffffffu, surv);
    if (!msurv) continue;
    surv_acc += __popc(msurv);
    int s[D + 1];
#pragma unroll
    for (int i = 0; i < D; ++i) s[i] = u[D - i];
    s[D] = v0;
    if (S.rows_out) {  // every survivor is a prefix row of dimension d+1
      const unsigned long long slot = warp_append(surv, S.rows_out_count);
      if (surv && slot < S.rows_out_cap) S.rows_out[slot] = pack_vertices<D>(s);
    }
    const uint64_t cidx = cbase + (uint64_t)v0;
    bool cleared = false;
    if (B.clr && surv) cleared = bit_test(B.clr, cidx);
    else if (B.clr_hash && surv) cleared = hash_has(B.clr_hash, B.clr_hash_mask, cidx);
    clr_acc += __popc(__ballot_sync(0xffffffffu, cleared));
    bool active = surv && !cleared;
    int hitv = -1, examined = 0;
    for (int j = 0; j < steps; ++j) {
      if (!__any_sync(0xffffffffu, active)) break;
      int v;
      uint32_t m;
      if (j < 32) {
        v = __shfl_sync(0xffffffffu, vwin, j);
        m = __shfl_sync(0xffffffffu, mwin, j);
      } else {
        v = (int)__ldg(L + j);
        m = 0;
#pragma unroll
        for (int i = 1; i <= D; ++i) m = (v == u[i]) ? VR_RINF : umax(m, rank_at(T, u[i], v));
      }
      examined += active;
      if (active && m <= rs && v != v0 && umax(m, rank_at(T, v, v0)) <= rs) {
        hitv = v;
        active = false;
      }
    }
    scan_acc += (unsigned long long)__reduce_add_sync(0xffffffffu, (unsigned)examined);
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
      const uint32_t b0 = rank_at(T, hitv, v0);
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
    const uint64_t key = ((uint64_t)(p.maxr - rs) << p.cbits) | cidx;
    const bool clrmode = B.clr || B.clr_hash;  // clearing decided above (else in phase 2)
    const bool to_resid = clrmode && hitv >= 0 && !app;
    const bool to_queue = active || (!clrmode && hitv >= 0 && !app);
    const unsigned long long rslot = warp_append(to_resid, &B.ctr->residual);
    if (to_resid && rslot < B.rcap) B.resid[rslot] = key;
    const unsigned long long qslot = warp_append(to_queue, &B.ctr->queued);
    if (to_queue && qslot < B.qcap) {
      B.qkey[qslot] = key;
      B.qvert[qslot] = pack_vertices<D>(s);
    }
  }
}

template <int D>
__global__ void __launch_bounds__(SP_THREADS, 8) k_enum_sparse(Tables T, DimParams p, HotBuffers B, SparseRows S) {
  const int lane = threadIdx.x & 31;
  unsigned long long surv_acc = 0, app_acc = 0, scan_acc = 0, clr_acc = 0;
  const uint64_t W = (uint64_t)p.shard_world;
  const uint64_t all = p.row_end - p.row_begin;
  const uint64_t nrows = all > (uint64_t)p.shard_rank ? (all - (uint64_t)p.shard_rank + W - 1) / W : 0;  // this shard's rows
  while (true) {
    unsigned long long g = 0;
    if (lane == 0) g = atomicAdd(&B.ctr->row_next, 1ull);
    g = __shfl_sync(0xffffffffu, g, 0);
    if (g >= nrows) break;
    const uint64_t r = p.row_begin + g * W + (uint64_t)p.shard_rank;
    int u[D + 2];
    if (S.rows_in == nullptr) {  // dimension 1: the rows are the vertices
      u[1] = (int)r;
    } else {                    // the (D-1)-simplex t[0] > ... > t[D-1]: u_i = t[D-i]
      int t[D];
      const uint4 pk = S.rows_in[r];
      const uint32_t w[4] = {pk.x, pk.y, pk.z, pk.w};
#pragma unroll
      for (int i = 0; i < D; ++i) t[i] = (int)((w[i >> 1] >> ((i & 1) * 16)) & 0xFFFFu);
#pragma unroll
      for (int i = 1; i <= D; ++i) u[i] = t[D - i];
    }
    u[0] = 0;
    u[D + 1] = T.n;
    sparse_row<D>(T, p, B, S, u, surv_acc, app_acc, scan_acc, clr_acc);
  }
  if (lane == 0) {
    if (surv_acc) atomicAdd(&B.ctr->survivors, surv_acc);
    if (app_acc) atomicAdd(&B.ctr->apparent1, app_acc);
    if (scan_acc) atomicAdd(&B.ctr->scanned, scan_acc);
    if (clr_acc) atomicAdd(&B.ctr->cleared, clr_acc);
  }
}

// ------------------------------------------------------------------ phase 2
// First neighbour v of `anchor` at list position >= start (descending) with v not in S and
// max_{w in S} R[w][v] <= r, or -1.  32 neighbours per step.
template <int K>
__device__ __forceinline__ int coop_scan_nbr(const Tables& T, const SparseRows& SR, const int (&S)[K], int anchor, uint32_t r,
                                             int start, unsigned long long& scan_acc) {
  const int lane = threadIdx.x & 31;
  const uint16_t* __restrict__ L = SR.adj + __ldg(SR.adj_off + anchor);
  const int deg = (int)(__ldg(SR.adj_off + anchor + 1) - __ldg(SR.adj_off + anchor));
  for (int base = start; base < deg; base += 32) {
    const int idx = base + lane;
    scan_acc += (unsigned long long)(deg - base < 32 ? deg - base : 32);
    bool ok = idx < deg;
    const int v = ok ? (int)__ldg(L + idx) : -1;
    uint32_t rt = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (ok) {
        if (v == S[k]) ok = false;
        else rt = umax(rt, rank_at(T, S[k], v));
      }
    }
    const uint32_t m = __ballot_sync(0xffffffffu, ok && rt <= r);
    if (m) return __shfl_sync(0xffffffffu, v, __ffs(m) - 1);
  }
  return -1;
}

template <int D>
__global__ void __launch_bounds__(SP_THREADS) k_resolve_sparse(Tables T, DimParams p, HotBuffers B, SparseRows SR, uint64_t qn) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t cmask = p.cbits >= 64 ? ~0ull : ((1ull << p.cbits) - 1);
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
    const int anchor = s[D - 1];  // u_1: the list phase 1 walked
    const bool clrmode = B.clr || B.clr_hash;
    const int v = coop_scan_nbr<D + 1>(T, SR, s, anchor, rs, clrmode ? p.steps : 0, scan_acc);
    bool app = false;
    if (v >= 0) {
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
      if (lane == 0 && (B.clr_next || B.clr_next_hash || B.app_pairs)) {
        const uint64_t tc = cofacet_cidx<D>(T, s, v);
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
      continue;
    }
    if (!clrmode) {
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
          cleared = coop_scan_nbr<D>(T, SR, f, f[D - 1], rs, 0, scan_acc) == w;
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

__global__ void k_hash_put(const uint64_t* __restrict__ list, int64_t m, uint64_t* __restrict__ t, uint64_t mask) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    hash_put(t, mask, __ldg(list + i));
}

// ------------------------------------------------------------------ launchers
static int sp_sms() {
  static int s = 0;
  if (!s) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
    if (s <= 0) s = 148;
  }
  return s;
}

void launch_adjacency(const uint32_t* rank, int n, uint32_t* deg, uint32_t* deg_below, uint32_t* off, uint16_t* adj,
                      void* scan_tmp, cudaStream_t st, int64_t* launches) {
  const unsigned blocks = (unsigned)(((uint64_t)n * 32 + SP_THREADS - 1) / SP_THREADS);
  k_adj_count<<<blocks, SP_THREADS, 0, st>>>(rank, n, deg, deg_below);
  exclusive_scan_u32(deg, off, (size_t)n + 1, scan_tmp, st, launches);  // deg[n] = 0
  k_adj_fill<<<blocks, SP_THREADS, 0, st>>>(rank, n, off, adj);
  *launches += 2;
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
  const uint64_t cap = (uint64_t)sp_sms() * 8;
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

}  // namespace vr

namespace vr {
void launch_hash_put(const uint64_t* list, int64_t m, uint64_t* table, uint64_t mask, cudaStream_t st, int64_t* launches) {
  if (m <= 0) return;
  const int64_t blocks = std::min<int64_t>((m + 255) / 256, 148 * 8);
  k_hash_put<<<(unsigned)blocks, 256, 0, st>>>(list, m, table, mask);
  if (launches) *launches += 1;
}
}  // namespace vr
