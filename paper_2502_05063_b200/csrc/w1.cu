// w1.cu — PDoptFlow (PAPER.md Ch.6, Alg 22): the (1+O(ε))-approximate 1-Wasserstein
// distance between persistence diagrams as a min-cost flow on a sparsified network.
// SURVEY.md §8(f) NEXT-4.
//
//   stage               where   paper
//   RWMD lower bound    GPU     Alg 20: brute-force nearest neighbours, fp64, one
//                               thread per point, the other diagram streamed through shared
//                               memory in tiles (O(nA nB) work — a few ms at 1e5 x 1e5)
//   δ-condensation      GPU     Alg 21: ε = 8/(s-4) (s >= 12) else 1,
//                               δ = 2εL/(√2 (|A|+|B|)), snap to the kδ-grid (k = 0.99), one
//                               node per occupied cell (hash table, atomic supply/flags),
//                               nodes ordered by cell key (radix sort), then a seeded random
//                               shift of at most (1-k)δ/2 per axis
//   0-condensation      GPU the same table keyed by the exact fp32 bits when
//                               condensation is off
//   split tree          host    §6.3.5: fair split of the bounding box's longer side
//   s-WSPD              GPU     Algs 23-25: one thread per internal node,
//                               count -> exclusive scan -> write, leftmost representatives
//                               ([170])
//   diagonal arcs       GPU     Alg 26: p -> ā for A-nodes, b̄ -> q for B-nodes, b̄ -> ā
//   arc sort (CSR)      GPU     §6.9.3: 64-bit keys (tail << 32 | head), our radix sort
//   min-cost flow       host    §6.3.7: netsimplex.cpp (block search)
//
// Readings: |A|, |B| in δ count points with multiplicity (the proof of
// Prop 6.3.2 counts matched and unmatched points); the diagonal arcs run Â -> ā and
// b̄ -> B̂ plus b̄ -> ā at cost 0 (Eq 6.37 and the proof of Thm 6.3.6, P:6616-6620 — the
// "arcs from Â^δ to b̄" wording of P:6662 is read as a garble); an A-point and a B-point
// in the same cell form one node with the net supply.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/vr.h"
#include "vr_common.cuh"
#include "vr_internal.h"

namespace vr {

namespace {

constexpr double kSnap = 0.99;  // k of Alg 21 (the grid is kδ)
constexpr unsigned long long kEmpty = ~0ull;

__device__ __forceinline__ double d_diag(double b, double d) { return fabs(d - b) * 0.70710678118654752440; }

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // splitmix64 finaliser
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// ------------------------------------------------------------------ RWMD (Alg 20)
constexpr int NN_THREADS = 256;
constexpr int NN_TILE = 1024;

// sum over u in U of min(min_v ||u - v||, d_Δ(u))  (Eq 6.40: the relaxed flow sends all of
// u's supply to its nearest node of B̂ ∪ {ā}; ā is at distance d_Δ(u))
__global__ void __launch_bounds__(NN_THREADS) k_rwmd(const float2* __restrict__ U, int64_t nu, const float2* __restrict__ V,
                                                     int64_t nv, double* __restrict__ out) {
  __shared__ double2 tile[NN_TILE];
  __shared__ double red[NN_THREADS / 32];
  const int64_t i = (int64_t)blockIdx.x * NN_THREADS + threadIdx.x;
  double ub = 0, ud = 0, best = INFINITY;
  if (i < nu) {
    const float2 p = U[i];
    ub = p.x;
    ud = p.y;
  }
  for (int64_t base = 0; base < nv; base += NN_TILE) {
    const int cnt = (nv - base < (int64_t)NN_TILE) ? (int)(nv - base) : NN_TILE;
    __syncthreads();
    for (int k = threadIdx.x; k < cnt; k += NN_THREADS) {
      const float2 q = V[base + k];
      tile[k] = make_double2(q.x, q.y);
    }
    __syncthreads();
    if (i < nu) {
#pragma unroll 8
      for (int k = 0; k < cnt; ++k) {
        const double dx = ub - tile[k].x, dy = ud - tile[k].y;
        best = fmin(best, fma(dx, dx, dy * dy));
      }
    }
  }
  double v = 0;
  if (i < nu) v = fmin(sqrt(best), d_diag(ub, ud));
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < NN_THREADS / 32; ++w) t += red[w];
    atomicAdd(out, t);
  }
}

// ------------------------------------------------------------------ condensation
struct CellParams {
  int exact;      // 1: key = the point's fp32 bits (0-condensation)
  double grid;    // kδ
  double shift;   // (1-k)δ/2
  uint64_t seed;
};

__device__ __forceinline__ uint64_t cell_key(float b, float d, const CellParams& cp) {
  if (cp.exact) return ((uint64_t)__float_as_uint(b) << 32) | (uint64_t)__float_as_uint(d);
  const long long cx = llround((double)b / cp.grid), cy = llround((double)d / cp.grid);
  return ((uint64_t)(uint32_t)(cx + 0x80000000ll) << 32) | (uint64_t)(uint32_t)(cy + 0x80000000ll);
}

__global__ void k_cells(const float2* __restrict__ P, int64_t n, int64_t nA, CellParams cp,
                        unsigned long long* __restrict__ tkey, long long* __restrict__ tsup, int* __restrict__ tflag,
                        uint64_t mask) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float2 p = P[i];
    const uint64_t key = cell_key(p.x, p.y, cp);
    uint64_t h = mix64(key) & mask;
    for (;;) {
      const unsigned long long prev = atomicCAS(tkey + h, kEmpty, (unsigned long long)key);
      if (prev == kEmpty || prev == key) break;
      h = (h + 1) & mask;
    }
    const bool isA = i < nA;
    atomicAdd((unsigned long long*)(tsup + h), (unsigned long long)(long long)(isA ? 1 : -1));
    atomicOr(tflag + h, isA ? 1 : 2);
  }
}

__global__ void k_compact_keys(const unsigned long long* __restrict__ tkey, uint64_t cap, uint64_t* __restrict__ keys,
                               unsigned long long* __restrict__ count) {
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < cap; base += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t h = base + threadIdx.x;
    const bool has = h < cap && tkey[h] != kEmpty;
    const unsigned long long slot = warp_append(has, count);
    if (has) keys[slot] = tkey[h];
  }
}

// node i = sorted key i: position, supply, flags (looked up in the table)
__global__ void k_nodes(const uint64_t* __restrict__ keys, int64_t N, CellParams cp, const unsigned long long* __restrict__ tkey,
                        const long long* __restrict__ tsup, const int* __restrict__ tflag, uint64_t mask,
                        double2* __restrict__ pos, long long* __restrict__ supply, int* __restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = keys[i];
    uint64_t h = mix64(key) & mask;
    while (tkey[h] != key) h = (h + 1) & mask;
    supply[i] = tsup[h];
    flag[i] = tflag[h];
    double x, y;
    if (cp.exact) {
      x = (double)__uint_as_float((uint32_t)(key >> 32));
      y = (double)__uint_as_float((uint32_t)key);
    } else {
      const long long cx = (long long)(uint32_t)(key >> 32) - 0x80000000ll;
      const long long cy = (long long)(uint32_t)key - 0x80000000ll;
      const uint64_t r = mix64(key ^ mix64(cp.seed));
      const double ux = (double)(uint32_t)(r >> 32) * (2.0 / 4294967296.0) - 1.0;  // [-1, 1)
      const double uy = (double)(uint32_t)r * (2.0 / 4294967296.0) - 1.0;
      x = (double)cx * cp.grid + ux * cp.shift;
      y = (double)cy * cp.grid + uy * cp.shift;
    }
    pos[i] = make_double2(x, y);
  }
}

// ------------------------------------------------------------------ s-WSPD (Algs 23-25)
struct TNode {
  double x0, y0, x1, y1;  // bounding box
  int32_t left, right;    // children (-1 for a leaf)
  int32_t rep;            // representative point (network node id): the leftmost point
  int32_t pad;
};

__device__ __forceinline__ bool well_separated(const TNode& a, const TNode& b, double s) {
  const double ax = 0.5 * (a.x0 + a.x1), ay = 0.5 * (a.y0 + a.y1);
  const double bx = 0.5 * (b.x0 + b.x1), by = 0.5 * (b.y0 + b.y1);
  const double ra = 0.5 * hypot(a.x1 - a.x0, a.y1 - a.y0), rb = 0.5 * hypot(b.x1 - b.x0, b.y1 - b.y0);
  const double r = fmax(ra, rb);
  return hypot(ax - bx, ay - by) - 2.0 * r >= s * r;
}

__device__ __forceinline__ double max_len(const TNode& a) { return fmax(a.x1 - a.x0, a.y1 - a.y0); }

// FIND-PAIRS of Algs 24/25, level-synchronous: the frontier holds node pairs (u, v) still
// to examine (initially (w.left, w.right) for every internal node w, Alg 23); a separated
// pair is emitted as (rep(u), rep(v)), otherwise the node with the longer box side is
// split and both child pairs go to the next frontier.  The pairs emitted are exactly those
// of the per-node recursion, and every level is one parallel pass, so the long chains of
// the nodes near the root (the load imbalance of one thread per node) disappear.
__global__ void k_wspd_level(const TNode* __restrict__ T, const int2* __restrict__ F, uint64_t nf, double s,
                             int2* __restrict__ Fn, unsigned long long* __restrict__ nfn, int2* __restrict__ P,
                             unsigned long long* __restrict__ np) {
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < nf; base += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = base + threadIdx.x;
    bool emit = false, split = false;
    int2 out = make_int2(0, 0), c0 = out, c1 = out;
    if (i < nf) {
      const int2 uv = F[i];
      const TNode& u = T[uv.x];
      const TNode& v = T[uv.y];
      if (well_separated(u, v, s)) {
        emit = true;
        out = make_int2(u.rep, v.rep);
      } else {
        split = true;
        if (max_len(u) > max_len(v)) { c0 = make_int2(u.left, uv.y); c1 = make_int2(u.right, uv.y); }
        else { c0 = make_int2(uv.x, v.left); c1 = make_int2(uv.x, v.right); }
      }
    }
    const unsigned long long pe = warp_append(emit, np);
    if (emit) P[pe] = out;
    const unsigned mask = __ballot_sync(0xffffffffu, split);
    unsigned long long fb = 0;
    const int lane = threadIdx.x & 31;
    if (lane == 0 && mask) fb = atomicAdd(nfn, 2ull * (unsigned long long)__popc(mask));
    fb = __shfl_sync(0xffffffffu, fb, 0);
    if (split) {
      const unsigned long long o = fb + 2ull * (unsigned long long)__popc(mask & lanemask_lt());
      Fn[o] = c0;
      Fn[o + 1] = c1;
    }
  }
}

// ------------------------------------------------------------------ arcs
// WSPD pairs -> biarcs; A-nodes -> ā; b̄ -> B-nodes; b̄ -> ā.  Keys tail << 32 | head.
__global__ void k_arc_keys(const int2* __restrict__ pairs, int64_t np, const int* __restrict__ flag, int64_t N,
                           uint64_t* __restrict__ keys) {
  const int64_t abar = N, bbar = N + 1;
  const int64_t total = 2 * np + N + 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t key;
    if (i < 2 * np) {
      const int2 pq = pairs[i >> 1];
      const int64_t t = (i & 1) ? pq.y : pq.x, h = (i & 1) ? pq.x : pq.y;
      key = ((uint64_t)t << 32) | (uint64_t)h;
    } else if (i < 2 * np + N) {
      const int64_t v = i - 2 * np;
      // a node with A points drains into ā; a pure B node is fed from b̄ (a mixed node
      // gets the b̄ arc in the exact-mode generator below and here through its B flag)
      key = (flag[v] & 1) ? (((uint64_t)v << 32) | (uint64_t)abar) : (((uint64_t)bbar << 32) | (uint64_t)v);
    } else {
      key = ((uint64_t)bbar << 32) | (uint64_t)abar;
    }
    keys[i] = key;
  }
}

// the b̄ -> v arcs of mixed nodes (flag 3), appended after the keys above
__global__ void k_mixed_keys(const int* __restrict__ flag, int64_t N, uint64_t* __restrict__ keys,
                             unsigned long long* __restrict__ count) {
  const int64_t bbar = N + 1;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < N; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = base + threadIdx.x;
    const bool mixed = v < N && flag[v] == 3;
    const unsigned long long slot = warp_append(mixed, count);
    if (mixed) keys[slot] = ((uint64_t)bbar << 32) | (uint64_t)v;
  }
}

// exact mode: every (A-node, B-node) pair, from the compacted lists (sorted, so the keys
// come out sorted by tail then head)
__global__ void k_bipartite_keys(const int32_t* __restrict__ LA, int64_t na, const int32_t* __restrict__ LB, int64_t nb,
                                 uint64_t* __restrict__ keys) {
  const int64_t total = na * nb;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = ((uint64_t)LA[i / nb] << 32) | (uint64_t)LB[i % nb];
}

__global__ void k_flag_lists(const int* __restrict__ flag, int64_t N, int32_t* __restrict__ LA, int32_t* __restrict__ LB,
                             unsigned long long* __restrict__ cnt) {
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < N; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = base + threadIdx.x;
    const int f = v < N ? flag[v] : 0;
    const unsigned long long sa = warp_append((f & 1) != 0, cnt);
    if (f & 1) LA[sa] = (int32_t)v;
    const unsigned long long sb = warp_append((f & 2) != 0, cnt + 1);
    if (f & 2) LB[sb] = (int32_t)v;
  }
}

// sorted keys -> unique arcs with costs (duplicates from repeated representatives and
// self-pairs dropped), order kept (keep flags -> exclusive scan -> write): tail, head, cost
__global__ void k_arc_keep(const uint64_t* __restrict__ keys, int64_t m, uint32_t* __restrict__ keep) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = keys[i];
    keep[i] = (i == 0 || keys[i - 1] != key) && (key >> 32) != (key & 0xffffffffull);
  }
}

__global__ void k_arcs_out(const uint64_t* __restrict__ keys, int64_t m, const uint32_t* __restrict__ keep,
                           const uint32_t* __restrict__ slot, const double2* __restrict__ pos, int64_t N,
                           int32_t* __restrict__ tail, int32_t* __restrict__ head, double* __restrict__ cost) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    if (!keep[i]) continue;
    const uint64_t key = keys[i];
    const int64_t t = (int64_t)(key >> 32), h = (int64_t)(key & 0xffffffffull);
    double c;
    if (t < N && h < N) {
      const double2 a = pos[t], b = pos[h];
      c = hypot(a.x - b.x, a.y - b.y);
    } else if (t < N) {
      c = d_diag(pos[t].x, pos[t].y);  // v -> ā
    } else if (h < N) {
      c = d_diag(pos[h].x, pos[h].y);  // b̄ -> v
    } else {
      c = 0.0;                         // b̄ -> ā
    }
    const uint32_t o = slot[i];
    tail[o] = (int32_t)t;
    head[o] = (int32_t)h;
    cost[o] = c;
  }
}

// ------------------------------------------------------------------ host helpers
// device blocks from the library's cache (vr_api.cu); every use below ends in a
// synchronous copy, so a block is idle when it goes back
struct Dev {
  void* p = nullptr;
  size_t bytes = 0;
  Dev() = default;
  explicit Dev(size_t b) { alloc(b); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  ~Dev() { if (p) dev_release(p, bytes); }
  void alloc(size_t b) {
    if (p) dev_release(p, bytes);
    bytes = b ? b : 16;
    p = dev_acquire(bytes);
  }
  template <class T> T* as() const { return (T*)p; }
};

void chk(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
}

double ms_since(std::chrono::steady_clock::time_point t) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
}

unsigned grid_for(int64_t n, int threads = 256) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, (int64_t)sms * 16));
}

// fair split tree (§6.3.5): split the bounding box's longer side in the middle; leaves are
// single points.  Iterative; returns the height.
int build_split_tree(const std::vector<double2>& P, std::vector<TNode>& T, std::vector<int32_t>& internal) {
  const int64_t N = (int64_t)P.size();
  T.clear();
  internal.clear();
  T.reserve((size_t)(2 * N));
  std::vector<int32_t> perm((size_t)N);
  for (int64_t i = 0; i < N; ++i) perm[(size_t)i] = (int32_t)i;
  struct Job { int64_t lo, hi; int32_t node; int depth; };
  std::vector<Job> stk;
  T.push_back(TNode{});
  stk.push_back({0, N, 0, 0});
  int height = 0;
  while (!stk.empty()) {
    const Job j = stk.back();
    stk.pop_back();
    height = std::max(height, j.depth);
    double x0 = INFINITY, y0 = INFINITY, x1 = -INFINITY, y1 = -INFINITY;
    int32_t rep = -1;
    for (int64_t k = j.lo; k < j.hi; ++k) {
      const double2 p = P[(size_t)perm[(size_t)k]];
      x0 = std::min(x0, p.x); x1 = std::max(x1, p.x);
      y0 = std::min(y0, p.y); y1 = std::max(y1, p.y);
      const int32_t id = perm[(size_t)k];
      if (rep < 0 || p.x < P[(size_t)rep].x || (p.x == P[(size_t)rep].x && p.y < P[(size_t)rep].y)) rep = id;
    }
    TNode& t = T[(size_t)j.node];
    t.x0 = x0; t.y0 = y0; t.x1 = x1; t.y1 = y1;
    t.rep = rep;
    t.pad = 0;
    if (j.hi - j.lo == 1) { t.left = t.right = -1; continue; }
    const bool sx = (x1 - x0) >= (y1 - y0);
    const double mid = sx ? 0.5 * (x0 + x1) : 0.5 * (y0 + y1);
    auto it = std::partition(perm.begin() + j.lo, perm.begin() + j.hi,
                             [&](int32_t id) { return (sx ? P[(size_t)id].x : P[(size_t)id].y) < mid; });
    int64_t m = it - perm.begin();
    if (m == j.lo || m == j.hi) m = (j.lo + j.hi) / 2;  // rounding left one side empty
    const int32_t l = (int32_t)T.size(), r = l + 1;
    T.push_back(TNode{});
    T.push_back(TNode{});
    T[(size_t)j.node].left = l;
    T[(size_t)j.node].right = r;
    internal.push_back(j.node);
    stk.push_back({j.lo, m, l, j.depth + 1});
    stk.push_back({m, j.hi, r, j.depth + 1});
  }
  return height;
}

}  // namespace

// The whole network of Alg 22 lines 1-5 (host arrays out).
struct W1Net {
  std::vector<double2> pos;       // N real nodes
  std::vector<int64_t> supply;    // N + 2 (ā = N, b̄ = N + 1)
  PinnedVec<int32_t> tail, head;  // page-locked: the arc arrays come back at full bandwidth
  PinnedVec<double> cost;
};

void w1_build(const float* A, int64_t nA, const float* B, int64_t nB, double s, uint64_t seed, int32_t flags, W1Net& net,
              vr_w1_stats& st) {
  const auto t_all = std::chrono::steady_clock::now();
  const int64_t n = nA + nB;
  st.points_a = nA;
  st.points_b = nB;
  const bool exact = (flags & VR_W1_EXACT) || !(s > 0);
  cudaStream_t cs = 0;
  // ---------------- H2D: the points, A then B
  auto t0 = std::chrono::steady_clock::now();
  Dev dP((size_t)std::max<int64_t>(n, 1) * sizeof(float2));
  if (nA) chk(cudaMemcpyAsync(dP.p, A, (size_t)nA * 8, cudaMemcpyHostToDevice, cs));
  if (nB) chk(cudaMemcpyAsync(dP.as<float2>() + nA, B, (size_t)nB * 8, cudaMemcpyHostToDevice, cs));
  chk(cudaStreamSynchronize(cs));
  st.ms_h2d = ms_since(t0);
  // ---------------- RWMD (Alg 20) and δ (Alg 21 lines 2-7)
  t0 = std::chrono::steady_clock::now();
  double L = 0;
  if (!exact) {
    Dev dL(2 * sizeof(double));
    chk(cudaMemsetAsync(dL.p, 0, 2 * sizeof(double), cs));
    if (nA) k_rwmd<<<(unsigned)((nA + NN_THREADS - 1) / NN_THREADS), NN_THREADS, 0, cs>>>(dP.as<float2>(), nA, dP.as<float2>() + nA, nB, dL.as<double>());
    if (nB) k_rwmd<<<(unsigned)((nB + NN_THREADS - 1) / NN_THREADS), NN_THREADS, 0, cs>>>(dP.as<float2>() + nA, nB, dP.as<float2>(), nA, dL.as<double>() + 1);
    chk(cudaGetLastError());
    double h[2];
    chk(cudaMemcpy(h, dL.p, sizeof h, cudaMemcpyDeviceToHost));
    L = std::max(h[0], h[1]);
  }
  st.rwmd = L;
  st.ms_rwmd = ms_since(t0);
  st.eps_condense = exact ? 0.0 : (s >= 12 ? 8.0 / (s - 4.0) : 1.0);
  st.eps_spanner = exact ? 0.0 : (s > 2 ? 4.0 / s + 4.0 / (s - 2.0) : INFINITY);
  double delta = exact || (flags & VR_W1_NO_CONDENSE) || n == 0 ? 0.0 : 2.0 * st.eps_condense * L / (std::sqrt(2.0) * (double)n);
  // the cell coordinates must fit 32 bits; otherwise condensation is skipped
  if (delta > 0) {
    double amax = 0;
    for (int64_t i = 0; i < nA; ++i) amax = std::max({amax, std::fabs((double)A[2 * i]), std::fabs((double)A[2 * i + 1])});
    for (int64_t i = 0; i < nB; ++i) amax = std::max({amax, std::fabs((double)B[2 * i]), std::fabs((double)B[2 * i + 1])});
    if (amax / (kSnap * delta) > 2.0e9) delta = 0;
  }
  st.delta = delta;
  st.condensed = delta > 0 ? 1 : 0;
  st.bound_lo = delta > 0 ? 1.0 - st.eps_condense : 1.0;
  st.bound_hi = (delta > 0 ? 1.0 + st.eps_condense : 1.0) * (exact ? 1.0 : 1.0 + st.eps_spanner);
  // ---------------- condensation: one node per occupied cell (or per distinct point)
  t0 = std::chrono::steady_clock::now();
  CellParams cp{delta > 0 ? 0 : 1, kSnap * delta, 0.5 * (1.0 - kSnap) * delta, seed};
  uint64_t cap = 1024;
  while (cap < (uint64_t)(2 * n)) cap <<= 1;
  const uint64_t mask = cap - 1;
  Dev dTk(cap * 8), dTs(cap * 8), dTf(cap * 4), dCnt(64);
  chk(cudaMemsetAsync(dTk.p, 0xff, cap * 8, cs));
  chk(cudaMemsetAsync(dTs.p, 0, cap * 8, cs));
  chk(cudaMemsetAsync(dTf.p, 0, cap * 4, cs));
  chk(cudaMemsetAsync(dCnt.p, 0, 64, cs));
  if (n) k_cells<<<grid_for(n), 256, 0, cs>>>(dP.as<float2>(), n, nA, cp, dTk.as<unsigned long long>(), dTs.as<long long>(), dTf.as<int>(), mask);
  Dev dKeys((size_t)std::max<int64_t>(n, 1) * 8), dAlt((size_t)std::max<int64_t>(n, 1) * 8);
  k_compact_keys<<<grid_for((int64_t)cap), 256, 0, cs>>>(dTk.as<unsigned long long>(), cap, dKeys.as<uint64_t>(), dCnt.as<unsigned long long>());
  unsigned long long Nn = 0;
  chk(cudaMemcpy(&Nn, dCnt.p, 8, cudaMemcpyDeviceToHost));
  const int64_t N = (int64_t)Nn;
  Dev dTmp(radix_sort_temp_bytes((size_t)std::max<int64_t>(N, 1)));
  uint64_t* sorted = radix_sort_u64(dKeys.as<uint64_t>(), dAlt.as<uint64_t>(), (size_t)N, 0, 64, dTmp.p, cs, nullptr);
  Dev dPos((size_t)std::max<int64_t>(N, 1) * 16), dSup((size_t)std::max<int64_t>(N, 1) * 8), dFlag((size_t)std::max<int64_t>(N, 1) * 4);
  if (N) k_nodes<<<grid_for(N), 256, 0, cs>>>(sorted, N, cp, dTk.as<unsigned long long>(), dTs.as<long long>(), dTf.as<int>(), mask,
                                               dPos.as<double2>(), dSup.as<long long>(), dFlag.as<int>());
  chk(cudaGetLastError());
  net.pos.resize((size_t)N);
  net.supply.resize((size_t)N + 2);
  std::vector<int> hflag((size_t)N);
  if (N) {
    chk(cudaMemcpy(net.pos.data(), dPos.p, (size_t)N * 16, cudaMemcpyDeviceToHost));
    chk(cudaMemcpy(net.supply.data(), dSup.p, (size_t)N * 8, cudaMemcpyDeviceToHost));
    chk(cudaMemcpy(hflag.data(), dFlag.p, (size_t)N * 4, cudaMemcpyDeviceToHost));
  }
  net.supply[(size_t)N] = -nA;     // ā absorbs every A point
  net.supply[(size_t)N + 1] = nB;  // b̄ feeds every B point
  st.nodes = N + 2;
  st.ms_condense = ms_since(t0);
  // ---------------- arcs
  uint64_t m_keys = 0;
  Dev dArcKeys, dArcAlt;
  t0 = std::chrono::steady_clock::now();
  if (exact) {
    Dev dLA((size_t)std::max<int64_t>(N, 1) * 4), dLB((size_t)std::max<int64_t>(N, 1) * 4), dC(16);
    chk(cudaMemsetAsync(dC.p, 0, 16, cs));
    if (N) k_flag_lists<<<grid_for(N), 256, 0, cs>>>(dFlag.as<int>(), N, dLA.as<int32_t>(), dLB.as<int32_t>(), dC.as<unsigned long long>());
    unsigned long long c2[2];
    chk(cudaMemcpy(c2, dC.p, 16, cudaMemcpyDeviceToHost));
    // the lists come out of warp-aggregated appends: sort them so the keys are ordered
    std::vector<int32_t> la(c2[0]), lb(c2[1]);
    if (c2[0]) chk(cudaMemcpy(la.data(), dLA.p, c2[0] * 4, cudaMemcpyDeviceToHost));
    if (c2[1]) chk(cudaMemcpy(lb.data(), dLB.p, c2[1] * 4, cudaMemcpyDeviceToHost));
    std::sort(la.begin(), la.end());
    std::sort(lb.begin(), lb.end());
    if (c2[0]) chk(cudaMemcpy(dLA.p, la.data(), c2[0] * 4, cudaMemcpyHostToDevice));
    if (c2[1]) chk(cudaMemcpy(dLB.p, lb.data(), c2[1] * 4, cudaMemcpyHostToDevice));
    const uint64_t nbip = (uint64_t)c2[0] * c2[1];
    m_keys = nbip + (uint64_t)N + 1 + (uint64_t)N;
    dArcKeys.alloc(std::max<uint64_t>(m_keys, 1) * 8);
    dArcAlt.alloc(std::max<uint64_t>(m_keys, 1) * 8);
    if (nbip) k_bipartite_keys<<<grid_for((int64_t)nbip), 256, 0, cs>>>(dLA.as<int32_t>(), (int64_t)c2[0], dLB.as<int32_t>(), (int64_t)c2[1], dArcKeys.as<uint64_t>());
    k_arc_keys<<<grid_for(N + 1), 256, 0, cs>>>(nullptr, 0, dFlag.as<int>(), N, dArcKeys.as<uint64_t>() + nbip);
    chk(cudaMemsetAsync(dC.p, 0, 8, cs));
    if (N) k_mixed_keys<<<grid_for(N), 256, 0, cs>>>(dFlag.as<int>(), N, dArcKeys.as<uint64_t>() + nbip + N + 1, dC.as<unsigned long long>());
    unsigned long long nm = 0;
    chk(cudaMemcpy(&nm, dC.p, 8, cudaMemcpyDeviceToHost));
    m_keys = nbip + (uint64_t)N + 1 + nm;
    st.ms_tree = 0;
    st.ms_wspd = 0;
  } else {
    // ---------------- split tree (host) and s-WSPD (GPU)
    auto tt = std::chrono::steady_clock::now();
    std::vector<TNode> T;
    std::vector<int32_t> internal;
    const int height = N ? build_split_tree(net.pos, T, internal) : 0;
    st.tree_height = height;
    st.ms_tree = ms_since(tt);
    tt = std::chrono::steady_clock::now();
    const int64_t ni = (int64_t)internal.size();
    Dev dT(std::max<size_t>(T.size(), 1) * sizeof(TNode)), dInt((size_t)std::max<int64_t>(ni, 1) * 4);
    if (!T.empty()) chk(cudaMemcpyAsync(dT.p, T.data(), T.size() * sizeof(TNode), cudaMemcpyHostToDevice, cs));
    if (ni) chk(cudaMemcpyAsync(dInt.p, internal.data(), (size_t)ni * 4, cudaMemcpyHostToDevice, cs));
    uint64_t npairs = 0;
    Dev dPairs;
    if (ni) {
      std::vector<int2> f0((size_t)ni);
      for (int64_t k = 0; k < ni; ++k) f0[(size_t)k] = make_int2(T[(size_t)internal[(size_t)k]].left, T[(size_t)internal[(size_t)k]].right);
      uint64_t nf = (uint64_t)ni, pcap = std::max<uint64_t>(4 * (uint64_t)ni, 1024);
      Dev dF(nf * sizeof(int2)), dCounters(16);
      dPairs.alloc(pcap * sizeof(int2));
      chk(cudaMemcpyAsync(dF.p, f0.data(), nf * sizeof(int2), cudaMemcpyHostToDevice, cs));
      chk(cudaMemsetAsync(dCounters.p, 0, 16, cs));
      while (nf) {
        if (npairs + nf > pcap) {  // at most one emitted pair per frontier pair
          const uint64_t ncap = std::max<uint64_t>(2 * pcap, npairs + nf);
          Dev grown(ncap * sizeof(int2));
          if (npairs) chk(cudaMemcpyAsync(grown.p, dPairs.p, npairs * sizeof(int2), cudaMemcpyDeviceToDevice, cs));
          std::swap(grown.p, dPairs.p);
          std::swap(grown.bytes, dPairs.bytes);
          pcap = ncap;
          chk(cudaStreamSynchronize(cs));
        }
        Dev dFn(2 * nf * sizeof(int2));
        chk(cudaMemsetAsync(dCounters.p, 0, 8, cs));  // next frontier size; [1] = pairs so far
        k_wspd_level<<<grid_for((int64_t)nf), 256, 0, cs>>>(dT.as<TNode>(), dF.as<int2>(), nf, s, dFn.as<int2>(),
                                                            dCounters.as<unsigned long long>(), dPairs.as<int2>(),
                                                            dCounters.as<unsigned long long>() + 1);
        chk(cudaGetLastError());
        unsigned long long c[2];
        chk(cudaMemcpy(c, dCounters.p, 16, cudaMemcpyDeviceToHost));
        nf = c[0];
        npairs = c[1];
        std::swap(dF.p, dFn.p);
        std::swap(dF.bytes, dFn.bytes);
        ++st.wspd_levels;
      }
    }
    st.wspd_pairs = (int64_t)npairs;
    st.ms_wspd = ms_since(tt);
    m_keys = 2 * npairs + (uint64_t)N + 1;
    dArcKeys.alloc((m_keys + (uint64_t)N) * 8);
    dArcAlt.alloc((m_keys + (uint64_t)N) * 8);
    k_arc_keys<<<grid_for((int64_t)m_keys), 256, 0, cs>>>(dPairs.as<int2>(), (int64_t)npairs, dFlag.as<int>(), N, dArcKeys.as<uint64_t>());
    chk(cudaMemsetAsync(dCnt.p, 0, 8, cs));
    if (N) k_mixed_keys<<<grid_for(N), 256, 0, cs>>>(dFlag.as<int>(), N, dArcKeys.as<uint64_t>() + m_keys, dCnt.as<unsigned long long>());
    unsigned long long nm = 0;
    chk(cudaMemcpy(&nm, dCnt.p, 8, cudaMemcpyDeviceToHost));
    m_keys += nm;
  }
  // ---------------- sort the arcs by (tail, head) (§6.9.3), drop duplicates, costs
  auto ts = std::chrono::steady_clock::now();
  int kb = 1;
  while (kb < 32 && ((uint64_t)(N + 1) >> kb)) ++kb;
  Dev dTmp2(radix_sort_temp_bytes((size_t)std::max<uint64_t>(m_keys, 1)));
  uint64_t* ak = radix_sort_u64(dArcKeys.as<uint64_t>(), dArcAlt.as<uint64_t>(), (size_t)m_keys, 0, 32 + kb, dTmp2.p, cs, nullptr);
  Dev dKeep(std::max<uint64_t>(m_keys, 1) * 4), dSlot(std::max<uint64_t>(m_keys, 1) * 4),
      dScanTmp(scan_temp_bytes((size_t)std::max<uint64_t>(m_keys, 1)));
  unsigned long long M = 0;
  if (m_keys) {
    if (m_keys >= (1ull << 32)) throw std::runtime_error("more than 2^32 arc keys");
    k_arc_keep<<<grid_for((int64_t)m_keys), 256, 0, cs>>>(ak, (int64_t)m_keys, dKeep.as<uint32_t>());
    exclusive_scan_u32(dKeep.as<uint32_t>(), dSlot.as<uint32_t>(), (size_t)m_keys, dScanTmp.p, cs, nullptr);
    uint32_t last[2];
    chk(cudaMemcpy(&last[0], dKeep.as<uint32_t>() + m_keys - 1, 4, cudaMemcpyDeviceToHost));
    chk(cudaMemcpy(&last[1], dSlot.as<uint32_t>() + m_keys - 1, 4, cudaMemcpyDeviceToHost));
    M = (unsigned long long)last[0] + last[1];
  }
  Dev dTail(std::max<unsigned long long>(M, 1) * 4), dHead(std::max<unsigned long long>(M, 1) * 4),
      dCost(std::max<unsigned long long>(M, 1) * 8);
  if (m_keys) k_arcs_out<<<grid_for((int64_t)m_keys), 256, 0, cs>>>(ak, (int64_t)m_keys, dKeep.as<uint32_t>(), dSlot.as<uint32_t>(),
                                                                    dPos.as<double2>(), N, dTail.as<int32_t>(), dHead.as<int32_t>(),
                                                                    dCost.as<double>());
  chk(cudaGetLastError());
  st.ms_arcs = ms_since(ts);
  auto td = std::chrono::steady_clock::now();
  net.tail.resize(M);
  net.head.resize(M);
  net.cost.resize(M);
  if (M) {
    chk(cudaMemcpy(net.tail.data(), dTail.p, M * 4, cudaMemcpyDeviceToHost));
    chk(cudaMemcpy(net.head.data(), dHead.p, M * 4, cudaMemcpyDeviceToHost));
    chk(cudaMemcpy(net.cost.data(), dCost.p, M * 8, cudaMemcpyDeviceToHost));
  }
  st.arcs = (int64_t)M;
  st.ms_d2h = ms_since(td);
  st.ms_build = ms_since(t_all);
}

}  // namespace vr

struct vr_w1_net {
  vr::W1Net net;
};

namespace {

int w1_checks(const float* A, int64_t nA, const float* B, int64_t nB) {
  if (nA < 0 || nB < 0 || (nA && !A) || (nB && !B)) return VR_EINVAL;
  if (nA + nB + 2 >= INT32_MAX) return VR_ECAPACITY;
  for (int64_t i = 0; i < 2 * nA; ++i) if (!std::isfinite(A[i])) return VR_EINPUT;
  for (int64_t i = 0; i < 2 * nB; ++i) if (!std::isfinite(B[i])) return VR_EINPUT;
  return VR_OK;
}
}  // namespace

extern "C" int vr_w1_network(const float* A, int64_t nA, const float* B, int64_t nB, double s, uint64_t seed, int32_t flags,
                             vr_w1_net** out, vr_w1_stats* stats) {
  if (!out) return VR_EINVAL;
  *out = nullptr;
  if (int e = w1_checks(A, nA, B, nB)) return e;
  try {
    std::unique_ptr<vr_w1_net> h(new vr_w1_net());
    vr_w1_stats st{};
    vr::w1_build(A, nA, B, nB, s, seed, flags, h->net, st);
    if (stats) *stats = st;
    *out = h.release();
    return VR_OK;
  } catch (const std::bad_alloc&) {
    return VR_ECAPACITY;
  } catch (const std::exception& e) {
    vr::set_last_error(e.what());
    return VR_EDEVICE;
  }
}

extern "C" int64_t vr_w1_net_nodes(const vr_w1_net* h) { return h ? (int64_t)h->net.supply.size() : 0; }
extern "C" int64_t vr_w1_net_arcs(const vr_w1_net* h) { return h ? (int64_t)h->net.tail.size() : 0; }
extern "C" void vr_w1_net_get(const vr_w1_net* h, double* xy, int64_t* supply, int32_t* tail, int32_t* head, double* cost) {
  if (!h) return;
  const auto& n = h->net;
  const size_t N = n.pos.size();
  if (xy) {
    for (size_t i = 0; i < N; ++i) { xy[2 * i] = n.pos[i].x; xy[2 * i + 1] = n.pos[i].y; }
    for (size_t i = N; i < N + 2; ++i) xy[2 * i] = xy[2 * i + 1] = NAN;  // ā, b̄
  }
  if (supply) std::copy(n.supply.begin(), n.supply.end(), supply);
  if (tail) std::copy(n.tail.data(), n.tail.data() + n.tail.size(), tail);
  if (head) std::copy(n.head.data(), n.head.data() + n.head.size(), head);
  if (cost) std::copy(n.cost.data(), n.cost.data() + n.cost.size(), cost);
}
extern "C" void vr_w1_net_free(vr_w1_net* h) { delete h; }

extern "C" int vr_w1(const float* A, int64_t nA, const float* B, int64_t nB, double s, uint64_t seed, int32_t flags,
                     int64_t max_blocks, double* w1, vr_w1_stats* stats) {
  if (!w1) return VR_EINVAL;
  if (int e = w1_checks(A, nA, B, nB)) return e;
  try {
    const auto t_all = std::chrono::steady_clock::now();
    vr::W1Net net;
    vr_w1_stats st{};
    vr::w1_build(A, nA, B, nB, s, seed, flags, net, st);
    const auto t0 = std::chrono::steady_clock::now();
    // optional warm start (VR_W1_WARM_DIAGONAL): the all-to-diagonal basis — every node with net supply > 0
    // drains into ā, every other node is fed from b̄, and b̄ -> ā carries the rest; rooted at
    // b̄, zero flows point away from the root (strongly feasible)
    const int64_t NN = (int64_t)net.supply.size();
    const int64_t N = NN - 2;
    std::vector<int32_t> pred((size_t)NN, -1), to_abar((size_t)std::max<int64_t>(N, 1), -1),
        from_bbar((size_t)std::max<int64_t>(N, 1), -1);
    int32_t bb_ab = -1;
    for (size_t a = 0; a < net.tail.size(); ++a) {
      const int32_t t = net.tail[a], h = net.head[a];
      if (h == N && t < N) to_abar[(size_t)t] = (int32_t)a;
      else if (t == N + 1 && h < N) from_bbar[(size_t)h] = (int32_t)a;
      else if (t == N + 1 && h == N) bb_ab = (int32_t)a;
    }
    bool ok = bb_ab >= 0 && (flags & VR_W1_WARM_DIAGONAL);
    pred[(size_t)N] = bb_ab;
    for (int64_t v = 0; v < N && ok; ++v) {
      pred[(size_t)v] = net.supply[(size_t)v] > 0 ? to_abar[(size_t)v] : from_bbar[(size_t)v];
      ok = pred[(size_t)v] >= 0;
    }
    const vr::McfResult r = vr::network_simplex(NN, net.supply.data(), (int64_t)net.tail.size(), net.tail.data(),
                                                net.head.data(), net.cost.data(), max_blocks, ok ? pred.data() : nullptr,
                                                ok ? (int32_t)(N + 1) : -1);
    st.warm_start = r.warm_start ? 1 : 0;
    st.ms_pricing = r.ms_pricing;
    st.ms_update = r.ms_update;
    st.ms_simplex = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    st.pivots = r.pivots;
    st.degenerate = r.degenerate;
    st.blocks = r.blocks;
    st.optimal = r.optimal ? 1 : 0;
    st.ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_all).count();
    *w1 = r.cost;
    if (stats) *stats = st;
    if (r.unbounded || r.infeasible) return VR_EINPUT;
    return VR_OK;
  } catch (const std::bad_alloc&) {
    return VR_ECAPACITY;
  } catch (const std::exception& e) {
    vr::set_last_error(e.what());
    return VR_EDEVICE;
  }
}
