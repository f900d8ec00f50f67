// netsimplex.cpp — uncapacitated min-cost flow by the primal network simplex with the
// block search pivot rule (§6.3.7; §6.10).
//
// Problem (Def 6.2.2 / Eq 6.38): nodes v with integer supply σ(v) (Σσ = 0), arcs a = (t, h)
// with cost c_a >= 0 and no capacity; minimise Σ c_a f_a with out(v) - in(v) = σ(v), f >= 0.
//
// Basis: a spanning tree over the nodes plus an artificial root r.  Start (big-M): node v
// hangs off r by an artificial arc v -> r if σ(v) > 0 (flow σ) and r -> v otherwise
// (flow -σ), each of cost M larger than any path of real arcs; zero-flow tree arcs point
// away from r, so the tree is strongly feasible and stays so (leaving-arc rule below),
// which prevents cycling.  Potentials π keep every tree arc at reduced cost
// c_a + π(t) - π(h) = 0.
//
// Pivot (block search, P:6644 / P:7076): scan the arcs cyclically in blocks of B = ⌈√m⌉
// and take the most negative reduced cost of the first block that has one.  The entering
// arc (p -> q) closes a cycle with the tree path q ~> join ~> p; the leaving arc is the
// blocking arc (flow decreasing around the cycle) with the least flow — on ties the last
// one met when walking the cycle from the join in the flow direction (strongly feasible
// rule).  The subtree cut off by the leaving arc is re-hung from the entering arc and its
// potentials shift by one constant.
//
// Stopping: optimal when no arc has a negative reduced cost (relative tolerance 1e-9 of
// the largest cost), or after `max_blocks` searched blocks (the C√(mn)+b
// criterion; 0 = no limit) — reported as not optimal.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <limits>
#include <new>
#if defined(__x86_64__)
#include <immintrin.h>
#endif
#include <vector>

#include "../../include/vr.h"
#include "vr_internal.h"

namespace vr {

namespace {

struct Tree {
  // per node (0..N, N = artificial root)
  std::vector<int32_t> parent, pred, first_child, next_sib, prev_sib, depth;
  std::vector<uint8_t> up;  // pred arc oriented node -> parent
  std::vector<double> pi;
  void detach(int32_t x) {
    const int32_t p = parent[(size_t)x];
    if (prev_sib[(size_t)x] >= 0) next_sib[(size_t)prev_sib[(size_t)x]] = next_sib[(size_t)x];
    else first_child[(size_t)p] = next_sib[(size_t)x];
    if (next_sib[(size_t)x] >= 0) prev_sib[(size_t)next_sib[(size_t)x]] = prev_sib[(size_t)x];
    next_sib[(size_t)x] = prev_sib[(size_t)x] = -1;
  }
  void attach(int32_t x, int32_t p) {
    parent[(size_t)x] = p;
    prev_sib[(size_t)x] = -1;
    next_sib[(size_t)x] = first_child[(size_t)p];
    if (first_child[(size_t)p] >= 0) prev_sib[(size_t)first_child[(size_t)p]] = x;
    first_child[(size_t)p] = x;
  }
};

// Minimum reduced cost over arcs [j0, j1) of one tail (potential pit): updates best/enter.
// Scalar reference and an AVX2 version (4 arcs per step: gathered head potentials, float
// costs widened to double, running vector minimum with its arc indices), picked at run time.
inline void price_segment_scalar(const float* c32, const int32_t* ah, const double* pi, double pit, int64_t j0, int64_t j1,
                                 double& best, int64_t& enter) {
  for (int64_t j = j0; j < j1; ++j) {
    const double r = (double)c32[j] + pit - pi[ah[j]];
    if (r < best) { best = r; enter = j; }
  }
}

#if defined(__x86_64__)
__attribute__((target("avx2,fma"))) void price_segment_avx2(const float* c32, const int32_t* ah, const double* pi, double pit,
                                                            int64_t j0, int64_t j1, double& best, int64_t& enter) {
  int64_t j = j0;
  if (j1 - j0 >= 8) {
    __m256d vbest = _mm256_set1_pd(best);
    __m256i vidx = _mm256_set1_epi64x(-1);
    const __m256d vpit = _mm256_set1_pd(pit);
    __m256i cur = _mm256_setr_epi64x(j, j + 1, j + 2, j + 3);
    const __m256i four = _mm256_set1_epi64x(4);
    for (; j + 4 <= j1; j += 4) {
      const __m128i h = _mm_loadu_si128((const __m128i*)(ah + j));
      const __m256d ph = _mm256_i32gather_pd(pi, h, 8);
      const __m256d c = _mm256_cvtps_pd(_mm_loadu_ps(c32 + j));
      const __m256d r = _mm256_sub_pd(_mm256_add_pd(c, vpit), ph);
      const __m256d lt = _mm256_cmp_pd(r, vbest, _CMP_LT_OQ);
      vbest = _mm256_blendv_pd(vbest, r, lt);
      vidx = _mm256_castpd_si256(_mm256_blendv_pd(_mm256_castsi256_pd(vidx), _mm256_castsi256_pd(cur), lt));
      cur = _mm256_add_epi64(cur, four);
    }
    alignas(32) double b[4];
    alignas(32) int64_t ix[4];
    _mm256_store_pd(b, vbest);
    _mm256_store_si256((__m256i*)ix, vidx);
    for (int k = 0; k < 4; ++k)  // lowest index among equal minima, like the scalar scan
      if (ix[k] >= 0 && (b[k] < best || (b[k] == best && enter >= 0 && ix[k] < enter) || (b[k] == best && enter < 0))) {
        if (b[k] < best || enter < 0 || ix[k] < enter) { best = b[k]; enter = ix[k]; }
      }
  }
  price_segment_scalar(c32, ah, pi, pit, j, j1, best, enter);
}
const bool g_has_avx2 = __builtin_cpu_supports("avx2") && __builtin_cpu_supports("fma");
#endif

inline void price_segment(const float* c32, const int32_t* ah, const double* pi, double pit, int64_t j0, int64_t j1,
                          double& best, int64_t& enter) {
#if defined(__x86_64__)
  if (g_has_avx2) { price_segment_avx2(c32, ah, pi, pit, j0, j1, best, enter); return; }
#endif
  price_segment_scalar(c32, ah, pi, pit, j0, j1, best, enter);
}

}  // namespace

McfResult network_simplex(int64_t nodes, const int64_t* supply, int64_t arcs, const int32_t* tail, const int32_t* head,
                          const double* cost, int64_t max_blocks, const int32_t* init_pred, int32_t init_root) {
  McfResult res;
  const int32_t N = (int32_t)nodes;
  const int64_t M = arcs;
  const int32_t root = N;
  double cmax = 0;
  for (int64_t a = 0; a < M; ++a) cmax = std::max(cmax, cost[a]);
  // artificial arc cost: larger than any simple path of real arcs
  const double big = (cmax + 1.0) * (double)(N + 1);
  // reduced costs carry rounding of potentials up to ~big; accept |rc| below 1e-9 of the
  // largest cost as zero (an objective error of at most 1e-9 cmax per unit of flow)
  const double eps = 1e-9 * (cmax > 0 ? cmax : 1.0);
  // arc arrays in tail-major (CSR) order, so the pricing stream reads the tail once per
  // node and per arc only the head (4 B) and a float copy of the cost (4 B); real arcs
  // 0..M-1, artificial arcs M..M+N-1 (node v's arc to/from the root)
  const int64_t MA = M + N;
  std::vector<int64_t> off((size_t)N + 1, 0);
  for (int64_t a = 0; a < M; ++a) ++off[(size_t)tail[a] + 1];
  for (int32_t v = 0; v < N; ++v) off[(size_t)v + 1] += off[(size_t)v];
  std::vector<int64_t> cur(off.begin(), off.end() - 1);
  std::vector<int32_t> pos((size_t)M);
  std::vector<int32_t> at((size_t)MA), ah((size_t)MA);
  std::vector<double> ac((size_t)MA, big), flow((size_t)MA, 0.0);
  std::vector<float> c32((size_t)std::max<int64_t>(M, 1));
  for (int64_t a = 0; a < M; ++a) {
    const int64_t i = cur[(size_t)tail[a]]++;
    pos[(size_t)a] = (int32_t)i;
    at[(size_t)i] = tail[a];
    ah[(size_t)i] = head[a];
    ac[(size_t)i] = cost[a];
    c32[(size_t)i] = (float)cost[a];
  }
  std::vector<uint8_t> in_tree((size_t)MA, 0);
  Tree T;
  const size_t NN = (size_t)N + 1;
  T.parent.assign(NN, -1);
  T.pred.assign(NN, -1);
  T.first_child.assign(NN, -1);
  T.next_sib.assign(NN, -1);
  T.prev_sib.assign(NN, -1);
  T.depth.assign(NN, 0);
  T.up.assign(NN, 0);
  T.pi.assign(NN, 0.0);
  // big-M start: every node on its artificial arc
  auto artificial_start = [&]() {
    for (int32_t v = 0; v < N; ++v) {
      const int64_t a = M + v;
      if (supply[v] > 0) {  // v -> root carries σ(v)
        at[(size_t)a] = v; ah[(size_t)a] = root; flow[(size_t)a] = (double)supply[v];
        T.up[(size_t)v] = 1;
        T.pi[(size_t)v] = -big;  // c + π(v) - π(r) = 0
      } else {              // root -> v carries -σ(v) (zero flow points away from the root)
        at[(size_t)a] = root; ah[(size_t)a] = v; flow[(size_t)a] = (double)(-supply[v]);
        T.up[(size_t)v] = 0;
        T.pi[(size_t)v] = big;   // c + π(r) - π(v) = 0
      }
      in_tree[(size_t)a] = 1;
      T.pred[(size_t)v] = (int32_t)a;
      T.depth[(size_t)v] = 1;
      T.attach(v, root);
    }
  };
  // caller's spanning tree (init_pred[v] = the real arc joining v to its parent, the
  // parent being the arc's other end; init_root hangs off the artificial root by a
  // zero-flow arc r -> init_root).  Tree flows follow from the supplies (leaves first);
  // a negative one means the tree is not a feasible basis -> big-M start instead.
  bool warm = false;
  if (init_pred && init_root >= 0 && init_root < N) {
    std::vector<int32_t> par((size_t)N, -1);
    std::vector<std::vector<int32_t>> kids((size_t)N + 1);
    bool ok = init_pred[init_root] < 0;
    for (int32_t v = 0; v < N && ok; ++v) {
      if (v == init_root) continue;
      const int32_t a0 = init_pred[v];
      if (a0 < 0 || a0 >= M || (tail[a0] != v && head[a0] != v)) { ok = false; break; }
      par[(size_t)v] = tail[a0] == v ? head[a0] : tail[a0];
    }
    std::vector<int32_t> order;
    if (ok) {
      for (int32_t v = 0; v < N; ++v)
        if (v != init_root) kids[(size_t)par[(size_t)v]].push_back(v);
      order.reserve((size_t)N);
      order.push_back(init_root);
      for (size_t k = 0; k < order.size(); ++k)
        for (int32_t c : kids[(size_t)order[k]]) order.push_back(c);
      ok = (int64_t)order.size() == N;  // connected, no cycle
    }
    std::vector<double> sub;
    if (ok) {
      sub.assign((size_t)N, 0.0);
      for (int32_t v = 0; v < N; ++v) sub[(size_t)v] = (double)supply[v];
      for (size_t k = order.size(); k-- > 1;) {
        const int32_t v = order[k];
        const int32_t a = pos[(size_t)init_pred[v]];
        const double f = at[(size_t)a] == v ? sub[(size_t)v] : -sub[(size_t)v];
        if (f < 0) { ok = false; break; }
        flow[(size_t)a] = f;
        sub[(size_t)par[(size_t)v]] += sub[(size_t)v];
      }
    }
    if (ok) {
      const int64_t ar = M + init_root;
      at[(size_t)ar] = root; ah[(size_t)ar] = init_root; flow[(size_t)ar] = 0;
      in_tree[(size_t)ar] = 1;
      T.pred[(size_t)init_root] = (int32_t)ar;
      T.up[(size_t)init_root] = 0;
      T.pi[(size_t)init_root] = big;
      T.depth[(size_t)init_root] = 1;
      T.attach(init_root, root);
      for (size_t k = 1; k < order.size(); ++k) {
        const int32_t v = order[k], p = par[(size_t)v];
        const int32_t a = pos[(size_t)init_pred[v]];
        in_tree[(size_t)a] = 1;
        T.pred[(size_t)v] = a;
        T.up[(size_t)v] = at[(size_t)a] == v;
        T.pi[(size_t)v] = T.up[(size_t)v] ? T.pi[(size_t)p] - ac[(size_t)a] : T.pi[(size_t)p] + ac[(size_t)a];
        T.depth[(size_t)v] = T.depth[(size_t)p] + 1;
        T.attach(v, p);
      }
      // the other artificial arcs exist but stay out of the basis (never priced)
      for (int32_t v = 0; v < N; ++v)
        if (v != init_root) { at[(size_t)(M + v)] = root; ah[(size_t)(M + v)] = v; }
      warm = true;
    } else {
      std::fill(flow.begin(), flow.end(), 0.0);
    }
  }
  res.warm_start = warm;
  if (!warm) artificial_start();
  double bf = 1.0;  // block = bf·√m (P:7076 uses √m); VR_MCF_BLOCK_FACTOR for experiments
  if (const char* e = std::getenv("VR_MCF_BLOCK_FACTOR")) bf = std::max(0.01, std::atof(e));
  const int64_t B = std::max<int64_t>(1, (int64_t)std::ceil(bf * std::sqrt((double)M)));
  int64_t next = 0;
  int32_t next_tail = 0;  // off[next_tail] <= next < off[next_tail + 1]
  while (next_tail < N && off[(size_t)next_tail + 1] <= 0) ++next_tail;
  std::vector<int32_t> path, stk;
  double t_price = 0, t_update = 0;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  // Pricing uses the float costs; when it finds no candidate, one full pass with the exact
  // costs confirms optimality (and pricing stays exact if that pass finds one).  Tree arcs
  // have reduced cost 0 up to rounding, far above -eps, so they need no membership test.
  bool exact_pricing = false;
  const double* pi = T.pi.data();
  for (;;) {
    const auto tp0 = now();
    // ---------------- block search pivot
    int64_t enter = -1;
    double best = -eps;
    int64_t scanned = 0;
    while (scanned < M) {
      int64_t left = std::min<int64_t>(B, M - scanned);
      scanned += left;
      while (left > 0) {
        const int64_t seg_end = std::min<int64_t>(off[(size_t)next_tail + 1], next + left);
        const double pit = pi[next_tail];
        if (exact_pricing) {
          for (int64_t j = next; j < seg_end; ++j) {
            const double r = ac[(size_t)j] + pit - pi[ah[(size_t)j]];
            if (r < best) { best = r; enter = j; }
          }
        } else {
          price_segment(c32.data(), ah.data(), pi, pit, next, seg_end, best, enter);
        }
        left -= seg_end - next;
        next = seg_end;
        if (next == off[(size_t)next_tail + 1]) {
          if (next == M) { next = 0; next_tail = 0; }
          while (next_tail < N && off[(size_t)next_tail + 1] <= next) ++next_tail;
        }
      }
      ++res.blocks;
      // the float cost may hide a tiny positive exact reduced cost: then keep searching
      if (enter >= 0 && !exact_pricing && ac[(size_t)enter] + pi[at[(size_t)enter]] - pi[ah[(size_t)enter]] >= -eps) {
        enter = -1;
        best = -eps;
      }
      if (enter >= 0) break;
    }
    if (enter < 0 && !exact_pricing) {
      exact_pricing = true;
      t_price += ms(tp0, now());
      continue;
    }
    const auto tp1 = now();
    t_price += ms(tp0, tp1);
    if (enter < 0) { res.optimal = true; break; }
    if (max_blocks > 0 && res.blocks >= max_blocks) break;
    // ---------------- cycle and leaving arc
    const int32_t p = at[(size_t)enter], q = ah[(size_t)enter];
    int32_t a1 = p, b1 = q;
    while (a1 != b1) {
      if (T.depth[(size_t)a1] >= T.depth[(size_t)b1]) a1 = T.parent[(size_t)a1];
      else b1 = T.parent[(size_t)b1];
    }
    const int32_t join = a1;
    double delta = std::numeric_limits<double>::infinity();
    int32_t leave_node = -1;  // the node whose pred arc leaves
    bool leave_on_p_side = false;
    // p side (walked from p up to the join = the cycle backwards): blocking if oriented
    // x -> parent(x); strict '<' keeps the one nearest p (last in cycle order)
    for (int32_t x = p; x != join; x = T.parent[(size_t)x]) {
      if (T.up[(size_t)x]) {
        const double f = flow[(size_t)T.pred[(size_t)x]];
        if (f < delta) { delta = f; leave_node = x; leave_on_p_side = true; }
      }
    }
    // q side (walked from q up to the join = the cycle forwards): blocking if oriented
    // parent(x) -> x; '<=' keeps the last one met, and beats a tie on the p side
    for (int32_t x = q; x != join; x = T.parent[(size_t)x]) {
      if (!T.up[(size_t)x]) {
        const double f = flow[(size_t)T.pred[(size_t)x]];
        if (f <= delta) { delta = f; leave_node = x; leave_on_p_side = false; }
      }
    }
    if (leave_node < 0) { res.unbounded = true; break; }  // a negative cycle of real arcs
    ++res.pivots;
    if (delta == 0) ++res.degenerate;
    // ---------------- flow update around the cycle
    if (delta > 0) {
      flow[(size_t)enter] += delta;
      for (int32_t x = p; x != join; x = T.parent[(size_t)x])
        flow[(size_t)T.pred[(size_t)x]] += T.up[(size_t)x] ? -delta : delta;
      for (int32_t x = q; x != join; x = T.parent[(size_t)x])
        flow[(size_t)T.pred[(size_t)x]] += T.up[(size_t)x] ? delta : -delta;
    }
    // ---------------- tree update: cut the leaving arc, re-hang its subtree from `enter`
    const int64_t leave_arc = T.pred[(size_t)leave_node];
    in_tree[(size_t)leave_arc] = 0;
    in_tree[(size_t)enter] = 1;
    const int32_t u_in = leave_on_p_side ? p : q;   // endpoint inside the cut subtree
    const int32_t v_in = leave_on_p_side ? q : p;   // endpoint outside
    // path u_in -> ... -> leave_node reverses its parent pointers
    path.clear();
    for (int32_t x = u_in;; x = T.parent[(size_t)x]) {
      path.push_back(x);
      if (x == leave_node) break;
    }
    T.detach(leave_node);
    for (size_t i = path.size() - 1; i >= 1; --i) {
      const int32_t x = path[i], y = path[i - 1];  // y is a child of x; x becomes a child of y
      T.detach(y);
      T.pred[(size_t)x] = T.pred[(size_t)y];
      T.up[(size_t)x] = !T.up[(size_t)y];
      T.attach(x, y);
    }
    T.pred[(size_t)u_in] = (int32_t)enter;
    T.up[(size_t)u_in] = at[(size_t)enter] == u_in;
    T.attach(u_in, v_in);
    // potentials and depths of the moved subtree (one DFS from u_in)
    stk.clear();
    stk.push_back(u_in);
    while (!stk.empty()) {
      const int32_t x = stk.back();
      stk.pop_back();
      const int32_t par = T.parent[(size_t)x];
      const int64_t a = T.pred[(size_t)x];
      T.pi[(size_t)x] = T.up[(size_t)x] ? T.pi[(size_t)par] - ac[(size_t)a] : T.pi[(size_t)par] + ac[(size_t)a];
      T.depth[(size_t)x] = T.depth[(size_t)par] + 1;
      for (int32_t c = T.first_child[(size_t)x]; c >= 0; c = T.next_sib[(size_t)c]) stk.push_back(c);
    }
    t_update += ms(tp1, now());
  }
  res.ms_pricing = t_price;
  res.ms_update = t_update;
  double total = 0;
  bool art = false;
  for (int64_t a = 0; a < M; ++a) total += ac[(size_t)a] * flow[(size_t)a];
  for (int64_t a = M; a < MA; ++a) art = art || flow[(size_t)a] > 0;
  res.cost = total;
  res.infeasible = res.optimal && art;
  return res;
}

}  // namespace vr

extern "C" int vr_min_cost_flow(int64_t nodes, const int64_t* supply, int64_t arcs, const int32_t* tail,
                                const int32_t* head, const double* cost, int64_t max_blocks, double* total_cost,
                                vr_mcf_stats* stats) {
  if (nodes < 0 || arcs < 0 || !total_cost || (nodes && !supply) || (arcs && (!tail || !head || !cost))) return VR_EINVAL;
  if (nodes + arcs >= INT32_MAX) return VR_ECAPACITY;  // tree arcs are indexed by int32
  int64_t sum = 0;
  for (int64_t v = 0; v < nodes; ++v) sum += supply[v];
  if (sum != 0) return VR_EINPUT;
  for (int64_t a = 0; a < arcs; ++a)
    if (tail[a] < 0 || tail[a] >= nodes || head[a] < 0 || head[a] >= nodes || !(cost[a] >= 0) || std::isinf(cost[a]))
      return VR_EINPUT;
  try {
    const vr::McfResult r = vr::network_simplex(nodes, supply, arcs, tail, head, cost, max_blocks, nullptr, -1);
    *total_cost = r.cost;
    if (stats) {
      stats->pivots = r.pivots;
      stats->degenerate = r.degenerate;
      stats->blocks = r.blocks;
      stats->optimal = r.optimal ? 1 : 0;
      stats->ms_pricing = r.ms_pricing;
      stats->ms_update = r.ms_update;
      stats->infeasible = r.infeasible ? 1 : 0;
    }
    if (r.unbounded || r.infeasible) return VR_EINPUT;
    return VR_OK;
  } catch (const std::bad_alloc&) {
    return VR_ECAPACITY;
  }
}
