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
#include <cmath>
#include <cstdint>
#include <limits>
#include <new>
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

}  // namespace

McfResult network_simplex(int64_t nodes, const int64_t* supply, int64_t arcs, const int32_t* tail, const int32_t* head,
                          const double* cost, int64_t max_blocks) {
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
  // arc arrays: real arcs 0..M-1, artificial arcs M..M+N-1 (node v's arc to/from the root)
  const int64_t MA = M + N;
  std::vector<int32_t> at(tail, tail + M), ah(head, head + M);
  std::vector<double> ac(cost, cost + M), flow((size_t)MA, 0.0);
  at.resize((size_t)MA);
  ah.resize((size_t)MA);
  ac.resize((size_t)MA, big);
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
  const int64_t B = std::max<int64_t>(1, (int64_t)std::ceil(std::sqrt((double)M)));
  int64_t next = 0;
  std::vector<int32_t> path, stk;
  auto rc = [&](int64_t a) { return ac[(size_t)a] + T.pi[(size_t)at[(size_t)a]] - T.pi[(size_t)ah[(size_t)a]]; };
  for (;;) {
    // ---------------- block search pivot
    int64_t enter = -1;
    double best = -eps;
    int64_t scanned = 0;
    while (scanned < M) {
      const int64_t len = std::min<int64_t>(B, M - scanned);
      for (int64_t k = 0; k < len; ++k) {
        const int64_t a = next;
        if (++next == M) next = 0;
        if (in_tree[(size_t)a]) continue;
        const double r = rc(a);
        if (r < best) { best = r; enter = a; }
      }
      scanned += len;
      ++res.blocks;
      if (enter >= 0) break;
    }
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
  }
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
    const vr::McfResult r = vr::network_simplex(nodes, supply, arcs, tail, head, cost, max_blocks);
    *total_cost = r.cost;
    if (stats) {
      stats->pivots = r.pivots;
      stats->degenerate = r.degenerate;
      stats->blocks = r.blocks;
      stats->optimal = r.optimal ? 1 : 0;
      stats->infeasible = r.infeasible ? 1 : 0;
    }
    if (r.unbounded || r.infeasible) return VR_EINPUT;
    return VR_OK;
  } catch (const std::bad_alloc&) {
    return VR_ECAPACITY;
  }
}
