// hypha_host.cpp — the host phase of HYPHA (PAPER.md Ch.4): compression (Algs 8-9,
// P:4411-4476) and the reduction of the columns the GPU-scan left unstable (Alg 2 with
// the GPU pivots pre-claimed; twist order, Lemma 4.2.3, when dimensions are given).
//
// Differences from the paper's host phase (same pivots):
//  * compression is applied lazily: a row is tested (FIND-COMPRESSIBLE, memoized) and
//    dropped when it surfaces as the low of the working column, so columns that the twist
//    order zeroes by clearing are never compressed, and rows that never surface are never
//    searched;
//  * the columns are reduced by a thread pool speculatively with in-order commit (below)
//    instead of the spectral-sequence tiles of HYPHA-SS;
//  * rows of every known destroyer (a column with a pivot, incl. the pivots found here)
//    are dropped when they surface — the lemma behind compression (such a row is never a
//    pivot row) applied to the destroyers discovered on the host as well.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/vr.h"
#include "vr_internal.h"

namespace vr {
namespace {

}  // namespace

void hypha_host_reduce(const int64_t* col_ptr, const int32_t* rows, int64_t n, const int32_t* dims, int32_t flags,
                       const int32_t* Left, int32_t* Lookup, const uint8_t* stable, const int32_t* u, int64_t nu,
                       vr_hypha_stats& st) {
  auto tq00 = std::chrono::steady_clock::now();
  const bool compress = (flags & VR_HYPHA_COMPRESSION) != 0;
  const size_t N = (size_t)std::max<int64_t>(n, 1);
  // GPU pivots: Lookup[row] = column; every pivot column and every leftmost-1 column is a
  // destroyer (Lemma 4.2.5: a column holding the leftmost 1 of a row ends with a pivot)
  std::vector<uint8_t> destroyer(N, 0), C(compress ? N : 0, 0);
  std::vector<uint8_t> is_pivot_col(N, 0);
  for (int64_t r = 0; r < n; ++r)
    if (Lookup[r] >= 0) is_pivot_col[(size_t)Lookup[r]] = 1;
  int64_t cleared = 0;
  for (int64_t j = 0; j < n; ++j) cleared += stable[j] && !is_pivot_col[(size_t)j] && col_ptr[j + 1] > col_ptr[j];
  st.stable = n - nu;
  st.unstable = nu;
  st.cleared = cleared;
  if (compress)
    for (int64_t r = 0; r < n; ++r) {
      if (Left[r] >= 0 && Left[r] < n) destroyer[(size_t)Left[r]] = 1;
      if (is_pivot_col[(size_t)r]) destroyer[(size_t)r] = 1;
    }
  // ---------------- FIND-COMPRESSIBLE (Alg 9), evaluated lazily for the rows that surface
  // as a low, memoized, explicit stack.  C[r] = 1: r is a destroyer found by the scan
  // (column r holds a leftmost 1 or a GPU pivot), or r is the pivot row of a GPU-stable
  // column all of whose other entries are compressible (adding that column removes r and
  // only adds compressible entries); 2: not compressible.  The answer depends only on the
  // scan's results (destroyer0, the GPU pivots), so threads racing on one memo entry
  // store the same value.
  const std::vector<uint8_t> destroyer0 = destroyer;
  auto c_ld = [&](int32_t r) { return __atomic_load_n(&C[(size_t)r], __ATOMIC_RELAXED); };
  auto c_st = [&](int32_t r, uint8_t v) { __atomic_store_n(&C[(size_t)r], v, __ATOMIC_RELAXED); };
  auto compressible = [&](int32_t r0, std::vector<std::pair<int32_t, int64_t>>& stk) -> bool {
    if (uint8_t c = c_ld(r0)) return c == 1;
    stk.clear();
    stk.push_back({r0, -1});
    while (!stk.empty()) {
      auto& top = stk.back();
      const int32_t r = top.first;
      if (top.second < 0) {
        if (c_ld(r)) { stk.pop_back(); continue; }
        if (destroyer0[(size_t)r]) { c_st(r, 1); stk.pop_back(); continue; }
        const int32_t pc = __atomic_load_n(&Lookup[r], __ATOMIC_RELAXED);
        if (pc < 0 || !stable[pc]) { c_st(r, 2); stk.pop_back(); continue; }  // GPU pivots only
        top.second = col_ptr[pc];
      }
      const int32_t pc = __atomic_load_n(&Lookup[r], __ATOMIC_RELAXED);
      bool pushed = false, bad = false;
      while (top.second < col_ptr[pc + 1]) {
        const int32_t k = rows[top.second];
        const uint8_t ck = k == r ? 1 : c_ld(k);
        if (ck == 2) { bad = true; break; }
        if (ck == 1) { ++top.second; continue; }
        stk.push_back({k, -1});  // decide k first (`top` is invalid from here)
        pushed = true;
        break;
      }
      if (pushed) continue;
      c_st(r, bad ? 2 : 1);
      stk.pop_back();
    }
    return c_ld(r0) == 1;
  };

  auto tq0 = std::chrono::steady_clock::now();
  // ---------------- reduction of the unstable columns (twist order with dims, else left to right)
  std::vector<int32_t> order(u, u + nu);
  std::sort(order.begin(), order.end());
  if (dims) std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return dims[a] > dims[b]; });
  // first position of each column's dimension group: a column waits for the groups before
  // it (a higher dimension) to commit, so that twist clearing has been applied
  std::vector<int64_t> group_start((size_t)std::max<int64_t>(nu, 1), 0);
  for (int64_t i = 1; i < nu; ++i)
    group_start[(size_t)i] = (dims && dims[order[(size_t)i]] != dims[order[(size_t)i - 1]]) ? i : group_start[(size_t)i - 1];
  // reduced columns that ended with a pivot (and parked ones), by position in `order`
  std::vector<std::vector<int32_t>> R((size_t)std::max<int64_t>(nu, 1));
  std::vector<int32_t> pos_of(N);
  for (int64_t i = 0; i < nu; ++i) pos_of[(size_t)order[(size_t)i]] = (int32_t)i;
  std::vector<uint8_t> zeroed(N, 0);

  // Speculative parallel reduction with in-order commit: a worker reduces its column with
  // every pivot already claimed (all claimed by columns earlier in the order, or by the
  // GPU); a column reaching zero is final at once; a column whose low has no pivot is
  // parked (state 2) and the thread moves on.  The committer (whoever holds `commit_mu`)
  // walks the positions in order and finishes each parked column with every earlier
  // column final — re-reading the tables, adding what appeared meanwhile, then claiming
  // the low — so the pivots are exactly those of the sequential order.
  std::atomic<int64_t> next{0}, committed{0};
  std::vector<uint8_t> state((size_t)std::max<int64_t>(nu, 1), 0);  // 0 running, 1 final, 2 parked
  std::atomic<int64_t> additions{0}, compressed{0};
  std::mutex commit_mu;
  auto ld8 = [](const uint8_t* p) { return __atomic_load_n(p, __ATOMIC_RELAXED); };
  struct Scratch {
    std::vector<int32_t> W, tmp;  // working column, ascending rows (low = back)
    std::vector<std::pair<int32_t, int64_t>> stk;  // FIND-COMPRESSIBLE's stack
    int64_t add = 0, comp = 0;
  };
  auto add_col = [](Scratch& sc, const int32_t* b, size_t nb) {
    auto& W = sc.W;
    auto& tmp = sc.tmp;
    tmp.clear();
    size_t i = 0, k = 0;
    while (i < W.size() && k < nb) {
      if (W[i] < b[k]) tmp.push_back(W[i++]);
      else if (W[i] > b[k]) tmp.push_back(b[k++]);
      else { ++i; ++k; }
    }
    tmp.insert(tmp.end(), W.begin() + (ptrdiff_t)i, W.end());
    tmp.insert(tmp.end(), b + k, b + nb);
    W.swap(tmp);
  };
  // reduce sc.W (column j) against the claimed pivots; returns the low without a pivot
  // (-1: the column is zero)
  auto reduce = [&](Scratch& sc, int32_t j) -> int32_t {
    (void)j;
    auto& W = sc.W;
    while (!W.empty()) {
      const int32_t lo = W.back();
      if (compress && (ld8(&destroyer[(size_t)lo]) || compressible(lo, sc.stk))) {
        W.pop_back();  // compression (Lemma 4.2.4): never a pivot row / eliminable
        ++sc.comp;
        continue;
      }
      const int32_t k = __atomic_load_n(&Lookup[lo], __ATOMIC_ACQUIRE);
      if (k < 0) return lo;
      if (stable[k]) add_col(sc, rows + col_ptr[k], (size_t)(col_ptr[k + 1] - col_ptr[k]));
      else {
        const auto& rk = R[(size_t)pos_of[(size_t)k]];
        add_col(sc, rk.data(), rk.size());
      }
      ++sc.add;
    }
    return -1;
  };
  auto try_commit = [&](Scratch& sc) {
    std::unique_lock<std::mutex> lk(commit_mu, std::try_to_lock);
    if (!lk.owns_lock()) return;
    int64_t c = committed.load(std::memory_order_relaxed);
    while (c < nu) {
      const uint8_t s8 = __atomic_load_n(&state[(size_t)c], __ATOMIC_ACQUIRE);
      if (s8 == 0) break;
      if (s8 == 2) {  // finish a parked column: every earlier column is final
        const int32_t j = order[(size_t)c];
        sc.W.assign(R[(size_t)c].begin(), R[(size_t)c].end());
        const int32_t lo = reduce(sc, j);
        if (lo >= 0) {
          R[(size_t)c] = sc.W;
          if (compress) __atomic_store_n(&destroyer[(size_t)j], (uint8_t)1, __ATOMIC_RELAXED);
          if (dims) __atomic_store_n(&zeroed[(size_t)lo], (uint8_t)1, __ATOMIC_RELAXED);  // Lemma 4.2.3
          __atomic_store_n(&Lookup[lo], j, __ATOMIC_RELEASE);
        } else {
          R[(size_t)c].clear();
        }
      }
      committed.store(++c, std::memory_order_release);
    }
  };
  auto worker = [&]() {
    Scratch sc;
    for (;;) {
      const int64_t i = next.fetch_add(1, std::memory_order_relaxed);
      if (i >= nu) break;
      const int32_t j = order[(size_t)i];
      // a column of a lower dimension starts after the higher one has committed (twist)
      for (int spins = 0; committed.load(std::memory_order_acquire) < group_start[(size_t)i];) {
        try_commit(sc);
        if (++spins > 64) std::this_thread::yield();
      }
      uint8_t s8 = 1;
      if (!ld8(&zeroed[(size_t)j])) {  // twist: cleared by a pivot of a higher dimension
        sc.W.assign(rows + col_ptr[j], rows + col_ptr[j + 1]);
        if (reduce(sc, j) >= 0) {
          R[(size_t)i] = sc.W;  // park (a copy: the scratch keeps its capacity)
          s8 = 2;
        }
      }
      __atomic_store_n(&state[(size_t)i], s8, __ATOMIC_RELEASE);
      try_commit(sc);
    }
    for (int spins = 0; committed.load(std::memory_order_acquire) < nu;) {  // drain the parked tail
      try_commit(sc);
      if (++spins > 64) std::this_thread::yield();
    }
    additions += sc.add;
    compressed += sc.comp;
  };
  int nthreads = (int)std::min<unsigned>(16u, std::max(1u, std::thread::hardware_concurrency()));
  if (const char* e = std::getenv("VR_HYPHA_THREADS")) nthreads = std::max(1, std::atoi(e));
  if (nu < 4096) nthreads = 1;
  std::vector<std::thread> pool;
  for (int t = 1; t < nthreads; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
  st.ms_compress_scan = std::chrono::duration<double, std::milli>(tq0 - tq00).count();
  st.ms_reduce = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tq0).count();
  st.threads = nthreads;
  st.additions = additions.load();
  st.compressed = compressed.load();
}

}  // namespace vr
