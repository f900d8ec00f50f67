// ripser_style.cpp — a single-threaded, Ripser-style CPU run of the Vietoris–Rips barcode.
//
// BASELINE ONLY.  BASELINE.json's north_star asks for "a single-threaded Ripser-style CPU
// run timed on the box's own host cores in the same run (core count stated; a baseline,
// not the target)".  bench.py times this program next to the GPU path; tests/ check it
// against the oracle.  The product (paper_2502_05063_b200, libvr.so) never loads it, and it
// shares no code, header or table with the product or with oracle/.
//
// What it does: the CPU algorithm PAPER.md §5.2 describes for Ripser, the program the paper
// accelerates (each step cited):
//   * dimension 0 by union-find over the edges in filtration order (H0 via
//     a union-find / Kruskal pass, the merging edges are the dimension-0 pivots);
//   * dimensions d >= 1 by cohomology (§5.2.2, Thm 5.2.3) with clearing (§5.2.3,
//     Thm 5.2.6): the columns of dimension d are the d-simplices with diam <= t that were
//     not a pivot of dimension d-1, processed in reverse filtration order;
//   * the coboundary matrix is implicit (§5.2.5): a column's cofacets are enumerated from
//     its vertices through the combinatorial number system (Eq 5.6) and the
//     distance matrix; the reduction matrix V is stored and coboundaries are regenerated
//     from it (§5.2.5, "implicit matrix reduction");
//   * the working column is a binary heap with Z/2 cancellation of equal entries (§5.2.8);
//   * the emergent-pair shortcut (§5.2.7 / Def 5.2.8): the first cofacet of equal
//     diameter met in descending-index order is the column's pivot; if no earlier column
//     owns it, the pair is recorded without building the column;
//   * filtration order (§5.1.4): diameter ascending, combinatorial index
//     DEscending among equal diameters; the pivot of a coboundary column is its oldest
//     cofacet (smallest diameter, then largest index);
//   * the enclosing-radius threshold (Prop 5.2.13) is the caller's business: `threshold`
//     is inclusive, +inf means the full complex.
// Output: the positive-persistence pairs per dimension (birth < death), essential bars
// with death = +inf, plus counters and per-dimension times.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

namespace {

struct Entry {
  float diam;
  uint64_t cidx;
};
inline bool same(const Entry& a, const Entry& b) { return a.cidx == b.cidx; }
// heap order: the top is the oldest entry (smallest diameter, then largest index)
struct Younger {
  bool operator()(const Entry& a, const Entry& b) const {
    return a.diam > b.diam || (a.diam == b.diam && a.cidx < b.cidx);
  }
};
// column order: reverse filtration (largest diameter first, then smallest index)
inline bool col_before(const Entry& a, const Entry& b) {
  return a.diam > b.diam || (a.diam == b.diam && a.cidx < b.cidx);
}

struct Binom {
  int64_t n;
  int kmax;
  std::vector<uint64_t> t;  // t[k * (n + 1) + x] = C(x, k)
  Binom(int64_t n_, int kmax_) : n(n_), kmax(kmax_), t((size_t)(kmax_ + 1) * (size_t)(n_ + 1), 0) {
    for (int64_t x = 0; x <= n; ++x) {
      t[x] = 1;
      for (int k = 1; k <= kmax; ++k) t[(size_t)k * (n + 1) + x] = x == 0 ? 0 : at(x - 1, k - 1) + at(x - 1, k);
    }
  }
  uint64_t at(int64_t x, int k) const { return t[(size_t)k * (n + 1) + x]; }
};

// open-addressing map: pivot cidx -> column tag (the simplex's cidx for a column whose V
// is itself, else VTAG | index of its stored V column)
constexpr uint64_t EMPTY = ~0ull;
constexpr uint64_t VTAG = 1ull << 63;
struct PivotMap {
  std::vector<uint64_t> key, val;
  uint64_t mask = 0;
  size_t used = 0;
  void reset(size_t expect) {
    size_t cap = 16;
    while (4 * cap < 5 * expect + 64) cap <<= 1;  // load <= 0.8 when `expect` keys land
    key.assign(cap, EMPTY);
    val.assign(cap, 0);
    mask = cap - 1;
    used = 0;
  }
  static uint64_t mix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
  }
  bool find(uint64_t k, uint64_t* v) const {
    for (uint64_t h = mix(k) & mask;; h = (h + 1) & mask) {
      if (key[h] == k) {
        *v = val[h];
        return true;
      }
      if (key[h] == EMPTY) return false;
    }
  }
  void insert(uint64_t k, uint64_t v) {
    if (10 * (used + 1) > 9 * key.size()) grow();
    for (uint64_t h = mix(k) & mask;; h = (h + 1) & mask) {
      if (key[h] == EMPTY) {
        key[h] = k;
        val[h] = v;
        ++used;
        return;
      }
    }
  }
  void grow() {
    std::vector<uint64_t> ok, ov;
    ok.swap(key);
    ov.swap(val);
    reset(ok.size());
    for (size_t i = 0; i < ok.size(); ++i)
      if (ok[i] != EMPTY) insert(ok[i], ov[i]);
  }
};

struct Pairs {
  std::vector<float> birth, death;
};

struct Ripser {
  int64_t n;
  int max_dim;
  float thr;
  std::vector<float> D;  // full n x n, diagonal 0
  // sparse mode (thresholds keeping <= 1/4 of the edges, as Ripser's sparse distance
  // matrices): each vertex's neighbours under the threshold, descending — a cofacet vertex
  // must be a neighbour of every vertex of the simplex
  bool sparse = false;
  std::vector<std::vector<int>> nbr;
  Binom B;
  std::vector<Pairs> out;
  std::vector<int64_t> n_columns, n_emergent, n_reduced, n_simplices;
  std::vector<double> ms_dim;

  Ripser(const float* lt, int64_t n_, int md, float t)
      : n(n_), max_dim(md), thr(t), D((size_t)n_ * (size_t)n_, 0.0f), B(n_, md + 2), out(md + 1),
        n_columns(md + 1, 0), n_emergent(md + 1, 0), n_reduced(md + 1, 0), n_simplices(md + 2, 0),
        ms_dim(md + 1, 0.0) {
    for (int64_t i = 1; i < n; ++i)
      for (int64_t j = 0; j < i; ++j) D[(size_t)i * n + j] = D[(size_t)j * n + i] = lt[i * (i - 1) / 2 + j];
    int64_t kept = 0;
    for (int64_t i = 1; i < n; ++i)
      for (int64_t j = 0; j < i; ++j) kept += D[(size_t)i * n + j] <= thr;
    if (n > 64 && 4 * kept <= n * (n - 1) / 2) {
      sparse = true;
      nbr.assign((size_t)n, {});
      for (int64_t i = 0; i < n; ++i)
        for (int64_t w = n - 1; w >= 0; --w)
          if (w != i && D[(size_t)i * n + w] <= thr) nbr[(size_t)i].push_back((int)w);
    }
  }
  float dist(int64_t i, int64_t j) const { return D[(size_t)i * n + j]; }

  // vertices of a d-simplex (d + 1 of them, ascending) from its index (Eq 5.6, inverted
  // greedily from the top vertex down)
  void vertices(uint64_t idx, int d, int* v) const {
    int64_t hi = n;
    for (int k = d + 1; k >= 1; --k) {
      int64_t lo = k - 1, h = hi - 1;  // largest x in [lo, hi) with C(x, k) <= idx
      while (lo < h) {
        int64_t mid = (lo + h + 1) >> 1;
        if (B.at(mid, k) <= idx) lo = mid;
        else h = mid - 1;
      }
      v[k - 1] = (int)lo;
      idx -= B.at(lo, k);
      hi = lo;
    }
  }
  float diameter(const int* v, int d) const {
    float m = 0.0f;
    for (int a = 0; a <= d; ++a)
      for (int b = 0; b < a; ++b) m = std::max(m, dist(v[a], v[b]));
    return m;
  }

  // cofacets of the d-simplex s (vertices v) in descending index order, diam <= thr.
  // f(Entry) returns false to stop.
  template <class F>
  void cofacets(const Entry& s, const int* v, int d, F&& f) const {
    if (sparse) {
      cofacets_sparse(s, v, d, f);
      return;
    }
    uint64_t above = 0, below = s.cidx;  // index parts of the vertices above / below w
    int j = d;                           // v[0..j] are below w
    for (int64_t w = n - 1; w >= 0; --w) {
      while (j >= 0 && v[j] >= w) {
        if (v[j] == w) break;
        below -= B.at(v[j], j + 1);
        above += B.at(v[j], j + 2);
        --j;
      }
      if (j >= 0 && v[j] == w) {  // w is a vertex of s: move it above and skip
        below -= B.at(v[j], j + 1);
        above += B.at(v[j], j + 2);
        --j;
        continue;
      }
      float dm = s.diam;
      const float* row = &D[(size_t)w * n];
      for (int a = 0; a <= d; ++a) dm = std::max(dm, row[v[a]]);
      if (dm > thr) continue;
      Entry c{dm, above + B.at(w, j + 2) + below};
      if (!f(c)) return;
    }
  }

  // the same, w running over the neighbours of v[0] (descending) only
  template <class F>
  void cofacets_sparse(const Entry& s, const int* v, int d, F&& f) const {
    uint64_t above = 0, below = s.cidx;
    int j = d;
    for (int w : nbr[(size_t)v[0]]) {
      while (j >= 0 && v[j] > w) {  // vertices of s above w move to the upper part
        below -= B.at(v[j], j + 1);
        above += B.at(v[j], j + 2);
        --j;
      }
      if (j >= 0 && v[j] == w) continue;  // w is a vertex of s (it moves up at the next w)
      float dm = s.diam;
      const float* row = &D[(size_t)w * n];
      for (int a = 0; a <= d; ++a) dm = std::max(dm, row[v[a]]);
      if (dm > thr) continue;
      Entry c{dm, above + B.at(w, j + 2) + below};
      if (!f(c)) return;
    }
  }

  // ---------------------------------------------------------------- dimension 0
  std::vector<Entry> dim0(PivotMap& piv) {
    std::vector<Entry> edges;
    for (int64_t i = 1; i < n; ++i)
      for (int64_t j = 0; j < i; ++j) {
        float x = dist(i, j);
        if (x <= thr) edges.push_back(Entry{x, (uint64_t)(i * (i - 1) / 2 + j)});
      }
    n_simplices[0] = n;
    n_simplices[1] = (int64_t)edges.size();
    // filtration order: diameter ascending, index descending
    std::sort(edges.begin(), edges.end(), [](const Entry& a, const Entry& b) {
      return a.diam < b.diam || (a.diam == b.diam && a.cidx > b.cidx);
    });
    std::vector<int64_t> parent(n);
    for (int64_t i = 0; i < n; ++i) parent[i] = i;
    auto find = [&](int64_t x) {
      while (parent[x] != x) {
        parent[x] = parent[parent[x]];
        x = parent[x];
      }
      return x;
    };
    piv.reset(n);
    std::vector<Entry> cols;
    for (const Entry& e : edges) {
      int v[2];
      vertices(e.cidx, 1, v);
      int64_t a = find(v[0]), b = find(v[1]);
      if (a != b) {
        parent[std::max(a, b)] = std::min(a, b);
        piv.insert(e.cidx, 0);
        if (e.diam > 0.0f) {
          out[0].birth.push_back(0.0f);
          out[0].death.push_back(e.diam);
        }
      } else {
        cols.push_back(e);
      }
    }
    for (int64_t i = 0; i < n; ++i)
      if (find(i) == i) {
        out[0].birth.push_back(0.0f);
        out[0].death.push_back(INFINITY);
      }
    std::reverse(cols.begin(), cols.end());  // reverse filtration order
    return cols;
  }

  // ---------------------------------------------------------------- dimension d >= 1
  // reduce the coboundary columns `cols` (d-simplices, reverse filtration order); the
  // pivots (d+1-simplices) land in piv.
  void reduce(int d, const std::vector<Entry>& cols, PivotMap& piv) {
    piv.reset(cols.size());
    std::vector<Entry> vstore;            // stored V columns, concatenated
    std::vector<uint64_t> vbeg{0};        // column k = vstore[vbeg[k], vbeg[k+1])
    std::vector<Entry> heap, work;        // working coboundary, working V
    Younger younger;
    int vv[16], vu[16];
    auto push_cob = [&](const Entry& s, const int* v) {
      cofacets(s, v, d, [&](const Entry& c) {
        heap.push_back(c);
        std::push_heap(heap.begin(), heap.end(), younger);
        return true;
      });
    };
    auto pop_pivot = [&](Entry* p) {
      while (!heap.empty()) {
        std::pop_heap(heap.begin(), heap.end(), younger);
        Entry e = heap.back();
        heap.pop_back();
        if (!heap.empty() && same(heap.front(), e)) {  // two copies cancel over Z/2
          std::pop_heap(heap.begin(), heap.end(), younger);
          heap.pop_back();
          continue;
        }
        *p = e;
        return true;
      }
      return false;
    };
    for (const Entry& s : cols) {
      vertices(s.cidx, d, vv);
      // emergent shortcut: the first equal-diameter cofacet in descending index order
      bool emergent = false, found = false;
      Entry first{0.0f, 0};
      cofacets(s, vv, d, [&](const Entry& c) {
        if (c.diam == s.diam) {
          found = true;
          first = c;
          return false;
        }
        return true;
      });
      uint64_t tag;
      if (found && !piv.find(first.cidx, &tag)) emergent = true;
      if (emergent) {
        piv.insert(first.cidx, s.cidx);
        ++n_emergent[d];
        continue;
      }
      ++n_reduced[d];
      heap.clear();
      work.clear();
      work.push_back(s);
      push_cob(s, vv);
      Entry p;
      bool has = pop_pivot(&p);
      while (has && piv.find(p.cidx, &tag)) {
        // add the stored column: V_j's simplices, their coboundaries regenerated
        auto add = [&](const Entry& u) {
          vertices(u.cidx, d, vu);
          push_cob(u, vu);
          work.push_back(u);
        };
        if (tag & VTAG) {
          uint64_t k = tag & ~VTAG;
          for (uint64_t q = vbeg[k]; q < vbeg[k + 1]; ++q) add(vstore[q]);
        } else {
          vertices(tag, d, vu);
          add(Entry{diameter(vu, d), tag});
        }
        // p was popped: its partner copy from the added coboundary cancels it
        heap.push_back(p);
        std::push_heap(heap.begin(), heap.end(), younger);
        has = pop_pivot(&p);
      }
      if (!has) {  // zero column: essential class (Thm 5.2.6 keeps it unpaired)
        out[d].birth.push_back(s.diam);
        out[d].death.push_back(INFINITY);
        continue;
      }
      if (p.diam > s.diam) {
        out[d].birth.push_back(s.diam);
        out[d].death.push_back(p.diam);
      }
      // store V (Z/2-cancelled)
      std::sort(work.begin(), work.end(), [](const Entry& a, const Entry& b) { return a.cidx < b.cidx; });
      size_t w0 = vstore.size();
      for (size_t q = 0; q < work.size();) {
        size_t r = q;
        while (r < work.size() && work[r].cidx == work[q].cidx) ++r;
        if ((r - q) & 1) vstore.push_back(work[q]);
        q = r;
      }
      if (vstore.size() - w0 == 1 && vstore[w0].cidx == s.cidx) {
        vstore.pop_back();
        piv.insert(p.cidx, s.cidx);
      } else {
        vbeg.push_back(vstore.size());
        piv.insert(p.cidx, VTAG | (uint64_t)(vbeg.size() - 2));
      }
    }
  }

  // the (d+1)-simplices with diam <= thr, from the d-simplices (each cofacet generated once,
  // by appending a vertex above the top one); `cols` gets those that are not pivots.
  void assemble(int d, const std::vector<Entry>& simp, const PivotMap& piv, std::vector<Entry>* next,
                std::vector<Entry>* cols, bool keep_next) {
    int v[16];
    int64_t count = 0;
    std::vector<int> ws;
    for (const Entry& s : simp) {
      vertices(s.cidx, d, v);
      ws.clear();
      if (sparse) {
        for (int w : nbr[(size_t)v[d]])
          if (w > v[d]) ws.push_back(w);
      } else {
        for (int64_t w = v[d] + 1; w < n; ++w) ws.push_back((int)w);
      }
      for (int w : ws) {
        float dm = s.diam;
        const float* row = &D[(size_t)w * n];
        for (int a = 0; a <= d; ++a) dm = std::max(dm, row[v[a]]);
        if (dm > thr) continue;
        Entry c{dm, s.cidx + B.at(w, d + 2)};
        ++count;
        if (keep_next) next->push_back(c);
        uint64_t tag;
        if (!piv.find(c.cidx, &tag)) cols->push_back(c);
      }
    }
    n_simplices[d + 1] = count;
    std::sort(cols->begin(), cols->end(), col_before);
  }

  void run() {
    using clk = std::chrono::steady_clock;
    auto t0 = clk::now();
    PivotMap piv;
    std::vector<Entry> cols = dim0(piv);
    std::vector<Entry> simp;  // the d-simplices (diam <= thr), needed for the next assembly
    if (max_dim >= 1) {
      for (int64_t i = 1; i < n; ++i)
        for (int64_t j = 0; j < i; ++j)
          if (dist(i, j) <= thr) simp.push_back(Entry{dist(i, j), (uint64_t)(i * (i - 1) / 2 + j)});
    }
    auto t1 = clk::now();
    ms_dim[0] = std::chrono::duration<double, std::milli>(t1 - t0).count();
    for (int d = 1; d <= max_dim; ++d) {
      auto a = clk::now();
      n_columns[d] = (int64_t)cols.size();
      reduce(d, cols, piv);
      if (d < max_dim) {
        std::vector<Entry> next, ncols;
        assemble(d, simp, piv, &next, &ncols, d + 1 < max_dim);
        simp.swap(next);
        cols.swap(ncols);
      } else {
        cols.clear();
        cols.shrink_to_fit();
      }
      ms_dim[d] = std::chrono::duration<double, std::milli>(clk::now() - a).count();
    }
  }
};

}  // namespace

extern "C" {

// Returns an opaque handle (nullptr on bad arguments or out of memory).
void* rs_barcode(const float* lt, int64_t n, int max_dim, float threshold) {
  if (!lt || n < 1 || max_dim < 0 || max_dim > 8) return nullptr;
  try {
    Ripser* r = new Ripser(lt, n, max_dim, threshold);
    r->run();
    return r;
  } catch (const std::bad_alloc&) {
    return nullptr;
  }
}
int64_t rs_num_pairs(void* h, int dim) {
  Ripser* r = (Ripser*)h;
  return (dim < 0 || dim > r->max_dim) ? 0 : (int64_t)r->out[dim].birth.size();
}
void rs_get_pairs(void* h, int dim, float* birth, float* death) {
  Ripser* r = (Ripser*)h;
  const Pairs& p = r->out[dim];
  std::memcpy(birth, p.birth.data(), p.birth.size() * sizeof(float));
  std::memcpy(death, p.death.data(), p.death.size() * sizeof(float));
}
// counters[dim] = {columns, emergent, reduced, simplices (dim), ms}
void rs_stats(void* h, int dim, double* c5) {
  Ripser* r = (Ripser*)h;
  c5[0] = (double)r->n_columns[dim];
  c5[1] = (double)r->n_emergent[dim];
  c5[2] = (double)r->n_reduced[dim];
  c5[3] = (double)r->n_simplices[dim];
  c5[4] = r->ms_dim[dim];
}
void rs_free(void* h) { delete (Ripser*)h; }

}  // extern "C"
