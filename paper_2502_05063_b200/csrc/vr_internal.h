// vr_internal.h — host-side interfaces between the libvr translation units (not exported).
#pragma once
#include <algorithm>
#include <cstdint>
#include <functional>
#include <string>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/vr.h"
#include "vr_types.h"

namespace vr {

// ---------------------------------------------------------------- sort.cu
size_t scan_temp_bytes(size_t n);
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t n, void* temp, cudaStream_t st, int64_t* launches);
size_t radix_sort_temp_bytes(size_t n);
// the residual column keys ((maxr - rank) << cbits | cidx, significant bits < end_bit)
// into ascending order: *mode 1 = a counting sort on the rank field (bins = maxr + 1) + an
// in-place sort of every run of equal rank (short runs), 0 = a radix sort on all bits, -1 =
// try 1 and set *mode (one synchronisation); d_flag: a device word.  Returns the buffer
// holding the result (keys or alt).
uint64_t* sort_columns(uint64_t* keys, uint64_t* alt, size_t n, int cbits, int end_bit, uint64_t bins, void* temp,
                       void* cnt_temp, int* mode, unsigned int* d_flag, cudaStream_t st, int64_t* launches);
size_t sort_columns_temp_bytes(uint64_t bins);  // cnt_temp of sort_columns (bins = maxr + 1)
// merge of `world` ascending lists of `cap` keys each (gathered[r*cap ..], padded with ~0;
// keys distinct across lists) into out (the non-padding keys, ascending)
void merge_gathered_u64(const uint64_t* gathered, int world, uint64_t cap, uint64_t* out, cudaStream_t st, int64_t* launches);
uint64_t* radix_sort_u64(uint64_t* keys, uint64_t* alt, size_t n, int begin_bit, int end_bit, void* temp,
                         cudaStream_t st, int64_t* launches);

// ---------------------------------------------------------------- tables.cu (a0)
struct TablesOut {
  uint32_t err;        // nonzero: a NaN or negative distance was found
  uint32_t tbits;      // fp32 bits of the threshold actually applied
  uint64_t m_le_t;     // number of edges with d <= t
  uint32_t rbits_pad;
};
// keys64 (n(n-1)/2) and alt64 ping-pong buffers, rowmax (n), rank (n*n), out (device),
// tb_temp (tables_temp_bytes(n)); m_known = the edge count under t when known (replays), or
// -1 (the first run: read back after the compaction, one stream synchronisation)
// g (optional): also build the threshold-graph bitmap and degrees (output-sensitive mode)
size_t tables_temp_bytes(int64_t n);
struct GraphOut {
  uint32_t* bm;
  int nw;
  uint32_t* deg;
  uint32_t* deg_below;
};
void launch_tables(const float* d_lt, int64_t n, float threshold, uint64_t* keys64, uint64_t* alt64, uint32_t* rowmax,
                   void* sort_temp, void* tb_temp, uint32_t* rank, TablesOut* d_out, int64_t m_known, uint64_t** sorted_out,
                   cudaStream_t st, int64_t* launches, const GraphOut* g = nullptr);
void launch_build_binom(uint64_t* binom, int64_t n, int kmax, cudaStream_t st, int64_t* launches);

// ---------------------------------------------------------------- hot path kernels
struct DimParams {
  int d;               // column dimension
  int64_t n;
  uint32_t maxr;       // largest rank <= t
  int cbits;           // bits of cidx of d-simplices
  int steps;           // phase-1 cofacet steps
  int grab;            // prefix rows per atomic grab in k_enumerate
  int variant;         // phase-1 scan loop variant (0: vote per vertex, 1: per 4 vertices)
  int shard_rank = 0;  // interleaved row shard: rows r with (row_end-1-r) % shard_world == shard_rank
  int shard_world = 1;
  uint64_t row_begin, row_end;  // prefix rows [row_begin, row_end) of the d-simplices
  int win = 0;         // 1: k_enumerate stages the 32-vertex scan window in shared memory
  int slices = 1;      // k_enum_sparse2: work items per row (each takes every slices-th x)
};
struct DimCounters {   // device counters (unsigned long long each)
  unsigned long long survivors, apparent1, apparent2, cleared, queued, residual, row_next, app_pairs, scanned, scanned2, rows_out;
  unsigned long long next_bound;  // sparse: sum over survivors s of deg_below(min s) (bounds the next dimension)
  unsigned long long exported;    // sharded sparse: apparent cofacets appended to exp_list
  unsigned long long cand_reads;  // sparse: rank reads of the candidate examination (a1)
};
struct HotBuffers {
  uint64_t* qkey;        // phase-2 queue: column keys
  uint4* qvert;          // phase-2 queue: packed vertices (16 bits each, s[0] > ... > s[d])
  uint64_t qcap;
  uint64_t* resid;       // residual (non-apparent, non-cleared) column keys
  uint64_t rcap;
  const uint32_t* clr;   // clearing bitmap over the d-simplices, or nullptr (recompute mode)
  uint32_t* clr_next;    // bitmap of dimension d+1 receiving apparent cofacets, or nullptr
  const uint64_t* deaths;// recompute mode: sorted residual deaths of dimension d-1
  int64_t ndeaths;
  DimCounters* ctr;
  uint64_t* app_pairs;   // debug (index-level output): (s, t) per apparent pair, or nullptr
  uint64_t app_cap;
  // sparse mode where no bitmap over C(n, d+1) is kept: the d-simplex pivots of dimension
  // d-1 as a hash set with a Bloom filter in front (vr_common.cuh ClearSet)
  ClearSet clr_set;       // table == nullptr: none
  ClearSet clr_next_set;  // receives this dimension's apparent cofacets
  uint64_t* exp_list;     // sharded: this rank's apparent cofacets (for the other ranks' sets), or nullptr
  uint64_t exp_cap;
};
void launch_set_put(const uint64_t* list, int64_t m, const ClearSet& c, cudaStream_t st, int64_t* launches);
// returns the VR_KERNEL_* flags of the kernel launched (vr_stats.kernels)
int launch_enumerate(const DimParams& p, const uint32_t* rank, const uint64_t* binom, int kmax, const HotBuffers& B,
                     cudaStream_t st, int64_t* launches);
void launch_resolve(const DimParams& p, const uint32_t* rank, const uint64_t* binom, int kmax, const HotBuffers& B,
                    uint64_t qn, cudaStream_t st, int64_t* launches);
void launch_set_bits(const uint64_t* list, int64_t m, uint32_t* bm, cudaStream_t st, int64_t* launches);

// ---------------------------------------------------------------- sparse.cu (output-sensitive mode)
struct SparseRows {
  const uint32_t* bm;             // threshold-graph bitmap, n rows of nw words (bit w of row v: d(v,w) <= t, v != w)
  int32_t nw;                     // words per bitmap row: ceil(n / 32) rounded up to a multiple of 4 (zero padding)
  const uint4* rows_in;           // packed row simplices (single level: survivors of d-1; two levels: of d-2),
                                  // nullptr = the vertices
  uint4* rows_out;                // survivors of dimension d (rows of a later dimension), or nullptr
  uint64_t rows_out_cap;
  unsigned long long* rows_out_count;
  const uint32_t* deg_below;      // #{w < v adjacent to v} per vertex (DimCounters.next_bound)
};
// bitmap + deg(v) + deg_below(v) = #{w < v adjacent to v} from the rank matrix
// (nw: words per row, >= ceil(n/32); the words past the last vertex are written as zeros)
void launch_threshold_bitmap(const uint32_t* rank, int n, int nw, uint32_t* bm, uint32_t* deg, uint32_t* deg_below,
                             cudaStream_t st, int64_t* launches);
// residual_prep.cu: the packed neighbour ranks of the threshold graph for the host, and the
// residual columns' first equal-diameter cofacets + apparent claims (ResidualHints);
// bm = nullptr: dense mode (scans over the rank rows)
void launch_neighbour_ranks(const uint32_t* rank, int n, const uint32_t* bm, int nw, const uint32_t* deg,
                            uint32_t* counter, uint32_t* nb_pre, uint32_t* nb_rank, cudaStream_t st, int64_t* launches);
void launch_residual_hints(const uint32_t* rank, const uint64_t* binom, int n, int kmax, int d, const uint32_t* bm,
                           int nw, const uint64_t* keys, uint64_t nkeys, uint32_t maxr, int cbits, uint64_t* first,
                           uint8_t* claimed, cudaStream_t st, int64_t* launches);
// rows of k vertices (packed) -> out, ordered by their smallest vertex descending (the
// two-level kernel's rows, largest work first); keys/alt: n u64 each, temp:
// order_rows_temp_bytes(n)
size_t order_rows_temp_bytes(uint64_t n);
void launch_order_rows(int k, const uint4* rows, uint64_t n, uint64_t* keys, uint64_t* alt, void* temp, uint4* out,
                       cudaStream_t st, int64_t* launches);
// two_level (d >= 2): rows are (d-2)-simplices extended by two vertices (k_enum_sparse2)
void launch_enumerate_sparse(const DimParams& p, const uint32_t* rank, const uint64_t* binom, int kmax, const HotBuffers& B,
                             const SparseRows& S, bool two_level, cudaStream_t st, int64_t* launches);
void launch_resolve_sparse(const DimParams& p, const uint32_t* rank, const uint64_t* binom, int kmax, const HotBuffers& B,
                           const SparseRows& S, uint64_t qn, cudaStream_t st, int64_t* launches);

// ---------------------------------------------------------------- host.cpp (off-path)
struct HostPairs {
  std::vector<float> birth, death;               // death = +inf for essential classes
  std::vector<uint64_t> birth_cidx, death_cidx;  // death_cidx = UINT64_MAX for essential
  void push(float b, float d, uint64_t bc, uint64_t dc) {
    birth.push_back(b); death.push_back(d); birth_cidx.push_back(bc); death_cidx.push_back(dc);
  }
};
// Page-locked host array (cudaHostAlloc) from a process-wide cache, so the n*n rank
// matrix comes back at full PCIe/C2C bandwidth and the next call reuses the pages.
void* pinned_acquire(size_t& bytes);
// COO input -> dense lower triangle on the device (+inf = absent edge)
void launch_coo_to_dense(const int32_t* ii, const int32_t* jj, const float* dd, int64_t nnz, int64_t n, float* lt,
                         cudaStream_t st);
// message returned by vr_last_error() (thread-local)
void set_last_error(const std::string& msg);
// Per-(current device, key) memo, thread-safe: f runs once per device and its value is
// returned afterwards (function attributes, occupancy and cluster probes apply to the current
// device's context only) (vr_api.cu)
int device_memo(const void* key, const std::function<int()>& f);
// NCCL communicators over devices 0..G-1 of this process (comm.cu; empty on failure)
std::vector<vr_comm*> comm_nccl_all(int G);
// device blocks from the process-wide cache (vr_api.cu); bytes is rounded up on return
void* dev_acquire(size_t& bytes);
void dev_release(void* p, size_t bytes);
void pinned_release(void* p, size_t bytes);
template <class T>
class PinnedVec {
 public:
  PinnedVec() = default;
  PinnedVec(const PinnedVec&) = delete;
  PinnedVec& operator=(const PinnedVec&) = delete;
  PinnedVec(PinnedVec&& o) noexcept { swap(o); }
  PinnedVec& operator=(PinnedVec&& o) noexcept { if (this != &o) { reset(); swap(o); } return *this; }
  ~PinnedVec() { reset(); }
  void resize(size_t n) {  // contents are not preserved nor initialised
    if (n * sizeof(T) > cap_) {
      reset();
      size_t b = n * sizeof(T);
      p_ = (T*)pinned_acquire(b);
      cap_ = b;
    }
    n_ = n;
  }
  template <class It> void assign(It a, It b) {
    resize((size_t)(b - a));
    std::copy(a, b, p_);
  }
  T* data() { return p_; }
  const T* data() const { return p_; }
  size_t size() const { return n_; }
  bool empty() const { return n_ == 0; }
  T& operator[](size_t i) { return p_[i]; }
  const T& operator[](size_t i) const { return p_[i]; }
  void reset() {
    if (p_) pinned_release(p_, cap_);
    p_ = nullptr; n_ = 0; cap_ = 0;
  }

 private:
  void swap(PinnedVec& o) { std::swap(p_, o.p_); std::swap(n_, o.n_); std::swap(cap_, o.cap_); }
  T* p_ = nullptr;
  size_t n_ = 0, cap_ = 0;
};

struct HostMatrix {
  int64_t n = 0;
  std::vector<float> value;     // value[rank] = the fp32 distance with that rank
  PinnedVec<uint32_t> rank;     // n*n
  std::vector<uint64_t> binom;  // (kmax+1)*(n+1)
  int kmax = 0;
  // output-sensitive mode: the threshold graph as bitmap rows (bit v of row u = {u, v}
  // under the threshold; empty = dense scans of the rank matrix), bmw 64-bit words per row;
  // the scans take the AND of the simplex's rows (common neighbours).  The ranks of each
  // row's neighbours are packed in ascending neighbour order (a few MB: they stay in the
  // host caches, unlike the n*n matrix, which is then not copied at all), and per (row,
  // word) nb_pre is the index in nb_rank of the word's first neighbour:
  // R(u, v) = nb_rank[nb_pre[u*bmw + v/64] + popc(word bits below v)]
  // (built on the device by residual_prep.cu; build_neighbour_ranks is the tools' copy).
  std::vector<uint64_t> bm;
  int64_t bmw = 0;
  std::vector<uint32_t> nb_rank;
  std::vector<uint32_t> nb_pre;
  void build_neighbour_ranks() {
    nb_pre.assign(bm.size(), 0);
    nb_rank.clear();
    for (int64_t u = 0; u < n; ++u)
      for (int64_t w = 0; w < bmw; ++w) {
        nb_pre[(size_t)(u * bmw + w)] = (uint32_t)nb_rank.size();
        uint64_t x = bm[(size_t)(u * bmw + w)];
        while (x) {
          const int b = __builtin_ctzll(x);
          x &= x - 1;
          nb_rank.push_back(R(u, w * 64 + b));
        }
      }
  }
  uint64_t C(int64_t v, int k) const { return binom[(size_t)k * (size_t)(n + 1) + (size_t)v]; }
  uint32_t R(int64_t i, int64_t j) const { return rank[(size_t)i * (size_t)n + (size_t)j]; }
};
// Dim 0 (§5.2.5): union-find over the edges in filtration order.  edges_sorted are the
// edge keys sorted ascending by (fp32 bits << 32 | ~cidx) (filtration order), first m.
void dim0_union_find(int64_t n, const uint64_t* edges_sorted, uint64_t m, int kbits, HostPairs& out,
                     std::vector<uint64_t>& deaths_sorted);
// Residual reduction of the non-apparent, non-cleared columns of dimension d given in
// coboundary order (keys ascending).  mode 0 = reduction matrix (V), 1 = oblivious.
struct ResidualStats {
  int64_t emergent = 0, additions = 0, coboundaries = 0, apparent_checks = 0;
};
// Per residual column c (keys order): first[c] = cidx of the first equal-diameter cofacet t
// (the lex-greatest cofacet with diam(t) = diam(σ); UINT64_MAX if none) and claimed[c] = 1
// iff t is the apparent cofacet of some column (Def 5.3.4).  With them the emergent check
// (§5.2.11) is one pivot-table lookup instead of a coboundary scan.
struct ResidualHints {
  const uint64_t* first;
  const uint8_t* claimed;
};
// deaths: the pivots (death cidx) of the columns with one, in no particular order.
void residual_reduce(const HostMatrix& M, int d, uint32_t maxr, int cbits, const uint64_t* keys, uint64_t nkeys,
                     int mode, HostPairs& out, std::vector<uint64_t>& deaths, ResidualStats& st,
                     const ResidualHints* hints = nullptr);
// the hints on the host (checks, tools/residual_bench.cpp)
void residual_hints_host(const HostMatrix& M, int d, uint32_t maxr, int cbits, const uint64_t* keys, uint64_t nkeys,
                         uint64_t* first, uint8_t* claimed);

// HYPHA host phase (hypha_host.cpp): compression + reduction of the unstable columns;
// Lookup (row -> pivot column, -1) holds the GPU pivots on entry and every pivot on exit.
void hypha_host_reduce(const int64_t* col_ptr, const int32_t* rows, int64_t n, const int32_t* dims, int32_t flags,
                       const int32_t* Left, int32_t* Lookup, const uint8_t* stable, const int32_t* u, int64_t nu,
                       vr_hypha_stats& st);

// Uncapacitated min-cost flow, primal network simplex with block search (netsimplex.cpp).
struct McfResult {
  double cost = 0;
  int64_t pivots = 0, degenerate = 0, blocks = 0;
  bool optimal = false, infeasible = false, unbounded = false, warm_start = false;
  double ms_pricing = 0, ms_update = 0;
};
// init_pred / init_root (optional): a feasible spanning tree to start from (see the .cpp)
McfResult network_simplex(int64_t nodes, const int64_t* supply, int64_t arcs, const int32_t* tail, const int32_t* head,
                          const double* cost, int64_t max_blocks, const int32_t* init_pred = nullptr,
                          int32_t init_root = -1);

}  // namespace vr
