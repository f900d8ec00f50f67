// vr_api.cu — the C ABI declared in include/vr.h and the per-call orchestration.
//
// Per call (SURVEY.md §3 "New vr_barcodes"):
//   a0  tables on the device (tables.cu): edge keys + radix sort, enclosing radius,
//       threshold, rank matrix; binomial table (host-built, copied once)
//   dim 0 on the host (union-find over the sorted edges, §5.2.5) -> death edges
//   for d = 1..max_dim:
//       k_enumerate (a1 + a5 phase 1 + a3)   -> queue of non-proven columns
//       k_resolve   (a5 phase 2 + a2 + a6)   -> residual columns (non-apparent, non-cleared)
//       radix sort of the residual columns into coboundary order (a4)
//       host residual reduction (off path)    -> pairs of dim d, deaths for d+1
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/vr.h"
#include "vr_common.cuh"
#include "vr_internal.h"

namespace {

thread_local std::string g_err;

struct VrError : std::runtime_error {
  int code;
  VrError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CUDA_TRY(x)                                                                                 \
  do {                                                                                              \
    cudaError_t e_ = (x);                                                                           \
    if (e_ != cudaSuccess) {                                                                        \
      int code_ = (e_ == cudaErrorMemoryAllocation) ? VR_ECAPACITY : VR_EDEVICE;                    \
      throw VrError(code_, std::string(#x) + ": " + cudaGetErrorString(e_));                        \
    }                                                                                               \
  } while (0)

// Process-wide cache of device blocks: cudaMalloc/cudaFree cost milliseconds each (and
// cudaFree synchronises the device), so a plan's buffers go back to this cache when the
// plan is freed and the next call of the same shape reuses them.  Best fit within 25% of
// the request; on an allocation failure the cache is emptied and the allocation retried.
class DevCache {
 public:
  static DevCache& get() {
    static DevCache c;
    return c;
  }
  void* alloc(size_t& b) {
    b = round(b);
    int dev = 0;
    cudaGetDevice(&dev);
    {
      std::lock_guard<std::mutex> g(mu_);
      auto it = free_.lower_bound(Key{dev, b});
      if (it != free_.end() && it->first.dev == dev && it->first.bytes <= b + b / 4) {
        void* p = it->second;
        b = it->first.bytes;
        cached_ -= b;
        free_.erase(it);
        return p;
      }
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, b);
    if (e != cudaSuccess) {
      cudaGetLastError();
      trim(dev);
      CUDA_TRY(cudaMalloc(&p, b));
    }
    return p;
  }
  void release(void* p, size_t b, int dev) {  // dev: the device the block was allocated on
    std::lock_guard<std::mutex> g(mu_);
    if (cached_ + b > kCap) {
      int cur = 0;
      cudaGetDevice(&cur);
      if (cur != dev) cudaSetDevice(dev);
      cudaFree(p);
      if (cur != dev) cudaSetDevice(cur);
      return;
    }
    free_.emplace(Key{dev, b}, p);
    cached_ += b;
  }
  void trim(int dev) {  // (called with `dev` current)
    std::lock_guard<std::mutex> g(mu_);
    for (auto it = free_.begin(); it != free_.end();) {
      if (it->first.dev == dev) {
        cudaFree(it->second);
        cached_ -= it->first.bytes;
        it = free_.erase(it);
      } else {
        ++it;
      }
    }
  }

 private:
  struct Key {
    int dev;
    size_t bytes;
    bool operator<(const Key& o) const { return dev != o.dev ? dev < o.dev : bytes < o.bytes; }
  };
  static size_t round(size_t b) {
    if (b < 256) return 256;
    if (b < (2u << 20)) return (b + 255) & ~(size_t)255;
    return (b + (2u << 20) - 1) & ~(size_t)((2u << 20) - 1);
  }
  static constexpr size_t kCap = (size_t)48 << 30;  // at most 48 GiB kept cached
  std::mutex mu_;
  std::multimap<Key, void*> free_;
  size_t cached_ = 0;
};

}  // namespace

namespace vr {
// pinned host blocks: exact-size reuse (the same workload repeats its shapes)
namespace {
std::mutex g_pin_mu;
std::multimap<size_t, void*> g_pin_free;
size_t g_pin_cached = 0;
constexpr size_t kPinCap = (size_t)16 << 30;
}  // namespace
void* pinned_acquire(size_t& bytes) {
  bytes = (bytes + 4095) & ~(size_t)4095;
  {
    std::lock_guard<std::mutex> g(g_pin_mu);
    auto it = g_pin_free.lower_bound(bytes);
    if (it != g_pin_free.end() && it->first <= bytes + bytes / 4) {
      void* p = it->second;
      bytes = it->first;
      g_pin_cached -= bytes;
      g_pin_free.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    p = std::malloc(bytes);  // pageable fallback (still correct, slower copies)
    if (!p) throw std::bad_alloc();
    bytes |= 1;              // low bit marks a malloc block
  }
  return p;
}
void pinned_release(void* p, size_t bytes) {
  if (bytes & 1) { std::free(p); return; }
  std::lock_guard<std::mutex> g(g_pin_mu);
  if (g_pin_cached + bytes > kPinCap) { cudaFreeHost(p); return; }
  g_pin_free.emplace(bytes, p);
  g_pin_cached += bytes;
}
}  // namespace vr

namespace {

}  // namespace

namespace vr {
void set_last_error(const std::string& msg) { g_err = msg; }
int device_memo(const void* key, const std::function<int()>& f) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> memo;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  auto it = memo.find({dev, key});
  if (it != memo.end()) return it->second;
  const int v = f();
  memo[{dev, key}] = v;
  return v;
}
void* dev_acquire(size_t& bytes) { return DevCache::get().alloc(bytes); }
void dev_release(void* p, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  DevCache::get().release(p, bytes, dev);
}
}  // namespace vr

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int dev = 0;  // the device the block belongs to
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes), dev(o.dev) { o.p = nullptr; o.bytes = 0; }  // (vector<DimRun>)
  DevBuf& operator=(DevBuf&&) = delete;
  ~DevBuf() { release(); }
  // the owner must have synchronised the stream that used the buffer; the block goes back
  // to the cache under its own device, whatever device is current
  void release() {
    if (p) DevCache::get().release(p, bytes, dev);
    p = nullptr;
    bytes = 0;
  }
  void ensure(size_t b) {
    if (b <= bytes && p) return;
    release();
    if (b == 0) b = 16;
    cudaGetDevice(&dev);
    p = DevCache::get().alloc(b);
    bytes = b;
  }
  template <class T> T* as() const { return (T*)p; }
};

int bits_for(uint64_t x) {
  int b = 0;
  while (b < 64 && (x >> b) != 0) ++b;
  return b ? b : 1;
}

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

struct Chunk {
  uint64_t row_begin, row_end, queued;
};

struct DimRun {
  vr::DimParams p{};
  std::vector<Chunk> chunks;
  uint64_t residual = 0;
  int sort_bits = 0;
  DevBuf deaths_in;  // sorted death cidx of dimension d-1 (clearing input)
  int64_t ndeaths_in = 0;
  DevBuf clr;        // clearing bitmap over the d-simplices (empty: recompute mode)
  size_t clr_words = 0;
  DevBuf hash, bloom;  // sparse mode without a bitmap: the clearing set (ClearSet) of d
  uint64_t hash_mask = 0;  // slots - 1; 0 = no set (recompute mode)
  uint32_t bloom_words = 0;
  bool two_level = false;  // sparse: k_enum_sparse2 (rows = survivors of d-2)
  int sort_mode = -1;      // residual-key sort: 1 rank bits + runs, 0 all bits (decided by the first run)
  // sharded runs (recorded by the first run, reused by replays): the largest per-rank count
  // of residual keys and of exported apparent cofacets, this rank's exported count, the sum
  std::vector<uint64_t> x_counts;
  uint64_t x_cap = 0, x_total = 0, exp_cap = 0, exp_local = 0;
  // algorithmic work of the first run: rank reads of
  // the enumeration (a1) and of the apparent test (a5, both phases), decode compares
  double reads_a1 = 0, reads_a5 = 0, reads_a5_phase2 = 0, decode = 0, decode_phase2 = 0;
  int64_t kernels = 0;
  bool active = false;
};

}  // namespace

struct vr_result {
  int32_t max_dim = 0;
  float tused = 0.0f;
  std::vector<std::vector<vr_pair>> pairs;
  std::vector<std::vector<vr_index_pair>> ipairs;
  std::vector<vr_stats> stats;
};

struct vr_plan {
  std::unique_ptr<vr_result> R{new vr_result()};
  vr::HostMatrix M;                  // host copies for the off-path steps
  std::vector<vr::HostPairs> hp;     // pairs per dimension
  std::vector<uint64_t> deaths;      // deaths of the last finished dimension
  int rbits = 1;
  cudaEvent_t ev[8] = {};
  uint64_t* local_sorted = nullptr;  // this rank's sorted residual keys of the last dimension run
  int32_t rank_id = 0, world = 1;    // shard of the rows (distributed driver)
  const vr_comm* comm = nullptr;     // the ranks' transport (world > 1)
  DevBuf x_counts, x_send, x_gather, x_merged, x_exp, x_expg, x_ser;  // exchange buffers
  int64_t n = 0;
  int32_t D = 0;
  float threshold = 0.0f;
  vr_options opt{};
  cudaStream_t st = nullptr;
  const float* d_lt = nullptr;
  uint64_t N = 0;
  int kbits = 1, kmax = 0;
  DevBuf rank, binom, keys, alt, rowmax, sort_tmp, tb_tmp, sort_flag, cnt_tmp, tout, ctrs, queue, qvert, resid, resid_alt, app_pairs, lt_copy;
  uint64_t qcap = 0, rcap = 0, app_cap = 0;
  uint32_t maxr = 0;
  uint64_t m = 0;
  std::vector<DimRun> dims;  // index d (1..D), dims[0] unused
  // output-sensitive mode: threshold-graph CSR and per-dimension survivor lists
  bool sparse = false;
  DevBuf bm, deg, deg_below, bound;  // threshold-graph bitmap (n x nw words), degrees
  int32_t nw = 0;
  DevBuf nb_pre, nb_rank, nb_ctr;     // packed neighbour ranks for the host (residual_prep.cu)
  DevBuf ord_keys, ord_alt, ord_tmp, ord_rows;  // two-level rows ordered by work (order_rows)
  int ord_dim = -1;                   // the dimension whose rows ord_rows holds
  // replay: the ordering of dimension d's rows runs on a side stream as soon as dimension
  // d-2 has written them, overlapping dimension d-1 (VR_NO_SIDE_ORDER: in line)
  cudaStream_t st_side = nullptr;
  cudaEvent_t ev_rows_ready = nullptr, ev_order_done = nullptr;
  int side_dim = -1;
  DevBuf h_first, h_claimed;          // residual hints of the current dimension
  std::vector<DevBuf> rows;           // rows[d] = packed d-simplex survivors (rows of d+1)
  std::vector<uint64_t> rows_count;   // survivors written per dimension
  std::vector<uint64_t> rows_cap;
  std::vector<uint64_t> next_bound;   // per dimension: sum over its survivors s of deg_below(min s)
  int64_t survivors_total = 0;
  int64_t apparent_total = 0, residual_total = 0;
  int64_t launches = 0;
  // work counters of the first run (for the roofline accounting)
  double work_candidates = 0, work_scanned = 0, work_rank_ops = 0, work_scanned2 = 0, work_rank_ops2 = 0;
  // replay timing: event pairs per stage (0 tables, 1 enumerate, 2 resolve, 3 sort)
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> stage_ev[4];
  std::vector<int> stage_dim[4];  // dimension of each event pair (0: tables; -d: per-dimension setup)
  int used_events[4] = {0, 0, 0, 0};
  ~vr_plan() {
    if (st) cudaStreamSynchronize(st);  // the device buffers go back to DevCache
    if (st_side) {
      cudaStreamSynchronize(st_side);
      cudaStreamDestroy(st_side);
    }
    if (ev_rows_ready) cudaEventDestroy(ev_rows_ready);
    if (ev_order_done) cudaEventDestroy(ev_order_done);
    for (auto& v : stage_ev)
      for (auto& e : v) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }
  uint32_t* clr_of(int d) {
    return (d >= 1 && d <= D && dims[(size_t)d].clr_words) ? dims[(size_t)d].clr.as<uint32_t>() : nullptr;
  }
  vr::ClearSet set_of(int d) {
    vr::ClearSet c{nullptr, 0, nullptr, 1};
    if (d >= 1 && d <= D && dims[(size_t)d].hash_mask) {
      c.table = dims[(size_t)d].hash.as<uint64_t>();
      c.mask = dims[(size_t)d].hash_mask;
      c.bloom = dims[(size_t)d].bloom.as<uint32_t>();
      c.bloom_words = dims[(size_t)d].bloom_words;
    }
    return c;
  }
  // the clearing-set fields of dimension d's HotBuffers
  void hash_fields(vr::HotBuffers& B, int d) {
    B.clr_set = set_of(d);
    B.clr_next_set = set_of(d + 1);
    // sharded: the apparent cofacets also go to the export list for the other ranks' sets
    B.exp_list = (world > 1 && B.clr_next_set.table) ? x_exp.as<uint64_t>() : nullptr;
    B.exp_cap = B.exp_list ? x_exp.bytes / 8 : 0;
  }
  // (the table is sized by the row bound, 2x rounded up to a power of two: most probes are
  // misses, and a low load keeps the few that reach it at one slot)
  void hash_reset(int d, cudaStream_t s) {
    const vr::ClearSet c = set_of(d);
    if (!c.table) return;
    cudaMemsetAsync(c.table, 0xFF, (c.mask + 1) * 8, s);
    cudaMemsetAsync(c.bloom, 0, (size_t)c.bloom_words * 4, s);
  }
  void hash_deaths(int d, cudaStream_t s) {  // deaths of dimension d-1 (deaths_in of d) into d's set
    const vr::ClearSet c = set_of(d);
    if (c.table) vr::launch_set_put(dims[(size_t)d].deaths_in.as<uint64_t>(), dims[(size_t)d].ndeaths_in, c, s, &launches);
  }
  // rows of dimension d: single level — the survivors of d-1 (vertices for d = 1); two
  // levels — the survivors of d-2 (vertices for d = 2).  Dimension d keeps its survivors
  // when a later dimension reads them as rows (rows_needed).
  bool rows_needed(int d) const {
    for (int k = d + 1; k <= D && k <= d + 2; ++k)
      if ((dims[(size_t)k].two_level ? k - 2 : k - 1) == d) return true;
    return false;
  }
  // Two-level rows of dimension d >= 3 (the survivors of d-2) ordered by their smallest
  // vertex, descending: the largest rows first (sparse.cu, launch_order_rows).
  // VR_NO_ROW_ORDER: the order the previous kernel wrote them in.
  void order_rows(int d, cudaStream_t s) {
    ord_dim = -1;
    if (!sparse || d < 3 || !dims[(size_t)d].two_level || std::getenv("VR_NO_ROW_ORDER")) return;
    const uint64_t nr = rows_count[(size_t)d - 2];
    if (nr < 2 || nr >= (1ull << 32)) return;
    ord_keys.ensure((size_t)nr * 8);
    ord_alt.ensure((size_t)nr * 8);
    ord_tmp.ensure(vr::order_rows_temp_bytes(nr));
    ord_rows.ensure((size_t)nr * 16);
    vr::launch_order_rows(d - 1, rows[(size_t)d - 2].as<uint4>(), nr, ord_keys.as<uint64_t>(), ord_alt.as<uint64_t>(),
                          ord_tmp.p, ord_rows.as<uint4>(), s, &launches);
    ord_dim = d;
  }
  vr::SparseRows sparse_rows(int d, vr::DimCounters* ctr) {
    vr::SparseRows SR{};
    if (sparse) {
      SR.bm = bm.as<uint32_t>();
      SR.nw = nw;
      const int src = dims[(size_t)d].two_level ? d - 2 : d - 1;
      SR.rows_in = src <= 0 ? nullptr : (ord_dim == d ? ord_rows.as<uint4>() : rows[(size_t)src].as<uint4>());
      const bool keep = rows_needed(d);
      SR.rows_out = keep ? rows[(size_t)d].as<uint4>() : nullptr;
      SR.rows_out_cap = keep ? rows_cap[(size_t)d] : 0;
      SR.rows_out_count = &ctr->rows_out;
      SR.deg_below = deg_below.as<uint32_t>();
    }
    return SR;
  }
};

namespace {

const int kDefaultSteps = 32;
const size_t kMaxBitmapBytes = (size_t)4 << 30;
const size_t kSparseBitmapBytes = (size_t)64 << 20;

uint64_t binom_host(uint64_t n, uint64_t k) {
  if (k > n) return 0;
  unsigned __int128 c = 1;
  for (uint64_t i = 1; i <= k; ++i) {
    c = c * (n - k + i) / i;
    if (c > ((unsigned __int128)1 << 64) - 1) return UINT64_MAX;
  }
  return (uint64_t)c;
}

void check_args(const void* lt, int64_t n, int32_t max_dim, float threshold) {
  if (n < 1) throw VrError(VR_EINVAL, "n must be >= 1");
  if (max_dim < 0 || max_dim > VR_MAX_DIM) throw VrError(VR_EINVAL, "max_dim must be in [0, VR_MAX_DIM]");
  if (std::isnan(threshold) || threshold < 0) throw VrError(VR_EINVAL, "threshold must be >= 0 or +inf");
  if (n >= 2 && !lt) throw VrError(VR_EINVAL, "dist_lower_tri is NULL");
  if (n > 65535) throw VrError(VR_ECAPACITY, "n > 65535 is not supported (rank matrix layout)");
  // C(n, max_dim + 2) < 2^63: every cofacet index must fit a signed 64-bit
  for (int k = 1; k <= max_dim + 2; ++k) {
    uint64_t c = binom_host((uint64_t)n, (uint64_t)k);
    if (c == UINT64_MAX || c >= (1ull << 63))
      throw VrError(VR_ECAPACITY, "C(n, max_dim+2) >= 2^63: simplex indices do not fit 64 bits");
  }
}

// Debug aid: write the inputs of residual_reduce for dimension d (tools/residual_bench).
void dump_residual(const char* dir, const vr::HostMatrix& M, int d, uint32_t maxr, int cbits,
                   const std::vector<uint64_t>& keys) {
  std::string base = std::string(dir) + "/";
  auto wr = [&](const std::string& f, const void* p, size_t b) {
    FILE* fp = std::fopen((base + f).c_str(), "wb");
    if (!fp) return;
    std::fwrite(p, 1, b, fp);
    std::fclose(fp);
  };
  if (d == 1) {
    wr("rank.bin", M.rank.data(), M.rank.size() * 4);
    wr("values.bin", M.value.data(), M.value.size() * 4);
  }
  wr("keys_d" + std::to_string(d) + ".bin", keys.data(), keys.size() * 8);
  FILE* fp = std::fopen((base + "meta_d" + std::to_string(d) + ".txt").c_str(), "w");
  if (fp) {
    std::fprintf(fp, "%lld %d %u %d %d\n", (long long)M.n, d, maxr, cbits, M.kmax);
    std::fclose(fp);
  }
}

struct SectionTimer {
  bool on = std::getenv("VR_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[vr] %-28s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// ------------------------------------------------------------------ the run, in stages
// stage_setup        binomials, a0 tables, host copies, dimension 0, sparse host graph,
//                    clearing bitmaps, dimension-1 clearing input
// stage_dim_local    this rank's shard of dimension d on the device (enumerate, apparent,
//                    clearing, compaction, local radix sort); leaves the sorted residual
//                    keys on the device
// stage_dim_finish   the host residual reduction of dimension d on the (merged) residual
//                    columns; deaths -> clearing input of d+1
// stage_result       barcode assembly
// A single-GPU run calls them in sequence; the distributed driver (paper_2502_05063_b200/
// dist.py) interleaves the two exchanges of SURVEY.md §8(e) between local and finish.
// ------------------------------------------------------------------ collectives (sharded runs)
void comm_ok(int rc, const char* what) {
  if (rc) throw VrError(rc, std::string(what) + ": " + g_err);
}
// every rank's value v (host), in rank order
std::vector<uint64_t> gather_u64(vr_plan& P, uint64_t v) {
  const int W = P.world;
  P.x_counts.ensure((size_t)(W + 1) * 8);
  uint64_t* d = P.x_counts.as<uint64_t>();
  CUDA_TRY(cudaMemcpyAsync(d, &v, 8, cudaMemcpyHostToDevice, P.st));
  comm_ok(P.comm->allgather_u64(P.comm->ctx, d, d + 1, 1, P.st), "all-gather (counts)");
  std::vector<uint64_t> all((size_t)W);
  CUDA_TRY(cudaMemcpyAsync(all.data(), d + 1, (size_t)W * 8, cudaMemcpyDeviceToHost, P.st));
  CUDA_TRY(cudaStreamSynchronize(P.st));
  return all;
}
// rank 0's host words to every rank (the count first)
void bcast_words(vr_plan& P, std::vector<uint64_t>& w) {
  P.x_counts.ensure((size_t)(P.world + 1) * 8);
  uint64_t* c = P.x_counts.as<uint64_t>();
  uint64_t n = w.size();
  CUDA_TRY(cudaMemcpyAsync(c, &n, 8, cudaMemcpyHostToDevice, P.st));
  comm_ok(P.comm->broadcast_u64(P.comm->ctx, c, 1, 0, P.st), "broadcast (count)");
  CUDA_TRY(cudaMemcpyAsync(&n, c, 8, cudaMemcpyDeviceToHost, P.st));
  CUDA_TRY(cudaStreamSynchronize(P.st));
  if (P.rank_id != 0) w.assign((size_t)n, 0);
  if (!n) return;
  P.x_ser.ensure((size_t)n * 8);
  uint64_t* b = P.x_ser.as<uint64_t>();
  if (P.rank_id == 0) CUDA_TRY(cudaMemcpyAsync(b, w.data(), (size_t)n * 8, cudaMemcpyHostToDevice, P.st));
  comm_ok(P.comm->broadcast_u64(P.comm->ctx, b, (int64_t)n, 0, P.st), "broadcast");
  if (P.rank_id != 0) CUDA_TRY(cudaMemcpyAsync(w.data(), b, (size_t)n * 8, cudaMemcpyDeviceToHost, P.st));
  CUDA_TRY(cudaStreamSynchronize(P.st));
}

void stage_setup(vr_plan& P) {
  SectionTimer ST;
  vr_result* R = P.R.get();
  const int64_t n = P.n;
  const int D = P.D;
  cudaStream_t st = P.st;
  P.N = (uint64_t)n * (uint64_t)(n - 1) / 2;
  P.kbits = bits_for(P.N ? P.N - 1 : 0);
  P.kmax = D + 2;

  // binomial table C(v, k), v in [0, n], k in [0, D+2], layout [k][v]
  std::vector<uint64_t> hb((size_t)(P.kmax + 1) * (size_t)(n + 1));
  for (int k = 0; k <= P.kmax; ++k)
    for (int64_t v = 0; v <= n; ++v) hb[(size_t)k * (size_t)(n + 1) + (size_t)v] = binom_host((uint64_t)v, (uint64_t)k);

  ST.mark("binomials");
  // ---------------- device memory for the tables
  size_t free_b = 0, total_b = 0;
  CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
  const size_t need_tables = (size_t)n * (size_t)n * 4 + 2 * (size_t)P.N * 8 + hb.size() * 8;
  if (need_tables > free_b) throw VrError(VR_ECAPACITY, "device memory too small for the tables");
  P.binom.ensure(hb.size() * 8);
  P.rank.ensure((size_t)n * (size_t)n * 4);
  P.keys.ensure(std::max<size_t>(P.N, 1) * 8);
  P.alt.ensure(std::max<size_t>(P.N, 1) * 8);
  P.rowmax.ensure((size_t)n * 4);
  P.tout.ensure(sizeof(vr::TablesOut));
  P.ctrs.ensure(sizeof(vr::DimCounters) * (size_t)(D + 1));
  P.sort_tmp.ensure(vr::radix_sort_temp_bytes(std::max<size_t>(P.N, 1)));
  P.tb_tmp.ensure(vr::tables_temp_bytes(n));
  CUDA_TRY(cudaMemcpyAsync(P.binom.p, hb.data(), hb.size() * 8, cudaMemcpyHostToDevice, st));
  for (auto& e : P.ev)
    if (!e) CUDA_TRY(cudaEventCreate(&e));

  ST.mark("allocate tables");
  // ---------------- a0
  uint64_t* sorted = nullptr;
  CUDA_TRY(cudaEventRecord(P.ev[0], st));
  vr::launch_tables(P.d_lt, n, P.threshold, P.keys.as<uint64_t>(), P.alt.as<uint64_t>(), P.rowmax.as<uint32_t>(),
                    P.sort_tmp.p, P.tb_tmp.p, P.rank.as<uint32_t>(), P.tout.as<vr::TablesOut>(), -1, &sorted, st,
                    &P.launches);
  CUDA_TRY(cudaGetLastError());
  vr::TablesOut to{};
  CUDA_TRY(cudaMemcpyAsync(&to, P.tout.p, sizeof to, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaEventRecord(P.ev[1], st));
  CUDA_TRY(cudaStreamSynchronize(st));
  ST.mark("tables (device)");
  if (to.err) throw VrError(VR_EINPUT, "dist_lower_tri holds a negative or NaN distance");
  float tms = 0;
  cudaEventElapsedTime(&tms, P.ev[0], P.ev[1]);
  float tused;
  std::memcpy(&tused, &to.tbits, 4);
  P.m = to.m_le_t;
  P.maxr = P.m ? (uint32_t)(P.m - 1) : 0;
  P.rbits = bits_for(P.maxr);

  R->max_dim = D;
  R->tused = tused;
  R->pairs.assign((size_t)D + 1, {});
  R->ipairs.assign((size_t)D + 1, {});
  R->stats.assign((size_t)D + 1, vr_stats{});
  P.hp.assign((size_t)D + 1, {});

  // ---------------- host copies for the off-path steps (sorted edges, rank matrix)
  auto tx0 = std::chrono::steady_clock::now();
  vr::HostMatrix& M = P.M;
  M = vr::HostMatrix();
  M.n = n;
  M.kmax = P.kmax;
  M.binom = hb;
  std::vector<uint64_t> h_edges((size_t)P.m);
  // (copies on the plan's stream: a legacy-default-stream cudaMemcpy does not wait for work
  // on the non-blocking streams the library uses)
  if (P.m) CUDA_TRY(cudaMemcpyAsync(h_edges.data(), sorted, (size_t)P.m * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  M.value.resize((size_t)P.m);
  for (uint64_t r = 0; r < P.m; ++r) {
    uint32_t fb = (uint32_t)(h_edges[(size_t)r] >> P.kbits);
    std::memcpy(&M.value[(size_t)r], &fb, 4);
  }
  const double ms_tx0 = ms_since(tx0);
  ST.mark("D2H edges");

  // ---------------- dimension 0 (replicated on every rank: cheap, §5.2.5)
  auto t0 = std::chrono::steady_clock::now();
  P.deaths.clear();
  vr::dim0_union_find(n, h_edges.data(), P.m, P.kbits, P.hp[0], P.deaths);
  {
    vr_stats& s0 = R->stats[0];
    s0.candidates = n;
    s0.survivors = n;
    s0.ms_residual = ms_since(t0);
    s0.ms_enumerate = tms;
    s0.ms_transfer = ms_tx0;
  }

  ST.mark("dim 0");
  // ---------------- output-sensitive mode?  (dense enumeration of
  // C(n, d+1) indices is wasted work when few edges are under the threshold)
  {
    const int mode = P.opt.sparse_mode;
    const uint64_t dense_rows = D >= 1 ? binom_host((uint64_t)n, (uint64_t)D) : 0;
    bool sp = (P.m * 4 <= P.N) || dense_rows > ((uint64_t)1 << 32);
    if (mode == 1) sp = false;
    if (mode == 2) sp = true;
    P.sparse = sp && D >= 1 && P.m > 0;
    if (P.sparse) {
      P.nw = (int32_t)(((n + 31) / 32 + 3) / 4 * 4);  // words per row, padded to 16-byte quads
      P.deg.ensure(((size_t)n + 1) * 4);
      P.deg_below.ensure(((size_t)n + 1) * 4);
      P.bm.ensure((size_t)n * (size_t)P.nw * 4);
      vr::launch_threshold_bitmap(P.rank.as<uint32_t>(), (int)n, P.nw, P.bm.as<uint32_t>(), P.deg.as<uint32_t>(),
                                  P.deg_below.as<uint32_t>(), st, &P.launches);
      CUDA_TRY(cudaGetLastError());
      P.rows.clear();
      P.rows.resize((size_t)D + 2);
      P.rows_count.assign((size_t)D + 2, 0);
      P.rows_cap.assign((size_t)D + 2, 0);
      P.next_bound.assign((size_t)D + 2, 0);
      // the host residual walks the same threshold graph: the bitmap rows (64-bit words)
      // and the packed neighbour ranks instead of the n x n rank matrix
      auto ta = std::chrono::steady_clock::now();
      const int64_t bmw = P.nw / 2;
      P.nb_pre.ensure((size_t)n * (size_t)bmw * 4);
      P.nb_rank.ensure(std::max<size_t>(2 * (size_t)P.m, 1) * 4);
      P.nb_ctr.ensure(4);
      vr::launch_neighbour_ranks(P.rank.as<uint32_t>(), (int)n, P.bm.as<uint32_t>(), P.nw, P.deg.as<uint32_t>(),
                                 P.nb_ctr.as<uint32_t>(), P.nb_pre.as<uint32_t>(), P.nb_rank.as<uint32_t>(), st,
                                 &P.launches);
      CUDA_TRY(cudaGetLastError());
      M.bmw = bmw;
      M.bm.resize((size_t)n * (size_t)bmw);
      M.nb_pre.resize((size_t)n * (size_t)bmw);
      M.nb_rank.resize(2 * (size_t)P.m);
      CUDA_TRY(cudaMemcpyAsync(M.bm.data(), P.bm.p, M.bm.size() * 8, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaMemcpyAsync(M.nb_pre.data(), P.nb_pre.p, M.nb_pre.size() * 4, cudaMemcpyDeviceToHost, st));
      if (P.m) CUDA_TRY(cudaMemcpyAsync(M.nb_rank.data(), P.nb_rank.p, M.nb_rank.size() * 4, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaStreamSynchronize(st));
      R->stats[0].ms_transfer += ms_since(ta);
    }
  }
  // dense mode: the host scans read the n x n rank matrix (also dumped for the tools)
  if (D >= 1 && P.m && (!P.sparse || std::getenv("VR_DUMP_RESIDUAL"))) {
    auto ta = std::chrono::steady_clock::now();
    M.rank.resize((size_t)n * (size_t)n);
    CUDA_TRY(cudaMemcpyAsync(M.rank.data(), P.rank.p, M.rank.size() * 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    R->stats[0].ms_transfer += ms_since(ta);
  }
  ST.mark("host graph");

  // ---------------- clearing bitmaps (one bit per d-simplex index) where they fit
  P.dims.clear();
  P.dims.resize((size_t)D + 2);
  // output-sensitive dimensions >= 2 extend the survivors of d-2 by two vertices
  // (k_enum_sparse2); VR_SPARSE_1LEVEL keeps the single-level kernel (A/B, tests)
  for (int d = 2; d <= D; ++d) P.dims[(size_t)d].two_level = P.sparse && !std::getenv("VR_SPARSE_1LEVEL");
  CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
  // (tests: VR_FORCE_CLEAR_HASH puts sparse dimensions >= 2 on the hash-set path)
  const bool force_hash = P.sparse && std::getenv("VR_FORCE_CLEAR_HASH") != nullptr;
  for (int d = 1; d <= D; ++d) {
    const uint64_t cand = binom_host((uint64_t)n, (uint64_t)d + 1);
    const size_t words = (size_t)((cand + 31) / 32);
    if (force_hash && d >= 2) continue;
    // output-sensitive mode on one GPU: a bitmap only while it stays small (its bits are
    // probed at random); beyond that the hash set of the pivots is smaller and L2-friendlier
    // (config 5: 1 MiB at dimension 1; 1.4 GiB at dimension 2 -> hash set)
    if (P.sparse && d >= 2 && words * 4 > kSparseBitmapBytes) continue;
    // (total, not free, memory: the decision must be the same on every rank)
    if (cand && P.m && words * 4 <= kMaxBitmapBytes && words * 4 <= total_b / 16) {
      const size_t w2 = (words + 1) & ~(size_t)1;  // even: summed as 64-bit words when sharded
      P.dims[(size_t)d].clr.ensure(w2 * 4);
      P.dims[(size_t)d].clr_words = w2;
    }
  }
  // deaths of dimension 0 -> clearing input of dimension 1
  {
    DimRun& d1 = P.dims[1];
    d1.deaths_in.ensure(std::max<size_t>(P.deaths.size(), 1) * 8);
    d1.ndeaths_in = (int64_t)P.deaths.size();
    if (!P.deaths.empty())
      CUDA_TRY(cudaMemcpyAsync(d1.deaths_in.p, P.deaths.data(), P.deaths.size() * 8, cudaMemcpyHostToDevice, st));
    if (D >= 1 && P.clr_of(1)) {
      CUDA_TRY(cudaMemsetAsync(P.clr_of(1), 0, d1.clr_words * 4, st));
      vr::launch_set_bits(d1.deaths_in.as<uint64_t>(), d1.ndeaths_in, P.clr_of(1), st, &P.launches);
    }
  }
  ST.mark("bitmaps");
}

// Runs this rank's shard of dimension d; returns the number of local residual columns,
// sorted on the device at P.local_sorted.
uint64_t stage_dim_local(vr_plan& P, int d) {
  SectionTimer ST;
  vr_result* R = P.R.get();
  const int64_t n = P.n;
  const int D = P.D;
  cudaStream_t st = P.st;
  DimRun& dr = P.dims[(size_t)d];
  vr_stats& stt = R->stats[(size_t)d];
  stt = vr_stats{};
  P.local_sorted = nullptr;
  const uint64_t cand = binom_host((uint64_t)n, (uint64_t)d + 1);
  stt.candidates = (int64_t)cand;
  dr.chunks.clear();
  dr.residual = 0;
  dr.active = !(cand == 0 || P.m == 0);
  if (!dr.active) return 0;
  const int cbits = bits_for(cand - 1);
  if (P.rbits + cbits > 64) throw VrError(VR_ECAPACITY, "column key (rank bits + cidx bits) does not fit 64 bits");
  const int steps = P.opt.apparent_steps > 0 ? P.opt.apparent_steps : kDefaultSteps;
  vr::DimParams& p = dr.p;
  p.d = d;
  p.n = n;
  p.maxr = P.maxr;
  p.cbits = cbits;
  p.steps = steps;
  // rows per atomic grab: 4 amortises the grab and the upper-prefix work at small n; few
  // rows (e.g. dimension 1: n rows) need every row on its own warp to fill the GPU
  p.grab = P.world > 1 ? 1
                       : (P.opt.rows_per_grab > 0 ? P.opt.rows_per_grab
                                                  : ((n < 384 && binom_host((uint64_t)n, (uint64_t)d) >= 8192) ? 4 : 1));
  p.variant = P.opt.scan_variant > 0 ? P.opt.scan_variant - 1 : 1;
  // shards: dense rows (and sparse vertex rows: dimension 1, or 2 with two levels) are
  // interleaved over the ranks; other sparse rows are this rank's own survivors of a lower
  // dimension, which already partition the d-simplices (each has exactly one prefix)
  const bool interleave = P.world > 1 && (!P.sparse || d == (dr.two_level ? 2 : 1));
  p.shard_rank = interleave ? P.rank_id : 0;
  p.shard_world = interleave ? P.world : 1;
  const uint64_t rows = binom_host((uint64_t)n, (uint64_t)d);
  dr.sort_bits = P.rbits + cbits;
  // the next dimension's bitmap receives this dimension's apparent cofacets
  uint32_t* clr_next = P.clr_of(d + 1);
  if (clr_next) CUDA_TRY(cudaMemsetAsync(clr_next, 0, P.dims[(size_t)d + 1].clr_words * 4, st));

  // sparse mode: the rows are the survivors of d-1 (single level; vertices for d = 1) or of
  // d-2 (two levels; vertices for d = 2).  The d-simplices number at most the bound the
  // dimension-(d-1) kernel accumulated, sum over its survivors s of deg_below(min s)
  uint64_t bound = cand;
  uint64_t nrows_sp = 0;
  if (P.sparse) {
    const int src = dr.two_level ? d - 2 : d - 1;
    nrows_sp = src <= 0 ? (uint64_t)n : P.rows_count[(size_t)src];
    if (dr.two_level && nrows_sp >= (1ull << 32))
      throw VrError(VR_ECAPACITY, "output-sensitive mode: more than 2^32 rows in one dimension");
    bound = d == 1 ? P.m : std::min<uint64_t>(cand, P.next_bound[(size_t)d - 1]);
    if (P.rows_needed(d)) {
      P.rows[(size_t)d].ensure(std::max<uint64_t>(bound, 1) * 16);
      P.rows_cap[(size_t)d] = std::max<uint64_t>(bound, 1);
    }
  }
  // sparse mode, no bitmap for dimension d+1 (C(n, d+2) bits too many), one GPU: the
  // pivots of this dimension (apparent cofacets + residual deaths, at most `bound`) go into a
  // hash set that dimension d+1 probes in phase 1 — instead of queueing every non-apparent
  // column for the phase-2 recomputation
  if (P.sparse && d < D && !P.clr_of(d + 1) && !std::getenv("VR_NO_CLEAR_HASH")) {
    DimRun& nx = P.dims[(size_t)d + 1];
    // sharded: every rank's set receives every rank's pivots — sized by the global bound
    uint64_t gbound = bound;
    if (P.world > 1) {
      gbound = 0;
      for (uint64_t b : gather_u64(P, bound)) gbound += b;
      P.x_exp.ensure(std::max<uint64_t>(bound, 1) * 8);  // this rank's apparent cofacets
    }
    uint64_t slots = 1024;
    while (slots < 2 * std::max<uint64_t>(gbound, 1) + 1024) slots <<= 1;
    size_t fb = 0, tb = 0;
    CUDA_TRY(cudaMemGetInfo(&fb, &tb));
    fb = tb;  // (the same decision on every rank)
    // Bloom filter: 16 bits per bounding key (3 bits set per key: ~0.1% false positives at
    // the pivots actually inserted)
    const uint64_t bw = std::min<uint64_t>(std::max<uint64_t>(gbound / 2, 1024), (uint64_t)UINT32_MAX);
    if (slots * 8 + bw * 4 <= fb / 8) {
      nx.hash.ensure(slots * 8);
      nx.hash_mask = slots - 1;
      nx.bloom.ensure(bw * 4);
      nx.bloom_words = (uint32_t)bw;
      P.hash_reset(d + 1, st);
    } else {
      nx.hash_mask = 0;
    }
  }
  ST.mark("  row bound");
  // queue / residual capacity: every candidate, bounded by a share of free device memory
  size_t free_b = 0, total_b = 0;
  CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
  const uint64_t qmax = std::max<uint64_t>((uint64_t)(free_b / 4 / 40), 1024);
  // (sparse mode with a clearing bitmap or set decides every column in the enumeration
  // kernel: no queue)
  const bool sp_decided = P.sparse && (P.clr_of(d) || P.set_of(d).table);
  const uint64_t qwant = sp_decided ? 1024 : std::min<uint64_t>(std::max<uint64_t>(bound, 1), qmax);
  if (P.sparse && !sp_decided && bound > qmax)
    throw VrError(VR_ECAPACITY, "output-sensitive mode: column bound exceeds device memory");
  if (P.qcap < qwant) {
    P.queue.ensure((size_t)qwant * 8);
    P.qvert.ensure((size_t)qwant * 16);
    P.qcap = qwant;
  }
  uint64_t rows_per_chunk = P.sparse ? nrows_sp : rows;
  const uint64_t rows_total = P.sparse ? nrows_sp : rows;
  if (!P.sparse && cand > P.qcap) rows_per_chunk = std::max<uint64_t>(1, P.qcap / (uint64_t)n);
  uint64_t app_cap = 0;
  uint64_t* app_ptr = nullptr;
  if (P.opt.index_pairs) {
    // index_pairs = 1: every apparent pair; k > 1: at most k of them (an arbitrary subset,
    // for sampled checks at full size)
    app_cap = std::max<uint64_t>(bound, 1);
    if (P.opt.index_pairs > 1) app_cap = std::min<uint64_t>(app_cap, (uint64_t)P.opt.index_pairs);
    P.app_pairs.ensure((size_t)app_cap * 16);
    app_ptr = P.app_pairs.as<uint64_t>();
  }
  ST.mark("  allocate queue");
  vr::DimCounters* ctr = P.ctrs.as<vr::DimCounters>() + d;
  CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(vr::DimCounters), st));
  float t_enum = 0, t_res = 0;
  int64_t kernels = 0;
  uint64_t resid_count = 0;
  for (uint64_t rb = 0; rb < rows_total; rb += rows_per_chunk) {
    const uint64_t re = std::min(rows_total, rb + rows_per_chunk);
    const uint64_t chunk_cand = P.sparse ? std::max<uint64_t>(bound, 1) : std::min<uint64_t>(cand, (re - rb) * (uint64_t)n);
    // residual capacity: what is there plus everything this chunk could add
    if (P.rcap < resid_count + chunk_cand || !P.resid.p) {
      const uint64_t ncap = std::max<uint64_t>(resid_count + chunk_cand, 1024);
      DevBuf nb;
      nb.ensure((size_t)ncap * 8);
      if (resid_count) CUDA_TRY(cudaMemcpyAsync(nb.p, P.resid.p, resid_count * 8, cudaMemcpyDeviceToDevice, st));
      CUDA_TRY(cudaStreamSynchronize(st));
      std::swap(P.resid.p, nb.p);
      std::swap(P.resid.bytes, nb.bytes);
      P.rcap = ncap;
    }
    vr::HotBuffers B{P.queue.as<uint64_t>(), P.qvert.as<uint4>(), P.qcap, P.resid.as<uint64_t>(), P.rcap,
                     P.clr_of(d), clr_next, dr.deaths_in.as<uint64_t>(), dr.ndeaths_in, ctr, app_ptr, app_cap};
    P.hash_fields(B, d);
    if (rb == 0) P.order_rows(d, st);  // (once per dimension, before its first chunk)
    vr::SparseRows SR = P.sparse_rows(d, ctr);
    p.row_begin = rb;
    p.row_end = re;
    CUDA_TRY(cudaMemsetAsync(&ctr->row_next, 0, 8, st));
    CUDA_TRY(cudaMemsetAsync(&ctr->queued, 0, 8, st));
    CUDA_TRY(cudaEventRecord(P.ev[2], st));
    if (P.sparse) {
      vr::launch_enumerate_sparse(p, P.rank.as<uint32_t>(), P.binom.as<uint64_t>(), P.kmax, B, SR, dr.two_level, st,
                                  &P.launches);
      kernels |= VR_KERNEL_SPARSE;
    } else {
      kernels |= vr::launch_enumerate(p, P.rank.as<uint32_t>(), P.binom.as<uint64_t>(), P.kmax, B, st, &P.launches);
    }
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(P.ev[3], st));
    unsigned long long q = 0;
    CUDA_TRY(cudaMemcpyAsync(&q, &ctr->queued, 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (q > P.qcap) throw VrError(VR_ECAPACITY, "apparent-phase queue overflow");
    float x = 0;
    cudaEventElapsedTime(&x, P.ev[2], P.ev[3]);
    t_enum += x;
    CUDA_TRY(cudaEventRecord(P.ev[4], st));
    if (P.sparse) vr::launch_resolve_sparse(p, P.rank.as<uint32_t>(), P.binom.as<uint64_t>(), P.kmax, B, SR, q, st, &P.launches);
    else vr::launch_resolve(p, P.rank.as<uint32_t>(), P.binom.as<uint64_t>(), P.kmax, B, q, st, &P.launches);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(P.ev[5], st));
    unsigned long long rc = 0;
    CUDA_TRY(cudaMemcpyAsync(&rc, &ctr->residual, 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    cudaEventElapsedTime(&x, P.ev[4], P.ev[5]);
    t_res += x;
    if (rc > P.rcap) throw VrError(VR_ECAPACITY, "residual list overflow");
    resid_count = rc;
    dr.chunks.push_back(Chunk{rb, re, q});
  }
  if (P.sparse) {
    vr::DimCounters c{};
    CUDA_TRY(cudaMemcpyAsync(&c, ctr, sizeof c, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (P.rows_needed(d) && c.rows_out > P.rows_cap[(size_t)d]) throw VrError(VR_ECAPACITY, "survivor list overflow");
    P.rows_count[(size_t)d] = P.rows_needed(d) ? c.rows_out : 0;
    P.next_bound[(size_t)d] = c.next_bound;
  }
  dr.residual = resid_count;
  ST.mark("  enumerate + resolve");
  // a4: sort the residual columns into coboundary order
  P.resid_alt.ensure(std::max<uint64_t>(resid_count, 1) * 8);
  size_t stmp = vr::radix_sort_temp_bytes(std::max<uint64_t>(resid_count, 1));
  if (P.sort_tmp.bytes < stmp) P.sort_tmp.ensure(stmp);
  CUDA_TRY(cudaEventRecord(P.ev[6], st));
  P.sort_flag.ensure(8);
  P.cnt_tmp.ensure(vr::sort_columns_temp_bytes((uint64_t)P.maxr + 1));
  dr.sort_mode = std::getenv("VR_FULL_SORT") ? 0 : -1;
  P.local_sorted = vr::sort_columns(P.resid.as<uint64_t>(), P.resid_alt.as<uint64_t>(), resid_count, dr.p.cbits,
                                    dr.sort_bits, (uint64_t)P.maxr + 1, P.sort_tmp.p, P.cnt_tmp.p, &dr.sort_mode,
                                    P.sort_flag.as<unsigned int>(), st, &P.launches);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaEventRecord(P.ev[7], st));
  vr::DimCounters hc{};
  CUDA_TRY(cudaMemcpyAsync(&hc, ctr, sizeof hc, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  float t_sort = 0;
  cudaEventElapsedTime(&t_sort, P.ev[6], P.ev[7]);
  if (P.opt.index_pairs && hc.app_pairs) {
    std::vector<uint64_t> app_h((size_t)std::min<uint64_t>(hc.app_pairs, app_cap) * 2);
    CUDA_TRY(cudaMemcpyAsync(app_h.data(), app_ptr, app_h.size() * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    for (size_t i = 0; i + 1 < app_h.size(); i += 2) R->ipairs[(size_t)d].push_back(vr_index_pair{app_h[i], app_h[i + 1]});
  }
  ST.mark("  sort");
  stt.survivors = (int64_t)hc.survivors;
  stt.apparent = (int64_t)(hc.apparent1 + hc.apparent2);
  stt.cleared = (int64_t)hc.cleared;
  stt.scanned = (int64_t)(hc.scanned + hc.scanned2);
  stt.queued = 0;
  for (auto& c : dr.chunks) stt.queued += (int64_t)c.queued;
  stt.ms_enumerate = t_enum;
  stt.ms_resolve = t_res;
  stt.ms_sort = t_sort;
  stt.kernels = kernels;
  // candidates the kernels examine: all C(n, d+1) dense; in the output-sensitive mode the
  // bitmap AND yields the survivors only
  const double cand_work = P.sparse ? (double)hc.survivors : (double)cand;
  P.work_candidates += cand_work;
  P.work_scanned += (double)hc.scanned;
  P.work_scanned2 += (double)hc.scanned2;
  // algorithmic integer work, SURVEY.md §8(d) per-unit figures: 2 ops per rank read;
  // a1 reads d ranks per candidate (hoisted prefix maxima); a5 reads (d+1) per scanned
  // cofacet vertex plus C(d+2,2) for the facet check, and decodes each tested column with
  // (d+1)·⌈log2 n⌉ compares
  {
    int lg = 0;
    while (((int64_t)1 << lg) < n) ++lg;
    const double tested = (double)hc.survivors - (double)hc.cleared;
    const double cd2 = (double)(d + 2) * (double)(d + 1) / 2.0;
    double queued = 0;
    for (auto& c : dr.chunks) queued += (double)c.queued;
    P.work_rank_ops += 2.0 * d * cand_work + 2.0 * (d + 1) * (double)hc.scanned + 2.0 * cd2 * tested +
                       (double)(d + 1) * lg * tested;
    P.work_rank_ops2 += 2.0 * (d + 1) * (double)hc.scanned2 + (double)(d + 1) * lg * queued;
    // a1 reads: dense — d per candidate index (hoisted prefix maxima); output-sensitive —
    // the reads the kernels' candidate examination made (list maxima, C(σ) compaction)
    dr.reads_a1 = P.sparse ? (double)hc.cand_reads : (double)d * cand_work;
    dr.reads_a5 = (double)(d + 1) * (double)hc.scanned + cd2 * tested;
    dr.reads_a5_phase2 = (double)(d + 1) * (double)hc.scanned2;
    dr.decode = (double)(d + 1) * lg * tested;
    dr.decode_phase2 = (double)(d + 1) * lg * queued;
    dr.kernels = kernels;
    stt.bytes_l2 = (int64_t)(4.0 * (dr.reads_a1 + dr.reads_a5 + dr.reads_a5_phase2));
    stt.bytes_hbm = (int64_t)(16.0 * (double)(P.sparse && P.rows_needed(d) ? P.rows_count[(size_t)d] : 0) +
                              24.0 * (double)resid_count + 24.0 * queued);
  }
  P.survivors_total += stt.survivors;
  P.apparent_total += stt.apparent;
  return resid_count;
}

// The deaths of dimension d (P.deaths, sorted) -> the clearing input of dimension d+1:
// the device death list, its bits in d+1's bitmap or its keys in d+1's clearing set.
void apply_deaths(vr_plan& P, int d) {
  if (d >= P.D) return;
  auto tx = std::chrono::steady_clock::now();
  cudaStream_t st = P.st;
  DimRun& nx = P.dims[(size_t)d + 1];
  nx.ndeaths_in = (int64_t)P.deaths.size();
  nx.deaths_in.ensure(std::max<size_t>(P.deaths.size(), 1) * 8);
  if (!P.deaths.empty())
    CUDA_TRY(cudaMemcpyAsync(nx.deaths_in.p, P.deaths.data(), P.deaths.size() * 8, cudaMemcpyHostToDevice, st));
  if (P.clr_of(d + 1)) vr::launch_set_bits(nx.deaths_in.as<uint64_t>(), nx.ndeaths_in, P.clr_of(d + 1), st, &P.launches);
  P.hash_deaths(d + 1, st);
  P.R->stats[(size_t)d].ms_transfer += ms_since(tx);
}

// The residual hints (residual_prep.cu) of dimension d's sorted columns dkeys (device),
// launched on the plan's stream and copied into first/claimed (the caller synchronises).
// VR_NO_RESIDUAL_HINTS=1: none (the host runs the emergent test itself).
bool residual_hints(vr_plan& P, int d, const uint64_t* dkeys, uint64_t nk, std::vector<uint64_t>& first,
                    std::vector<uint8_t>& claimed) {
  if (std::getenv("VR_NO_RESIDUAL_HINTS") || nk == 0) return false;
  first.resize((size_t)nk);
  claimed.resize((size_t)nk);
  P.h_first.ensure((size_t)nk * 8);
  P.h_claimed.ensure((size_t)nk);
  vr::launch_residual_hints(P.rank.as<uint32_t>(), P.binom.as<uint64_t>(), (int)P.n, P.kmax, d,
                            P.sparse ? P.bm.as<uint32_t>() : nullptr, P.nw, dkeys, nk, P.maxr, P.dims[(size_t)d].p.cbits,
                            P.h_first.as<uint64_t>(), P.h_claimed.as<uint8_t>(), P.st, &P.launches);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(first.data(), P.h_first.p, (size_t)nk * 8, cudaMemcpyDeviceToHost, P.st));
  CUDA_TRY(cudaMemcpyAsync(claimed.data(), P.h_claimed.p, (size_t)nk, cudaMemcpyDeviceToHost, P.st));
  return true;
}

// Host residual of dimension d on the sorted residual columns (all ranks' columns when
// distributed); deaths -> the clearing input of dimension d+1.
void stage_dim_finish(vr_plan& P, int d, const uint64_t* keys, uint64_t nkeys, const vr::ResidualHints* hints,
                      double ms_prep) {
  SectionTimer ST;
  vr_result* R = P.R.get();
  const int D = P.D;
  DimRun& dr = P.dims[(size_t)d];
  vr_stats& stt = R->stats[(size_t)d];
  if (!dr.active) {
    P.deaths.clear();
    if (d < D) {
      P.dims[(size_t)d + 1].ndeaths_in = 0;
    }
    return;
  }
  if (hints && std::getenv("VR_CHECK_HINTS")) {  // tests: the device hints against the host's own scans
    std::vector<uint64_t> f((size_t)nkeys);
    std::vector<uint8_t> c((size_t)nkeys);
    vr::residual_hints_host(P.M, d, P.maxr, dr.p.cbits, keys, nkeys, f.data(), c.data());
    for (uint64_t i = 0; i < nkeys; ++i)
      if (f[(size_t)i] != hints->first[i] || c[(size_t)i] != hints->claimed[i])
        throw VrError(VR_EDEVICE, "residual hints differ from the host scan (dimension " + std::to_string(d) + ", column " +
                                      std::to_string(i) + ")");
  }
  auto tr = std::chrono::steady_clock::now();
  vr::ResidualStats rst;
  vr::residual_reduce(P.M, d, P.maxr, dr.p.cbits, keys, nkeys, P.opt.residual_mode, P.hp[(size_t)d], P.deaths, rst,
                      hints);
  if (d < D) std::sort(P.deaths.begin(), P.deaths.end());  // the clearing input of d+1 (binary searches)
  stt.ms_residual = ms_since(tr) + ms_prep;
  ST.mark("  residual (host)");
  if (std::getenv("VR_TIMING"))
    std::fprintf(stderr, "[vr]   residual d=%d: columns %llu emergent %lld additions %lld coboundaries %lld apparent checks %lld\n", d,
                 (unsigned long long)nkeys, (long long)rst.emergent, (long long)rst.additions, (long long)rst.coboundaries,
                 (long long)rst.apparent_checks);
  if (const char* dump = std::getenv("VR_DUMP_RESIDUAL")) {
    std::vector<uint64_t> kv(keys, keys + nkeys);
    dump_residual(dump, P.M, d, P.maxr, dr.p.cbits, kv);
  }
  apply_deaths(P, d);
  stt.residual_columns = (int64_t)nkeys;
  stt.emergent = rst.emergent;
  P.residual_total += (int64_t)nkeys;
}

void stage_result(vr_plan& P) {
  vr_result* R = P.R.get();
  for (int d = 0; d <= P.D; ++d) {
    const vr::HostPairs& h = P.hp[(size_t)d];
    vr_stats& s = R->stats[(size_t)d];
    auto& out = R->pairs[(size_t)d];
    out.clear();
    s.essential = s.pairs_all = s.pairs_positive = 0;
    for (size_t i = 0; i < h.birth.size(); ++i) {
      const bool ess = std::isinf(h.death[i]);
      if (ess) ++s.essential;
      else {
        ++s.pairs_all;
        if (h.birth[i] < h.death[i]) ++s.pairs_positive;
      }
      if (ess || h.birth[i] < h.death[i] || P.opt.include_zero) out.push_back(vr_pair{h.birth[i], h.death[i]});
      if (P.opt.index_pairs) R->ipairs[(size_t)d].push_back(vr_index_pair{h.birth_cidx[i], h.death_cidx[i]});
    }
    if (d >= 1) s.pairs_all += s.apparent;  // apparent pairs: zero-length, counted only
    std::sort(out.begin(), out.end(), [](const vr_pair& a, const vr_pair& b) {
      return a.birth < b.birth || (a.birth == b.birth && a.death < b.death);
    });
  }
}

// Exchange A of a sharded dimension d (include/vr.h "Multi-GPU"): the clearing input of
// d+1 from every rank — the SUM all-reduce of the bitmap (disjoint bits, reading R3), or
// the all-gather of every rank's apparent cofacets into each rank's clearing set.
// `replay`: the counts are the first run's (no host synchronisation).
void exchange_clearing(vr_plan& P, int d, bool replay) {
  if (P.world == 1 || d >= P.D) return;
  DimRun& dr = P.dims[(size_t)d];
  cudaStream_t st = P.st;
  if (uint32_t* bm = P.clr_of(d + 1)) {
    comm_ok(P.comm->allreduce_sum_u64(P.comm->ctx, (uint64_t*)bm, (int64_t)(P.dims[(size_t)d + 1].clr_words / 2), st),
            "all-reduce (clearing bitmap)");
    return;
  }
  const vr::ClearSet c = P.set_of(d + 1);
  if (!c.table) return;
  if (!replay) {
    vr::DimCounters hc{};
    CUDA_TRY(cudaMemcpyAsync(&hc, P.ctrs.as<vr::DimCounters>() + d, sizeof hc, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (hc.exported * 8 > P.x_exp.bytes) throw VrError(VR_ECAPACITY, "export list overflow");
    dr.exp_local = hc.exported;
    dr.exp_cap = 0;
    for (uint64_t v : gather_u64(P, dr.exp_local)) dr.exp_cap = std::max(dr.exp_cap, v);
  }
  if (!dr.exp_cap) return;
  P.x_exp.ensure((size_t)dr.exp_cap * 8);
  uint64_t* L = P.x_exp.as<uint64_t>();
  if (dr.exp_cap > dr.exp_local) CUDA_TRY(cudaMemsetAsync(L + dr.exp_local, 0xFF, (dr.exp_cap - dr.exp_local) * 8, st));
  P.x_expg.ensure((size_t)P.world * dr.exp_cap * 8);
  comm_ok(P.comm->allgather_u64(P.comm->ctx, L, P.x_expg.as<uint64_t>(), (int64_t)dr.exp_cap, st),
          "all-gather (apparent cofacets)");
  vr::launch_set_put(P.x_expg.as<uint64_t>(), (int64_t)(P.world * dr.exp_cap), c, st, &P.launches);
}

// Exchange B: every rank's sorted residual keys of dimension d, all-gathered (padded with ~0
// to the largest count) and merged on the device into P.x_merged; returns the total.
uint64_t exchange_residual(vr_plan& P, int d, uint64_t nk_local, bool replay) {
  DimRun& dr = P.dims[(size_t)d];
  if (P.world == 1) return nk_local;
  cudaStream_t st = P.st;
  if (!replay) {
    dr.x_counts = gather_u64(P, nk_local);
    dr.x_cap = 0;
    dr.x_total = 0;
    for (uint64_t v : dr.x_counts) {
      dr.x_cap = std::max(dr.x_cap, v);
      dr.x_total += v;
    }
  }
  if (!dr.x_total) return 0;
  P.x_send.ensure((size_t)dr.x_cap * 8);
  uint64_t* snd = P.x_send.as<uint64_t>();
  if (dr.x_cap > nk_local) CUDA_TRY(cudaMemsetAsync(snd + nk_local, 0xFF, (dr.x_cap - nk_local) * 8, st));
  if (nk_local) CUDA_TRY(cudaMemcpyAsync(snd, P.local_sorted, nk_local * 8, cudaMemcpyDeviceToDevice, st));
  P.x_gather.ensure((size_t)P.world * dr.x_cap * 8);
  comm_ok(P.comm->allgather_u64(P.comm->ctx, snd, P.x_gather.as<uint64_t>(), (int64_t)dr.x_cap, st),
          "all-gather (residual keys)");
  P.x_merged.ensure((size_t)dr.x_total * 8);
  vr::merge_gathered_u64(P.x_gather.as<uint64_t>(), P.world, dr.x_cap, P.x_merged.as<uint64_t>(), st, &P.launches);
  return dr.x_total;
}

// The apparent index pairs of dimension d (debug output) from every rank to rank 0.
void gather_index_pairs(vr_plan& P, int d) {
  auto& ip = P.R->ipairs[(size_t)d];
  std::vector<uint64_t> counts = gather_u64(P, ip.size());
  uint64_t cap = 0;
  for (uint64_t v : counts) cap = std::max(cap, v);
  if (!cap) return;
  std::vector<uint64_t> mine((size_t)cap * 2, ~0ull);
  for (size_t i = 0; i < ip.size(); ++i) { mine[2 * i] = ip[i].birth_cidx; mine[2 * i + 1] = ip[i].death_cidx; }
  P.x_send.ensure((size_t)cap * 16);
  P.x_gather.ensure((size_t)P.world * cap * 16);
  CUDA_TRY(cudaMemcpyAsync(P.x_send.p, mine.data(), (size_t)cap * 16, cudaMemcpyHostToDevice, P.st));
  comm_ok(P.comm->allgather_u64(P.comm->ctx, P.x_send.as<uint64_t>(), P.x_gather.as<uint64_t>(), (int64_t)cap * 2, P.st),
          "all-gather (index pairs)");
  std::vector<uint64_t> all((size_t)P.world * cap * 2);
  CUDA_TRY(cudaMemcpyAsync(all.data(), P.x_gather.p, all.size() * 8, cudaMemcpyDeviceToHost, P.st));
  CUDA_TRY(cudaStreamSynchronize(P.st));
  ip.clear();
  for (size_t i = 0; i + 1 < all.size(); i += 2)
    if (all[i] != ~0ull) ip.push_back(vr_index_pair{all[i], all[i + 1]});
}

// Rank 0's result to every rank: stats, pairs and index pairs of every dimension, and the
// threshold applied, serialised as 64-bit words.
void bcast_result(vr_plan& P) {
  vr_result* R = P.R.get();
  const size_t sw = (sizeof(vr_stats) + 7) / 8;
  std::vector<uint64_t> w;
  if (P.rank_id == 0) {
    uint32_t tb;
    std::memcpy(&tb, &R->tused, 4);
    w.push_back(tb);
    for (int d = 0; d <= P.D; ++d) {
      const size_t o = w.size();
      w.resize(o + sw, 0);
      std::memcpy(&w[o], &R->stats[(size_t)d], sizeof(vr_stats));
      w.push_back(R->pairs[(size_t)d].size());
      for (const vr_pair& q : R->pairs[(size_t)d]) {
        uint32_t b, e;
        std::memcpy(&b, &q.birth, 4);
        std::memcpy(&e, &q.death, 4);
        w.push_back((uint64_t)b | ((uint64_t)e << 32));
      }
      w.push_back(R->ipairs[(size_t)d].size());
      for (const vr_index_pair& q : R->ipairs[(size_t)d]) { w.push_back(q.birth_cidx); w.push_back(q.death_cidx); }
    }
  }
  bcast_words(P, w);
  if (P.rank_id == 0) return;
  size_t k = 0;
  const uint32_t tb = (uint32_t)w[k++];
  std::memcpy(&R->tused, &tb, 4);
  for (int d = 0; d <= P.D; ++d) {
    std::memcpy(&R->stats[(size_t)d], &w[k], sizeof(vr_stats));
    k += sw;
    const uint64_t np = w[k++];
    R->pairs[(size_t)d].resize((size_t)np);
    for (uint64_t i = 0; i < np; ++i, ++k) {
      const uint32_t b = (uint32_t)w[k], e = (uint32_t)(w[k] >> 32);
      std::memcpy(&R->pairs[(size_t)d][(size_t)i].birth, &b, 4);
      std::memcpy(&R->pairs[(size_t)d][(size_t)i].death, &e, 4);
    }
    const uint64_t ni = w[k++];
    R->ipairs[(size_t)d].resize((size_t)ni);
    for (uint64_t i = 0; i < ni; ++i, k += 2) R->ipairs[(size_t)d][(size_t)i] = vr_index_pair{w[k], w[k + 1]};
  }
}

// A sharded run (P.comm, world > 1): every rank runs its shard of each dimension's hot path,
// exchanges A and B, rank 0 the host residual and the deaths go to every rank (exchange C);
// at the end the counters are summed and rank 0's result is broadcast.
void run_distributed(vr_plan& P) {
  stage_setup(P);
  for (int d = 1; d <= P.D; ++d) {
    const uint64_t nk = stage_dim_local(P, d);
    const bool active = P.dims[(size_t)d].active;
    auto tx = std::chrono::steady_clock::now();
    if (active) {
      exchange_clearing(P, d, false);
      if (P.opt.index_pairs) gather_index_pairs(P, d);
    }
    const uint64_t total = active ? exchange_residual(P, d, nk, false) : 0;
    CUDA_TRY(cudaStreamSynchronize(P.st));
    double ms_x = ms_since(tx);
    if (P.rank_id == 0) {
      std::vector<uint64_t> hkeys((size_t)total), hfirst;
      std::vector<uint8_t> hclaimed;
      auto tx = std::chrono::steady_clock::now();
      const bool hinted = active && residual_hints(P, d, P.x_merged.as<uint64_t>(), total, hfirst, hclaimed);
      if (total) CUDA_TRY(cudaMemcpyAsync(hkeys.data(), P.x_merged.p, total * 8, cudaMemcpyDeviceToHost, P.st));
      CUDA_TRY(cudaStreamSynchronize(P.st));
      const vr::ResidualHints hints{hfirst.data(), hclaimed.data()};
      stage_dim_finish(P, d, hkeys.data(), total, hinted ? &hints : nullptr, ms_since(tx));
    }
    // exchange C: rank 0's deaths of dimension d to every rank
    std::vector<uint64_t> deaths;
    if (P.rank_id == 0) deaths = P.deaths;
    tx = std::chrono::steady_clock::now();
    bcast_words(P, deaths);
    ms_x += ms_since(tx);
    P.R->stats[(size_t)d].ms_exchange = ms_x;
    if (P.rank_id != 0) {
      P.deaths = deaths;
      if (active) apply_deaths(P, d);
      else if (d < P.D) P.dims[(size_t)d + 1].ndeaths_in = 0;
      P.R->stats[(size_t)d].residual_columns = (int64_t)total;
      P.residual_total += (int64_t)total;
    }
  }
  // the counters the ranks accumulated locally, summed
  std::vector<uint64_t> c((size_t)(P.D + 1) * 5, 0);
  for (int d = 1; d <= P.D; ++d) {
    const vr_stats& s = P.R->stats[(size_t)d];
    uint64_t* q = &c[(size_t)d * 5];
    q[0] = (uint64_t)s.survivors; q[1] = (uint64_t)s.apparent; q[2] = (uint64_t)s.cleared; q[3] = (uint64_t)s.queued;
    q[4] = (uint64_t)s.scanned;
  }
  P.x_ser.ensure(c.size() * 8);
  CUDA_TRY(cudaMemcpyAsync(P.x_ser.p, c.data(), c.size() * 8, cudaMemcpyHostToDevice, P.st));
  comm_ok(P.comm->allreduce_sum_u64(P.comm->ctx, P.x_ser.as<uint64_t>(), (int64_t)c.size(), P.st), "all-reduce (counters)");
  CUDA_TRY(cudaMemcpyAsync(c.data(), P.x_ser.p, c.size() * 8, cudaMemcpyDeviceToHost, P.st));
  CUDA_TRY(cudaStreamSynchronize(P.st));
  P.survivors_total = P.apparent_total = 0;
  for (int d = 1; d <= P.D; ++d) {
    vr_stats& s = P.R->stats[(size_t)d];
    const uint64_t* q = &c[(size_t)d * 5];
    s.survivors = (int64_t)q[0]; s.apparent = (int64_t)q[1]; s.cleared = (int64_t)q[2]; s.queued = (int64_t)q[3];
    s.scanned = (int64_t)q[4];
    P.survivors_total += s.survivors;
    P.apparent_total += s.apparent;
  }
  if (P.rank_id == 0) stage_result(P);
  bcast_result(P);
}

void run_full(vr_plan& P) {
  if (P.comm && P.world > 1) {
    run_distributed(P);
    return;
  }
  stage_setup(P);
  for (int d = 1; d <= P.D; ++d) {
    const uint64_t nk = stage_dim_local(P, d);
    if (P.opt.hot_path_only) {  // diagnostics: no host residual, no deaths
      P.R->stats[(size_t)d].residual_columns = (int64_t)nk;
      P.residual_total += (int64_t)nk;
      P.deaths.clear();
      if (P.dims[(size_t)d].active) apply_deaths(P, d);
      else if (d < P.D) P.dims[(size_t)d + 1].ndeaths_in = 0;
      continue;
    }
    std::vector<uint64_t> hkeys((size_t)nk), hfirst;
    std::vector<uint8_t> hclaimed;
    auto tx = std::chrono::steady_clock::now();
    const bool hinted = P.dims[(size_t)d].active && residual_hints(P, d, P.local_sorted, nk, hfirst, hclaimed);
    if (nk) CUDA_TRY(cudaMemcpyAsync(hkeys.data(), P.local_sorted, nk * 8, cudaMemcpyDeviceToHost, P.st));
    CUDA_TRY(cudaStreamSynchronize(P.st));
    const vr::ResidualHints hints{hfirst.data(), hclaimed.data()};
    stage_dim_finish(P, d, hkeys.data(), nk, hinted ? &hints : nullptr, ms_since(tx));
  }
  stage_result(P);
}

// Re-launch the GPU hot path of every dimension with the recorded sizes (no host sync).
// Each stage is bracketed by CUDA events on the plan's stream (vr_plan_timing).  The
// clearing inputs are the device death lists recorded by the full run.
void replay(vr_plan& P) {
  cudaStream_t st = P.st;
  int used[4] = {0, 0, 0, 0};
  int cur_dim = 0;
  auto ev = [&](int stage) -> std::pair<cudaEvent_t, cudaEvent_t>& {
    auto& v = P.stage_ev[stage];
    if ((int)v.size() <= used[stage]) {
      std::pair<cudaEvent_t, cudaEvent_t> e;
      CUDA_TRY(cudaEventCreate(&e.first));
      CUDA_TRY(cudaEventCreate(&e.second));
      v.push_back(e);
      P.stage_dim[stage].push_back(0);
    }
    P.stage_dim[stage][(size_t)used[stage]] = cur_dim;
    return v[(size_t)used[stage]++];
  };
  auto clr_of = [&](int d) -> uint32_t* { return P.clr_of(d); };
  uint64_t* sorted = nullptr;
  {
    auto& e = ev(0);
    cudaEventRecord(e.first, st);
    const vr::GraphOut g{P.bm.as<uint32_t>(), P.nw, P.deg.as<uint32_t>(), P.deg_below.as<uint32_t>()};
    vr::launch_tables(P.d_lt, P.n, P.threshold, P.keys.as<uint64_t>(), P.alt.as<uint64_t>(), P.rowmax.as<uint32_t>(),
                      P.sort_tmp.p, P.tb_tmp.p, P.rank.as<uint32_t>(), P.tout.as<vr::TablesOut>(), (int64_t)P.m, &sorted, st,
                      &P.launches, P.sparse ? &g : nullptr);
    if (P.D >= 1 && clr_of(1)) {
      cudaMemsetAsync(clr_of(1), 0, P.dims[1].clr_words * 4, st);
      vr::launch_set_bits(P.dims[1].deaths_in.as<uint64_t>(), P.dims[1].ndeaths_in, clr_of(1), st, &P.launches);
    }
    cudaEventRecord(e.second, st);
  }
  for (int d = 1; d <= P.D; ++d) {
    DimRun& dr = P.dims[(size_t)d];
    if (dr.chunks.empty()) continue;
    vr::DimCounters* ctr = P.ctrs.as<vr::DimCounters>() + d;
    uint32_t* clr_next = clr_of(d + 1);
    cur_dim = -d;  // the dimension's setup: counters, next clearing bitmap / set reset
    auto& e1 = ev(1);
    cur_dim = d;
    cudaEventRecord(e1.first, st);
    cudaMemsetAsync(ctr, 0, sizeof(vr::DimCounters), st);
    if (clr_next) cudaMemsetAsync(clr_next, 0, P.dims[(size_t)d + 1].clr_words * 4, st);
    P.hash_reset(d + 1, st);
    cudaEventRecord(e1.second, st);
    vr::DimParams p = dr.p;
    {
      auto& eo = ev(1);  // (timed with the enumeration stage)
      cudaEventRecord(eo.first, st);
      if (P.side_dim == d) {  // ordered on the side stream during dimension d-1
        cudaStreamWaitEvent(st, P.ev_order_done, 0);
        P.ord_dim = d;
        P.side_dim = -1;
      } else {
        P.order_rows(d, st);
      }
      cudaEventRecord(eo.second, st);
    }
    for (const Chunk& c : dr.chunks) {
      vr::HotBuffers B{P.queue.as<uint64_t>(), P.qvert.as<uint4>(), P.qcap, P.resid.as<uint64_t>(), P.rcap,
                       clr_of(d), clr_next, dr.deaths_in.as<uint64_t>(), dr.ndeaths_in, ctr, nullptr, 0};
      P.hash_fields(B, d);
      vr::SparseRows SR = P.sparse_rows(d, ctr);
      p.row_begin = c.row_begin;
      p.row_end = c.row_end;
      auto& e2 = ev(1);
      cudaEventRecord(e2.first, st);
      cudaMemsetAsync(&ctr->row_next, 0, 8, st);
      cudaMemsetAsync(&ctr->queued, 0, 8, st);
      if (P.sparse)
        vr::launch_enumerate_sparse(p, P.rank.as<uint32_t>(), P.binom.as<uint64_t>(), P.kmax, B, SR, dr.two_level, st,
                                    &P.launches);
      else vr::launch_enumerate(p, P.rank.as<uint32_t>(), P.binom.as<uint64_t>(), P.kmax, B, st, &P.launches);
      cudaEventRecord(e2.second, st);
      auto& e3 = ev(2);
      cudaEventRecord(e3.first, st);
      if (P.sparse) vr::launch_resolve_sparse(p, P.rank.as<uint32_t>(), P.binom.as<uint64_t>(), P.kmax, B, SR, c.queued, st, &P.launches);
      else vr::launch_resolve(p, P.rank.as<uint32_t>(), P.binom.as<uint64_t>(), P.kmax, B, c.queued, st, &P.launches);
      cudaEventRecord(e3.second, st);
    }
    if (P.world > 1) {  // exchange A (timed with the enumeration stage)
      auto& ex = ev(1);
      cudaEventRecord(ex.first, st);
      exchange_clearing(P, d, true);
      cudaEventRecord(ex.second, st);
    }
    // rows of dimension d are complete: order them for dimension d+2 on the side stream
    if (d + 2 <= P.D && P.sparse && P.dims[(size_t)d + 2].two_level && !std::getenv("VR_NO_SIDE_ORDER")) {
      if (!P.st_side) {
        CUDA_TRY(cudaStreamCreateWithFlags(&P.st_side, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&P.ev_rows_ready, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&P.ev_order_done, cudaEventDisableTiming));
      }
      cudaEventRecord(P.ev_rows_ready, st);
      cudaStreamWaitEvent(P.st_side, P.ev_rows_ready, 0);
      P.order_rows(d + 2, P.st_side);
      if (P.ord_dim == d + 2) {
        cudaEventRecord(P.ev_order_done, P.st_side);
        P.side_dim = d + 2;
      }
      P.ord_dim = -1;  // (dimension d+1 reads its own rows)
    }
    auto& e4 = ev(3);
    cudaEventRecord(e4.first, st);
    P.local_sorted = vr::sort_columns(P.resid.as<uint64_t>(), P.resid_alt.as<uint64_t>(), dr.residual, dr.p.cbits,
                                      dr.sort_bits, (uint64_t)P.maxr + 1, P.sort_tmp.p, P.cnt_tmp.p, &dr.sort_mode,
                                      P.sort_flag.as<unsigned int>(), st, &P.launches);
    if (P.world > 1) exchange_residual(P, d, dr.residual, true);  // exchange B (timed with the sort)
    if (d < P.D && clr_next)
      vr::launch_set_bits(P.dims[(size_t)d + 1].deaths_in.as<uint64_t>(), P.dims[(size_t)d + 1].ndeaths_in, clr_next,
                          st, &P.launches);
    if (d < P.D) P.hash_deaths(d + 1, st);
    cudaEventRecord(e4.second, st);
  }
  P.used_events[0] = used[0]; P.used_events[1] = used[1]; P.used_events[2] = used[2]; P.used_events[3] = used[3];
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return VR_OK;
  } catch (const VrError& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host out of memory";
    return VR_ECAPACITY;
  } catch (const std::exception& e) {
    g_err = e.what();
    return VR_EDEVICE;
  }
}

vr_options default_options(const vr_options* o) {
  vr_options d{};
  if (o) d = *o;
  return d;
}

}  // namespace

extern "C" {

int vr_barcodes_device(const float* d_lt, int64_t n, int32_t max_dim, float threshold, const vr_options* opt, void* stream,
                       vr_result** out) {
  if (out) *out = nullptr;
  return guarded([&] {
    if (!out) throw VrError(VR_EINVAL, "out is NULL");
    check_args(d_lt, n, max_dim, threshold);
    vr_plan P;
    P.n = n; P.D = max_dim; P.threshold = threshold; P.opt = default_options(opt);
    P.st = (cudaStream_t)stream; P.d_lt = d_lt;
    run_full(P);
    *out = P.R.release();
  });
}

int vr_barcodes_coo(int64_t n, int64_t nnz, const int32_t* rows, const int32_t* cols, const float* dist, int32_t max_dim,
                    float threshold, const vr_options* opt, vr_result** out) {
  if (out) *out = nullptr;
  return guarded([&] {
    if (!out) throw VrError(VR_EINVAL, "out is NULL");
    if (nnz < 0 || (nnz && (!rows || !cols || !dist))) throw VrError(VR_EINVAL, "COO arrays are NULL");
    check_args(n >= 2 ? (const void*)1 : nullptr, n, max_dim, threshold);
    for (int64_t k = 0; k < nnz; ++k) {
      if (rows[k] < 0 || rows[k] >= n || cols[k] < 0 || cols[k] >= n || rows[k] == cols[k])
        throw VrError(VR_EINPUT, "COO entry out of range or on the diagonal");
      if (!(dist[k] >= 0.0f) || std::isinf(dist[k])) throw VrError(VR_EINPUT, "COO distance negative, NaN or infinite");
    }
    vr_options o = default_options(opt);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) throw VrError(VR_EDEVICE, "no CUDA device");
    if (o.device < 0 || o.device >= ndev) throw VrError(VR_EINVAL, "options.device out of range");
    CUDA_TRY(cudaSetDevice(o.device));
    std::unique_ptr<vr_plan> P(new vr_plan());
    P->n = n; P->D = max_dim; P->threshold = threshold; P->opt = o;
    CUDA_TRY(cudaStreamCreateWithFlags(&P->st, cudaStreamNonBlocking));
    struct SG { cudaStream_t s; ~SG() { cudaStreamDestroy(s); } } sg{P->st};
    const size_t bytes = (size_t)n * (size_t)(n - 1) / 2 * sizeof(float);
    P->lt_copy.ensure(std::max<size_t>(bytes, 4));
    DevBuf dr, dc, dd;
    dr.ensure(std::max<int64_t>(nnz, 1) * 4);
    dc.ensure(std::max<int64_t>(nnz, 1) * 4);
    dd.ensure(std::max<int64_t>(nnz, 1) * 4);
    if (nnz) {
      CUDA_TRY(cudaMemcpyAsync(dr.p, rows, (size_t)nnz * 4, cudaMemcpyHostToDevice, P->st));
      CUDA_TRY(cudaMemcpyAsync(dc.p, cols, (size_t)nnz * 4, cudaMemcpyHostToDevice, P->st));
      CUDA_TRY(cudaMemcpyAsync(dd.p, dist, (size_t)nnz * 4, cudaMemcpyHostToDevice, P->st));
    }
    vr::launch_coo_to_dense(dr.as<int32_t>(), dc.as<int32_t>(), dd.as<float>(), nnz, n, P->lt_copy.as<float>(), P->st);
    CUDA_TRY(cudaGetLastError());
    P->d_lt = P->lt_copy.as<float>();
    run_full(*P);
    CUDA_TRY(cudaStreamSynchronize(P->st));
    std::unique_ptr<vr_result> R(std::move(P->R));
    P.reset();
    *out = R.release();
  });
}

// restores the caller's current device on scope exit
struct DeviceGuard {
  int dev = -1;
  DeviceGuard() { if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); dev = -1; } }
  ~DeviceGuard() { if (dev >= 0) cudaSetDevice(dev); }
};

// The host-pointer computation on the current device, sharded when comm is given.
void barcodes_host(const float* lt, int64_t n, int32_t max_dim, float threshold, const vr_options& o, const vr_comm* comm,
                   vr_result** out) {
  SectionTimer ST;
  std::unique_ptr<vr_plan> P(new vr_plan());
  P->n = n; P->D = max_dim; P->threshold = threshold; P->opt = o;
  if (comm) {
    P->comm = comm;
    P->rank_id = comm->rank;
    P->world = comm->world;
  }
  CUDA_TRY(cudaStreamCreateWithFlags(&P->st, cudaStreamNonBlocking));
  struct SG { cudaStream_t s; ~SG() { cudaStreamDestroy(s); } } sg{P->st};
  const size_t bytes = (size_t)n * (size_t)(n - 1) / 2 * sizeof(float);
  P->lt_copy.ensure(std::max<size_t>(bytes, 4));
  if (bytes) CUDA_TRY(cudaMemcpyAsync(P->lt_copy.p, lt, bytes, cudaMemcpyHostToDevice, P->st));
  P->d_lt = P->lt_copy.as<float>();
  ST.mark("H2D input");
  run_full(*P);
  CUDA_TRY(cudaStreamSynchronize(P->st));
  ST.mark("run_full");
  std::unique_ptr<vr_result> R(std::move(P->R));
  P.reset();
  ST.mark("release device buffers");
  *out = R.release();
}

int vr_barcodes_comm(const float* lt, int64_t n, int32_t max_dim, float threshold, const vr_options* opt,
                     const vr_comm* comm, vr_result** out) {
  if (out) *out = nullptr;
  DeviceGuard dg;
  return guarded([&] {
    if (!out || !comm) throw VrError(VR_EINVAL, "out / comm is NULL");
    if (comm->world < 1 || comm->rank < 0 || comm->rank >= comm->world) throw VrError(VR_EINVAL, "bad rank / world");
    check_args(lt, n, max_dim, threshold);
    barcodes_host(lt, n, max_dim, threshold, default_options(opt), comm, out);
  });
}

int vr_barcodes(const float* lt, int64_t n, int32_t max_dim, float threshold, const vr_options* opt, vr_result** out) {
  if (out) *out = nullptr;
  DeviceGuard dg;
  int rc = guarded([&] {
    if (!out) throw VrError(VR_EINVAL, "out is NULL");
    check_args(lt, n, max_dim, threshold);
    vr_options o = default_options(opt);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) throw VrError(VR_EDEVICE, "no CUDA device");
    if (o.num_gpus > 1) {  // one process over devices 0..G-1: a host thread per device, NCCL
      const int G = o.num_gpus;
      if (G > ndev) throw VrError(VR_EINVAL, "options.num_gpus exceeds the visible devices");
      std::vector<vr_comm*> comms = vr::comm_nccl_all(G);
      if ((int)comms.size() != G) throw VrError(VR_EDEVICE, "ncclCommInitAll failed: " + g_err);
      std::vector<vr_result*> res((size_t)G, nullptr);
      std::vector<int> rcs((size_t)G, VR_OK);
      std::vector<std::string> errs((size_t)G);
      std::vector<std::thread> th;
      for (int g = 0; g < G; ++g)
        th.emplace_back([&, g] {
          cudaSetDevice(g);
          rcs[(size_t)g] = guarded([&] { barcodes_host(lt, n, max_dim, threshold, o, comms[(size_t)g], &res[(size_t)g]); });
          if (rcs[(size_t)g]) errs[(size_t)g] = g_err;
        });
      for (auto& t : th) t.join();
      for (vr_comm* c : comms) vr_comm_free(c);
      for (int g = 1; g < G; ++g) delete res[(size_t)g];
      for (int g = 0; g < G; ++g)
        if (rcs[(size_t)g]) {
          delete res[0];
          throw VrError(rcs[(size_t)g], "rank " + std::to_string(g) + ": " + errs[(size_t)g]);
        }
      *out = res[0];
      return;
    }
    if (o.device < 0 || o.device >= ndev) throw VrError(VR_EINVAL, "options.device out of range");
    CUDA_TRY(cudaSetDevice(o.device));
    barcodes_host(lt, n, max_dim, threshold, o, nullptr, out);
  });
  return rc;
}

int32_t vr_max_dim(const vr_result* r) { return r ? r->max_dim : -1; }
int64_t vr_num_pairs(const vr_result* r, int32_t dim) {
  return (r && dim >= 0 && dim <= r->max_dim) ? (int64_t)r->pairs[(size_t)dim].size() : 0;
}
const vr_pair* vr_pairs(const vr_result* r, int32_t dim) {
  return (r && dim >= 0 && dim <= r->max_dim && !r->pairs[(size_t)dim].empty()) ? r->pairs[(size_t)dim].data() : nullptr;
}
int64_t vr_num_index_pairs(const vr_result* r, int32_t dim) {
  return (r && dim >= 0 && dim <= r->max_dim) ? (int64_t)r->ipairs[(size_t)dim].size() : 0;
}
const vr_index_pair* vr_index_pairs(const vr_result* r, int32_t dim) {
  return (r && dim >= 0 && dim <= r->max_dim && !r->ipairs[(size_t)dim].empty()) ? r->ipairs[(size_t)dim].data() : nullptr;
}
int vr_stats_get(const vr_result* r, int32_t dim, vr_stats* s) {
  if (!r || !s || dim < 0 || dim > r->max_dim) {
    g_err = "vr_stats_get: bad arguments";
    return VR_EINVAL;
  }
  *s = r->stats[(size_t)dim];
  return VR_OK;
}
float vr_threshold_used(const vr_result* r) { return r ? r->tused : NAN; }
void vr_free(vr_result* r) { delete r; }
const char* vr_last_error(void) { return g_err.c_str(); }

int vr_plan_create(const float* d_lt, int64_t n, int32_t max_dim, float threshold, const vr_options* opt, void* stream,
                   vr_plan** plan, vr_result** out) {
  if (plan) *plan = nullptr;
  if (out) *out = nullptr;
  return guarded([&] {
    if (!plan) throw VrError(VR_EINVAL, "plan is NULL");
    check_args(d_lt, n, max_dim, threshold);
    std::unique_ptr<vr_plan> P(new vr_plan());
    P->n = n; P->D = max_dim; P->threshold = threshold; P->opt = default_options(opt);
    P->opt.index_pairs = 0;
    P->st = (cudaStream_t)stream; P->d_lt = d_lt;
    run_full(*P);
    CUDA_TRY(cudaStreamSynchronize(P->st));
    P->launches = 0;
    std::unique_ptr<vr_result> R(std::move(P->R));
    P->R.reset(new vr_result(*R));
    *plan = P.release();
    if (out) *out = R.release();
  });
}

int vr_plan_create_comm(const float* d_lt, int64_t n, int32_t max_dim, float threshold, const vr_options* opt,
                        const vr_comm* comm, void* stream, vr_plan** plan, vr_result** out) {
  if (plan) *plan = nullptr;
  if (out) *out = nullptr;
  return guarded([&] {
    if (!plan || !comm) throw VrError(VR_EINVAL, "plan / comm is NULL");
    if (comm->world < 1 || comm->rank < 0 || comm->rank >= comm->world) throw VrError(VR_EINVAL, "bad rank / world");
    check_args(d_lt, n, max_dim, threshold);
    std::unique_ptr<vr_plan> P(new vr_plan());
    P->n = n; P->D = max_dim; P->threshold = threshold; P->opt = default_options(opt);
    P->opt.index_pairs = 0;
    P->st = (cudaStream_t)stream; P->d_lt = d_lt;
    P->comm = comm;
    P->rank_id = comm->rank;
    P->world = comm->world;
    run_full(*P);
    CUDA_TRY(cudaStreamSynchronize(P->st));
    P->launches = 0;
    std::unique_ptr<vr_result> R(std::move(P->R));
    P->R.reset(new vr_result(*R));
    *plan = P.release();
    if (out) *out = R.release();
  });
}

int vr_plan_replay(vr_plan* P, int64_t* launches) {
  return guarded([&] {
    if (!P) throw VrError(VR_EINVAL, "plan is NULL");
    const int64_t before = P->launches;
    replay(*P);
    CUDA_TRY(cudaGetLastError());
    if (launches) *launches = P->launches - before;
  });
}

int64_t vr_plan_survivors(const vr_plan* P) { return P ? P->survivors_total : 0; }

int vr_plan_check(vr_plan* P, int64_t* apparent_total, int64_t* residual_total) {
  return guarded([&] {
    if (!P) throw VrError(VR_EINVAL, "plan is NULL");
    std::vector<vr::DimCounters> h((size_t)P->D + 1);
    CUDA_TRY(cudaMemcpyAsync(h.data(), P->ctrs.p, h.size() * sizeof(vr::DimCounters), cudaMemcpyDeviceToHost, P->st));
    CUDA_TRY(cudaStreamSynchronize(P->st));
    int64_t a = 0, r = 0;
    for (int d = 1; d <= P->D; ++d) {
      if (P->dims[(size_t)d].chunks.empty()) continue;
      a += (int64_t)(h[(size_t)d].apparent1 + h[(size_t)d].apparent2);
      r += (int64_t)h[(size_t)d].residual;
    }
    if (apparent_total) *apparent_total = a;
    if (residual_total) *residual_total = r;
  });
}

int vr_plan_timing(vr_plan* P, double out[9]) {
  return guarded([&] {
    if (!P || !out) throw VrError(VR_EINVAL, "plan/out is NULL");
    CUDA_TRY(cudaStreamSynchronize(P->st));
    for (int k = 0; k < 4; ++k) {
      double t = 0;
      for (int i = 0; i < P->used_events[k]; ++i) {
        float x = 0;
        CUDA_TRY(cudaEventElapsedTime(&x, P->stage_ev[k][(size_t)i].first, P->stage_ev[k][(size_t)i].second));
        t += x;
      }
      out[k] = t;
    }
    out[4] = P->work_candidates;
    out[5] = (double)P->survivors_total;
    out[6] = P->work_scanned + P->work_scanned2;
    out[7] = P->work_rank_ops;
    out[8] = P->work_rank_ops2;
  });
}

int vr_plan_dim_timing(vr_plan* P, int32_t d, double out[10]) {
  return guarded([&] {
    if (!P || !out || d < 1 || d > P->D) throw VrError(VR_EINVAL, "bad plan / dimension");
    CUDA_TRY(cudaStreamSynchronize(P->st));
    double t[4] = {0, 0, 0, 0};
    for (int k = 0; k < 4; ++k)
      for (int i = 0; i < P->used_events[k]; ++i) {
        const int dd = P->stage_dim[k][(size_t)i];
        if (dd != d && !(k == 1 && dd == -d)) continue;
        float x = 0;
        CUDA_TRY(cudaEventElapsedTime(&x, P->stage_ev[k][(size_t)i].first, P->stage_ev[k][(size_t)i].second));
        t[dd == -d ? 0 : k] += x;
      }
    const DimRun& dr = P->dims[(size_t)d];
    out[0] = t[1];  // enumeration kernel(s)
    out[1] = t[2];  // phase-2 kernel(s)
    out[2] = t[3];  // sort (+ the next dimension's death bits / set inserts)
    out[3] = t[0];  // setup (counter reset, next clearing bitmap / set reset)
    out[4] = (double)P->R->stats[(size_t)d].survivors;
    out[5] = dr.reads_a1;
    out[6] = dr.reads_a5;
    out[7] = dr.reads_a5_phase2;
    out[8] = dr.decode + dr.decode_phase2;
    out[9] = (double)dr.kernels;
  });
}

void vr_plan_free(vr_plan* P) { delete P; }

int vr_radix_sort_u64(uint64_t* keys, int64_t n, int32_t begin_bit, int32_t end_bit) {
  return guarded([&] {
    if (n < 0 || (n > 0 && !keys) || begin_bit < 0 || end_bit > 64 || begin_bit > end_bit)
      throw VrError(VR_EINVAL, "vr_radix_sort_u64: bad arguments");
    if (n <= 1) return;
    DevBuf a, b, t;
    a.ensure((size_t)n * 8);
    b.ensure((size_t)n * 8);
    t.ensure(vr::radix_sort_temp_bytes((size_t)n));
    CUDA_TRY(cudaMemcpy(a.p, keys, (size_t)n * 8, cudaMemcpyHostToDevice));
    int64_t launches = 0;
    uint64_t* r = vr::radix_sort_u64(a.as<uint64_t>(), b.as<uint64_t>(), (size_t)n, begin_bit, end_bit, t.p, 0, &launches);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpy(keys, r, (size_t)n * 8, cudaMemcpyDeviceToHost));
  });
}

int vr_sort_columns_u64(uint64_t* keys, int64_t n, int32_t cbits, int32_t end_bit, uint64_t bins, int32_t* mode) {
  return guarded([&] {
    if (n < 0 || (n > 0 && !keys) || cbits < 0 || end_bit > 64 || cbits > end_bit || !mode || bins < 1)
      throw VrError(VR_EINVAL, "vr_sort_columns_u64: bad arguments");
    if (n <= 1) return;
    DevBuf a, b, t, c, f;
    a.ensure((size_t)n * 8);
    b.ensure((size_t)n * 8);
    t.ensure(vr::radix_sort_temp_bytes((size_t)n));
    c.ensure(vr::sort_columns_temp_bytes(bins));
    f.ensure(8);
    CUDA_TRY(cudaMemcpy(a.p, keys, (size_t)n * 8, cudaMemcpyHostToDevice));
    int64_t launches = 0;
    int m = *mode;
    uint64_t* r = vr::sort_columns(a.as<uint64_t>(), b.as<uint64_t>(), (size_t)n, cbits, end_bit, bins, t.p, c.p, &m,
                                   f.as<unsigned int>(), 0, &launches);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpy(keys, r, (size_t)n * 8, cudaMemcpyDeviceToHost));
    *mode = m;
  });
}

int64_t vr_plan_launches(const vr_plan* P) { return P ? P->launches : 0; }

int vr_host_residual(const uint32_t* rank, const float* values, int64_t nvalues, int64_t n, int32_t d, uint32_t maxr,
                     int32_t cbits, const uint64_t* keys, int64_t nkeys, int32_t mode, float* birth, float* death,
                     uint64_t* birth_cidx, uint64_t* death_cidx, int64_t* emergent) {
  return guarded([&] {
    if (!rank || !values || n < 2 || d < 1 || d > VR_MAX_DIM || nkeys < 0 || (nkeys && !keys))
      throw VrError(VR_EINVAL, "vr_host_residual: bad arguments");
    vr::HostMatrix M;
    M.n = n;
    M.kmax = d + 2;
    M.rank.assign(rank, rank + (size_t)n * (size_t)n);
    M.value.assign(values, values + nvalues);
    M.binom.resize((size_t)(M.kmax + 1) * (size_t)(n + 1));
    for (int k = 0; k <= M.kmax; ++k)
      for (int64_t v = 0; v <= n; ++v) M.binom[(size_t)k * (size_t)(n + 1) + (size_t)v] = binom_host((uint64_t)v, (uint64_t)k);
    vr::HostPairs hp;
    std::vector<uint64_t> deaths;
    vr::ResidualStats st;
    vr::residual_reduce(M, d, maxr, cbits, keys, (uint64_t)nkeys, mode, hp, deaths, st);
    for (size_t i = 0; i < hp.birth.size(); ++i) {
      birth[i] = hp.birth[i];
      death[i] = hp.death[i];
      birth_cidx[i] = hp.birth_cidx[i];
      death_cidx[i] = hp.death_cidx[i];
    }
    if (emergent) *emergent = st.emergent;
  });
}

}  // extern "C"
