// hypha.cu — HYPHA (PAPER.md Ch.4, ICS'19): pivots of an EXPLICIT Z/2 boundary matrix.
// SURVEY.md §8(f) NEXT-3.
//
//   GPU-scan (Alg 3), one thread per CSC column:
//     k_set_leftmost  (Alg 4)  Left[row] = atomicMin over the columns with a 1 in
//                     that row (reading A19: indexed by the entry's row, not its position);
//                     an empty column is stable
//     k_set_lookup    (Alg 5)  if low(j) is the leftmost 1 of its row, (low(j), j)
//                     is a pivot of a 0-addition column: Lookup[low] = j, stable j, and
//                     column low(j) is cleared (Lemma 4.2.3)
//     k_set_unstable  (Alg 6)  warp-aggregated append of the unstable columns
//   host: compression (Algs 8-9; reading A20: SEARCH visits every entry, the
//   early `return true` of Alg 9 line 4 is a garble), then the standard reduction (Alg 2) of
//   the unstable columns with the GPU pivots pre-claimed — twist order (higher dimensions
//   first, clearing each found pivot's row column, Lemma 4.2.3) when dimensions are given.
//   Pre-claiming is exact: no column left of a stable pivot column j has a 1 in row low(j),
//   so no reduction of a left column can reach that row.
#include <algorithm>
#include <chrono>
#include <memory>
#include <mutex>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/vr.h"
#include "vr_common.cuh"
#include "vr_internal.h"

namespace vr {

// also validates the matrix (rows strictly above the diagonal and ascending): a bad entry
// raises *bad and is skipped, and the call returns VR_EINPUT
// (also writes low(j), the last row of column j or -1, so k_set_lookup reads it coalesced)
__global__ void k_set_leftmost(const int64_t* __restrict__ col_ptr, const int32_t* __restrict__ rows, int64_t n,
                               int32_t* __restrict__ left, uint8_t* __restrict__ stable, int32_t* __restrict__ low,
                               int* __restrict__ bad) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = col_ptr[j], b = col_ptr[j + 1];
    if (a == b) stable[j] = 1;
    int32_t prev = -1;
    for (int64_t k = a; k < b; ++k) {
      const int32_t r = rows[k];
      if (r <= prev || r >= j) { atomicOr(bad, 1); break; }
      prev = r;
      atomicMin(left + r, (int32_t)j);
    }
    low[j] = prev;
  }
}

__global__ void k_set_lookup(const int32_t* __restrict__ lows, int64_t n, const int32_t* __restrict__ left,
                             int32_t* __restrict__ lookup, uint8_t* __restrict__ stable, int clearing) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t low = lows[j];  // rows ascending: the last is low(j); -1 = empty column
    if (low < 0) continue;
    if (left[low] == (int32_t)j) {
      lookup[low] = (int32_t)j;
      stable[j] = 1;
      if (clearing) stable[low] = 1;  // clearing: column low(j) is zero in the reduced matrix
    }
  }
}

__global__ void k_set_unstable(const uint8_t* __restrict__ stable, int64_t n, int32_t* __restrict__ u,
                               unsigned long long* __restrict__ count) {
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = base + threadIdx.x;
    const bool un = j < n && stable[j] == 0;
    const unsigned long long slot = warp_append(un, count);
    if (un) u[slot] = (int32_t)j;
  }
}

}  // namespace vr

namespace {

// device workspace kept across calls (grown on demand), one per device
struct HyphaWs {
  std::mutex mu;
  void* p[8] = {};
  size_t cap[8] = {};
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  void* get(int i, size_t bytes) {
    if (cap[i] < bytes) {
      if (p[i]) cudaFree(p[i]);
      p[i] = nullptr;
      cap[i] = 0;
      if (cudaMalloc(&p[i], bytes) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
      cap[i] = bytes;
    }
    return p[i];
  }
};
HyphaWs& hypha_ws(int dev) {
  static std::mutex m;
  static std::vector<std::unique_ptr<HyphaWs>> ws;
  std::lock_guard<std::mutex> g(m);
  if ((int)ws.size() <= dev) ws.resize((size_t)dev + 1);
  if (!ws[(size_t)dev]) ws[(size_t)dev].reset(new HyphaWs());
  return *ws[(size_t)dev];
}
}

extern "C" int vr_hypha_pivots(const int64_t* col_ptr, const int32_t* rows, int64_t ncols, const int32_t* dims,
                               int32_t flags, int32_t* low_out, vr_hypha_stats* stats) {
  using namespace vr;
  const auto t_call = std::chrono::steady_clock::now();
  try {
    if (ncols < 0 || !col_ptr || !low_out || (ncols && col_ptr[ncols] > 0 && !rows)) return VR_EINVAL;
    if (ncols && col_ptr[0] != 0) return VR_EINVAL;
    for (int64_t j = 0; j < ncols; ++j)
      if (col_ptr[j + 1] < col_ptr[j]) return VR_EINVAL;
    // the rows themselves are validated by k_set_leftmost on the device
    vr_hypha_stats st{};
    const int64_t n = ncols;
    const int64_t nnz = n ? col_ptr[n] : 0;
    std::vector<int32_t> Left((size_t)std::max<int64_t>(n, 1)), Lookup((size_t)std::max<int64_t>(n, 1));
    std::vector<uint8_t> stable((size_t)std::max<int64_t>(n, 1));
    std::vector<int32_t> u;
    if (n) {
      // ---------------- GPU-scan (Alg 3)
      auto chk = [](cudaError_t e) { if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e)); };
      int dev = 0, sms = 148;
      chk(cudaGetDevice(&dev));
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      HyphaWs& ws = hypha_ws(dev);
      std::lock_guard<std::mutex> lk(ws.mu);
      auto* d_ptr = (int64_t*)ws.get(0, (size_t)(n + 1) * 8);
      auto* d_rows = (int32_t*)ws.get(1, (size_t)std::max<int64_t>(nnz, 1) * 4);
      auto* d_left = (int32_t*)ws.get(2, (size_t)n * 4);
      auto* d_lookup = (int32_t*)ws.get(3, (size_t)n * 4);
      auto* d_stable = (uint8_t*)ws.get(4, (size_t)n);
      auto* d_u = (int32_t*)ws.get(5, (size_t)n * 4);
      auto* d_cnt = (unsigned long long*)ws.get(6, 16);
      auto* d_low = (int32_t*)ws.get(7, (size_t)n * 4);
      int* d_bad = (int*)(d_cnt + 1);
      if (!ws.e0) { chk(cudaEventCreate(&ws.e0)); chk(cudaEventCreate(&ws.e1)); }
      chk(cudaMemcpyAsync(d_ptr, col_ptr, (size_t)(n + 1) * 8, cudaMemcpyHostToDevice, 0));
      if (nnz) chk(cudaMemcpyAsync(d_rows, rows, (size_t)nnz * 4, cudaMemcpyHostToDevice, 0));
      st.ms_prepare = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_call).count();
      cudaEventRecord(ws.e0, 0);
      cudaMemsetAsync(d_left, 0x7f, (size_t)n * 4, 0);  // +inf
      cudaMemsetAsync(d_lookup, 0xff, (size_t)n * 4, 0);  // -1
      cudaMemsetAsync(d_stable, 0, (size_t)n, 0);
      cudaMemsetAsync(d_cnt, 0, 16, 0);
      const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)sms * 16);
      k_set_leftmost<<<grid, 256>>>(d_ptr, d_rows, n, d_left, d_stable, d_low, d_bad);
      k_set_lookup<<<grid, 256>>>(d_low, n, d_left, d_lookup, d_stable, (flags & VR_HYPHA_CLEARING) ? 1 : 0);
      k_set_unstable<<<grid, 256>>>(d_stable, n, d_u, d_cnt);
      cudaEventRecord(ws.e1, 0);
      chk(cudaGetLastError());
      unsigned long long cnt[2] = {0, 0};
      chk(cudaMemcpy(cnt, d_cnt, 16, cudaMemcpyDeviceToHost));
      if ((int)cnt[1]) return VR_EINPUT;  // a row not strictly above the diagonal, or not ascending
      float ms = 0;
      cudaEventElapsedTime(&ms, ws.e0, ws.e1);
      st.ms_gpu_scan = ms;
      u.resize((size_t)cnt[0]);
      chk(cudaMemcpy(Left.data(), d_left, (size_t)n * 4, cudaMemcpyDeviceToHost));
      chk(cudaMemcpy(Lookup.data(), d_lookup, (size_t)n * 4, cudaMemcpyDeviceToHost));
      chk(cudaMemcpy(stable.data(), d_stable, (size_t)n, cudaMemcpyDeviceToHost));
      if (cnt[0]) chk(cudaMemcpy(u.data(), d_u, (size_t)cnt[0] * 4, cudaMemcpyDeviceToHost));
    }
    auto t0 = std::chrono::steady_clock::now();
    hypha_host_reduce(col_ptr, rows, n, dims, flags, Left.data(), Lookup.data(), stable.data(), u.data(),
                      (int64_t)u.size(), st);
    st.ms_host = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    for (int64_t j = 0; j < n; ++j) low_out[j] = -1;
    for (int64_t r = 0; r < n; ++r)
      if (Lookup[(size_t)r] >= 0) low_out[Lookup[(size_t)r]] = (int32_t)r;
    st.ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_call).count();
    if (stats) *stats = st;
    return VR_OK;
  } catch (const std::exception& e) {
    vr::set_last_error(e.what());
    return VR_EDEVICE;
  }
}
