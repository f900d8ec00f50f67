// sort.cu — LSD radix sort of 64-bit keys and an exclusive scan, hand-written for sm_100a.
//
// "ascending radix sort of key = ((maxrank - rank(diam)) << cbits) |
// cidx, which gives diam desc, cidx asc. LSD, only the significant bits".  The paper's
// Alg 18 line 5 calls an unnamed library GPU-sort; this is our own.
//
// Up to 131072 keys (RS_CL_MAX x RS_SMALL_CAP): ONE launch of one thread-block cluster,
// every pass in distributed shared memory (rs_cluster; rs_small below 8192 keys).  Larger:
// one cooperative launch (rs_coop) or, past its co-residency limit,
// one pass per 8-bit digit, three launches per pass:
//   rs_hist     per-tile digit histogram  (reads 8 B/key)
//   scan        exclusive scan of the digit-major [256][tiles] histogram
//   rs_scatter  stable in-tile ranking (warp __match_any_sync multisplit over contiguous
//               per-warp segments), staging in shared memory sorted by digit, then
//               coalesced runs written to the digit's global offset (reads 8 + writes 8 B/key)
// Stability: inside a tile order is (digit, position); across tiles the digit-major scan
// orders tiles — so each pass is a stable counting sort, as LSD requires.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>

#include "vr_common.cuh"
#include "vr_internal.h"

namespace vr {

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;  // 4096 keys
constexpr int RS_BINS = 256;
constexpr int RS_SEG = RS_TILE / RS_WARPS;      // 512 keys per warp segment

constexpr int SC_THREADS = 256;
constexpr int SC_ITEMS = 16;
constexpr int SC_TILE = SC_THREADS * SC_ITEMS;

// ------------------------------------------------------------------ scan
__device__ __forceinline__ uint32_t block_exclusive_scan_256(uint32_t x, uint32_t* warp_tot, uint32_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) warp_tot[w] = inc;
  __syncthreads();
  if (w == 0) {
    uint32_t t = lane < (SC_THREADS / 32) ? warp_tot[lane] : 0u;
    uint32_t ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    if (lane < (SC_THREADS / 32)) warp_tot[lane] = ti - t;
    if (lane == (SC_THREADS / 32) - 1) *total = ti;
  }
  __syncthreads();
  uint32_t r = warp_tot[w] + inc - x;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(SC_THREADS) scan_tile_sums(const uint32_t* __restrict__ in, size_t n, uint32_t* __restrict__ sums) {
  __shared__ uint32_t red[SC_THREADS / 32];
  size_t base = (size_t)blockIdx.x * SC_TILE;
  uint32_t acc = 0;
  for (int i = 0; i < SC_ITEMS; ++i) {
    size_t k = base + (size_t)i * SC_THREADS + threadIdx.x;
    if (k < n) acc += in[k];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < SC_THREADS / 32; ++w) t += red[w];
    sums[blockIdx.x] = t;
  }
}

// exclusive scan of one tile, plus an optional per-tile carry
// (in and out may alias: exclusive_scan_u32 scans in place — no __restrict__ on them)
__global__ void __launch_bounds__(SC_THREADS) scan_tile_apply(const uint32_t* in, uint32_t* out, size_t n,
                                                              const uint32_t* __restrict__ carry) {
  __shared__ uint32_t warp_tot[SC_THREADS / 32];
  __shared__ uint32_t total;
  size_t base = (size_t)blockIdx.x * SC_TILE;
  uint32_t run = carry ? carry[blockIdx.x] : 0u;
  for (int i = 0; i < SC_ITEMS; ++i) {
    size_t k = base + (size_t)i * SC_THREADS + threadIdx.x;
    uint32_t x = k < n ? in[k] : 0u;
    uint32_t e = block_exclusive_scan_256(x, warp_tot, &total);
    if (k < n) out[k] = run + e;
    run += total;
    __syncthreads();
  }
}

size_t scan_temp_bytes(size_t n) {
  size_t b = 0;
  while (n > (size_t)SC_TILE) {
    n = (n + SC_TILE - 1) / SC_TILE;
    b += ((n * sizeof(uint32_t) + 255) / 256) * 256;
  }
  return b + 256;
}

// out may alias in.  temp: scan_temp_bytes(n).
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t n, void* temp, cudaStream_t st, int64_t* launches) {
  if (n == 0) return;
  if (n <= (size_t)SC_TILE) {
    scan_tile_apply<<<1, SC_THREADS, 0, st>>>(in, out, n, nullptr);
    if (launches) *launches += 1;
    return;
  }
  size_t nb = (n + SC_TILE - 1) / SC_TILE;
  uint32_t* sums = (uint32_t*)temp;
  void* rest = (char*)temp + ((nb * sizeof(uint32_t) + 255) / 256) * 256;
  scan_tile_sums<<<(unsigned)nb, SC_THREADS, 0, st>>>(in, n, sums);
  exclusive_scan_u32(sums, sums, nb, rest, st, launches);
  scan_tile_apply<<<(unsigned)nb, SC_THREADS, 0, st>>>(in, out, n, sums);
  if (launches) *launches += 2;
}

// ------------------------------------------------------------------ radix sort
__global__ void __launch_bounds__(RS_THREADS) rs_hist(const uint64_t* __restrict__ keys, size_t n, int shift,
                                                      uint32_t* __restrict__ tile_hist, uint32_t ntiles, uint32_t dmask) {
  __shared__ uint32_t h[RS_BINS];
  h[threadIdx.x] = 0;
  __syncthreads();
  size_t base = (size_t)blockIdx.x * RS_TILE;
#pragma unroll 4
  for (int i = 0; i < RS_ITEMS; ++i) {
    size_t k = base + (size_t)i * RS_THREADS + threadIdx.x;
    if (k < n) atomicAdd(&h[(uint32_t)(__ldg(keys + k) >> shift) & dmask], 1u);
  }
  __syncthreads();
  tile_hist[(size_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(RS_THREADS) rs_scatter(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, size_t n, int shift,
                                                         const uint32_t* __restrict__ offsets, uint32_t ntiles, uint32_t dmask) {
  extern __shared__ __align__(16) unsigned char rs_smem[];
  uint64_t* keys_s = (uint64_t*)rs_smem;                 // tile keys, input order
  uint64_t* sorted_s = keys_s + RS_TILE;                 // tile keys, digit order
  uint32_t* whist = (uint32_t*)(sorted_s + RS_TILE);     // [RS_WARPS][RS_BINS]
  uint32_t* dstart = whist + RS_WARPS * RS_BINS;         // [RS_BINS]
  uint32_t* gofs = dstart + RS_BINS;                     // [RS_BINS]
  __shared__ uint32_t warp_tot[SC_THREADS / 32];
  __shared__ uint32_t total;

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const size_t base = (size_t)blockIdx.x * RS_TILE;
  const int cnt = (int)((n - base) < (size_t)RS_TILE ? (n - base) : (size_t)RS_TILE);

  for (int i = threadIdx.x; i < RS_TILE; i += RS_THREADS) keys_s[i] = i < cnt ? in[base + i] : ~0ull;
  for (int i = threadIdx.x; i < RS_WARPS * RS_BINS; i += RS_THREADS) whist[i] = 0;
  __syncthreads();

  // per-warp digit counts over the warp's contiguous segment
  const int seg0 = w * RS_SEG;
  for (int i = seg0 + lane; i < seg0 + RS_SEG; i += 32)
    if (i < cnt) atomicAdd(&whist[w * RS_BINS + ((uint32_t)(keys_s[i] >> shift) & dmask)], 1u);
  __syncthreads();

  // thread b: exclusive prefix over warps of digit b; tile total of digit b
  {
    const int b = threadIdx.x;
    uint32_t run = 0;
#pragma unroll
    for (int q = 0; q < RS_WARPS; ++q) {
      uint32_t t = whist[q * RS_BINS + b];
      whist[q * RS_BINS + b] = run;
      run += t;
    }
    uint32_t e = block_exclusive_scan_256(run, warp_tot, &total);
    dstart[b] = e;
    gofs[b] = offsets[(size_t)b * ntiles + blockIdx.x];
  }
  __syncthreads();

  // stable ranking: each warp walks its segment in order, 32 keys per step
  for (int i0 = seg0; i0 < seg0 + RS_SEG; i0 += 32) {
    const int i = i0 + lane;
    const bool valid = i < cnt;
    const uint64_t k = keys_s[i];
    const uint32_t dg = valid ? ((uint32_t)(k >> shift) & dmask) : (RS_BINS + lane);
    const uint32_t peers = __match_any_sync(0xffffffffu, dg);
    uint32_t pos = 0;
    if (valid) pos = dstart[dg] + whist[w * RS_BINS + dg] + __popc(peers & lanemask_lt());
    __syncwarp();
    if (valid && (lane == 31 - __clz(peers))) whist[w * RS_BINS + dg] += __popc(peers);
    if (valid) sorted_s[pos] = k;
    __syncwarp();
  }
  __syncthreads();

  for (int j = threadIdx.x; j < cnt; j += RS_THREADS) {
    const uint64_t k = sorted_s[j];
    const uint32_t dg = (uint32_t)(k >> shift) & dmask;
    out[(size_t)gofs[dg] + (size_t)(j - (int)dstart[dg])] = k;
  }
}


// Tile ranking shared by the kernels below: stable per-warp-segment multisplit of keys_s
// (cnt valid keys) on digit `shift`, writing the keys in digit order to sorted_s and the
// tile's digit starts to dstart.  All 256 threads of the block must call it.
// Stable in-shared-memory counting pass over cnt keys.  The keys are cut into RS_WARPS
// contiguous warp segments of `seg` = cnt/RS_WARPS rounded up to whole warps, so a short
// tile costs only the iterations it needs (the histogram, the prefix over warps and the
// multisplit ranking all stay stable: earlier segments = earlier warps).
__device__ __forceinline__ void rs_tile_rank(const uint64_t* keys_s, uint64_t* sorted_s, int cnt, int shift, uint32_t dmask,
                                             uint32_t* whist, uint32_t* dstart, uint32_t* warp_tot, uint32_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int seg = ((cnt + RS_WARPS * 32 - 1) / (RS_WARPS * 32)) * 32;
  for (int i = threadIdx.x; i < RS_WARPS * RS_BINS; i += RS_THREADS) whist[i] = 0;
  __syncthreads();
  const int seg0 = w * seg;
  for (int i = seg0 + lane; i < seg0 + seg; i += 32)
    if (i < cnt) atomicAdd(&whist[w * RS_BINS + ((uint32_t)(keys_s[i] >> shift) & dmask)], 1u);
  __syncthreads();
  {
    const int b = threadIdx.x;
    uint32_t run = 0;
#pragma unroll
    for (int q = 0; q < RS_WARPS; ++q) {
      uint32_t t = whist[q * RS_BINS + b];
      whist[q * RS_BINS + b] = run;
      run += t;
    }
    dstart[b] = block_exclusive_scan_256(run, warp_tot, total);
  }
  __syncthreads();
  for (int i0 = seg0; i0 < seg0 + seg && i0 < cnt; i0 += 32) {
    const int i = i0 + lane;
    const bool valid = i < cnt;
    const uint64_t k = valid ? keys_s[i] : 0ull;
    const uint32_t dg = valid ? ((uint32_t)(k >> shift) & dmask) : (RS_BINS + lane);
    const uint32_t peers = __match_any_sync(0xffffffffu, dg);
    uint32_t pos = 0;
    if (valid) pos = dstart[dg] + whist[w * RS_BINS + dg] + __popc(peers & lanemask_lt());
    __syncwarp();
    if (valid && (lane == 31 - __clz(peers))) whist[w * RS_BINS + dg] += __popc(peers);
    if (valid) sorted_s[pos] = k;
    __syncwarp();
  }
  __syncthreads();
}

// Digit b's total over all tiles and the part in tiles before `me`, from the digit-major
// tile histogram.  Loads are issued 8 at a time (independent, from L2 — the histogram was
// written by other CTAs of this pass), so a pass waits one L2 latency per 8 tiles instead of
// one per tile.
__device__ __forceinline__ void digit_totals(const uint32_t* th, int b, uint32_t ntiles, uint32_t me, uint32_t& tot,
                                             uint32_t& before) {
  const uint32_t* row = th + (size_t)b * ntiles;
  tot = 0;
  before = 0;
  uint32_t t = 0;
  for (; t + 8 <= ntiles; t += 8) {
    uint32_t c[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = __ldcg(row + t + k);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      tot += c[k];
      before += (t + (uint32_t)k < me) ? c[k] : 0u;
    }
  }
  for (; t < ntiles; ++t) {
    const uint32_t c = __ldcg(row + t);
    tot += c;
    before += t < me ? c : 0u;
  }
}

// Whole sort of n <= RS_SMALL_CAP keys in one CTA, every pass in shared memory, one launch.
constexpr int RS_SMALL_CAP = 2 * RS_TILE;
__global__ void __launch_bounds__(RS_THREADS) rs_small(uint64_t* __restrict__ keys, int n, int begin_bit, int end_bit) {
  extern __shared__ __align__(16) unsigned char rs_smem[];
  uint64_t* A = (uint64_t*)rs_smem;
  uint64_t* Bk = A + RS_SMALL_CAP;
  uint32_t* whist = (uint32_t*)(Bk + RS_SMALL_CAP);
  uint32_t* dstart = whist + RS_WARPS * RS_BINS;
  __shared__ uint32_t warp_tot[SC_THREADS / 32];
  __shared__ uint32_t total;
  for (int i = threadIdx.x; i < n; i += RS_THREADS) A[i] = keys[i];
  __syncthreads();
  for (int shift = begin_bit; shift < end_bit; shift += 8) {
    const uint32_t dmask = end_bit - shift >= 8 ? 0xFFu : ((1u << (end_bit - shift)) - 1u);
    rs_tile_rank(A, Bk, n, shift, dmask, whist, dstart, warp_tot, &total);
    uint64_t* t = A; A = Bk; Bk = t;
  }
  for (int i = threadIdx.x; i < n; i += RS_THREADS) keys[i] = A[i];
}

// Whole sort of n <= RS_CL_MAX * RS_SMALL_CAP keys by ONE thread-block cluster (up to 16
// CTAs of 1024 threads, one per SM): the keys stay in the cluster's distributed shared
// memory for every pass.  Per pass: each CTA counts the digits of its tile per warp segment
// and publishes the tile's counts in its own shared memory; cluster barrier; every CTA reads
// all tiles' counts over DSMEM (digit totals + the counts of lower-ranked CTAs = the stable
// global start of each of its digits) and ranks its keys (warp multisplit, stable) straight
// into the owning CTA's next-pass buffer (DSMEM stores); cluster barrier.  No grid-wide
// barrier and no global-memory round trip between passes.
constexpr int RS_CL_MAX = 16;
constexpr int CL_THREADS = 1024;
constexpr int CL_WARPS = CL_THREADS / 32;

__device__ __forceinline__ uint32_t block_exclusive_scan_1024(uint32_t x, uint32_t* warp_tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) warp_tot[w] = inc;
  __syncthreads();
  if (w == 0) {
    const uint32_t t = warp_tot[lane];
    uint32_t ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    warp_tot[lane] = ti - t;
  }
  __syncthreads();
  const uint32_t r = warp_tot[w] + inc - x;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(CL_THREADS, 1) rs_cluster(uint64_t* __restrict__ keys, int n, int begin_bit, int end_bit,
                                                            int tile) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int me = (int)cl.block_rank();
  const int csize = (int)cl.num_blocks();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  extern __shared__ __align__(16) unsigned char rs_smem[];
  uint64_t* A = (uint64_t*)rs_smem;            // this pass's input tile
  uint64_t* Bk = A + RS_SMALL_CAP;             // this pass's output tile (written by every CTA)
  uint32_t* whist = (uint32_t*)(Bk + RS_SMALL_CAP);  // [CL_WARPS][RS_BINS]
  uint32_t* hist = whist + CL_WARPS * RS_BINS;  // this tile's digit counts (read by the cluster)
  uint32_t* gofs = hist + RS_BINS;              // global start of this tile's keys of each digit
  __shared__ uint32_t warp_tot[CL_WARPS];
  const int base = me * tile;
  const int cnt = n - base < tile ? (n - base > 0 ? n - base : 0) : tile;
  const int seg = ((cnt + CL_WARPS * 32 - 1) / (CL_WARPS * 32)) * 32;  // keys per warp segment
  const int seg0 = w * seg;
  for (int i = threadIdx.x; i < cnt; i += CL_THREADS) A[i] = keys[base + i];
  for (int shift = begin_bit; shift < end_bit; shift += 8) {
    const uint32_t dmask = end_bit - shift >= 8 ? 0xFFu : ((1u << (end_bit - shift)) - 1u);
    for (int i = threadIdx.x; i < CL_WARPS * RS_BINS; i += CL_THREADS) whist[i] = 0;
    __syncthreads();
    for (int i = seg0 + lane; i < seg0 + seg; i += 32)
      if (i < cnt) atomicAdd(&whist[w * RS_BINS + ((uint32_t)(A[i] >> shift) & dmask)], 1u);
    __syncthreads();
    if (threadIdx.x < RS_BINS) {  // prefix over warp segments (stability) and the tile count
      const int b = threadIdx.x;
      uint32_t run = 0;
      for (int q = 0; q < CL_WARPS; ++q) {
        const uint32_t t = whist[q * RS_BINS + b];
        whist[q * RS_BINS + b] = run;
        run += t;
      }
      hist[b] = run;
    }
    cl.sync();  // every tile's counts published; the previous pass's scatter is complete
    uint32_t tot = 0, before = 0;
    if (threadIdx.x < RS_BINS) {
      const int b = threadIdx.x;
      for (int c = 0; c < csize; ++c) {
        const uint32_t h = cl.map_shared_rank(hist, c)[b];
        tot += h;
        before += c < me ? h : 0u;
      }
    }
    const uint32_t dig_start = block_exclusive_scan_1024(threadIdx.x < RS_BINS ? tot : 0u, warp_tot);
    if (threadIdx.x < RS_BINS) gofs[threadIdx.x] = dig_start + before;
    __syncthreads();
    for (int i0 = seg0; i0 < seg0 + seg && i0 < cnt; i0 += 32) {
      const int i = i0 + lane;
      const bool valid = i < cnt;
      const uint64_t k = valid ? A[i] : 0ull;
      const uint32_t dg = valid ? ((uint32_t)(k >> shift) & dmask) : (RS_BINS + lane);
      const uint32_t peers = __match_any_sync(0xffffffffu, dg);
      int pos = 0;
      if (valid) pos = (int)(gofs[dg] + whist[w * RS_BINS + dg] + __popc(peers & lanemask_lt()));
      __syncwarp();
      if (valid && (lane == 31 - __clz(peers))) whist[w * RS_BINS + dg] += __popc(peers);
      if (valid) {
        const int dst = pos / tile;
        cl.map_shared_rank(Bk, dst)[pos - dst * tile] = k;
      }
      __syncwarp();
    }
    cl.sync();  // the next pass's tiles are complete
    uint64_t* t = A; A = Bk; Bk = t;
  }
  for (int i = threadIdx.x; i < cnt; i += CL_THREADS) keys[base + i] = A[i];
}

// Scatter for up to RS_FUSED_TILES tiles: the block computes its own digit offsets from
// the per-tile histogram (no separate scan launch).
constexpr uint32_t RS_FUSED_TILES = 256;
__global__ void __launch_bounds__(RS_THREADS) rs_scatter_fused(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                                                               size_t n, int shift, const uint32_t* __restrict__ tile_hist,
                                                               uint32_t ntiles, uint32_t dmask) {
  extern __shared__ __align__(16) unsigned char rs_smem[];
  uint64_t* keys_s = (uint64_t*)rs_smem;
  uint64_t* sorted_s = keys_s + RS_TILE;
  uint32_t* whist = (uint32_t*)(sorted_s + RS_TILE);
  uint32_t* dstart = whist + RS_WARPS * RS_BINS;
  uint32_t* gofs = dstart + RS_BINS;
  __shared__ uint32_t warp_tot[SC_THREADS / 32];
  __shared__ uint32_t total;
  const size_t base = (size_t)blockIdx.x * RS_TILE;
  const int cnt = (int)((n - base) < (size_t)RS_TILE ? (n - base) : (size_t)RS_TILE);
  for (int i = threadIdx.x; i < RS_TILE; i += RS_THREADS) keys_s[i] = i < cnt ? in[base + i] : ~0ull;
  // global offset of digit b for this tile = sum over digits < b of all tiles
  //                                          + sum over earlier tiles of digit b
  {
    const int b = threadIdx.x;
    uint32_t tot_b, before;
    digit_totals(tile_hist, b, ntiles, blockIdx.x, tot_b, before);
    const uint32_t dig_start = block_exclusive_scan_256(tot_b, warp_tot, &total);
    gofs[b] = dig_start + before;
  }
  __syncthreads();
  rs_tile_rank(keys_s, sorted_s, cnt, shift, dmask, whist, dstart, warp_tot, &total);
  for (int j = threadIdx.x; j < cnt; j += RS_THREADS) {
    const uint64_t k = sorted_s[j];
    const uint32_t dg = (uint32_t)(k >> shift) & dmask;
    out[(size_t)gofs[dg] + (size_t)(j - (int)dstart[dg])] = k;
  }
}


// Every pass in ONE cooperative launch (one CTA per tile, all co-resident): per-tile
// histogram -> grid sync -> offsets + stable scatter -> grid sync, per 8-bit digit.
__global__ void __launch_bounds__(RS_THREADS) rs_coop(uint64_t* __restrict__ a, uint64_t* __restrict__ b, size_t n,
                                                     int begin_bit, int end_bit, uint32_t* __restrict__ tile_hist,
                                                     uint32_t ntiles, int tile) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char rs_smem[];
  uint64_t* keys_s = (uint64_t*)rs_smem;
  uint64_t* sorted_s = keys_s + RS_TILE;
  uint32_t* whist = (uint32_t*)(sorted_s + RS_TILE);
  uint32_t* dstart = whist + RS_WARPS * RS_BINS;
  uint32_t* gofs = dstart + RS_BINS;
  __shared__ uint32_t warp_tot[SC_THREADS / 32];
  __shared__ uint32_t total;
  __shared__ uint32_t h[RS_BINS];
  // tile <= RS_TILE keys per CTA: smaller tiles put more SMs on a mid-size sort
  const size_t base = (size_t)blockIdx.x * (size_t)tile;
  const int cnt = (int)((n - base) < (size_t)tile ? (n - base) : (size_t)tile);
  uint64_t* src = a;
  uint64_t* dst = b;
  for (int shift = begin_bit; shift < end_bit; shift += 8) {
    const uint32_t dmask = end_bit - shift >= 8 ? 0xFFu : ((1u << (end_bit - shift)) - 1u);
    for (int i = threadIdx.x; i < cnt; i += RS_THREADS) keys_s[i] = src[base + i];
    h[threadIdx.x] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += RS_THREADS) atomicAdd(&h[(uint32_t)(keys_s[i] >> shift) & dmask], 1u);
    __syncthreads();
    tile_hist[(size_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
    grid.sync();
    {
      const int bb = threadIdx.x;
      uint32_t tot_b, before;
      digit_totals(tile_hist, bb, ntiles, blockIdx.x, tot_b, before);
      const uint32_t dig_start = block_exclusive_scan_256(tot_b, warp_tot, &total);
      gofs[bb] = dig_start + before;
    }
    __syncthreads();
    rs_tile_rank(keys_s, sorted_s, cnt, shift, dmask, whist, dstart, warp_tot, &total);
    for (int j = threadIdx.x; j < cnt; j += RS_THREADS) {
      const uint64_t k = sorted_s[j];
      const uint32_t dg = (uint32_t)(k >> shift) & dmask;
      dst[(size_t)gofs[dg] + (size_t)(j - (int)dstart[dg])] = k;
    }
    grid.sync();  // the next pass reads dst, and tile_hist is rewritten
    uint64_t* t = src; src = dst; dst = t;
  }
}

static size_t align256(size_t b) { return (b + 255) / 256 * 256; }

size_t radix_sort_temp_bytes(size_t n) {
  size_t ntiles = (n + 1023) / 1024;  // the cooperative path may use tiles down to 1024 keys
  size_t hist = (size_t)RS_BINS * ntiles;
  return align256(hist * sizeof(uint32_t)) + scan_temp_bytes(hist);
}


// Sorts keys[0..n) ascending on bits [begin_bit, end_bit).  alt is a ping-pong buffer of
// n keys.  Returns the buffer holding the result (keys or alt).
uint64_t* radix_sort_u64(uint64_t* keys, uint64_t* alt, size_t n, int begin_bit, int end_bit, void* temp,
                         cudaStream_t st, int64_t* launches) {
  if (n <= 1 || end_bit <= begin_bit) return keys;
  const size_t smem = 2 * RS_TILE * sizeof(uint64_t) + (RS_WARPS * RS_BINS + 2 * RS_BINS) * sizeof(uint32_t);
  const size_t smem_small = 2 * RS_SMALL_CAP * sizeof(uint64_t) + (RS_WARPS * RS_BINS + 2 * RS_BINS) * sizeof(uint32_t);
  static const char attr_tag = 0, cl_tag = 0, coop_tag = 0;  // per-device memo keys
  device_memo(&attr_tag, [&] {
    cudaFuncSetAttribute(rs_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(rs_scatter_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(rs_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_small);
    return 1;
  });
  // one cluster, all passes in distributed shared memory
  const size_t smem_cl = 2 * RS_SMALL_CAP * sizeof(uint64_t) + (CL_WARPS * RS_BINS + 2 * RS_BINS) * sizeof(uint32_t);
  const int cl_max = device_memo(&cl_tag, [&] {
    int cl_max = 0;
    if (!std::getenv("VR_NO_CLUSTER_SORT") &&
        cudaFuncSetAttribute(rs_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cl) == cudaSuccess &&
        cudaFuncSetAttribute(rs_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
      for (int c = RS_CL_MAX; c >= 2 && cl_max == 0; c /= 2) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)c;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3((unsigned)c);
        cfg.blockDim = dim3(CL_THREADS);
        cfg.dynamicSmemBytes = smem_cl;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, (void*)rs_cluster, &cfg) == cudaSuccess && ncl > 0) cl_max = c;
      }
    }
    cudaGetLastError();
    return cl_max;
  });
  // one CTA, all passes in shared memory: up to RS_SMALL_CAP keys without clusters, else
  // up to VR_SMALL_SORT_MAX (default 2048) keys — above that a cluster of 2-4 CTAs of 1024
  // threads sorts faster than one 256-thread CTA
  static const size_t small_max = []() {
    const char* e = std::getenv("VR_SMALL_SORT_MAX");
    const long long v = e ? std::atoll(e) : 2048;
    return (size_t)(v >= 0 && v <= RS_SMALL_CAP ? v : 2048);
  }();
  if (n <= (size_t)RS_SMALL_CAP && (cl_max == 0 || n <= small_max)) {
    rs_small<<<1, RS_THREADS, smem_small, st>>>(keys, (int)n, begin_bit, end_bit);
    if (launches) *launches += 1;
    return keys;
  }
  if (cl_max > 0 && n <= (size_t)cl_max * RS_SMALL_CAP) {
    // the smallest power-of-two cluster whose CTAs hold at most `per` keys each (capped at the
    // largest cluster; VR_CL_TILE overrides `per`)
    static const size_t per = []() {
      const char* e = std::getenv("VR_CL_TILE");
      const long long v = e ? std::atoll(e) : 0;
      return (size_t)(v >= 256 && v <= RS_SMALL_CAP ? v : 1024);  // 1024: measured best (tools/ab_sort_sweep.sh)
    }();
    int c = 2;
    while ((size_t)c * per < n && c < cl_max) c *= 2;
    int tile = (int)((n + (size_t)c - 1) / (size_t)c);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)c;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)c);
    cfg.blockDim = dim3(CL_THREADS);
    cfg.dynamicSmemBytes = smem_cl;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nn = (int)n;
    cudaLaunchKernelEx(&cfg, rs_cluster, keys, nn, begin_bit, end_bit, tile);
    if (launches) *launches += 1;
    return keys;
  }
  const uint32_t ntiles = (uint32_t)((n + RS_TILE - 1) / RS_TILE);
  uint32_t* hist = (uint32_t*)temp;
  const int coop_cap = device_memo(&coop_tag, [&] {
    int dev = 0, sms = 0, per = 0, coop = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    cudaFuncSetAttribute(rs_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, rs_coop, RS_THREADS, smem);
    return coop ? sms * per : 0;
  });
  if ((int)ntiles <= coop_cap) {  // every pass in one cooperative launch
    const int passes = (end_bit - begin_bit + 7) / 8;
    // halve the tile while the grid stays small: a pass's latency scales with the keys per
    // CTA, but every CTA also walks all ntiles histograms, so stop at 32 tiles
    int tile = RS_TILE;
    uint32_t nt = ntiles;
    int sms = 148;
    {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    while (tile > 1024) {
      const uint32_t nt2 = (uint32_t)((n + (size_t)(tile / 2) - 1) / (size_t)(tile / 2));
      if ((int)nt2 > coop_cap || (int)nt2 > sms || nt2 > 32) break;
      tile /= 2;
      nt = nt2;
    }
    void* args[] = {(void*)&keys, (void*)&alt, (void*)&n, (void*)&begin_bit, (void*)&end_bit, (void*)&hist, (void*)&nt,
                    (void*)&tile};
    cudaLaunchCooperativeKernel((void*)rs_coop, dim3(nt), dim3(RS_THREADS), args, smem, st);
    if (launches) *launches += 1;
    return (passes & 1) ? alt : keys;
  }
  void* scan_tmp = (char*)temp + align256((size_t)RS_BINS * ntiles * sizeof(uint32_t));
  uint64_t* src = keys;
  uint64_t* dst = alt;
  for (int shift = begin_bit; shift < end_bit; shift += 8) {
    const uint32_t dmask = end_bit - shift >= 8 ? 0xFFu : ((1u << (end_bit - shift)) - 1u);
    rs_hist<<<ntiles, RS_THREADS, 0, st>>>(src, n, shift, hist, ntiles, dmask);
    if (ntiles <= RS_FUSED_TILES) {
      rs_scatter_fused<<<ntiles, RS_THREADS, smem, st>>>(src, dst, n, shift, hist, ntiles, dmask);
    } else {
      exclusive_scan_u32(hist, hist, (size_t)RS_BINS * ntiles, scan_tmp, st, launches);
      rs_scatter<<<ntiles, RS_THREADS, smem, st>>>(src, dst, n, shift, hist, ntiles, dmask);
    }
    if (launches) *launches += 2;
    uint64_t* t = src; src = dst; dst = t;
  }
  return src;
}

// ------------------------------------------------------------------ k-way merge (a7)
// Every key's output position = its index in its own list + the number of smaller keys in
// each other list (binary search; keys are distinct, so positions are distinct) — the
// merge path of each element computed directly, no sequential cursor.
__global__ void k_merge_gathered(const uint64_t* __restrict__ g, int world, uint64_t cap, uint64_t* __restrict__ out) {
  const uint64_t total = (uint64_t)world * cap;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = __ldg(g + e);
    if (x == ~0ull) continue;
    const int r = (int)(e / cap);
    uint64_t pos = e - (uint64_t)r * cap;
    for (int h = 0; h < world; ++h) {
      if (h == r) continue;
      const uint64_t* L = g + (uint64_t)h * cap;
      uint64_t lo = 0, hi = cap;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (__ldg(L + mid) < x) lo = mid + 1; else hi = mid;
      }
      pos += lo;
    }
    VR_ASSERT(pos < total);
    out[pos] = x;
  }
}

void merge_gathered_u64(const uint64_t* gathered, int world, uint64_t cap, uint64_t* out, cudaStream_t st, int64_t* launches) {
  const uint64_t total = (uint64_t)world * cap;
  if (!total) return;
  const uint64_t blocks = std::min<uint64_t>((total + 255) / 256, 148ull * 8);
  k_merge_gathered<<<(unsigned)blocks, 256, 0, st>>>(gathered, world, cap, out);
  if (launches) *launches += 1;
}

// ------------------------------------------------------------------ column keys (a4)
// Column keys are ((maxr - rank) << cbits) | cidx.  Residual columns rarely share a
// diameter, so they are counting-sorted on the rank field (a histogram over the maxr + 1
// values, a scan, an atomic placement: 3 short kernels instead of 8 radix passes at config
// 5, dimension 3) and every run of equal rank is then sorted by cidx in place — valid while
// no run is longer than FIX_RUN_MAX (checked on the first run; past it the full sort).
constexpr int FIX_RUN_MAX = 4096;  // (config 5, dimension 3: 552K keys, longest run 60)
constexpr int FIX_RUN_REG = 16;    // runs up to this length are sorted in registers
constexpr uint64_t FIX_LONG_CAP = 1 << 16;  // long runs listed per sort

// Runs of up to FIX_RUN_REG keys: one thread, in registers; longer ones (up to FIX_RUN_MAX)
// are listed (d_long[0] = count, then run starts) for k_fix_long_runs; longer still: flag.
__global__ void k_fix_runs(uint64_t* __restrict__ k, uint64_t n, int cbits, unsigned int* __restrict__ overflow,
                           uint64_t* __restrict__ d_long, uint64_t long_cap) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t hi = k[i] >> cbits;
    if (i > 0 && (k[i - 1] >> cbits) == hi) continue;  // not the start of a run
    uint64_t e = i + 1;
    while (e < n && (k[e] >> cbits) == hi && e - i <= (uint64_t)FIX_RUN_MAX) ++e;
    const int len = (int)(e - i);
    if (len == 1) continue;
    if (len > FIX_RUN_MAX) {  // too long: the caller falls back to the full sort
      atomicOr(overflow, 1u);
      continue;
    }
    if (len > FIX_RUN_REG) {
      const unsigned long long slot = atomicAdd((unsigned long long*)d_long, 1ull);
      if (slot < long_cap) d_long[1 + slot] = i;
      else atomicOr(overflow, 1u);
      continue;
    }
    if (len <= 4) {  // the common case (config 5, dimension 3: mean run 2.4): a 4-key network
      uint64_t a0 = k[i], a1 = k[i + 1], a2 = len > 2 ? k[i + 2] : ~0ull, a3 = len > 3 ? k[i + 3] : ~0ull;
#define VR_CS(x, y) { const uint64_t lo_ = x < y ? x : y, hi_ = x < y ? y : x; x = lo_; y = hi_; }
      VR_CS(a0, a1) VR_CS(a2, a3) VR_CS(a0, a2) VR_CS(a1, a3) VR_CS(a1, a2)
#undef VR_CS
      k[i] = a0;
      k[i + 1] = a1;
      if (len > 2) k[i + 2] = a2;
      if (len > 3) k[i + 3] = a3;
      continue;
    }
    uint64_t v[FIX_RUN_REG];
#pragma unroll
    for (int a = 0; a < FIX_RUN_REG; ++a) v[a] = a < len ? k[i + (uint64_t)a] : ~0ull;
    // odd-even transposition network on the fixed-size register array (no local memory);
    // the ~0 padding sorts to the end
#pragma unroll
    for (int r = 0; r < FIX_RUN_REG; ++r)
#pragma unroll
      for (int a = r & 1; a + 1 < FIX_RUN_REG; a += 2)
        if (v[a] > v[a + 1]) { const uint64_t t = v[a]; v[a] = v[a + 1]; v[a + 1] = t; }
#pragma unroll
    for (int a = 0; a < FIX_RUN_REG; ++a)
      if (a < len) k[i + (uint64_t)a] = v[a];
  }
}

// one warp per listed long run: every key's place = the number of smaller keys in the run
__global__ void k_fix_long_runs(uint64_t* __restrict__ k, uint64_t n, int cbits, const uint64_t* __restrict__ d_long,
                                uint64_t long_cap, uint64_t* __restrict__ tmp) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t cnt = d_long[0] < long_cap ? d_long[0] : long_cap;  // (past the cap: the caller re-sorts)
  for (uint64_t q = warp; q < cnt; q += nw) {
    const uint64_t i = d_long[1 + q];
    const uint64_t hi = k[i] >> cbits;
    uint64_t e = i + 1;
    while (e < n && (k[e] >> cbits) == hi) ++e;
    const int len = (int)(e - i);
    for (int a = lane; a < len; a += 32) {
      const uint64_t x = k[i + (uint64_t)a];
      int pos = 0;
      for (int b = 0; b < len; ++b) pos += k[i + (uint64_t)b] < x;
      VR_ASSERT(i + (uint64_t)len <= n && pos < len);
      tmp[i + (uint64_t)pos] = x;
    }
    __syncwarp();
    for (int a = lane; a < len; a += 32) k[i + (uint64_t)a] = tmp[i + (uint64_t)a];
    __syncwarp();
  }
}

__global__ void k_count_hi(const uint64_t* __restrict__ k, uint64_t n, int cbits, uint32_t* __restrict__ cnt) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + (__ldg(k + i) >> cbits), 1u);
}
__global__ void k_place_hi(const uint64_t* __restrict__ k, uint64_t n, int cbits, uint32_t* __restrict__ off,
                           uint64_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = __ldg(k + i);
    out[atomicAdd(off + (x >> cbits), 1u)] = x;  // (order within a run: fixed by k_fix_runs)
  }
}

size_t sort_columns_temp_bytes(uint64_t bins) {  // counts, offsets, scan temp, the long-run list
  return 2 * (((bins + 1) * 4 + 255) / 256 * 256) + (scan_temp_bytes(bins + 1) + 255) / 256 * 256 + (FIX_LONG_CAP + 1) * 8;
}

uint64_t* sort_columns(uint64_t* keys, uint64_t* alt, size_t n, int cbits, int end_bit, uint64_t bins, void* temp,
                       void* cnt_temp, int* mode, unsigned int* d_flag, cudaStream_t st, int64_t* launches) {
  if (n <= 1) return keys;
  // (worth it for many keys with short runs — few keys per rank; up to 131072 keys the
  // one-cluster radix sort is a single launch)
  if (*mode < 0 && ((uint64_t)n > 4 * bins || n <= 131072)) *mode = 0;
  if (*mode == 0 || cbits >= end_bit || !cnt_temp) return radix_sort_u64(keys, alt, n, 0, end_bit, temp, st, launches);
  // a counting sort on the rank field (bins = maxr + 1 values), then the runs
  const size_t cb = ((bins + 1) * 4 + 255) / 256 * 256;
  uint32_t* cnt = (uint32_t*)cnt_temp;
  uint32_t* off = (uint32_t*)((char*)cnt_temp + cb);
  void* scan_tmp = (char*)cnt_temp + 2 * cb;
  const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, 148ull * 8);
  cudaMemsetAsync(cnt, 0, (bins + 1) * 4, st);
  k_count_hi<<<(unsigned)blocks, 256, 0, st>>>(keys, n, cbits, cnt);
  exclusive_scan_u32(cnt, off, bins + 1, scan_tmp, st, launches);
  k_place_hi<<<(unsigned)blocks, 256, 0, st>>>(keys, n, cbits, off, alt);
  uint64_t* out = alt;
  if (launches) *launches += 2;
  if (*mode < 0) cudaMemsetAsync(d_flag, 0, 4, st);
  uint64_t* d_long = (uint64_t*)((char*)cnt_temp + sort_columns_temp_bytes(bins) - (FIX_LONG_CAP + 1) * 8);
  cudaMemsetAsync(d_long, 0, 8, st);
  k_fix_runs<<<(unsigned)blocks, 256, 0, st>>>(out, n, cbits, d_flag, d_long, FIX_LONG_CAP);
  k_fix_long_runs<<<148 * 4, 256, 0, st>>>(out, n, cbits, d_long, FIX_LONG_CAP, keys);
  if (launches) *launches += 2;
  if (*mode < 0) {  // the first run decides
    unsigned int f = 0;
    cudaMemcpyAsync(&f, d_flag, 4, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    *mode = f ? 0 : 1;
    if (f) return radix_sort_u64(out, keys, n, 0, end_bit, temp, st, launches);
  }
  return out;
}

}  // namespace vr
