// tables.cu — step a0: the device tables every later kernel reads.
//
//   1. tb_rowmax    : row maxima of the symmetric matrix (enclosing radius, §5.2.12), by
//                     32 x 32 tiles of the lower triangle (row and column maxima).
//   2. tb_threshold : R = min_i rowmax_i, t = threshold or R when threshold is
//                     +inf (Prop 5.2.13).
//   3. tb_edge_count / scan / tb_edge_compact : validate the fp32 lower-distance input
//                     (VR_EINPUT on NaN / negative) and write one 64-bit key per edge with
//                     d <= t (inclusive, Eq 5.3), (fp32 bits << kbits) | (N-1-k), k = lower-
//                     distance index = edge cidx (Eq 5.6: C(i,2) + j), in DEscending k order; m = their
//                     number.  (A sparse threshold keeps few edges: config 5 sorts 234K keys
//                     instead of 8.4M.)
//   4. radix sort of the m keys on the 31 distance bits (stable) — ascending = diameter
//                     ascending, cidx DEscending: exactly the §5.1.4 filtration order of the
//                     edges (dimension 0 walks it for union-find) and the sorted distance
//                     list the ranks index.
//   5. tb_rank_scatter : rank[i][j] = index of the first sorted edge with the value d(i,j)
//                     (a lower bound, computed once per edge under t and scattered to (i, j)
//                     and (j, i) of a matrix pre-filled with RINF), or RINF when d(i,j) > t or
//                     i = j; in the output-sensitive mode also the threshold-graph bitmap.  Equal distances get equal
//                     ranks and the order is kept, so rank comparisons are the paper's
//                     diameter comparisons, exactly (reading A11: no arithmetic on values).
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "vr_common.cuh"
#include "vr_internal.h"

namespace vr {

__device__ __forceinline__ float lt_at(const float* __restrict__ lt, int64_t i, int64_t j) {
  if (i == j) return 0.0f;
  if (i < j) { int64_t t = i; i = j; j = t; }
  return __ldg(lt + i * (i - 1) / 2 + j);
}

__device__ __forceinline__ uint32_t dist_bits(float x) {
  // non-negative fp32 values order like their uint32 bit patterns; map -0.0 to +0.0
  return x == 0.0f ? 0u : __float_as_uint(x);
}

// The symmetric matrix in 32 x 32 tiles (I, J), I >= J, of the lower triangle: a tile's rows
// i = 32I + a are contiguous runs of the lower-distance vector (coalesced reads); its column
// maxima are row maxima of the transposed tile (symmetry), and its ranks are written to
// both (i, j) and (j, i) through a transpose in shared memory (coalesced writes).
__device__ __forceinline__ void tile_of(uint32_t b, int& I, int& J) {
  int t = (int)((sqrtf(8.0f * (float)b + 1.0f) - 1.0f) * 0.5f);
  while ((uint64_t)(t + 1) * (uint64_t)(t + 2) / 2 <= b) ++t;
  while ((uint64_t)t * (uint64_t)(t + 1) / 2 > b) --t;
  I = t;
  J = (int)(b - (uint32_t)((uint64_t)t * (uint64_t)(t + 1) / 2));
}

// rowmax[] must be zero on entry (atomicMax of the non-negative fp32 bit patterns)
__global__ void tb_rowmax(const float* __restrict__ lt, int64_t n, uint32_t* __restrict__ rowmax) {
  __shared__ uint32_t cmax[8][32];
  int I, J;
  tile_of(blockIdx.x, I, J);
  const int bx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads, 4 rows each
  const int64_t j = 32 * (int64_t)J + bx;
  uint32_t cm = 0;
  for (int a = ty; a < 32; a += 8) {
    const int64_t i = 32 * (int64_t)I + a;
    uint32_t x = 0;
    if (i < n && j < i) x = dist_bits(__ldg(lt + i * (i - 1) / 2 + j));
    cm = x > cm ? x : cm;
    uint32_t rm = x;
#pragma unroll
    for (int o = 16; o; o >>= 1) { const uint32_t y = __shfl_xor_sync(0xffffffffu, rm, o); rm = y > rm ? y : rm; }
    if (bx == 0 && i < n && rm) atomicMax(rowmax + i, rm);
  }
  cmax[ty][bx] = cm;
  __syncthreads();
  if (ty == 0) {
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) m = cmax[k][bx] > m ? cmax[k][bx] : m;
    if (j < n && m) atomicMax(rowmax + j, m);
  }
}

__global__ void tb_threshold(const uint32_t* __restrict__ rowmax, int64_t n, float threshold, TablesOut* __restrict__ out) {
  __shared__ uint32_t red[32];
  uint32_t m = 0xFFFFFFFFu;
  if (isinf(threshold))  // (rowmax is only computed for the enclosing radius)
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = rowmax[i] < m ? rowmax[i] : m;
#pragma unroll
  for (int o = 16; o; o >>= 1) { uint32_t y = __shfl_xor_sync(0xffffffffu, m, o); m = y < m ? y : m; }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t R = 0xFFFFFFFFu;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) R = red[w] < R ? red[w] : R;
    if (n < 2) R = 0;  // A27: n = 1 -> R = 0
    // +inf entries are absent edges (a sparse input): never in the complex.  With such
    // entries R is +inf as well, and then every finite edge is kept (no enclosing-radius cut)
    const uint32_t tb0 = isinf(threshold) ? R : dist_bits(threshold);
    out->tbits = tb0 < 0x7F800000u ? tb0 : 0x7F7FFFFFu;
  }
}

// edges in DEscending index order k = N-1-j, j = TB_TILE * block + ...: a block counts the
// edges with d <= t of its tile (and validates the input)
constexpr int TB_THREADS = 256;
constexpr int TB_TILE = 8192;
__global__ void tb_edge_count(const float* __restrict__ lt, uint64_t N, TablesOut* __restrict__ out,
                              uint32_t* __restrict__ blk_count) {
  __shared__ uint32_t red[TB_THREADS / 32];
  const uint32_t tb = out->tbits;
  const uint64_t j0 = (uint64_t)blockIdx.x * TB_TILE;
  uint32_t c = 0;
  for (int i = threadIdx.x; i < TB_TILE; i += TB_THREADS) {
    const uint64_t j = j0 + (uint64_t)i;
    if (j >= N) break;
    const float x = __ldg(lt + (N - 1 - j));
    if (!(x >= 0.0f)) atomicOr(&out->err, 1u);  // NaN or negative
    c += dist_bits(x) <= tb;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < TB_THREADS / 32; ++w) t += red[w];
    blk_count[blockIdx.x] = t;
  }
}

// the keys of the edges with d <= t, order kept (descending k), at the block's offset
__global__ void tb_edge_compact(const float* __restrict__ lt, uint64_t N, int kbits, TablesOut* __restrict__ out,
                                const uint32_t* __restrict__ blk_off, uint32_t nblk, uint64_t* __restrict__ keys) {
  __shared__ uint32_t wsum[TB_THREADS / 32];
  const uint32_t tb = out->tbits;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t j0 = (uint64_t)blockIdx.x * TB_TILE;
  uint32_t base = blk_off[blockIdx.x];
  if (blockIdx.x == 0 && threadIdx.x == 0) out->m_le_t = blk_off[nblk];
  for (int i0 = 0; i0 < TB_TILE; i0 += TB_THREADS) {
    const uint64_t j = j0 + (uint64_t)(i0 + threadIdx.x);
    uint32_t b = 0;
    bool keep = false;
    if (j < N) {
      b = dist_bits(__ldg(lt + (N - 1 - j)));
      keep = b <= tb;
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) wsum[wid] = __popc(bal);
    __syncthreads();
    uint32_t before = 0, total = 0;
    for (int w = 0; w < TB_THREADS / 32; ++w) {
      const uint32_t x = wsum[w];
      before += w < wid ? x : 0;
      total += x;
    }
    if (keep) keys[base + before + __popc(bal & lanemask_lt())] = ((uint64_t)b << kbits) | j;  // j = N-1-k
    base += total;
    __syncthreads();
  }
}

// The ranks from the sorted edges (replaces the per-entry binary search over the whole
// matrix): the edge at sorted position p has rank = the first position of its distance
// (a lower bound over the prefix [0, p]); it is written to (i, j) and (j, i) of the rank
// matrix (pre-filled with RINF) and, when `bm` is given, to the threshold-graph bitmap.
__global__ void tb_rank_scatter(const uint64_t* __restrict__ sorted, uint64_t m, uint64_t N, int kbits, int64_t n,
                                uint32_t* __restrict__ rank, uint32_t* __restrict__ bm, int nw) {
  const uint64_t kmask = (1ull << kbits) - 1;
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t key = __ldg(sorted + p);
    const uint64_t x = key & ~kmask;  // the distance bits
    uint64_t lo = 0, hi = p;          // first position whose distance equals this one's
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if ((__ldg(sorted + mid) & ~kmask) < x) lo = mid + 1; else hi = mid;
    }
    const uint64_t k = N - 1 - (key & kmask);  // lower-distance index: k = i(i-1)/2 + j, i > j
    int64_t i = (int64_t)((1.0 + sqrt(1.0 + 8.0 * (double)k)) * 0.5);
    while (i * (i - 1) / 2 > (int64_t)k) --i;
    while ((i + 1) * i / 2 <= (int64_t)k) ++i;
    const int64_t j = (int64_t)k - i * (i - 1) / 2;
    VR_ASSERT(i < n && j >= 0 && j < i);
    rank[(size_t)i * (size_t)n + (size_t)j] = (uint32_t)lo;
    rank[(size_t)j * (size_t)n + (size_t)i] = (uint32_t)lo;
    if (bm) {
      atomicOr(bm + (size_t)i * (size_t)nw + (size_t)(j >> 5), 1u << (j & 31));
      atomicOr(bm + (size_t)j * (size_t)nw + (size_t)(i >> 5), 1u << (i & 31));
    }
  }
}

// deg(v) and deg_below(v) = #{w < v adjacent} from the bitmap (one warp per row)
__global__ void tb_bitmap_degrees(const uint32_t* __restrict__ bm, int n, int nw, uint32_t* __restrict__ deg,
                                  uint32_t* __restrict__ deg_below) {
  const int lane = threadIdx.x & 31;
  const int v = (int)(((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (v >= n) return;
  uint32_t c = 0, cb = 0;
  for (int k = lane; k < nw; k += 32) {
    const uint32_t w = __ldg(bm + (size_t)v * (size_t)nw + (size_t)k);
    c += __popc(w);
    if (32 * k + 31 < v) cb += __popc(w);
    else if (32 * k < v) cb += __popc(w & ((1u << (v - 32 * k)) - 1));
  }
  c = __reduce_add_sync(0xffffffffu, c);
  cb = __reduce_add_sync(0xffffffffu, cb);
  if (lane == 0) {
    deg[v] = c;
    deg_below[v] = cb;
  }
}

// sparse (COO) input -> dense lower triangle: +inf everywhere, then each entry (i, j, d),
// i != j, at i(i-1)/2 + j for i > j; repeated pairs keep the smallest distance
__global__ void coo_fill_inf(float* __restrict__ lt, uint64_t N) {
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < N; k += (uint64_t)gridDim.x * blockDim.x)
    lt[k] = __int_as_float(0x7F800000);
}
__global__ void coo_scatter(const int32_t* __restrict__ ii, const int32_t* __restrict__ jj, const float* __restrict__ dd,
                            int64_t nnz, float* __restrict__ lt) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = ii[k], b = jj[k];
    if (a < b) { const int64_t t = a; a = b; b = t; }
    const float x = dd[k] == 0.0f ? 0.0f : dd[k];
    atomicMin(reinterpret_cast<unsigned int*>(lt) + a * (a - 1) / 2 + b, __float_as_uint(x));
  }
}
void launch_coo_to_dense(const int32_t* ii, const int32_t* jj, const float* dd, int64_t nnz, int64_t n, float* lt,
                         cudaStream_t st) {
  const uint64_t N = (uint64_t)n * (uint64_t)(n - 1) / 2;
  if (N) coo_fill_inf<<<(unsigned)((N + 255) / 256 < 148u * 16u ? (N + 255) / 256 : 148u * 16u), 256, 0, st>>>(lt, N);
  if (nnz > 0)
    coo_scatter<<<(unsigned)(((uint64_t)nnz + 255) / 256 < 148u * 16u ? ((uint64_t)nnz + 255) / 256 : 148u * 16u), 256, 0, st>>>(
        ii, jj, dd, nnz, lt);
}

static int bits_for(uint64_t x) {  // number of bits to represent values 0..x
  int b = 0;
  while (b < 64 && (x >> b) != 0) ++b;
  return b ? b : 1;
}

size_t tables_temp_bytes(int64_t n) {
  const uint64_t N = (uint64_t)n * (uint64_t)(n - 1) / 2;
  const size_t nblk = (size_t)((N + TB_TILE - 1) / TB_TILE);
  return 2 * (((nblk + 1) * 4 + 255) / 256 * 256) + scan_temp_bytes(nblk + 1);
}

void launch_tables(const float* d_lt, int64_t n, float threshold, uint64_t* keys64, uint64_t* alt64, uint32_t* rowmax,
                   void* sort_temp, void* tb_temp, uint32_t* rank, TablesOut* d_out, int64_t m_known, uint64_t** sorted_out,
                   cudaStream_t st, int64_t* launches, const GraphOut* g) {
  const uint64_t N = (uint64_t)n * (uint64_t)(n - 1) / 2;
  const int kbits = bits_for(N ? N - 1 : 0);
  cudaMemsetAsync(d_out, 0, sizeof(TablesOut), st);
  const int T = (int)((n + 31) / 32);
  const unsigned tiles = (unsigned)((int64_t)T * (T + 1) / 2);
  if (isinf(threshold)) {  // the enclosing radius needs the row maxima (Prop 5.2.13)
    cudaMemsetAsync(rowmax, 0, (size_t)n * 4, st);
    tb_rowmax<<<tiles, 256, 0, st>>>(d_lt, n, rowmax);
    *launches += 1;
  }
  tb_threshold<<<1, 1024, 0, st>>>(rowmax, n, threshold, d_out);
  *launches += 1;
  uint64_t* sorted = keys64;
  uint64_t m = 0;
  if (N) {
    const uint32_t nblk = (uint32_t)((N + TB_TILE - 1) / TB_TILE);
    const size_t cb = (((size_t)nblk + 1) * 4 + 255) / 256 * 256;
    uint32_t* blk_count = (uint32_t*)tb_temp;
    uint32_t* blk_off = (uint32_t*)((char*)tb_temp + cb);
    void* scan_tmp = (char*)tb_temp + 2 * cb;
    cudaMemsetAsync(blk_count + nblk, 0, 4, st);
    tb_edge_count<<<nblk, TB_THREADS, 0, st>>>(d_lt, N, d_out, blk_count);
    exclusive_scan_u32(blk_count, blk_off, (size_t)nblk + 1, scan_tmp, st, launches);
    tb_edge_compact<<<nblk, TB_THREADS, 0, st>>>(d_lt, N, kbits, d_out, blk_off, nblk, keys64);
    *launches += 2;
    m = (uint64_t)m_known;
    if (m_known < 0) {  // first run: the count decides the sort size
      TablesOut h{};
      cudaMemcpyAsync(&h, d_out, sizeof h, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      m = h.m_le_t;
    }
    sorted = radix_sort_u64(keys64, alt64, (size_t)m, kbits, 31 + kbits, sort_temp, st, launches);
  }
  // the rank matrix: RINF, then the m edges under t scattered with their ranks
  cudaMemsetAsync(rank, 0xFF, (size_t)n * (size_t)n * 4, st);
  if (g && g->bm) cudaMemsetAsync(g->bm, 0, (size_t)n * (size_t)g->nw * 4, st);
  if (m) {
    const uint64_t blocks = std::min<uint64_t>((m + 255) / 256, 148ull * 16);
    tb_rank_scatter<<<(unsigned)blocks, 256, 0, st>>>(sorted, m, N, kbits, n, rank, g ? g->bm : nullptr, g ? g->nw : 0);
    *launches += 1;
  }
  if (g && g->bm) {
    tb_bitmap_degrees<<<(unsigned)(((uint64_t)n * 32 + 255) / 256), 256, 0, st>>>(g->bm, (int)n, g->nw, g->deg, g->deg_below);
    *launches += 1;
  }
  *sorted_out = sorted;
}

}  // namespace vr
