// probe.cu — micro-benchmarks of the two on-chip peaks the hot path is measured against
// (SURVEY.md §8(d) "Roofline": MEASURED_PEAKS.json holds only the HBM copy and bf16 GEMM
// peaks, so the integer-ALU and L2 peaks are measured on the box by bench.py through
// vr_probe_peaks).
//
//   integer ALU : every thread runs 8 independent chains of (IMNMX, LOP3) — the max/compare
//                 and logic ops the enumeration kernels are made of — for 2 ops per chain
//                 step; 148 x 8 CTAs of 256 threads.
//   L2 read     : a 48 MiB buffer (well inside the 126 MB L2) read with 16-byte loads by
//                 every SM, after one untimed pass that makes it L2-resident.
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/vr.h"
#include "vr_internal.h"

namespace vr {

constexpr int PR_ITERS = 4096;
constexpr int PR_CHAINS = 8;

__global__ void __launch_bounds__(256) k_probe_alu(uint32_t seed, uint32_t* __restrict__ sink) {
  uint32_t a[PR_CHAINS], v[PR_CHAINS], c[PR_CHAINS];
#pragma unroll
  for (int k = 0; k < PR_CHAINS; ++k) {
    a[k] = seed * (threadIdx.x + 1) + k;
    v[k] = seed ^ (blockIdx.x * 977u + k * 131u);
    c[k] = seed * 0x9E3779B9u + (uint32_t)k * 0x85EBCA6Bu;
  }
  for (int it = 0; it < PR_ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < PR_CHAINS; ++k) {
      a[k] = a[k] > v[k] ? a[k] : v[k];  // IMNMX
      v[k] = v[k] ^ a[k] ^ c[k];         // LOP3
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int k = 0; k < PR_CHAINS; ++k) x ^= a[k] ^ v[k];
  if (x == 0x9E3779B9u) sink[blockIdx.x] = x;  // keeps the chains alive
}

__global__ void __launch_bounds__(256) k_probe_l2(const uint4* __restrict__ buf, uint64_t n16, int reps,
                                                  uint32_t* __restrict__ sink) {
  uint32_t x = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
      const uint4 t = __ldcg(buf + i);  // L2 (bypass L1)
      x ^= t.x ^ t.y ^ t.z ^ t.w;
    }
  if (x == 0x9E3779B9u) sink[blockIdx.x] = x;
}

}  // namespace vr

extern "C" int vr_probe_peaks(int32_t device, double* alu_ops_per_s, double* l2_bytes_per_s) {
  if (!alu_ops_per_s || !l2_bytes_per_s) return VR_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) { cudaGetLastError(); return VR_EDEVICE; }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const size_t bytes = (size_t)48 << 20;
  void* buf = nullptr;
  uint32_t* sink = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int rc = VR_OK;
  do {
    if (cudaMalloc(&buf, bytes) != cudaSuccess || cudaMalloc(&sink, 4096 * 4) != cudaSuccess) { rc = VR_ECAPACITY; break; }
    cudaMemset(buf, 1, bytes);
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const unsigned blocks = (unsigned)sms * 8;
    // integer ALU: warm-up, then best of 5
    vr::k_probe_alu<<<blocks, 256>>>(12345u, sink);
    float best = 1e30f;
    for (int t = 0; t < 5; ++t) {
      cudaEventRecord(e0);
      vr::k_probe_alu<<<blocks, 256>>>(12345u + t, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    *alu_ops_per_s = 2.0 * vr::PR_CHAINS * (double)vr::PR_ITERS * (double)blocks * 256.0 / (best * 1e-3);
    // L2: one pass to make the buffer resident, then best of 5 passes of 8 reads each
    const uint64_t n16 = bytes / 16;
    vr::k_probe_l2<<<blocks, 256>>>((const uint4*)buf, n16, 1, sink);
    best = 1e30f;
    for (int t = 0; t < 5; ++t) {
      cudaEventRecord(e0);
      vr::k_probe_l2<<<blocks, 256>>>((const uint4*)buf, n16, 8, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    *l2_bytes_per_s = 8.0 * (double)bytes / (best * 1e-3);
    if (cudaGetLastError() != cudaSuccess) rc = VR_EDEVICE;
  } while (0);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (buf) cudaFree(buf);
  if (sink) cudaFree(sink);
  return rc;
}
