// residual_bench.cpp — time libvr's host residual reduction on inputs dumped by a GPU run
// (VR_DUMP_RESIDUAL=<dir>).  Diagnostics only.
//   g++ -O3 -std=c++17 -I /usr/local/cuda/include -I paper_2502_05063_b200/csrc tools/residual_bench.cpp
//       paper_2502_05063_b200/csrc/host.cpp -o /tmp/residual_bench && /tmp/residual_bench <dir> <d> [mode]
// env: VR_BM=1 output-sensitive host graph, VR_HINTS=1 residual hints (computed untimed),
//      VR_RESIDUAL_THREADS, VR_RESIDUAL_BLOCK
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "vr_internal.h"

template <class T>
static std::vector<T> rd(const std::string& f) {
  std::vector<T> v;
  FILE* fp = std::fopen(f.c_str(), "rb");
  if (!fp) { std::perror(f.c_str()); std::exit(1); }
  std::fseek(fp, 0, SEEK_END);
  long b = std::ftell(fp);
  std::fseek(fp, 0, SEEK_SET);
  v.resize((size_t)b / sizeof(T));
  if (std::fread(v.data(), 1, (size_t)b, fp) != (size_t)b) std::exit(2);
  std::fclose(fp);
  return v;
}

// the library's pinned-host cache lives in vr_api.cu; plain heap blocks here
namespace vr {
void* pinned_acquire(size_t& bytes) { return std::malloc(bytes); }
void pinned_release(void* p, size_t) { std::free(p); }
}  // namespace vr

int main(int argc, char** argv) {
  std::string dir = argv[1];
  int d = std::atoi(argv[2]);
  int mode = argc > 3 ? std::atoi(argv[3]) : 0;
  long long n; int dd, cbits, kmax; unsigned maxr;
  FILE* fp = std::fopen((dir + "/meta_d" + std::to_string(d) + ".txt").c_str(), "r");
  if (std::fscanf(fp, "%lld %d %u %d %d", &n, &dd, &maxr, &cbits, &kmax) != 5) return 3;
  std::fclose(fp);
  vr::HostMatrix M;
  M.n = n; M.kmax = kmax;
  {
    auto v = rd<uint32_t>(dir + "/rank.bin");
    M.rank.assign(v.begin(), v.end());
  }
  M.value = rd<float>(dir + "/values.bin");
  M.binom.resize((size_t)(kmax + 1) * (size_t)(n + 1));
  for (int k = 0; k <= kmax; ++k)
    for (long long v = 0; v <= n; ++v) {
      unsigned __int128 c = 1;
      if (k > v) c = 0;
      else for (int i = 1; i <= k; ++i) c = c * (unsigned __int128)(v - k + i) / (unsigned)i;
      M.binom[(size_t)k * (size_t)(n + 1) + (size_t)v] = (uint64_t)c;
    }
  if (std::getenv("VR_BM")) {  // threshold-graph bitmap + packed ranks, as the output-sensitive mode builds them
    M.bmw = (n + 63) / 64;
    M.bm.assign((size_t)n * M.bmw, 0);
    for (long long v = 0; v < n; ++v)
      for (long long w = 0; w < n; ++w)
        if (w != v && M.rank[(size_t)v * n + w] != 0xFFFFFFFFu) M.bm[(size_t)v * M.bmw + w / 64] |= 1ull << (w % 64);
    M.build_neighbour_ranks();
  }
  auto keys = rd<uint64_t>(dir + "/keys_d" + std::to_string(d) + ".bin");
  vr::HostPairs hp; std::vector<uint64_t> deaths; vr::ResidualStats st;
  std::vector<uint64_t> hfirst(keys.size());
  std::vector<uint8_t> hclaimed(keys.size());
  vr::ResidualHints hints{hfirst.data(), hclaimed.data()};
  const bool use_hints = std::getenv("VR_HINTS") != nullptr;  // precomputed (untimed), as the GPU emits them
  if (use_hints) vr::residual_hints_host(M, d, maxr, cbits, keys.data(), keys.size(), hfirst.data(), hclaimed.data());
  auto t0 = std::chrono::steady_clock::now();
  vr::residual_reduce(M, d, maxr, cbits, keys.data(), keys.size(), mode, hp, deaths, st, use_hints ? &hints : nullptr);
  double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  size_t pos = 0;
  for (size_t i = 0; i < hp.birth.size(); ++i) pos += hp.birth[i] < hp.death[i];
  if (const char* f = std::getenv("VR_PAIRS_OUT")) {  // per column: death cidx (UINT64_MAX: zero column)
    FILE* fo = std::fopen(f, "wb");
    if (fo) {
      std::fwrite(hp.death_cidx.data(), 8, hp.death_cidx.size(), fo);
      std::fclose(fo);
    }
  }
  if (const char* c = std::getenv("VR_COL")) {
    size_t i = (size_t)std::atoll(c);
    std::printf("col %zu: birth %.7g death %.7g bcidx %llu dcidx %llu\n", i, hp.birth[i], hp.death[i],
                (unsigned long long)hp.birth_cidx[i], (unsigned long long)hp.death_cidx[i]);
    uint64_t cm = (1ull << cbits) - 1;
    std::printf("key rank %u\n", maxr - (unsigned)(keys[i] >> cbits));
    (void)cm;
  }
  uint64_t h = 0;
  for (size_t i = 0; i < hp.birth.size(); ++i) h = h * 1000003ull + hp.birth_cidx[i] * 31 + hp.death_cidx[i];
  std::printf("hash %016llx\n", (unsigned long long)h);
  std::printf("d=%d mode=%d columns=%zu emergent=%lld additions=%lld coboundaries=%lld apparent_checks=%lld pairs=%zu positive=%zu ms=%.1f\n",
              d, mode, keys.size(), (long long)st.emergent, (long long)st.additions, (long long)st.coboundaries, (long long)st.apparent_checks,
              hp.birth.size(), pos, ms);
  return 0;
}
// (debug) print the pair produced by a given column: VR_COL=<index>
