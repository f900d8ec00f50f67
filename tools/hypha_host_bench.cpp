// hypha_host_bench.cpp — time HYPHA's host phase on CPU (diagnostics only): the GPU-scan
// (Algs 4-6) is emulated serially here, then vr::hypha_host_reduce runs as in the library.
//   g++ -O3 -std=c++17 -I /usr/local/cuda/include -I paper_2502_05063_b200/csrc tools/hypha_host_bench.cpp
//       paper_2502_05063_b200/csrc/hypha_host.cpp -o /tmp/hypha_host_bench
//   /tmp/hypha_host_bench <dir with ptr.i64 rows.i32 dims.i32 [low.i32]> [flags]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../include/vr.h"
#include "vr_internal.h"

template <class T>
static std::vector<T> rd(const std::string& f) {
  std::vector<T> v;
  FILE* fp = std::fopen(f.c_str(), "rb");
  if (!fp) return v;
  std::fseek(fp, 0, SEEK_END);
  long b = std::ftell(fp);
  std::fseek(fp, 0, SEEK_SET);
  v.resize((size_t)b / sizeof(T));
  if (std::fread(v.data(), 1, (size_t)b, fp) != (size_t)b) std::exit(2);
  std::fclose(fp);
  return v;
}

int main(int argc, char** argv) {
  std::string dir = argv[1];
  int flags = argc > 2 ? std::atoi(argv[2]) : 3;
  auto ptr = rd<int64_t>(dir + "/ptr.i64");
  auto rows = rd<int32_t>(dir + "/rows.i32");
  auto dims = rd<int32_t>(dir + "/dims.i32");
  auto exp = rd<int32_t>(dir + "/low.i32");
  const int64_t n = (int64_t)ptr.size() - 1;
  std::vector<int32_t> Left(n, INT32_MAX), Lookup(n, -1), u;
  std::vector<uint8_t> stable(n, 0);
  for (int64_t j = 0; j < n; ++j) {
    if (ptr[j] == ptr[j + 1]) stable[j] = 1;
    for (int64_t k = ptr[j]; k < ptr[j + 1]; ++k) Left[rows[k]] = std::min<int32_t>(Left[rows[k]], (int32_t)j);
  }
  for (int64_t j = 0; j < n; ++j) {
    if (ptr[j] == ptr[j + 1]) continue;
    int32_t lo = rows[ptr[j + 1] - 1];
    if (Left[lo] == j) { Lookup[lo] = (int32_t)j; stable[j] = 1; if (flags & 2) stable[lo] = 1; }
  }
  for (int64_t j = 0; j < n; ++j) if (!stable[j]) u.push_back((int32_t)j);
  vr_hypha_stats st{};
  auto t0 = std::chrono::steady_clock::now();
  vr::hypha_host_reduce(ptr.data(), rows.data(), n, dims.empty() ? nullptr : dims.data(), flags, Left.data(), Lookup.data(),
                        stable.data(), u.data(), (int64_t)u.size(), st);
  double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  std::vector<int32_t> low(n, -1);
  for (int64_t r = 0; r < n; ++r) if (Lookup[r] >= 0) low[Lookup[r]] = (int32_t)r;
  long bad = 0;
  if (!exp.empty()) for (int64_t j = 0; j < n; ++j) bad += low[j] != exp[j];
  std::printf("n=%ld unstable=%ld additions=%ld compressed=%ld host_ms=%.1f mismatches=%ld\n", (long)n,
              (long)st.unstable, (long)st.additions, (long)st.compressed, ms, bad);
}
