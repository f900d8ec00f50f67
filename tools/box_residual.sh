#!/bin/bash
# Box-side A/B timing of the host residual on a fresh dump (diagnostics):
#   A_FLAGS="" B_FLAGS="-DVR_BINARY_RADIX" bash tools/box_residual.sh [cfg D dims...]
# Builds tools/residual_bench.cpp with each flag set and times each dimension on 1 and 16
# threads, twice each (B_FLAGS default: the binary radix heap; e.g. -DVR_NO_PREFETCH;
# B_SRC: another host.cpp for B).
cfg=${1:-c5_o3_4096}; D=${2:-3}; shift 2; dims=${@:-1 2 3}
A_FLAGS=${A_FLAGS:-}; B_FLAGS=${B_FLAGS:--DVR_BINARY_RADIX}; B_SRC=${B_SRC:-paper_2502_05063_b200/csrc/host.cpp}
mkdir -p /tmp/dumpx
VR_DUMP_RESIDUAL=/tmp/dumpx python tools/dim_stats.py $cfg $D 1 > /dev/null 2>&1
g++ -O3 -march=native $A_FLAGS -std=c++17 -I /usr/local/cuda/include -I paper_2502_05063_b200/csrc tools/residual_bench.cpp paper_2502_05063_b200/csrc/host.cpp -o /tmp/rb_A -lpthread
g++ -O3 -march=native $B_FLAGS -std=c++17 -I /usr/local/cuda/include -I paper_2502_05063_b200/csrc tools/residual_bench.cpp $B_SRC -o /tmp/rb_B -lpthread
for d in $dims; do for t in 1 16; do for v in A B; do for r in 1 2; do
  echo "$cfg d=$d T=$t $v $(VR_BM=1 VR_HINTS=1 VR_RESIDUAL_THREADS=$t /tmp/rb_$v /tmp/dumpx $d | tail -1 | grep -o 'ms=.*')"
done; done; done; done
