#!/bin/bash
# Box-side timing of the host residual on fresh dumps (diagnostics): bash tools/box_residual.sh [cfg D dims...]
# Builds tools/residual_bench.cpp twice (byte-digit radix heap = default, binary radix heap =
# -DVR_BINARY_RADIX) and times each dimension on 1 and 16 threads.
cfg=${1:-c5_o3_4096}; D=${2:-3}; shift 2; dims=${@:-1 2 3}
mkdir -p /tmp/dumpx
VR_DUMP_RESIDUAL=/tmp/dumpx python tools/dim_stats.py $cfg $D 1 > /dev/null 2>&1
for v in B bin; do
  f=""; [ $v = bin ] && f="-DVR_BINARY_RADIX"
  g++ -O3 -march=native $f -std=c++17 -I /usr/local/cuda/include -I paper_2502_05063_b200/csrc tools/residual_bench.cpp paper_2502_05063_b200/csrc/host.cpp -o /tmp/rb_$v -lpthread
done
for d in $dims; do for t in 1 16; do for v in B bin; do for r in 1 2; do
  echo "$cfg d=$d T=$t heap=$v $(VR_BM=1 VR_HINTS=1 VR_RESIDUAL_THREADS=$t /tmp/rb_$v /tmp/dumpx $d | tail -1 | grep -o 'ms=.*')"
done; done; done; done
