#!/bin/bash
# Box-side timing of the host residual on a fresh dump of config 5 (diagnostics): bash tools/box_residual.sh
mkdir -p /tmp/dump5
VR_DUMP_RESIDUAL=/tmp/dump5 python tools/dim_stats.py c5_o3_4096 3 1 > /dev/null 2>&1
g++ -O3 -march=native -std=c++17 -I /usr/local/cuda/include -I paper_2502_05063_b200/csrc tools/residual_bench.cpp paper_2502_05063_b200/csrc/host.cpp -o /tmp/rb -lpthread
nproc; lscpu | grep -E "Model name|Thread|Core|Socket|MHz" | head
for d in 1 2 3; do for t in 1 4 8 16; do echo "d=$d T=$t"; VR_BM=1 VR_HINTS=1 VR_RESIDUAL_THREADS=$t /tmp/rb /tmp/dump5 $d | tail -1; done; done
