#!/bin/bash
# Builds the micro-benchmark binaries (not part of librk); run from anywhere.
set -e
D=$(cd "$(dirname "$0")" && pwd)
R=$D/../..
NV="nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -I $R/include -I $R/paper_1501_03358_b200/csrc"
$NV -o $D/chain_bench $D/chain_bench.cu $R/paper_1501_03358_b200/csrc/chain.cu
$NV -DRK_CHAIN_LOADONLY=1 -o $D/chain_bench_lo $D/chain_bench.cu $R/paper_1501_03358_b200/csrc/chain.cu
$NV -o $D/bdot_bench $D/bdot_bench.cu
$NV -o $D/blockops_prod $D/blockops_prod.cu -L $R/paper_1501_03358_b200 -lrk -Xlinker -rpath -Xlinker '$ORIGIN/../../paper_1501_03358_b200'
