#!/bin/bash
# Build a library variant with extra -D flags into ablibs/<name>.so (A/B runs):
#   tools/build_variant.sh k1pf2 "-DTAFV_K1_PF=2"
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=$ROOT/paper_1704_01144_b200/csrc
mkdir -p $ROOT/ablibs
/usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false \
  -Xcompiler -fPIC,-ffp-contract=off -I$ROOT/include $2 -shared -o $ROOT/ablibs/$1.so \
  $C/solver.cu $C/meshgen.cpp $C/shard.cpp $C/io.cpp -lnccl
