#!/bin/bash
# Build an A/B variant of the library with extra defines: tools/build_variant.sh NAME -DFOO=1 ...
# -> ablibs/NAME.so (travels to the GPU box; git-ignored); time with tools/ab.sh ablibs/*.so
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
mkdir -p "$ROOT/ablibs"
cd "$ROOT/paper_1607_04091_b200/csrc"
nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-pthread "$@" \
  -shared -o "$ROOT/ablibs/$name.so" gs_capi.cu gs_ndft.cu gs_plan.cu host_inputs.cpp gs_voronoi.cu
