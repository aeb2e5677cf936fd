#!/bin/bash
# Build an experimental libgmr variant: scripts/build_variant.sh NAME [nvcc -D flags...]
# Output: variants/libgmr_NAME.so (git-ignored, travels to the GPU box).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
mkdir -p "$ROOT/variants"
cd "$ROOT/paper_2602_14493_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  "$@" -o "$ROOT/variants/libgmr_$NAME.so" gmr_capi.cu
