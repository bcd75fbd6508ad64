#!/bin/bash
# Build the C-ABI library from an alternative csrc tree into build/ab/<name>.so (A/B runs:
# FSBM_LIB_PATH=build/ab/<name>.so python bench.py ...).  usage: build_variant.sh <name> <csrc dir> [nvcc flags]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; src=$2; shift 2
mkdir -p "$ROOT/build/ab"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared \
  --expt-relaxed-constexpr -I "$ROOT/include" "$@" "$src/fsbm_coal.cu" -o "$ROOT/build/ab/$name.so" -ldl
