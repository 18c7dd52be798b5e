#!/bin/bash
# Build a variant of libadi.so with extra nvcc defines (same-box A/B with tools/ab_lib.py):
#   bash tools/build_variant.sh NAME -DADI_NSUB=1 ...   ->  paper_2006_07583_b200/ab/NAME.so
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
mkdir -p "$ROOT/paper_2006_07583_b200/ab"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -diag-suppress 177 "$@" -I "$ROOT/include" -o "$ROOT/paper_2006_07583_b200/ab/$NAME.so" \
  "$ROOT/paper_2006_07583_b200/csrc/adi_runtime.cu"
