#!/bin/bash
# Build the CUDA library under another name for A/B timing (bench.py reads M3E_LIB):
#   tools/build_variant.sh NAME [extra nvcc flags...]  ->  paper_2206_11535_b200/lib/variants/libm3e_NAME.so
cd "$(dirname "$0")/.." || exit 1
N=$1; shift
mkdir -p paper_2206_11535_b200/lib/variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -Iinclude \
  -Ipaper_2206_11535_b200/csrc "$@" -o paper_2206_11535_b200/lib/variants/libm3e_$N.so \
  paper_2206_11535_b200/csrc/m3e_kernels.cu paper_2206_11535_b200/csrc/m3e_runtime.cu
