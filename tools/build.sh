#!/bin/bash
# fast rebuild of the CUDA library only (full build: python __graft_entry__.py)
cd "$(dirname "$0")/.." && nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC \
  -shared -diag-suppress 128 "$@" -o paper_2605_24584_b200/liblaplex_b200.so paper_2605_24584_b200/csrc/lx_capi.cu
