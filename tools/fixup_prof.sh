#!/bin/bash
# Build the library with fixup phase timers (BR_FIXUP_PROF) into tools/micro/proflib (dev only).
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr \
  -DBR_FIXUP_PROF -shared -o "$HERE/micro/proflib/libbatchrand_b200.so" "$HERE/../paper_2408_06213_b200/csrc/capi.cu"
