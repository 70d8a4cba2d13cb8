#!/bin/bash
# Diagnostic: build variants of the library with SPGEMM_ABLATE_* macros into
# tools/abl_<name>/ (used with tools/abl_run.sh; never shipped).
set -e
cd "$(dirname "$0")/.."
for v in "$@"; do
  mkdir -p tools/abl_$v
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -fmad=false \
    -DSPGEMM_ABLATE_${v^^} $EXTRA -I include -o tools/abl_$v/libspgemm_b200.so \
    paper_2206_07244_b200/csrc/capi.cu paper_2206_07244_b200/lib/cxx_api.cpp.o paper_2206_07244_b200/lib/multi.cpp.o &
done
wait
