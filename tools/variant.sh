#!/bin/bash
# Build a flag variant of the library into variants/lib_<name>.so (development aid).
# usage: tools/variant.sh <name> [-Dflags...]; on the box: cp variants/lib_<name>.so paper_1908_09378_b200/libpbh_gpu.so
name=$1; shift
D=$(dirname "$0")/../paper_1908_09378_b200
nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 "$@" -shared \
  $D/csrc/pbh_gpu.cu $D/csrc/pbh_gen.cpp $D/csrc/pbh_trace_io.cpp -o $(dirname "$0")/../variants/lib_$name.so
