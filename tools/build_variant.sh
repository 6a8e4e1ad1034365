#!/bin/bash
# build a scan-parameter variant of the library: tools/build_variant.sh OUT.so -DSKM_SCAN_DEPTH=8 ...
out=$1; shift
cd "$(dirname "$0")/../paper_2603_20009_b200" && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared "$@" -o "$out" csrc/skm_abi.cu
