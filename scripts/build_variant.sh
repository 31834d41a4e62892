#!/bin/bash
# Build a libpaircount variant with extra -D flags for A/B timing:  scripts/build_variant.sh NAME [-DFOO=1 ...]
# -> build/ab/NAME.so  (select it with PAIRCOUNT_LIB=build/ab/NAME.so)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build/ab
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared "$@" \
    paper_1901_11204_b200/csrc/paircount.cu -o build/ab/$name.so
