#!/bin/bash
# build_variant.sh OUT.so [extra nvcc flags...] -- libslora with experiment macros (parallel per-file compile)
set -e
OUT=$1; shift
D=$(cd "$(dirname "$0")/../paper_2311_03285_b200" && pwd)
T=$(mktemp -d)
F="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC"
for s in kernels mbgmm; do nvcc $F "$@" -c $D/csrc/$s.cu -o $T/$s.o & done
g++ -O2 -std=c++17 -fPIC -I/usr/local/cuda/include "$@" -c $D/csrc/api.cpp -o $T/api.o 2>/dev/null || nvcc $F "$@" -c $D/csrc/api.cpp -o $T/api.o &
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT" $T/*.o -lcuda
rm -rf $T
