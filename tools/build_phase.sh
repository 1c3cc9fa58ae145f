#!/bin/bash
# diagnostic build of liblmm with per-phase clock64 instrumentation of the meta-mesh kernel
set -e
D=$(mktemp -d); R=$(cd "$(dirname "$0")/.." && pwd)
A="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC"
for f in lmm_api lattice scan triangulate; do /usr/local/cuda/bin/nvcc $A -c $R/paper_2405_15197_b200/csrc/$f.cu -o $D/$f.o & done
/usr/local/cuda/bin/nvcc $A -fmad=false -DLMM_PHASE_TIMING -c $R/paper_2405_15197_b200/csrc/metamesh.cu -o $D/metamesh.o
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/tools/liblmm_phase.so $D/*.o
rm -rf $D
