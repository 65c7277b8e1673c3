#!/bin/bash
# Developer helper: build a variant of the library with extra nvcc flags into
# scripts/_exp/<name>.so (git-ignored; travels with the gpurun snapshot) for A/B runs:
#   scripts/build_variant.sh p6 -DVQNQS_TCA_PARTS=6
# On the GPU box: cp scripts/_exp/p6.so paper_2212_11296_b200/_lib/libvqnqs_b200.so
set -e
cd "$(dirname "$0")/.."
name=$1; shift
L=paper_2212_11296_b200/_lib
mkdir -p scripts/_exp/obj_$name
nvcc -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -Xptxas -v "$@" -O3 -std=c++17 -lineinfo \
  -Xcompiler -fPIC -Xcompiler -O3 -I include -c paper_2212_11296_b200/csrc/engine.cu \
  -o scripts/_exp/obj_$name/engine.cu.o 2> scripts/_exp/obj_$name/ptxas.log
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scripts/_exp/$name.so scripts/_exp/obj_$name/engine.cu.o \
  $L/grad.cu.o $L/capi.cpp.o $L/host_model.cpp.o $L/comm.cpp.o -lcudart -ldl
grep -A2 'k_tc_attention' scripts/_exp/obj_$name/ptxas.log | head -8
