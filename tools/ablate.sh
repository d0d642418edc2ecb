#!/bin/bash
# Timing ablations of the compact step kernel (numerics are NOT valid in these builds):
#   bit 1: tanh -> identity   bit 4: no DSMEM pushes   bit 8: allreduce fold -> one leaf
# builds _abl/lib_<mask>.so here; run the printed command lines under gpurun.
set -e
cd "$(dirname "$0")/.."
mkdir -p _abl
F="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -fmad=false -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off --expt-relaxed-constexpr"
for m in "$@"; do
  mkdir -p _abl/$m
  for s in bt_capi bt_reduce bt_data; do cp paper_2208_14228_b200/_build/$s.cu.o _abl/$m/; done
  nvcc $F -DBT_ABL=$m -c paper_2208_14228_b200/csrc/bt_mlp.cu -o _abl/$m/bt_mlp.cu.o
  nvcc -shared -gencode arch=compute_100a,code=sm_100a _abl/$m/*.o -o _abl/lib_$m.so -lcudart
done
