#!/bin/bash
# Build experiment variants of the fused pass (SN_EXP=1 no stores, 2 no
# pass H, 3 no pass V, 4 neither pass, 5 stores only, 6 loads only) into exp/ and time each with
# tools/time_fused.py.  Not part of the product.
set -e
cd "$(dirname "$0")/../paper_2504_15121_b200/csrc"
mkdir -p ../../exp
FLAGS="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -I../../include"
for v in ${VARIANTS:-1 2 3 4}; do
  nvcc $FLAGS -DSN_EXP=$v -c sn_fixed.cu -o ../../exp/sn_fixed_$v.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../exp/libsn_exp$v.so sn_api.o ../../exp/sn_fixed_$v.o sn_ccl.o sn_cloud.o sn_adaptive.o sn_eval.o sn_codec.o -Xcompiler -fvisibility=hidden
done
