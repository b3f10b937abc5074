#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab_fused.log
for so in exp/*.so; do
  for rep in 1 2; do
    echo "== $so" >> gpurun_out/ab_fused.log
    SN_B200_LIB=$so timeout 300 python tools/time_fused.py 64 >> gpurun_out/ab_fused.log 2>&1
  done
done
cat gpurun_out/ab_fused.log
