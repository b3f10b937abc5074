#!/bin/bash
# A/B of bits-kernel variants in exp/*.so (tools/time_ccl.py: bits and labels separately)
mkdir -p gpurun_out
: > gpurun_out/ab_bits.log
for so in exp/*.so; do
  echo "== $so" >> gpurun_out/ab_bits.log
  SN_B200_LIB=$so timeout 300 python tools/time_ccl.py ${B:-64} >> gpurun_out/ab_bits.log 2>&1
done
cat gpurun_out/ab_bits.log
