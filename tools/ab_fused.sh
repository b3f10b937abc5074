#!/bin/bash
# A/B of the fused-pass variants in exp/*.so (tools/time_fused.py, 64 C3 frames);
# PARITY=1 also runs the fixed-pass parity tests against each variant
mkdir -p gpurun_out
: > gpurun_out/ab_fused.log
for so in exp/*.so; do
  for rep in 1 2; do
    echo "== $so" >> gpurun_out/ab_fused.log
    SN_B200_LIB=$so timeout 300 python tools/time_fused.py 64 >> gpurun_out/ab_fused.log 2>&1
  done
  if [ -n "$PARITY" ]; then
    SN_B200_LIB=$so timeout 600 python -m pytest tests -m gpu -x -q -k "fixed or pipeline or points" 2>&1 | tail -2 >> gpurun_out/ab_fused.log
  fi
done
cat gpurun_out/ab_fused.log
