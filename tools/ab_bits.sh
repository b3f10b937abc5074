#!/bin/bash
# A/B of bits-kernel variants in exp/*.so (tools/time_ccl.py: bits and labels
# separately); PARITY=1 also runs the predicate / label parity tests per variant
mkdir -p gpurun_out
: > gpurun_out/ab_bits.log
for so in exp/*.so; do
  echo "== $so" >> gpurun_out/ab_bits.log
  SN_B200_LIB=$so timeout 300 python tools/time_ccl.py ${B:-64} >> gpurun_out/ab_bits.log 2>&1
  if [ -n "$PARITY" ]; then
    SN_B200_LIB=$so timeout 900 python -m pytest tests -m gpu -x -q -k "label or ccl or pipeline or passable or parallel or f64 or bits" 2>&1 | tail -2 >> gpurun_out/ab_bits.log
  fi
done
cat gpurun_out/ab_bits.log
