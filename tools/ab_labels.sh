#!/bin/bash
# A/B of labeller variants in exp/*.so through tools/time_labels.py (C3);
# PARITY=1 also runs the label parity tests against each variant
mkdir -p gpurun_out
: > gpurun_out/ab_labels.log
for so in exp/*.so; do
  for rep in 1 2; do
    echo "== $so" >> gpurun_out/ab_labels.log
    SN_B200_LIB=$so timeout 300 python tools/time_labels.py ${B:-128} >> gpurun_out/ab_labels.log 2>&1
  done
  if [ -n "$PARITY" ]; then
    SN_B200_LIB=$so timeout 900 python -m pytest tests -m gpu -x -q -k "label or ccl or pipeline or passable or parallel" 2>&1 | tail -2 >> gpurun_out/ab_labels.log
  fi
done
cat gpurun_out/ab_labels.log
