#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab_generic.log
for so in exp/*.so; do
  echo "== $so" >> gpurun_out/ab_generic.log
  SN_B200_LIB=$so timeout 600 python tools/time_generic.py >> gpurun_out/ab_generic.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -x -k "generic or affine or kernel or pattern or unaligned or kats or golden or pitched" > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_tests.log
cat gpurun_out/ab_generic.log; tail -3 gpurun_out/ab_tests.log
