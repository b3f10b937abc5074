#!/bin/bash
# A/B of labeller variants: each exp/*.so through tools/time_ccl.py, then the
# parity tests of the labeller on the default library.
mkdir -p gpurun_out
for so in exp/*.so; do
  echo "== $so" >> gpurun_out/ab_ccl.log
  SN_B200_LIB=$so timeout 300 python tools/time_ccl.py 64 >> gpurun_out/ab_ccl.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -x ${TESTS:+-k "$TESTS"} > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_tests.log
cat gpurun_out/ab_ccl.log; tail -3 gpurun_out/ab_tests.log
