#!/bin/bash
# The GPU test suite against the bounds-checked build (make -C
# paper_2504_15121_b200/csrc check: SN_ASSERT on shared / global indices and
# union-find link monotonicity, trap on failure) -- the memory-safety evidence
# in place of compute-sanitizer, which the pool does not run.
mkdir -p gpurun_out
make -C paper_2504_15121_b200/csrc check -j8 > /dev/null  # incremental: rebuilt when a source changed
export SN_B200_LIB=$PWD/paper_2504_15121_b200/libsn_b200_check.so
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/checked_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/checked_pytest.log
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-extras --no-configs \
  > gpurun_out/checked_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/checked_bench.log
grep -c "SN_ASSERT failed" gpurun_out/checked_pytest.log gpurun_out/checked_bench.log
tail -3 gpurun_out/checked_pytest.log
