#!/bin/bash
# GPU-box check: full parity suite, smoke, a short bench line.  Outputs under gpurun_out/.
#   TAG=r2a bash tools/gpu_check.sh
set -u
O=gpurun_out
mkdir -p $O
TAG=${TAG:-chk}
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -x ${TESTS:+-k "$TESTS"} > $O/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_$TAG.log
tail -3 $O/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $O/smoke_$TAG.log
tail -2 $O/smoke_$TAG.log
if [ "${BENCH:-1}" = "1" ]; then
timeout 600 python bench.py ${BENCH_ARGS:---steps 10 --warmup 3} > $O/bench_$TAG.json 2> $O/bench_$TAG.err; echo "bench rc=$?" >> $O/bench_$TAG.err
tail -c 3000 $O/bench_$TAG.json
fi
