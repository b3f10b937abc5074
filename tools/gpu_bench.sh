#!/bin/bash
# GPU-box bench session: our arm (default flags + extras), the reference arm,
# lscpu.  TAG=r2b bash tools/gpu_bench.sh
set -u
O=gpurun_out
mkdir -p $O
TAG=${TAG:-b}
timeout 1200 python bench.py ${BENCH_ARGS:---steps 20 --warmup 5} > $O/bench_$TAG.json 2> $O/bench_$TAG.err; echo "rc=$?" >> $O/bench_$TAG.err
if [ "${REF:-1}" = "1" ]; then
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_$TAG.json 2> $O/bench_ref_$TAG.err
fi
lscpu > $O/lscpu.txt 2>&1
tail -c 5000 $O/bench_$TAG.json; tail -5 $O/bench_$TAG.err; cut -c1-400 $O/bench_ref_$TAG.json 2>/dev/null
