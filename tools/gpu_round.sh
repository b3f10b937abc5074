#!/bin/bash
# One GPU-box session: parity tests, smoke, bench, ncu launch list, ncu --set full
# captures of the fused pass and the labeller.  Outputs under gpurun_out/.
#   TAG=r1x NCU=1 BENCH_ARGS="..." bash tools/gpu_round.sh
set -u
O=gpurun_out
mkdir -p $O
TAG=${TAG:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi_$TAG.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" >> $O/smi_$TAG.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $O/smoke_$TAG.log
timeout 900 python bench.py --extras ${BENCH_ARGS:-} > $O/bench_$TAG.json 2> $O/bench_$TAG.err; echo "bench rc=$?" >> $O/bench_$TAG.err
if [ "${REF:-0}" = "1" ]; then
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_$TAG.json 2> $O/bench_ref_$TAG.err
fi
if [ "${NCU:-1}" = "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-extras --no-configs > $O/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fixed_square -c 1 \
  -o $O/fused_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-extras --no-configs > $O/ncu_fused_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ccl_|passable_bits" -c 4 \
  -o $O/ccl_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-extras --no-configs > $O/ncu_ccl_$TAG.log 2>&1
fi
ls -la $O
