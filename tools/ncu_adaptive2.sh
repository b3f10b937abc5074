#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"adaptive_kernel" -s ${SKIP:-7} -c 1 \
  -o gpurun_out/ncu_${TAG:-adp} -f python tools/time_adaptive.py 4 > gpurun_out/ncu_${TAG:-adp}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_${TAG:-adp}.log; tail -2 gpurun_out/ncu_${TAG:-adp}.log
