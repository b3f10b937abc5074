#!/bin/bash
# ncu --set full of the passable-bits kernel and the labeller on C3 frames
mkdir -p gpurun_out
TAG=${TAG:-bits}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-passable_bits}" -s ${SKIP:-2} -c ${COUNT:-1} \
  -o gpurun_out/ncu_$TAG -f python tools/time_ccl.py 16 > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$TAG.log
tail -3 gpurun_out/ncu_$TAG.log
