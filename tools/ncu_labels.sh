#!/bin/bash
# Labeller kernels at C3 (tools/time_labels.py): the launch list (per-kernel
# times) and --set full captures of the tile and resolve kernels at t = 0.2
mkdir -p gpurun_out
TAG=${TAG:-labels}
B=${B:-32}
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python tools/time_labels.py $B > gpurun_out/launches_$TAG.log 2>&1
for k in ccl_tile ccl_resolve passable_bits; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 9 -c 1 \
    -o gpurun_out/ncu_${TAG}_$k -f python tools/time_labels.py $B > gpurun_out/ncu_${TAG}_$k.log 2>&1
  echo "$k rc=$?"
done
