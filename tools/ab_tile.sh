#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab_tile.log
for so in exp/*.so; do
  echo "== $so" >> gpurun_out/ab_tile.log
  SN_B200_LIB=$so timeout 300 python tools/time_tile.py >> gpurun_out/ab_tile.log 2>&1
done
cat gpurun_out/ab_tile.log
