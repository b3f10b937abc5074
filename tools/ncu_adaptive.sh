# ncu --set full of the adaptive kernels (tools/time_adaptive.py, 2 frames)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adaptive_kernel -c 2 -o gpurun_out/adaptive_full -f python tools/time_adaptive.py 2 > gpurun_out/ncu_adaptive.log 2>&1
tail -2 gpurun_out/ncu_adaptive.log
