# ncu --set full of the fused PNG16 pass (tools/time_codecs.py at 8 frames)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:Png16 -c 1 -o gpurun_out/png16_full -f python tools/time_codecs.py 8 > gpurun_out/ncu_png.log 2>&1
tail -3 gpurun_out/ncu_png.log
