mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
nvidia-smi --query-gpu=name,driver_version --format=csv > gpurun_out/san_env.txt 2>&1
$S --version >> gpurun_out/san_env.txt 2>&1
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 $S --tool $t --error-exitcode 9 --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitize_$t.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$t.log
done
tail -3 gpurun_out/sanitize_*.log
