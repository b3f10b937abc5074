# quick GPU check: parity tests of the touched area + bench stages
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x ${TESTS:+-k "$TESTS"} > gpurun_out/quick_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/quick_tests.log
tail -2 gpurun_out/quick_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/quick_bench.json 2>gpurun_out/quick_bench.err
python -c "import json; d=json.load(open('gpurun_out/quick_bench.json')); print(round(d['value']), {k: round(v*1000,2) for k,v in d['stages_ms_per_frame'].items()})"
