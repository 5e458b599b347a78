# GPU tests + bench (no CPU baseline) + stage times
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 300 python bench.py --no-cpu-baseline $BENCH_ARGS > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('ms/step', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step']); print({k: round(v,3) for k,v in d['stage_ms'].items()})"
