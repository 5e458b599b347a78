timeout 900 python -m pytest tests -m gpu -x -q -s -k "map or nnf" > gpurun_out/gpu_map.log 2>&1; echo "map rc=$?"; tail -15 gpurun_out/gpu_map.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('ms/step', d['ms_per_step'], 'setup_s', d['config']['engine_setup_s'])"
