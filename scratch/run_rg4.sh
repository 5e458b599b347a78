timeout 900 python -m pytest tests -m gpu -x -q -k "neighbor or sharded or golden or filter or stages" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('global f', d['ms_per_step'], d['stage_ms']['refresh_gather_ms'])"
SMCL_RG_PLAIN=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench2.json')); print('global plain', d['ms_per_step'], d['stage_ms']['refresh_gather_ms'])"
