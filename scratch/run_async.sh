timeout 900 python -m pytest tests/test_gpu_scan_prep.py -x -q > gpurun_out/gpu_async.log 2>&1; echo "async rc=$?"; tail -15 gpurun_out/gpu_async.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e_raw_points'], d['scan_prep_ms'])"
