# round 2: full GPU test suite + default bench line
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02_gputests.log
timeout 600 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench.json')); print(round(d['ms_per_step'],3), d['e2e']['ms_per_step'], {k:round(v,3) for k,v in d['stage_ms'].items()})"
