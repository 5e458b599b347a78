# round 2: GPU suite + default bench after the launch-bound / guard / solve changes
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_gputests5.log 2>&1; tail -2 gpurun_out/r02_gputests5.log
timeout 900 python bench.py > gpurun_out/r02_bench_default2.json 2> gpurun_out/r02_bench_default2.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench_default2.json')); print(round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['value'], d['hash_guard']['flagged'], {k:round(v,3) for k,v in d['stage_ms'].items()})"
