# round 2: final validation: GPU suite + default bench (with CPU baseline) + kidnap + reference arm
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_gputests8.log 2>&1; tail -2 gpurun_out/r02_gputests8.log
timeout 900 python bench.py > gpurun_out/r02_bench_default5.json 2> gpurun_out/r02_bench_default5.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench_default5.json')); print(round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['value'], d['hash_guard']['flagged'], round(d['roofline']['frac'],3), round(d['roofline_gather']['frac'],3), d['clocks'], {k:round(v,3) for k,v in d['stage_ms'].items()})"
timeout 900 python bench.py --workload kidnap --steps 30 --warmup 25 --no-cpu-baseline --profile-json gpurun_out/r02_kid_prof.json > gpurun_out/r02_bench_kidnap3.json 2> gpurun_out/r02_bench_kidnap3.err; echo "kidnap rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench_kidnap3.json')); print(round(d['ms_per_step'],3), d['frame_ms'], round(d['roofline_gather']['frac'],3))"
