# round 2: final validation after the gate split: GPU suite, default bench (CPU baseline), kidnap
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_gputests10.log 2>&1; tail -2 gpurun_out/r02_gputests10.log
timeout 900 python bench.py > gpurun_out/r02_bench_default7.json 2> gpurun_out/r02_bench_default7.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench_default7.json')); print(round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['value'], d['gpu_launches'], d['hash_guard']['flagged'], round(d['roofline']['frac'],3), round(d['roofline_gather']['frac'],3), d['clocks'], {k:round(v,3) for k,v in d['stage_ms'].items()})"
timeout 900 python bench.py --workload kidnap --steps 30 --warmup 25 --no-cpu-baseline > gpurun_out/r02_bench_kidnap5.json 2> gpurun_out/r02_bench_kidnap5.err; echo "kidnap rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench_kidnap5.json')); print(round(d['ms_per_step'],3), d['frame_ms'], round(d['roofline_gather']['frac'],3))"
