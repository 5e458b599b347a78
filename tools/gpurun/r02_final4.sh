# round 2: GPU suite + default bench + kidnap after the K1 queue rework
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_gputests7.log 2>&1; tail -2 gpurun_out/r02_gputests7.log
timeout 900 python bench.py > gpurun_out/r02_bench_default4.json 2> gpurun_out/r02_bench_default4.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench_default4.json')); print(round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['value'], d['hash_guard']['flagged'], d['roofline']['frac'], d['roofline_gather']['frac'], {k:round(v,3) for k,v in d['stage_ms'].items()})"
timeout 900 python bench.py --workload kidnap --steps 30 --warmup 25 --no-cpu-baseline --profile-json gpurun_out/r02_kid_prof.json > gpurun_out/r02_bench_kidnap2.json 2> gpurun_out/r02_bench_kidnap2.err; echo "kidnap rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench_kidnap2.json')); print(round(d['ms_per_step'],3), d['frame_ms'], d['roofline_gather']['frac'])"
