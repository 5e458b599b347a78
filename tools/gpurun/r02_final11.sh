# round 2 closing run (after the K1 fraction-bits change): GPU suite, default bench, kidnap, configs[4] problem on one GPU,
# then the launch list and --set full captures of the final kernels (profiles/)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_gputests12.log 2>&1; tail -2 gpurun_out/r02_gputests11.log
timeout 900 python bench.py > gpurun_out/r02_bench_default11.json 2> gpurun_out/r02_bench_default11.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench_default11.json')); print(round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['value'], d['gpu_launches'], d['hash_guard']['flagged'], round(d['roofline']['frac'],3), round(d['roofline_gather']['frac'],3), d['clocks'], {k:round(v,3) for k,v in d['stage_ms'].items()})"
timeout 900 python bench.py --workload kidnap --steps 30 --warmup 25 --no-cpu-baseline > gpurun_out/r02_bench_kidnap7.json 2> gpurun_out/r02_bench_kidnap7.err; echo "kidnap rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench_kidnap7.json')); print(round(d['ms_per_step'],3), d['frame_ms'], round(d['roofline_gather']['frac'],3))"
timeout 900 python bench.py --particles 4194304 --scan-points 1024 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_4m3.json 2> gpurun_out/r02_bench_4m3.err; echo "4m rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench_4m3.json')); print(round(d['ms_per_step'],3), d['value'])"
bash tools/gpurun/r02_finalprof2.sh
