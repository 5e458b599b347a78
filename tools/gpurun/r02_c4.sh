# round 2: configs[4]'s problem size on one B200 (4,194,304 particles x 1,024-pt scans)
timeout 1200 python bench.py --particles 4194304 --scan-points 1024 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_4m.json 2> gpurun_out/r02_bench_4m.err; echo "rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench_4m.json')); print(round(d['ms_per_step'],3), d['value'], {k:round(v,3) for k,v in d['stage_ms'].items()})"
tail -3 gpurun_out/r02_bench_4m.err
