# round 2: full GPU suite + default bench (SVGD prefetch, lazy stage times, cheaper odometry marshalling)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputests3.log 2>&1; tail -3 gpurun_out/r02_gputests3.log
timeout 900 python bench.py > gpurun_out/r02_bench3.json 2> gpurun_out/r02_bench3.err || tail -5 gpurun_out/r02_bench3.err
python -c "import json; d=json.load(open('gpurun_out/r02_bench3.json')); print(round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items()}, d['clocks'])"
