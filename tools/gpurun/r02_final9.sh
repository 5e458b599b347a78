# round 2 closing bench: default line (CPU baseline) with the final profiles/r02_dram_traffic.json
timeout 900 python bench.py > gpurun_out/r02_bench_default9.json 2> gpurun_out/r02_bench_default9.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench_default9.json')); print(round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['value'], d['gpu_launches'], round(d['roofline']['frac'],3), round(d['roofline_gather']['frac'],3), d['clocks'], {k:round(v,3) for k,v in d['stage_ms'].items()})"
