# round 2 closing bench (raw-points leg with the preparation pipeline set up before the timed region)
timeout 900 python bench.py > gpurun_out/r02_bench_default10.json 2> gpurun_out/r02_bench_default10.err; echo "bench rc=$?"
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02_bench_nocpu10.json 2> gpurun_out/r02_bench_nocpu10.err; echo "bench rc=$?"
for f in gpurun_out/r02_bench_default10.json gpurun_out/r02_bench_nocpu10.json; do
python -c "import json; d=json.load(open('$f')); print(round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), round(d['e2e_raw_points']['ms_per_step'],3), d['value'], d['gpu_launches'], round(d['roofline']['frac'],3), d['clocks'])"
done
