timeout 600 python bench.py --workload tracking --particles 65536 --no-cpu-baseline > gpurun_out/bench_track.json 2> gpurun_out/bench_track.err; echo "track rc=$?"; tail -2 gpurun_out/bench_track.err
python -c "import json; d=json.load(open('gpurun_out/bench_track.json')); print(d['ms_per_step'], d['value'], d['e2e']['ms_per_step']); print({k: round(v,3) for k,v in d['stage_ms'].items()})"
timeout 600 python bench.py --particles 4194304 --scan-points 1024 --steps 5 --no-cpu-baseline > gpurun_out/bench_4m.json 2> gpurun_out/bench_4m.err; echo "4m rc=$?"; tail -2 gpurun_out/bench_4m.err
python -c "import json; d=json.load(open('gpurun_out/bench_4m.json')); print(d['ms_per_step'], d['value'], d['e2e']['ms_per_step']); print({k: round(v,3) for k,v in d['stage_ms'].items()})"
