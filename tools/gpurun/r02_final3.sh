# round 2: GPU suite + default bench + launch list / ncu of the queue K1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_gputests6.log 2>&1; tail -2 gpurun_out/r02_gputests6.log
timeout 900 python bench.py > gpurun_out/r02_bench_default3.json 2> gpurun_out/r02_bench_default3.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench_default3.json')); print(round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['value'], d['hash_guard']['flagged'], {k:round(v,3) for k,v in d['stage_ms'].items()})"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio --clock-control none --csv --log-file gpurun_out/r02_p5_launches.csv $CMD > gpurun_out/r02_p5_launches.log 2>&1; echo "launch rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_gicp|k_ll_count|k_refresh_gather|k_svgd" -s 15 -c 5 -o gpurun_out/r02_p5_full $CMD > gpurun_out/r02_p5_full.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_smooth|k_chunk_serial|k_reorder" -s 40 -c 3 -o gpurun_out/r02_p5_small $CMD > gpurun_out/r02_p5_small.log 2>&1; echo "ncu2 rc=$?"
