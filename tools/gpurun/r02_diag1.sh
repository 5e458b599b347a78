# round 2: refresh-pass statistics, launch list, --set full of the hot kernels
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
SMCL_RG_STATS=1 timeout 300 $CMD > gpurun_out/r02_rgstats.json 2> gpurun_out/r02_rgstats.err; echo "stats rc=$?"
grep "\[rg\]" gpurun_out/r02_rgstats.err | head -12
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio --clock-control none --csv --log-file gpurun_out/r02_launches.csv $CMD > gpurun_out/r02_launches.log 2>&1; echo "launch rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_gicp|k_ll_count|k_refresh_gather|k_svgd|k_smooth" -s 12 -c 7 -o gpurun_out/r02_full1 $CMD > gpurun_out/r02_full1.log 2>&1; echo "ncu rc=$?"
