# round 2 final (after the K1 epilogue and smoothing PDL changes): launch list + --set full captures
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio --clock-control none --csv --log-file gpurun_out/r02_final4_launches.csv $CMD > gpurun_out/r02_final4_launches.log 2>&1; echo "launch rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_gicp|k_ll_count|k_refresh_gather|k_svgd" -s 15 -c 5 -o gpurun_out/r02_final4_full $CMD > gpurun_out/r02_final4_full.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_smooth|k_chunk_serial|k_reorder" -s 40 -c 3 -o gpurun_out/r02_final4_small $CMD > gpurun_out/r02_final4_small.log 2>&1; echo "ncu2 rc=$?"
