timeout 600 python scratch/occ_stats.py > gpurun_out/occ_stats.log 2>&1; echo "occ rc=$?"; cat gpurun_out/occ_stats.log | tail -9
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_rg.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_refresh_gather|k_gicp" -s 3 -c 3 -o gpurun_out/prof_r3 $CMD > gpurun_out/ncu_r3.log 2>&1; echo "ncu rc=$?"
