CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_rg.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_refresh_gather|k_svgd" -s 2 -c 2 -o gpurun_out/prof_rg4 $CMD > gpurun_out/ncu_rg4.log 2>&1; echo "ncu rc=$?"
