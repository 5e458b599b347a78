CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_k.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gicp|k_refresh_gather" -s 3 -c 3 -o gpurun_out/prof_full $CMD > gpurun_out/ncu_k.log 2>&1; echo "ncu rc=$?"
