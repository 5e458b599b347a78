CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_k1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gicp_fast" -s 1 -c 1 -o gpurun_out/prof_k1b $CMD > gpurun_out/ncu_k1b.log 2>&1; echo "ncu rc=$?"
