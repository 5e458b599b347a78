set -x
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain2.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_gicp_fast|k_refresh_gather|k_svgd" -s 3 -c 3 -o gpurun_out/prof_r01 $CMD > gpurun_out/ncu2.log 2>&1; echo "ncu rc=$?"
