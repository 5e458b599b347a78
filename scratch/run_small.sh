CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_s.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_smooth_round|k_svgd|k_solve|k_reorder_k|k_chunk|k_bayes|k_seg_stats" -s 20 -c 12 -o gpurun_out/prof_small $CMD > gpurun_out/ncu_s.log 2>&1; echo "ncu rc=$?"
