# round 2: fresh ncu --set full of the three hot kernels on the current code
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/r02_plain.log 2>&1; echo "plain rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_gicp|k_refresh_gather|k_svgd|k_smooth" -s 6 -c 6 -o gpurun_out/r02_prof0 $CMD > gpurun_out/r02_ncu0.log 2>&1; echo "ncu rc=$?"
