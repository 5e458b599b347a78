# round 2: ncu --set full (with source) of K6/K7, K1, K8, K2 of the third step
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gicp|k_refresh_gather|k_svgd" -s 8 -c 4 -o gpurun_out/r02_prof1 $CMD > gpurun_out/r02_ncu1.log 2>&1; echo "ncu rc=$?"
