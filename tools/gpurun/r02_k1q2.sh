# round 2: queue K1 as default: parity + one ncu --set full capture of it
timeout 900 python -m pytest tests/test_gpu_likelihood.py tests/test_gpu_parity_step.py tests/test_gpu_filter.py tests/test_gpu_golden.py tests/test_gpu_fullsize.py tests/test_gpu_acceptance_c2.py -x -q 2>&1 | tail -2
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gicp_fast_q" -s 3 -c 1 -o gpurun_out/r02_k1q $CMD > gpurun_out/r02_k1q_ncu.log 2>&1; echo "ncu rc=$?"
