for v in "" "SMCL_NO_LL_GATE=1"; do
  env $v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_b6.json 2> gpurun_out/r02_b6.err; echo "bench [$v] rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/r02_b6.json')); print(d['ms_per_step'], {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('gn_kernel_ms','ll_kernel_ms','svgd_ms','refresh_gather_ms')})"
done
timeout 600 python -m pytest tests/test_gpu_likelihood.py tests/test_gpu_parity_step.py -x -q -k "not exact_ten" > gpurun_out/r02_t6.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02_t6.log
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active -k regex:"k_ll_count|k_gicp_ll_lanes" -s 4 -c 2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "k_ll|k_gicp|duration|inst_exec|warps_active" | head -12
