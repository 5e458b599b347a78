for v in "X=1" "SMCL_SVGD_F64=1"; do
  env $v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_b10.json 2> gpurun_out/r02_b10.err
  python -c "import json; d=json.load(open('gpurun_out/r02_b10.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('gn_kernel_ms','ll_kernel_ms','svgd_ms')})"
done
timeout 900 python -m pytest tests/test_gpu_parity_step.py -x -q -s -k "whole_step" 2>&1 | grep -E "whole step|passed|failed|Error" | cut -c1-400
