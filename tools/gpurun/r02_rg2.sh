# round 2: GN 4x20 default; refresh/gather evaluation-loop prefetch variant; ncu of K1 and RG
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "X=1" "SMCL_RG_EVPF=1"; do
  env $v timeout 600 $B > gpurun_out/r02_rg2.json 2> gpurun_out/r02_rg2.err || tail -5 gpurun_out/r02_rg2.err
  python -c "import json; d=json.load(open('gpurun_out/r02_rg2.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('gn_kernel_ms','refresh_gather_ms','svgd_ms','total_ms')})"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gicp_fast|k_refresh_gather" -s 4 -c 2 -o gpurun_out/r02_full2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02_full2.log 2>&1; echo "ncu rc=$?"
