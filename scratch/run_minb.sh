for mb in 1 10 12; do
  touch paper_2404_16370_b200/csrc/kernels/lsh.cu
  make -j16 EXTRA_NVFLAGS="-DSMCL_RG_MINB=$mb" > /dev/null 2>&1 || { echo "build fail $mb"; continue; }
  timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/bench_mb$mb.json 2> /dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/bench_mb$mb.json').read().strip().splitlines()[-1])
print('minb $mb', d['ms_per_step'], d['stage_ms']['refresh_gather_ms'], d['stage_ms']['svgd_ms'])"
done
