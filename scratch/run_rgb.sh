for b in 64 32 128; do
  touch paper_2404_16370_b200/csrc/kernels/lsh.cu
  make -j16 EXTRA_NVFLAGS="-DSMCL_RG_BLOCK=$b" > /dev/null 2>&1 || { echo "build fail $b"; continue; }
  timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_rg.json 2> /dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/b_rg.json').read().strip().splitlines()[-1])
print('block $b', round(d['ms_per_step'],3), round(d['stage_ms']['refresh_gather_ms'],3))"
done
