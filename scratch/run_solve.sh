for mb in 1 4 6; do
  touch paper_2404_16370_b200/csrc/kernels/likelihood.cu
  make -j16 EXTRA_NVFLAGS="-DSMCL_SOLVE_MINB=$mb" > /dev/null 2>&1 || { echo "build fail $mb"; continue; }
  timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_sv.json 2> /dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/b_sv.json').read().strip().splitlines()[-1])
print('minb $mb', round(d['ms_per_step'],3), round(d['stage_ms']['solve_ms'],3))"
done
