for v in "-DSMCL_SVGD_MINB=5" "-DSMCL_SVGD_MINB=7" "-DSMCL_SVGD_MINB=8" "-DSMCL_SVGD_VEC -DSMCL_SVGD_MINB=6" "-DSMCL_SVGD_VEC -DSMCL_SVGD_MINB=8"; do
  touch paper_2404_16370_b200/csrc/kernels/particles.cu
  make -j16 EXTRA_NVFLAGS="$v" > /dev/null 2>&1 || { echo "build fail $v"; continue; }
  timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/bench_sv.json 2> /dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/bench_sv.json').read().strip().splitlines()[-1])
print('$v', d['ms_per_step'], d['stage_ms']['svgd_ms'])"
done
