python scratch/ll_dump.py gpurun_out/ll_base.npy
SMCL_LL_COMPACT=2x8:3 python scratch/ll_dump.py gpurun_out/ll_cmp.npy
python -c "
import numpy as np
a=np.load('gpurun_out/ll_base.npy'); b=np.load('gpurun_out/ll_cmp.npy'); print('bitwise equal:', np.array_equal(a,b), (a!=b).sum())"
run() {
  timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_c.json 2> gpurun_out/b_c.err
  python -c "
import json
d=json.loads(open('gpurun_out/b_c.json').read().strip().splitlines()[-1])
print('$1', round(d['ms_per_step'],3), round(d['stage_ms']['ll_kernel_ms'],3))" || tail -3 gpurun_out/b_c.err
}
run base
for c in 2x8:3 2x8:2 4x8:2 2x4:6 4x4:4; do SMCL_LL_COMPACT=$c run $c; done
