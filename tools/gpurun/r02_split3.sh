# round 2: gate split statistics
SMCL_LL_SPLIT_STATS=1 timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/r02_split3.err; grep "ll-gate" gpurun_out/r02_split3.err | head -8
SMCL_LL_SPLIT_STATS=1 SMCL_NO_LL_SPLIT=1 timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/r02_split3b.err; grep "ll-gate" gpurun_out/r02_split3b.err | head -8
