# round 2: functional check of bench.py's multi-rank path (2 ranks, gloo, one GPU; not a measurement)
SMCL_BENCH_GLOO=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --particles 262144 > gpurun_out/r02_mrank.json 2> gpurun_out/r02_mrank.err; echo "rc=$?"
grep -v "^\[" gpurun_out/r02_mrank.json | head -2 | cut -c1-600
tail -5 gpurun_out/r02_mrank.err
timeout 900 python bench.py --steps 3 --warmup 3 --particles 262144 --no-cpu-baseline > gpurun_out/r02_mrank1.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/r02_mrank1.json')); print('single', d['config']['pp_per_step'], d['hash_guard'])"
