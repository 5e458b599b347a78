timeout 1500 python -m pytest tests -m gpu -q -s -k "not outdoor" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python - <<'P'
import json
d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print("ms", d["ms_per_step"], {k: round(v,3) for k,v in d["stage_ms"].items()})
P
timeout 900 python -m pytest tests/test_gpu_scenario.py -q -s -k outdoor > gpurun_out/outdoor.log 2>&1; echo "outdoor rc=$?"; grep "outdoor kidnap" gpurun_out/outdoor.log
