# round 2: compute-sanitizer memcheck / racecheck on a small engine run (if the pool allows it)
cat > /tmp/small_step.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
from paper_2404_16370_b200 import workload
from paper_2404_16370_b200.api import FilterEngine
wl = workload.build("global_init", n_particles=4096, scan_points=512, n_frames=4)
e = FilterEngine(wl.map, wl.cfg, device=0)
e.init_uniform(wl.bounds)
for f in range(3):
    e.step(wl.scans[f], *wl.odometry[f])
print("ok")
PY
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python /tmp/small_step.py > gpurun_out/r02_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -5 gpurun_out/r02_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python /tmp/small_step.py > gpurun_out/r02_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -5 gpurun_out/r02_racecheck.log
