import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2404_16370_b200 import workload, api
from paper_2404_16370_b200.api import FilterEngine
wl = workload.build("global_init", n_particles=4096, scan_points=512, n_frames=4)
cfg = wl.cfg
cfg.n_scan_max = 512
e = FilterEngine(wl.map, cfg)
for i in range(4):
    t0 = time.perf_counter(); e.scan_prepare(1, wl.raw[i]); t1 = time.perf_counter()
    print("prepare total", (t1 - t0) * 1e3, "ms", file=sys.stderr)
