import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2404_16370_b200 import workload
from paper_2404_16370_b200.api import FilterEngine
wl = workload.build("global_init", n_particles=1 << 20, scan_points=512, n_frames=10)
e = FilterEngine(wl.map, wl.cfg); e.init_uniform(wl.bounds)
for f in range(8):
    d, c, v = wl.odometry[f]
    e.step(wl.scans[f], d, c, v)
    if f in (2, 5, 7):
        p = e.particles()
        valid = np.arange(p.k)[None, :] < p.count[:, None]
        kv = p.kval[valid]
        print(f, "count mean", p.count.mean(), "kval==0 frac", np.mean(kv == 0), "kval<1e-30", np.mean(kv < 1e-30), "median", np.median(kv))
