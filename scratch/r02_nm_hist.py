# Fraction of particles that pass the likelihood gate (n_matched >= ceil(0.5 S)) in the bench workload
import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2404_16370_b200 import workload
from paper_2404_16370_b200.api import FilterEngine
for kind, n in (("global_init", 1 << 20), ("tracking", 1 << 16), ("kidnap", 1 << 20)):
    wl = workload.build(kind, n_particles=n, scan_points=512, n_frames=14 if kind != "kidnap" else 32)
    e = FilterEngine(wl.map, wl.cfg)
    e.init_uniform(wl.bounds)
    nf = 12 if kind != "kidnap" else 28
    for f in range(nf):
        d, c, v = wl.odometry[f]
        e.step(wl.scans[f], d, c, v)
        if f in (0, 1, 2, 5, 11, 27):
            sc = wl.scans[f + 1]
            if len(sc) == 0:
                continue
            ll, nm = e.evaluate_likelihoods(sc)
            S = len(sc); mm = -(-S // 2)
            print(kind, "frame", f, "S", S, "live frac %.3f" % np.mean(nm >= mm), "mean nm %.1f" % nm.mean(),
                  "hist", np.histogram(nm, bins=8, range=(0, S))[0].tolist(), flush=True)
