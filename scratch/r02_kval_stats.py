import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2404_16370_b200 import workload
from paper_2404_16370_b200.api import FilterEngine
wl = workload.build("global_init", n_particles=1 << 20, scan_points=512, n_frames=10)
e = FilterEngine(wl.map, wl.cfg); e.init_uniform(wl.bounds)
for f in range(8):
    d, c, v = wl.odometry[f]
    r = e.step(wl.scans[f], d, c, v)
    if f in (2, 4, 7):
        p = e.particles()
        valid = np.arange(p.k)[None, :] < p.count[:, None]
        kv = p.kval[valid]
        print("frame", f, "count mean %.2f" % p.count.mean(), "kval==0 %.3f" % np.mean(kv == 0), "kval<1e-30 %.3f" % np.mean(kv < 1e-30),
              "kval<1e-6 %.3f" % np.mean(kv < 1e-6), "nonzero per row %.2f" % ((p.kval > 0) & valid).sum(1).mean(),
              "stats", r["neighbor_stats"]["buckets_used"], r["neighbor_stats"]["occupancy_hist"][:12], flush=True)
