import sys, numpy as np
sys.path.insert(0, '.')
from paper_2404_16370_b200 import workload
from paper_2404_16370_b200.api import FilterEngine
wl = workload.build("global_init", n_particles=1 << 20, scan_points=512, n_frames=6)
eng = FilterEngine(wl.map, wl.cfg)
eng.init_uniform(wl.bounds)
for f in range(6):
    d, c, v = wl.odometry[f]
    r = eng.step(wl.scans[f], d, c, v)
    h = np.array(r["neighbor_stats"]["occupancy_hist"], dtype=np.float64)
    s = np.arange(len(h))
    parts = h * s  # particles in buckets of size s
    win = np.minimum(s, 64) - 1
    print(f"frame {f}: mean window/particle {(parts * win).sum() / parts.sum():.2f}  buckets used {r['neighbor_stats']['buckets_used']}"
          f"  mean kernel {r['neighbor_stats']['mean_kernel']:.4f}  matched {r['mean_n_matched']:.1f}")
p = eng.particles()
cnt = p.count
print("list count mean", cnt.mean(), "full frac", (cnt == p.k).mean())
