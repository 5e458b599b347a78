import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, oracle as O
from paper_2404_16370_b200 import workload
from paper_2404_16370_b200.api import FilterEngine
wl = workload.build("tracking", n_particles=1 << 16, scan_points=512, n_frames=12)
cfg = wl.cfg; cfg.likelihood_mode = 1; cfg.n_svgd_iters = 2
e = FilterEngine(wl.map, cfg); e.init_uniform(wl.bounds)
o = O.FilterEngine(wl.map.mu, wl.map.sigma, cfg, wl.map.bounds); o.init_uniform(wl.bounds)
for f in range(10):
    d, c, v = wl.odometry[f]; sc = wl.scans[f]
    rg = e.step(sc, d, c, v); ro = o.step(sc.mu, sc.sigma, d, c, v)
    G, R = e.particles(), o.particles()
    bad = np.argwhere(G.kval != R.kval)
    print("frame", f, "ids eq", np.array_equal(G.id, R.id), "idx eq", np.array_equal(G.idx, R.idx), "kval diff", len(bad),
          "pose maxdiff", np.abs(G.poses - R.poses).max())
    for i, s in bad[:5]:
        j = G.idx[i, s]
        kk = O.kernel(R.poses[i], R.poses[j], cfg.sigma_r, cfg.sigma_t)
        kg = O.kernel(G.poses[i], G.poses[j], cfg.sigma_r, cfg.sigma_t)
        print("   ", i, s, j, repr(G.kval[i, s]), repr(R.kval[i, s]), "oracle kernel on R poses", repr(kk), "on G poses", repr(kg),
              "float", repr(np.float32(kk)), "posediff i", np.abs(G.poses[i]-R.poses[i]).max(), "j", np.abs(G.poses[j]-R.poses[j]).max())
