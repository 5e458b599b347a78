import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle as O
from helpers import random_cube_set
from paper_2404_16370_b200.abi import make_config
from paper_2404_16370_b200.api import FilterEngine
n, side, ang, off = 600, 6.0, 0.3, 5000.0
g = random_cube_set(n, side, ang, 20, 71)
g.poses[:, 9:] += off
bounds = [off, off, off, off + side, off + side, off + side]
cfg = make_config()
r = g.copy()
e = FilterEngine(None, cfg); e.set_particles(g)
for p in range(4):
    seed = O.mix_seed(73, p)
    st = e.update_neighbors(seed, bounds)
    sr = O.update_neighbors(r, cfg, seed, bounds)
    got = e.particles()
    bad = np.nonzero((got.idx != r.idx).any(1) | (got.kval != r.kval).any(1) | (got.count != r.count))[0]
    print("pass", p, "mismatched particles", len(bad), st["buckets_used"], sr["buckets_used"])
    if len(bad):
        i = bad[0]
        print(" gpu", got.count[i], got.idx[i][:got.count[i]], got.kval[i][:got.count[i]])
        print(" ora", r.count[i], r.idx[i][:r.count[i]], r.kval[i][:r.count[i]])
        break
