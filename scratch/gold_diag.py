import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, 'tests/golden'); sys.path.insert(0, 'tests')
import numpy as np
import make_golden as G
from paper_2404_16370_b200.abi import make_config
from paper_2404_16370_b200.api import FilterEngine, GaussianCloud
GOLD = np.load('tests/golden/configs0_smoke.npz')
rects, mapc, pts, cfg, mu, sg = G.configs0()
e = FilterEngine(mapc, cfg); e.init_uniform(mapc.bounds)
steps, ll, nm = e.evaluate_all(GaussianCloud(mu, sg))
d = np.flatnonzero(ll != GOLD['ea_ll'])
print('ll mismatches', len(d), 'nm mismatches', np.count_nonzero(nm != GOLD['ea_nm']))
for i in d[:10]:
    print(i, nm[i], ll[i], GOLD['ea_ll'][i], (ll[i]-GOLD['ea_ll'][i])/abs(GOLD['ea_ll'][i]))
ds = np.flatnonzero(np.any(steps != GOLD['ea_steps'], 1)); print('step mismatches', len(ds))
p = e.particles(); print('poses equal init?', np.abs(p.poses).sum())
