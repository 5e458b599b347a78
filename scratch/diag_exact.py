import sys, numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import oracle as O
from test_gpu_filter import SmallWorld, I12
from paper_2404_16370_b200 import sim
from paper_2404_16370_b200.abi import make_config
from paper_2404_16370_b200.api import FilterEngine
w = SmallWorld()
cfg = make_config(n_particles=500, seed=42, nnf_resolution=0.2, likelihood_mode=1)
g = FilterEngine(w.map, cfg); r = O.FilterEngine(w.map.mu, w.map.sigma, cfg, w.map.bounds)
g.init_uniform(w.map.bounds); r.init_uniform(w.map.bounds)
gt = I12.copy(); gt[9:] = [5.0, 4.0, 1.5]
delta = I12.copy(); delta[9] = 0.05
cov = np.diag([1e-4] * 6).reshape(36)
for f in range(6):
    gt = sim.compose(gt, delta)
    scan = w.scan_at(gt, cfg, 100 + f)
    a = g.step(scan, delta, cov, True); b = r.step(scan.mu, scan.sigma, delta, cov, True)
    pg, pr = g.particles(), r.particles()
    print(f, a["rep_id"], b["rep_id"], a["rep_log_post"], b["rep_log_post"], a["mean_n_matched"], b["mean_n_matched"])
    for nm in ("poses", "log_post", "id", "idx", "kval", "count"):
        x, y = getattr(pg, nm), getattr(pr, nm)
        d = np.abs(x.astype(np.float64) - y.astype(np.float64))
        print("  ", nm, "maxdiff", d.max(), "n_diff", int((d > 0).sum()))
