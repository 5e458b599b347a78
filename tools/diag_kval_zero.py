"""Diagnostic: share of zero kernel values in the neighbour lists after the
bench's warm-up frames (configs[2] global_init at 1M)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_16370_b200 import workload  # noqa: E402
from paper_2404_16370_b200.api import FilterEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
wl = workload.build("global_init", n_particles=n, scan_points=512, n_frames=12)
eng = FilterEngine(wl.map, wl.cfg, device=0)
eng.init_uniform(wl.bounds)
for f in range(10):
    d, c, v = wl.odometry[f]
    eng.step(wl.scans[f], d, c, v)
    p = eng.particles()
    m = np.arange(p.k)[None, :] < p.count[:, None]
    kv = p.kval[m]
    print(f"frame {f}: entries/particle {m.sum() / p.n:.2f} zero {np.mean(kv == 0):.3f} "
          f"tiny(<1e-30) {np.mean(kv < 1e-30):.3f} one {np.mean(kv == 1):.3f}", flush=True)
