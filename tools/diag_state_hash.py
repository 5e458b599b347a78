"""Diagnostic: hash of the particle state after a few filter steps (configs[2]
global init, default 65,536 particles), to compare kernel variants selected by
environment switches bit for bit across two processes."""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_16370_b200 import workload  # noqa: E402
from paper_2404_16370_b200.api import FilterEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 5
wl = workload.build("global_init", n_particles=n, scan_points=512, n_frames=frames)
eng = FilterEngine(wl.map, wl.cfg, device=0)
eng.init_uniform(wl.bounds)
for f in range(frames):
    d, c, v = wl.odometry[f]
    r = eng.step(wl.scans[f], d, c, v)
p = eng.particles()
h = hashlib.sha256()
for a in (p.poses, p.log_post, p.id, p.idx, p.kval, p.count):
    h.update(np.ascontiguousarray(a).tobytes())
print(f"n {n} frames {frames} rep_log_post {r['rep_log_post']!r} state {h.hexdigest()[:16]}")
