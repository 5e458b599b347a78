"""Host time between steps at configs[2]: wall clock per step_slot call vs the
step's device span (E_START..E_END), with and without the per-step profile read."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2404_16370_b200 import workload
from paper_2404_16370_b200.api import FilterEngine

wl = workload.build("global_init", n_particles=1 << 20, scan_points=512, n_frames=24)
eng = FilterEngine(wl.map, wl.cfg, device=0)
eng.init_uniform(wl.bounds)
for f in range(24):
    eng.scan_upload(f, wl.scans[f])
for f in range(3):
    eng.step_slot(f, *wl.odometry[f])
import os as _os
for label, with_prof in (("step_slot+profile", True), ("step_slot only", False)):
    eng.timer_start()
    t0 = time.perf_counter()
    tot = []
    for f in range(3, 13) if with_prof else range(13, 23):
        r = eng.step_slot(f, *wl.odometry[f])
        tot.append(r["total_ms"])
        if with_prof:
            eng.last_step_profile()
    wall = (time.perf_counter() - t0) * 1e3 / 10
    dev = eng.timer_stop() / 10
    print(f"{label}: wall {wall:.3f} ms/step, device timer {dev:.3f}, step span {np.mean(tot):.3f}")
t0 = time.perf_counter()
for _ in range(100):
    eng.last_step_profile()
print(f"last_step_profile: {(time.perf_counter() - t0) * 1e4:.1f} us")
# per-call wall time between step_slot entries (host gap = wall - device span)
t_prev = time.perf_counter()
gaps = []
for f in range(3, 13):
    r = eng.step_slot(f, *wl.odometry[f])
    t = time.perf_counter()
    gaps.append((t - t_prev) * 1e3 - r["total_ms"])
    t_prev = t
print("wall - span per call (ms):", np.round(gaps[1:], 3))
