"""Seeded synthetic workloads of BASELINE.json's configs.

* ``global_init``  — configs[2]: corridor_world (4 identical rooms, 100 pts/m^2,
  NNF 0.1 m), N particles uniform over the map with full SO3, 512-point scans
  along the corridor_easy trajectory.
* ``tracking``     — configs[1]: box_easy room with the corridor.cfg desk
  calibration, 65,536 particles, 512-point scans.
* ``kidnap``       — configs[3]: builder-defined outdoor world (280 x 200 x
  30 m city grid, 10 pts/m^2, NNF 0.2 m / 2.0 m max query = 2.2e8 cells), a
  street drive with a 20-frame scan blackout and a teleport (empty scans
  exercise the kidnap branch of filter.cpp:174-187).

Scans: 2,048 rays (256 azimuths x 8 elevations in [-30, 30] deg, 30 m range,
1 cm range noise), voxel-downsampled at the reference's 5 cm leaf, then
subsampled evenly to exactly S points (the reference bench truncates raw points
to S, bench.cpp:40-42), kNN(10) plane-model covariances + sensor noise^2 I
(filter.cpp:86-100).
"""
import numpy as np

from . import sim
from .abi import CORRIDOR_CFG, make_config
from .api import GaussianCloud, downsample_to, estimate_covariances


def bench_sensor():
    return sim.sensor_spec(n_azimuth=256, elevations_deg=list(np.linspace(-30.0, 30.0, 8)), max_range=30.0,
                           noise_sigma=0.01)


def scan_of_points(pts, n_points, cfg):
    if len(pts) < max(cfg.covariance_k + 1, 5):  # occluded frame: empty scan (filter.cpp:87-89)
        return GaussianCloud(np.zeros((0, 3)), np.zeros((0, 9)))
    d = downsample_to(pts, 1 << 20, cfg.scan_voxel_leaf)
    if len(d) > n_points:
        d = d[np.linspace(0, len(d) - 1, n_points).astype(np.int64)]
    sig = estimate_covariances(d, min(cfg.covariance_k, len(d) - 1), cfg.epsilon_plane)
    nv = cfg.sensor_noise_sigma ** 2
    sig[:, [0, 4, 8]] += nv
    return GaussianCloud(d, sig)


class Workload:
    def __init__(self, name, cfg, mapc, rects, scans, odometry, truth, raw=None):
        self.name, self.cfg, self.map, self.rects = name, cfg, mapc, rects
        self.scans, self.odometry, self.truth = scans, odometry, truth
        self.raw = raw or []  # raw sensor points per frame (make_scan_cloud input)

    @property
    def bounds(self):
        return self.map.bounds


def build(kind="global_init", n_particles=1 << 20, scan_points=512, n_frames=13, seed=1):
    if kind == "global_init":
        sc = sim.scenario_preset("corridor_easy", seed=seed)
        cfg = make_config(n_particles=n_particles, seed=seed)
    elif kind == "kidnap":
        # configs[3]: outdoor world 280 x 200 x 30 m, NNF 0.2 m, max query 2.0 m
        sc = sim.scenario_preset("outdoor_kidnap", seed=seed)
        cfg = make_config(n_particles=n_particles, seed=seed, nnf_resolution=0.2, nnf_max_query_dist=2.0)
    elif kind == "tracking":
        sc = sim.scenario_preset("box_easy", seed=seed)
        cfg = make_config(n_particles=n_particles, seed=seed, **CORRIDOR_CFG)
    else:
        raise ValueError(kind)
    sc.sensor = bench_sensor()
    rects, mapc = sim.scenario_map(sc, cfg)
    sc.n_frames = max(sc.n_frames, n_frames)
    truth = sim.build_trajectory(sc)[:n_frames]
    odo = sim.build_odometry(sc, truth)
    scans, raw = [], []
    for f in range(n_frames):
        pts = sim.scan_points_for_frame(sc, rects, truth, f)
        raw.append(pts)
        scans.append(scan_of_points(pts, scan_points, cfg))
    return Workload(kind, cfg, mapc, rects, scans, odo, truth, raw)
