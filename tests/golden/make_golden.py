"""Regenerate tests/golden/configs0_smoke.npz: the CPU-ref smoke config of
BASELINE.json (configs[0]) run through the oracle (oracle/, the C++
restatement of /root/reference/proj), so the GPU parity tests and the
oracle's own regression test compare against committed vectors.

configs[0]: box_room(10, 10, 3) sampled at 100 pts/m^2, NNF
0.1 m (pad 0.5, max query 1.0); 4,096 particles init_uniform over the map
bounds with full SO3 (seed 1); one scan from (5, 5, 1.5): 256 azimuths x 8
elevations (2,048 rays, sigma 0.01) -> downsample_to(256) -> kNN(10)
covariances + 0.01^2 I; then one LSH neighbour pass and one full step.

Usage: python tests/golden/make_golden.py   (writes next to this script)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402
from paper_2404_16370_b200 import sim  # noqa: E402
from paper_2404_16370_b200.abi import make_config  # noqa: E402


def configs0():
    rects = sim.box_room([10.0, 10.0, 3.0])
    mapc = sim.sample_world(rects, 100.0, sim.mix_seed(1, 13))
    sensor = sim.sensor_spec(n_azimuth=256, elevations_deg=list(np.linspace(-30.0, 30.0, 8)), noise_sigma=0.01)
    pose = np.zeros(12)
    pose[[0, 4, 8]] = 1.0
    pose[9:] = [5.0, 5.0, 1.5]
    pts, _ = sim.simulate_scan_points(rects, pose, sensor, sim.mix_seed(1, 11, 0))
    cfg = make_config(n_particles=4096, seed=1, nnf_resolution=0.1, nnf_padding=0.5, nnf_max_query_dist=1.0,
                      n_scan_max=256, likelihood_mode=1)
    mu, sg = O.make_scan_cloud(pts, cfg)
    return rects, mapc, pts, cfg, mu, sg


def compute():
    rects, mapc, pts, cfg, mu, sg = configs0()
    parts0 = O.init_uniform(cfg.n_particles, cfg.k_neighbors, mapc.bounds, True, 1)
    om = O.OracleMap(mapc.mu, mapc.sigma, mapc.bounds, cfg.nnf_resolution, cfg.nnf_padding, cfg.nnf_max_query_dist)
    steps, ll, nm = O.evaluate_all(om, mu, sg, parts0.poses, cfg)
    import copy
    pn = copy.deepcopy(parts0)
    nbst = O.update_neighbors(pn, cfg, 0x5EED, mapc.bounds)  # in place: reorder + lists
    eng = O.FilterEngine(mapc.mu, mapc.sigma, cfg, mapc.bounds)
    eng.init_uniform(mapc.bounds)
    fr = eng.step(mu, sg, None, np.diag([1e-4] * 6).reshape(36), True)
    p1 = eng.particles()
    import hashlib

    def digest(a):
        return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), np.uint8)

    return dict(
        # inputs are regenerated from their seeds; their digests pin them
        map_mu_sha256=digest(mapc.mu), map_sigma_sha256=digest(mapc.sigma), scan_points_sha256=digest(pts),
        init_poses_sha256=digest(parts0.poses),
        scan_mu=mu, scan_sigma=sg,
        ea_steps=steps, ea_ll=ll, ea_nm=nm,
        nb_id=pn.id, nb_idx=pn.idx, nb_kval=pn.kval, nb_count=pn.count,
        nb_buckets_used=np.array(nbst["buckets_used"]), nb_mean_kernel=np.array(nbst["mean_kernel"]),
        step_rep=fr["representative"], step_rep_id=np.array(fr["rep_id"]),
        step_rep_log_post=np.array(fr["rep_log_post"]), step_mean_n_matched=np.array(fr["mean_n_matched"]),
        p1_poses=p1.poses, p1_log_post=p1.log_post, p1_id=p1.id, p1_idx=p1.idx, p1_kval=p1.kval,
        p1_count=p1.count,
    )


if __name__ == "__main__":
    out = compute()
    np.savez_compressed(os.path.join(HERE, "configs0_smoke.npz"), **out)
    print({k: v.shape for k, v in out.items()})
