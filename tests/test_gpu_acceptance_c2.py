"""Acceptance criterion C2 (proj/tests/acceptance.cpp:83-134): a one-particle
engine reduces to a directly coded damped Gauss-Newton tracker.

The GPU engine (N = 1) runs 50 FilterEngine::step calls on a 10 x 8 x 3 m box
room (density 60, seed 7, cfg.seed 3); the tracker applies the same odometry,
then one damped GN step per frame built from the oracle's evaluate /
solve_step / se3_exp / renormalize (gicp.cpp:11-75, se3.hpp). The reference
requires a deviation below 1e-9 in translation and rotation entries.

* exact mode (likelihood_mode = 1): <= 1e-9, as the reference;
* fast mode (the benchmarked fp32 algebra): the same trajectory within the
  fp32 GN tolerance (TOL_FAST).
"""
import math

import numpy as np
import pytest

import oracle as O
from paper_2404_16370_b200 import sim
from paper_2404_16370_b200.abi import identity_pose, make_config
from paper_2404_16370_b200.api import FilterEngine, make_scan_cloud

pytestmark = pytest.mark.gpu
TOL_FAST = 1e-5


def run_c2(mode):
    room = sim.box_room([10.0, 8.0, 3.0])
    mapc = sim.sample_world(room, 60.0, 7)
    cfg = make_config(n_particles=1, seed=3, likelihood_mode=mode)
    e = FilterEngine(mapc, cfg)
    e.init_uniform([4.9, 3.9, 1.4, 5.1, 4.1, 1.6])
    start = identity_pose()
    start[9:] = [5.0, 4.0, 1.5]
    p = e.particles()
    p.poses[0] = start
    e.set_particles(p)  # engine.mutable_particles().poses[0] = start
    om = O.OracleMap(mapc.mu, mapc.sigma, mapc.bounds, cfg.nnf_resolution, cfg.nnf_padding, cfg.nnf_max_query_dist)

    tracker = start.copy()
    gt = start.copy()
    delta = identity_pose()
    delta[9:] = [0.03, 0.01, 0.0]
    c, s = math.cos(0.008), math.sin(0.008)  # AngleAxisd(0.008, UnitZ)
    delta[:9] = [c, -s, 0.0, s, c, 0.0, 0.0, 0.0, 1.0]
    sensor = sim.sensor_spec(noise_sigma=0.0)
    zero_cov = np.zeros(36)
    worst = 0.0
    for f in range(50):
        gt = O.compose(gt, delta)
        pts, _ = sim.simulate_scan_points(room, gt, sensor, O.mix_seed(11, f))
        scan = make_scan_cloud(pts, cfg)
        fr = e.step(scan, delta, zero_cov, True)
        tracker = O.compose(tracker, delta)
        steps, ll, nm = O.evaluate_all(om, scan.mu, scan.sigma, tracker[None, :], cfg)
        if nm[0] > 0:  # solve_step(sys, damping * trace / 6, limits) is evaluate_all's step
            tracker = O.renormalize(O.compose(tracker, O.se3_exp(steps[0])[0]))
        rep = fr["representative"]
        worst = max(worst, float(np.linalg.norm(rep[9:] - tracker[9:])), float(np.abs(rep[:9] - tracker[:9]).max()))
    return worst


def test_c2_exact_single_particle_is_gn_tracker():
    worst = run_c2(1)
    print(f"C2 exact: max engine-vs-tracker deviation {worst:.3g} over 50 steps")
    assert worst < 1e-9


def test_c2_fast_single_particle_tracks_gn_tracker():
    worst = run_c2(2)
    print(f"C2 fast: max engine-vs-tracker deviation {worst:.3g} over 50 steps")
    assert worst < TOL_FAST
