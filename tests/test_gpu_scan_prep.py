"""Device scan input pipeline: make_scan_cloud
(filter.cpp:86-100) on the GPU must equal the host product path
(smcl_make_scan_cloud, pinned to the oracle in test_abi.py) bit for bit:
voxel downsample with leaf doubling (gaussian_cloud.cpp:110-144), kNN
plane-model covariances (gaussian_cloud.cpp:36-90) and the sensor-noise term.
A step on raw points (step_points) must equal step() on the host-prepared scan.
"""
import numpy as np
import pytest

import oracle as O
from helpers import config, room_scene
from paper_2404_16370_b200 import api, sim
from paper_2404_16370_b200.api import FilterEngine

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def raw():
    rects, mapc, _ = room_scene()
    pose = np.zeros(12)
    pose[[0, 4, 8]] = 1.0
    pose[9:] = [4.0, 3.0, 1.5]
    pts, _ = sim.simulate_scan_points(rects, pose, sim.sensor_spec(n_azimuth=256), 9)
    return mapc, pts


@pytest.mark.parametrize("kw", [dict(), dict(n_scan_max=200), dict(n_scan_max=64, scan_voxel_leaf=0.2),
                                dict(n_scan_max=5000), dict(covariance_k=6, sensor_noise_sigma=0.0),
                                dict(covariance_k=15, epsilon_plane=1e-2)])
def test_device_scan_prep_is_bitwise(raw, kw):
    mapc, pts = raw
    cfg = config(n_particles=64, nnf_resolution=0.2, **kw)
    e = FilterEngine(mapc, cfg)
    e.scan_prepare(3, pts)
    got = e.scan_get(3)
    want = api.make_scan_cloud(pts, cfg)
    assert len(got) == len(want) > 0
    assert np.array_equal(got.mu, want.mu)
    assert np.array_equal(got.sigma, want.sigma)
    mu, sg = O.make_scan_cloud(pts, cfg)
    assert np.array_equal(got.sigma, sg)


def test_lattice_ties_and_small_inputs(raw):
    mapc, _ = raw
    g = np.arange(0.0, 1.0, 0.1)
    lat = np.stack(np.meshgrid(g, g, [0.0, 0.1], indexing="ij"), -1).reshape(-1, 3)  # equidistant neighbours
    cfg = config(n_particles=64, nnf_resolution=0.2, n_scan_max=1000)
    e = FilterEngine(mapc, cfg)
    e.scan_prepare(0, lat)
    got, want = e.scan_get(0), api.make_scan_cloud(lat, cfg)
    assert np.array_equal(got.mu, want.mu) and np.array_equal(got.sigma, want.sigma)
    e.scan_prepare(1, lat[:8])  # fewer than k+1 points: empty scan (filter.cpp:87-89)
    assert len(e.scan_get(1)) == 0


def test_step_points_equals_host_prepared_step(raw):
    mapc, pts = raw
    cfg = config(n_particles=2048, nnf_resolution=0.2, seed=5)
    a, b = FilterEngine(mapc, cfg), FilterEngine(mapc, cfg)
    a.init_uniform(mapc.bounds)
    b.init_uniform(mapc.bounds)
    cov = np.diag([1e-4] * 6).reshape(36)
    for _ in range(2):
        ra = a.step_points(pts, None, cov, True)
        rb = b.step(api.make_scan_cloud(pts, cfg), None, cov, True)
        assert np.array_equal(ra["representative"], rb["representative"])
        assert ra["rep_log_post"] == rb["rep_log_post"] and ra["mean_n_matched"] == rb["mean_n_matched"]
    pa, pb = a.particles(), b.particles()
    assert np.array_equal(pa.poses, pb.poses) and np.array_equal(pa.log_post, pb.log_post)
    assert np.array_equal(pa.idx, pb.idx) and np.array_equal(pa.kval, pb.kval)


def test_async_pipeline_matches_synchronous(raw):
    """smcl_scan_prepare_async on the preparation stream, one frame ahead of
    the step (the bench's raw-points pipeline), gives bit-identical frames to
    the synchronous step_points sequence."""
    mapc, pts = raw
    rects = sim.box_room([8.0, 6.0, 3.0])
    frames = []
    for f in range(4):
        pose = np.zeros(12)
        pose[[0, 4, 8]] = 1.0
        pose[9:] = [3.0 + 0.3 * f, 3.0, 1.5]
        p, _ = sim.simulate_scan_points(rects, pose, sim.sensor_spec(n_azimuth=256), 30 + f)
        frames.append(p)
    cfg = config(n_particles=4096, nnf_resolution=0.2, seed=9, n_scan_max=200)
    a, b = FilterEngine(mapc, cfg), FilterEngine(mapc, cfg)
    a.init_uniform(mapc.bounds)
    b.init_uniform(mapc.bounds)
    cov = np.diag([1e-4] * 6).reshape(36)
    a.scan_prepare_async(0, frames[0])
    for i in range(4):
        if i + 1 < 4:
            a.scan_prepare_async((i + 1) % 2, frames[i + 1])
        ra = a.step_slot(i % 2, None, cov, True)
        rb = b.step_points(frames[i], None, cov, True)
        assert np.array_equal(ra["representative"], rb["representative"])
        assert ra["rep_log_post"] == rb["rep_log_post"]
    pa, pb = a.particles(), b.particles()
    assert np.array_equal(pa.poses, pb.poses) and np.array_equal(pa.idx, pb.idx)
    a.scan_prepare_async(5, frames[1])
    a.scan_prepare(6, frames[1])
    g5, g6 = a.scan_get(5), a.scan_get(6)
    assert np.array_equal(g5.mu, g6.mu) and np.array_equal(g5.sigma, g6.sigma)
