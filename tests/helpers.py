"""Seeded fixtures mirroring /root/reference/proj/tests/test_helpers.hpp and the
scene builders of the reference suites (test_gicp.cpp, test_parallel_consistency.cpp,
test_neighbor_search.cpp). Random streams come from the oracle's SplitMix64 so
the fixtures are the reference's own seeded inputs."""
import math

import numpy as np

import oracle as O
from paper_2404_16370_b200 import sim
from paper_2404_16370_b200.abi import Particles, make_config
from paper_2404_16370_b200.api import GaussianCloud, estimate_covariances


def random_tangent(rng, max_angle, max_trans):  # test_helpers.hpp:10-17
    axis = np.array([rng.normal01(), rng.normal01(), rng.normal01()])
    axis /= np.sqrt((axis[0] * axis[0] + axis[1] * axis[1]) + axis[2] * axis[2])
    xi = np.zeros(6)
    xi[:3] = axis * rng.uniform_range(0.0, max_angle)
    for a in range(3):
        xi[3 + a] = rng.uniform_range(-max_trans, max_trans)
    return xi


def random_pose(rng, max_angle=math.pi - 0.2, max_trans=5.0):  # test_helpers.hpp:19-22
    return O.se3_exp(random_tangent(rng, max_angle, max_trans))[0]


def cube_set(n, seed, k, side=6.0, max_angle=0.3):
    """test_parallel_consistency.cpp:13-26 (random_pose(rng, 0.3, 0) then t ~ U[0,6]^3)."""
    rng = O.SplitMix64(seed)
    poses = np.empty((n, 12))
    for i in range(n):
        p = random_pose(rng, max_angle, 0.0)
        for a in range(3):
            p[9 + a] = rng.uniform_range(0.0, side)
        poses[i] = p
    return Particles.from_poses(poses, k)


def random_cube_set(n, side, max_angle, k, seed):
    """test_neighbor_search.cpp:24-37."""
    rng = O.SplitMix64(seed)
    poses = np.empty((n, 12))
    for i in range(n):
        axis = np.array([rng.normal01(), rng.normal01(), rng.normal01()])
        axis /= np.sqrt((axis[0] * axis[0] + axis[1] * axis[1]) + axis[2] * axis[2])
        xi = np.zeros(6)
        xi[:3] = axis * rng.uniform_range(0.0, max_angle)
        p = O.se3_exp(xi)[0]
        for a in range(3):
            p[9 + a] = rng.uniform_range(0.0, side)
        poses[i] = p
    return Particles.from_poses(poses, k)


def room_scene(size=(8.0, 6.0, 3.0), density=60.0, map_seed=3, scan_seed=5, center=(4.0, 3.0, 1.5),
               sensor=None, noise_sigma=0.01):
    """Box room, sampled map and a ray-cast scan with kNN covariances
    (test_parallel_consistency.cpp:31-41)."""
    rects = sim.box_room(size)
    mapc = sim.sample_world(rects, density, map_seed)
    pose = np.zeros(12)
    pose[[0, 4, 8]] = 1.0
    pose[9:] = center
    sensor = sensor if sensor is not None else sim.sensor_spec(noise_sigma=noise_sigma)
    pts, _ = sim.simulate_scan_points(rects, pose, sensor, scan_seed)
    scan = GaussianCloud(pts, estimate_covariances(pts, 10))
    return rects, mapc, scan


def config(**kw):
    return make_config(**kw)
