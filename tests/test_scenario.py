"""Trajectory evaluation and I/O of the scenario harness (eval.cpp:32-116,
trajectory_io.cpp:10-92), re-expressing test_eval.cpp-style known answers."""
import math

import numpy as np

from paper_2404_16370_b200 import scenario as S
from paper_2404_16370_b200 import sim


def _traj(n, off=0.0, yaw=0.0):
    return [(0.1 * f, sim.pose_of(sim.yaw_rotation(yaw), np.array([0.5 * f + off, 1.0, 0.0]))) for f in range(n)]


def test_identical_trajectories():
    t = _traj(30)
    r = S.evaluate_ate(t, t)
    assert r.ate_rmse == 0.0 and r.ate_max == 0.0 and r.convergence_frame == 0
    assert r.ate_rmse_post_convergence == 0.0


def test_constant_offset_and_convergence():
    truth = _traj(40)
    est = [(s, p.copy()) for s, p in truth]
    for f in range(12):  # far away for 12 frames, then exact
        est[f][1][9] += 5.0
    r = S.evaluate_ate(est, truth)
    assert r.convergence_frame == 12
    assert abs(r.ate_max - 5.0) < 1e-12
    assert abs(r.ate_rmse - math.sqrt(12 * 25.0 / 40)) < 1e-12
    assert r.ate_rmse_post_convergence == 0.0
    # rotation threshold: 20 degrees of yaw never converges
    bad = [(s, sim.pose_of(sim.yaw_rotation(math.radians(20)), p[9:])) for s, p in truth]
    assert S.evaluate_ate(bad, truth).convergence_frame == -1


def test_recovery_frames_and_alignment():
    truth = _traj(60)
    est = [(s, p.copy()) for s, p in truth]
    for f in range(20, 35):  # lost during and a little after the occlusion [20, 30)
        est[f][1][10] += 3.0
    r = S.evaluate_ate(est, truth, 0, S.AteOptions(occlusions=[(20, 30)]))
    assert r.recovery_frames == [5]
    shifted = [(s, sim.compose(sim.pose_of(sim.yaw_rotation(0.3), np.array([2.0, -1.0, 0.5])), p))
               for s, p in truth]
    assert S.evaluate_ate(shifted, truth).ate_rmse > 1.0
    assert S.evaluate_ate(shifted, truth, 0, S.AteOptions(align=True)).ate_rmse < 1e-9


def test_tum_and_odometry_round_trip(tmp_path):
    rng = np.random.default_rng(2)
    traj = []
    for f in range(25):
        xi = np.concatenate([rng.normal(size=3) * 1.2, rng.normal(size=3)])
        traj.append((0.1 * f, sim.se3_exp(xi)))
    p = tmp_path / "t.tum"
    S.write_tum(str(p), traj)
    back = S.read_tum(str(p))
    for (s0, a), (s1, b) in zip(traj, back):
        assert abs(s0 - s1) < 1e-6 and np.abs(a - b).max() < 1e-8
    odo = [(traj[f][1], np.diag(np.arange(1.0, 7.0) * 1e-4).reshape(36), f % 3 != 0) for f in range(25)]
    q = tmp_path / "o.txt"
    S.write_odometry(str(q), odo)
    for (d0, c0, v0), (d1, c1, v1) in zip(odo, S.read_odometry(str(q))):
        assert np.abs(d0 - d1).max() < 1e-9 and np.abs(c0 - c1).max() < 1e-15 and v0 == v1
    with open(q, "a") as f:
        f.write("1 2 3\n")
    try:
        S.read_odometry(str(q))
        raise AssertionError("malformed line accepted")
    except RuntimeError:
        pass
