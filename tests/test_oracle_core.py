"""Pins the CPU oracle against the reference's own known-answer tests
(re-expressed from /root/reference/proj/tests/test_se3.cpp, test_svgd.cpp,
test_gicp.cpp, test_posterior.cpp). The reference ships no golden-vector
files; these closed-form / finite-difference / fixed-point assertions are its
pins for the hot path."""
import math

import numpy as np
import pytest

import oracle as O
from helpers import random_pose, random_tangent, room_scene
from paper_2404_16370_b200 import sim
from paper_2404_16370_b200.abi import identity_pose, make_config

I12 = identity_pose()


def R(p):
    return np.asarray(p)[:9].reshape(3, 3)


def T(p):
    return np.asarray(p)[9:]


# ---------------------------------------------------------------- se3 (test_se3.cpp)
def test_exp_zero_is_identity():
    p = O.se3_exp(np.zeros(6))[0]
    assert np.array_equal(p, I12)


def test_exp_quarter_turn_z():
    xi = np.zeros(6)
    xi[2] = math.pi / 2
    p = O.se3_exp(xi)[0]
    assert np.abs(R(p) @ [1, 0, 0] - [0, 1, 0]).max() < 1e-12
    assert np.all(T(p) == 0)


def test_exp_pure_translation():
    p = O.se3_exp([0, 0, 0, 1, 2, 3])[0]
    assert np.abs(R(p) - np.eye(3)).max() <= 1e-15 and np.linalg.norm(T(p) - [1, 2, 3]) < 1e-15


def test_log_identity_and_translation():
    assert np.linalg.norm(O.se3_log(I12)[0]) == 0.0
    p = I12.copy()
    p[9] = 2.0
    xi = O.se3_log(p)[0]
    assert np.linalg.norm(xi[:3]) == 0.0 and np.linalg.norm(xi[3:] - [2, 0, 0]) < 1e-12


def test_log_inverts_exp():
    xi = np.array([0.1, -0.2, 0.3, 1.0, -1.0, 0.5])
    assert np.linalg.norm(O.se3_log(O.se3_exp(xi))[0] - xi) < 1e-9
    rng = O.SplitMix64(11)
    for _ in range(300):
        xi = random_tangent(rng, math.pi - 0.1, 10.0)
        assert np.linalg.norm(O.se3_log(O.se3_exp(xi))[0] - xi) < 1e-9


def test_compose_identity_inverse_associative():
    rng = O.SplitMix64(7)
    p = random_pose(rng)
    assert np.array_equal(O.compose(p, I12), p)
    r = O.inverse(O.inverse(p))
    assert np.abs(r - p).max() < 1e-12
    rng = O.SplitMix64(13)
    for _ in range(100):
        a, b, c = random_pose(rng), random_pose(rng), random_pose(rng)
        assert np.abs(O.compose(O.compose(a, b), c) - O.compose(a, O.compose(b, c))).max() < 1e-12


def test_log_pi_branch():
    xi = np.zeros(6)
    xi[:3] = (math.pi - 1e-3) * np.array([1, 2, 2]) / 3.0
    assert np.linalg.norm(O.se3_log(O.se3_exp(xi))[0] - xi) < 1e-6
    at = np.array([0, 0, math.pi, 0.5, -0.2, 0.1])
    p = O.se3_exp(at)[0]
    a, b = O.se3_log(p)[0], O.se3_log(p)[0]
    assert np.all(np.isfinite(a)) and np.array_equal(a, b)
    assert abs(np.linalg.norm(a[:3]) - math.pi) < 1e-6
    q = O.se3_exp(a)[0]
    assert np.abs(q - p).max() < 1e-6


def test_long_chain_stays_orthonormal():
    rng = O.SplitMix64(17)
    p = I12.copy()
    for _ in range(3000):
        p = O.renormalize(O.compose(p, O.se3_exp(random_tangent(rng, 0.05, 0.05))[0]))
    assert O.rotation_drift(p) < 1e-9 and np.linalg.det(R(p)) > 0


# ---------------------------------------------------------------- kernel / SVGD (test_svgd.cpp)
def test_kernel_self_one_and_one_meter():
    rng = O.SplitMix64(3)
    for _ in range(20):
        p = random_pose(rng)
        assert O.kernel(p, p) == 1.0
    b = I12.copy()
    b[9] = 1.0
    assert abs(O.kernel(I12, b) - math.exp(-2.5)) <= 1e-12 * math.exp(-2.5)


def test_kernel_symmetry_bounds_and_gradient():
    rng = O.SplitMix64(5)
    for _ in range(200):
        a, b = random_pose(rng, 2.0, 2.0), random_pose(rng, 2.0, 2.0)
        kab, kba = O.kernel(a, b), O.kernel(b, a)
        assert abs(kab - kba) < 1e-12 and 0.0 < kab <= 1.0
    rng = O.SplitMix64(11)
    h = 1e-6
    for _ in range(50):
        a = random_pose(rng, 1.0, 2.0)
        d = random_tangent(rng, 0.2, 0.25)
        if np.linalg.norm(d) >= 0.5:
            d *= 0.4 / np.linalg.norm(d)
        b = O.compose(a, O.se3_exp(d)[0])
        g = O.kernel_grad(a, b)
        for c in range(6):
            dp, dm = d.copy(), d.copy()
            dp[c] += h
            dm[c] -= h
            fd = (O.kernel(a, O.compose(a, O.se3_exp(dp)[0])) - O.kernel(a, O.compose(a, O.se3_exp(dm)[0]))) / (2 * h)
            assert abs(g[c] - fd) < 1e-4


def test_phi_self_only_and_single_particle_gn():
    rng = O.SplitMix64(17)
    p = random_pose(rng)
    psi = random_tangent(rng, 0.3, 0.5)
    phi = O.compute_phis([p], [psi], [[0]], [1])[0]
    assert np.array_equal(phi, psi)
    rng = O.SplitMix64(31)
    start = random_pose(rng)
    psi = random_tangent(rng, 0.2, 0.5)
    phi = O.compute_phis([start], [psi], [[0]], [1])
    got = O.apply_updates([start], phi)[0]
    assert np.array_equal(got, O.compose(start, O.se3_exp(psi)[0]))


def test_repulsion_sign_and_coincident():
    a, b = I12.copy(), I12.copy()
    b[9] = 0.2
    phi = O.compute_phis([a, b], np.zeros((2, 6)), [[0, 1], [0, 1]], [2, 2])
    assert phi[0][3] < 0.0 and phi[1][3] > 0.0
    rng = O.SplitMix64(37)
    p = random_pose(rng)
    n = 50
    poses = np.tile(p, (n, 1))
    idx = np.tile(np.arange(n, dtype=np.int32), (n, 1))
    phis = O.compute_phis(poses, np.zeros((n, 6)), idx, np.full(n, n))
    out = O.apply_updates(poses, phis)
    assert np.all(out == out[0]) and np.linalg.norm(T(out[0]) - T(p)) < 1e-12


def test_apply_zero_phi_noop():
    rng = O.SplitMix64(23)
    poses = np.array([random_pose(rng) for _ in range(10)])
    assert np.array_equal(O.apply_updates(poses, np.zeros((10, 6))), poses)


# ---------------------------------------------------------------- solve_step (test_gicp.cpp:130-173)
def test_solve_step_known_answers():
    Hm = np.eye(6)
    assert np.linalg.norm(O.solve_step(Hm, np.zeros(6), 0.0)) == 0.0
    b = np.zeros(6)
    b[3] = 1.0
    s = O.solve_step(Hm, b, 0.0)
    assert abs(s[3] + 1.0) < 1e-12 and np.linalg.norm(s[:3]) < 1e-12
    rng = O.SplitMix64(5)
    for _ in range(50):
        a = np.array([[rng.normal01() for _ in range(6)] for _ in range(6)])
        Hs = a.T @ a + 0.1 * np.eye(6)
        bb = np.array([rng.normal01() for _ in range(6)])
        s = O.solve_step(Hs, bb, 1e-3, 100.0, 100.0)
        assert np.linalg.norm((Hs + 1e-3 * np.eye(6)) @ s + bb) < 1e-9
    s = O.solve_step(np.eye(6), [3, -3, 3, 5, -5, 5], 0.0)
    assert np.allclose(np.abs(s[:3]), 0.5) and np.allclose(np.abs(s[3:]), 1.0)
    b = np.zeros(6)
    b[0] = 1.0
    assert np.linalg.norm(O.solve_step(np.zeros((6, 6)), b, 0.0)) == 0.0
    with pytest.raises(ValueError):
        O.solve_step(np.eye(6), b, -1.0)


# ---------------------------------------------------------------- GICP (test_gicp.cpp)
def sparse_grid_cloud(per_axis, seed, sigma_iso=1e-4):  # test_gicp.cpp:24-44
    rng = O.SplitMix64(seed)
    pts = []
    for x in range(per_axis):
        for y in range(per_axis):
            for z in range(per_axis):
                pts.append([x * 0.4 + rng.uniform_range(-0.01, 0.01), y * 0.4 + rng.uniform_range(-0.01, 0.01),
                            z * 0.4 + rng.uniform_range(-0.01, 0.01)])
    mu = np.array(pts)
    sig = np.tile((sigma_iso * np.eye(3)).reshape(9), (len(mu), 1))
    return mu, sig


def test_gicp_zero_residual_and_offset_recovery():
    mu, sig = sparse_grid_cloud(7, 1)
    om = O.OracleMap(mu, sig, None, 0.1, 0.5, 1.0)
    steps, ll, nm, H, b = O.evaluate_all(om, mu, sig, [I12], make_config(min_match_fraction=0.0, miss_cost=0.0),
                                         want_system=True)
    assert nm[0] == len(mu) and ll[0] == 0.0 and np.linalg.norm(b[0]) == 0.0
    mu, sig = sparse_grid_cloud(7, 3)
    om = O.OracleMap(mu, sig, None, 0.1, 0.5, 1.0)
    off = I12.copy()
    off[9] = 0.05
    steps, ll, nm, H, b = O.evaluate_all(om, mu, sig, [off], make_config(), want_system=True)
    assert nm[0] > 300
    s = O.solve_step(H[0], b[0], 1e-3 * np.trace(H[0]) / 6.0)
    assert np.linalg.norm(s[3:] - [-0.05, 0, 0]) < 1e-3


def test_gicp_unmatched_sentinel():
    rng = O.SplitMix64(51)
    mu = np.array([[rng.uniform_range(0, 2) for _ in range(3)] for _ in range(100)])
    sig = np.tile((1e-4 * np.eye(3)).reshape(9), (100, 1))
    om = O.OracleMap(mu, sig, None, 0.1, 0.5, 1.0)
    far = I12.copy()
    far[9] = 500.0
    steps, ll, nm, H, b = O.evaluate_all(om, mu, sig, [far], make_config(), want_system=True)
    assert nm[0] == 0 and ll[0] == -1e30 and np.all(H[0] == 0) and np.all(b[0] == 0)


def test_gicp_descent_in_basin():
    rects = sim.box_room([8.0, 6.0, 3.0])
    mapc = sim.sample_world(rects, 80.0, 23)
    truth = I12.copy()
    truth[9:] = [4.0, 3.0, 1.5]
    pts, _ = sim.simulate_scan_points(rects, truth, sim.sensor_spec(noise_sigma=0.0), O.mix_seed(23, 7))
    ssig = O.estimate_covariances(pts, 10)
    om = O.OracleMap(mapc.mu, mapc.sigma, None, 0.1, 0.5, 1.0)
    rng = O.SplitMix64(29)
    starts = []
    for _ in range(100):
        axis = np.array([rng.normal01(), rng.normal01(), rng.normal01()])
        axis /= np.linalg.norm(axis)
        xi = np.zeros(6)
        xi[:3] = axis * rng.uniform_range(0.0, 10.0 * math.pi / 180.0)
        for a in range(3):
            xi[3 + a] = rng.uniform_range(-0.2, 0.2)
        starts.append(O.compose(truth, O.se3_exp(xi)[0]))
    starts = np.array(starts)
    cfg = make_config(min_match_fraction=0.0, miss_cost=0.0)
    steps, ll0, nm0 = O.evaluate_all(om, pts, ssig, starts, cfg)
    moved = np.array([O.compose(s, O.se3_exp(st)[0]) for s, st in zip(starts, steps)])
    ll1, _ = O.evaluate_likelihoods(om, pts, ssig, moved, cfg)
    improved = np.sum((ll1 > ll0) & (nm0 > 0))
    assert improved >= 0.95 * np.sum(nm0 > 0)


def test_parallel_equals_serial_bitwise():
    """test_parallel_consistency.cpp:86-95: OpenMP oracle == serial twin."""
    from helpers import cube_set
    rects, mapc, scan = room_scene()
    parts = cube_set(300, 7, 20)
    om = O.OracleMap(mapc.mu, mapc.sigma, None, 0.2, 0.5, 1.0)
    a = O.evaluate_all(om, scan.mu, scan.sigma, parts.poses, make_config(), serial=False)
    b = O.evaluate_all(om, scan.mu, scan.sigma, parts.poses, make_config(), serial=True)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


# ---------------------------------------------------------------- posterior (test_posterior.cpp)
def lse(v):
    m = np.max(v)
    return m + math.log(np.sum(np.exp(v - m)))


def test_bayes_uniform_and_ratio():
    post, rej = O.bayes_update(np.full(64, -math.log(64)), np.full(64, -12.5), np.full(64, 40), 2.0)
    assert not rej and np.allclose(post, -math.log(64), rtol=1e-12) and abs(lse(post)) < 1e-9
    post, _ = O.bayes_update(np.full(2, -math.log(2)), [0.0, -1.7], [1, 1], 1.0)
    assert abs((post[0] - post[1]) - 1.7) < 1e-12
    post, _ = O.bayes_update(np.full(2, -math.log(2)), [-10.0, -10.0], [10, 5], 1.0)
    assert abs((post[0] - post[1]) - 1.0) < 1e-12


def test_bayes_beta_zero_and_rejection():
    p0 = O.normalize_log_post([-0.5, -2.0, -1.2])
    post, _ = O.bayes_update(p0, [-5.0, -50.0, -2.0], [3, 3, 3], 0.0)
    assert np.allclose(post, p0, rtol=1e-12)
    p0 = O.normalize_log_post([-0.1, -3.0, -2.0, -5.0])
    post, rej = O.bayes_update(p0, np.full(4, -1e30), np.zeros(4, np.int32), 2.0)
    assert rej and np.allclose(post, -math.log(4), rtol=1e-12)


def full_graph(n, kv):
    idx = np.full((n, n), -1, np.int32)
    kval = np.zeros((n, n), np.float32)
    for i in range(n):
        idx[i] = [i] + [j for j in range(n) if j != i]
        kval[i] = [1.0] + [kv] * (n - 1)
    return idx, kval, np.full(n, n, np.int32)


def test_smooth_fixed_points():
    p0 = O.normalize_log_post([-0.2, -1.0, -2.5, -3.0, -4.0])
    idx = np.full((5, 4), -1, np.int32)
    idx[:, 0] = np.arange(5)
    kv = np.zeros((5, 4), np.float32)
    kv[:, 0] = 1.0
    assert np.allclose(O.smooth(p0, idx, kv, np.ones(5, np.int32), 7), p0, rtol=1e-12)
    idx, kv, cnt = full_graph(16, 0.37)
    out = O.smooth(np.full(16, -math.log(16)), idx, kv, cnt, 10)
    assert np.allclose(out, -math.log(16), rtol=1e-12)
    idx, kv, cnt = full_graph(3, 1.0)
    out = O.smooth([0.0, -80.0, -80.0], idx, kv, cnt, 1)
    assert np.allclose(np.exp(out), 1.0 / 3.0, rtol=1e-12)


def test_representative_ties():
    assert O.representative([-3.0, -1.0, -2.0, -1.0, -1.0, -4.0])[0] == 1
    assert O.representative([math.log(0.1), math.log(0.7), math.log(0.2)])[0] == 1


def test_normalization_after_operations():
    rng = O.SplitMix64(33)
    post = O.normalize_log_post([rng.uniform_range(-40.0, 0.0) for _ in range(500)])
    assert abs(lse(post)) < 1e-9
    lik = [rng.uniform_range(-500.0, 0.0) for _ in range(500)]
    nm = [1 + rng() % 60 for _ in range(500)]
    post, _ = O.bayes_update(post, lik, nm, 2.0)
    assert abs(lse(post)) < 1e-9
    idx, kv, cnt = full_graph(32, 0.5)
    p32 = O.smooth(O.normalize_log_post(post[:32]), idx, kv, cnt, 10)
    assert abs(lse(p32)) < 1e-9 and np.all(p32 >= -80.0)
