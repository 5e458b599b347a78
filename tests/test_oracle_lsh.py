"""The reference's own LSH / neighbour-graph and GICP Jacobian fixtures,
ported line by line against the oracle (CPU, no GPU needed).

* proj/tests/test_neighbor_search.cpp:55-63    lsh_hash is deterministic
* proj/tests/test_neighbor_search.cpp:65-107   near poses collide, far poses do not
* proj/tests/test_neighbor_search.cpp:109-136  random_lsh_frame properties (+ octant chi^2)
* proj/tests/test_neighbor_search.cpp:139-149  a lone particle keeps a self-only list
* proj/tests/test_neighbor_search.cpp:151-181  widely separated particles: pure GN updates
* proj/tests/test_neighbor_search.cpp:183-202  offer known answer {0, 5, 9}, never evicts self
* proj/tests/test_neighbor_search.cpp:204-236  iterative search approaches brute-force kNN
* proj/tests/test_neighbor_search.cpp:238-263  passes deterministic, equal to the serial twin
* proj/tests/test_neighbor_search.cpp:265-276  stats are coherent
* proj/tests/test_gicp.cpp:104-128             analytic Jacobian vs central finite differences
* proj/tests/test_gicp.cpp:196-224             log-likelihood invariant under a joint rigid transform

Random streams are the reference's (SplitMix64 seeds of each TEST_CASE, the
same draw order), through the oracle's rng.hpp restatement.
"""
import math

import numpy as np

import oracle as O
from helpers import random_cube_set, random_pose, random_tangent
from paper_2404_16370_b200.abi import Particles, identity_pose, make_config

SR, ST = 5.0, 2.5  # KernelParams defaults (svgd.hpp:13-15)
ALPHA, NOISE = 0.1, 0.5  # LshConfig defaults (neighbor_search.hpp:13-21)


def W():  # KernelParams::weights() (svgd.hpp:23-27)
    return np.array([SR, SR, SR, ST, ST, ST])


def hash_of(pose, frame, noise):
    return O.lsh_hash(pose, frame, noise, ALPHA, SR, ST)


def zeta(pose, frame, noise):
    return ALPHA * W() * O.se3_log(O.compose(O.inverse(frame), pose))[0] + noise


def test_lsh_hash_is_deterministic():  # :55-63
    rng = O.SplitMix64(3)
    p = random_pose(rng)
    frame = random_pose(rng)
    noise = 0.5 * rng.normal6()
    assert hash_of(p, frame, noise) == hash_of(p, frame, noise)


def test_near_poses_collide_far_poses_do_not():  # :65-107
    rng = O.SplitMix64(5)
    n_buckets = 509
    w = ALPHA * W()
    box = [-5.0, -5.0, -5.0, 5.0, 5.0, 5.0]
    near_col = near_tr = far_col = far_tr = 0
    for _ in range(10000):
        frame = rng.random_lsh_frame(box)
        noise = NOISE * rng.normal6()  # one draw per frame
        a = random_pose(rng, 1.5, 4.0)
        budget = rng.uniform_range(0.0, 0.1)
        dz = np.array([rng.uniform_range(-1.0, 1.0) for _ in range(6)])
        dz *= budget / np.abs(dz).sum()
        b = O.compose(a, O.se3_exp(dz / w)[0])
        ha = hash_of(a, frame, noise) % n_buckets
        hb = hash_of(b, frame, noise) % n_buckets
        if np.abs(zeta(a, frame, noise) - zeta(b, frame, noise)).sum() < 0.1:
            near_tr += 1
            near_col += int(ha == hb)
        c = a.copy()
        c[9:] += [50.0, -30.0, 40.0]  # far beyond one cell
        hc = hash_of(c, frame, noise) % n_buckets
        far_tr += 1
        far_col += int(ha == hc)
    assert near_tr > 5000
    assert near_col / near_tr > 0.9
    assert far_col / far_tr <= 2.0 / n_buckets + 0.01


def test_random_lsh_frame_properties():  # :109-136
    box = [-2.0, -3.0, 0.0, 2.0, 3.0, 1.0]
    fa = O.SplitMix64(1).random_lsh_frame(box)
    fb = O.SplitMix64(2).random_lsh_frame(box)
    assert np.abs(fa[:9] - fb[:9]).max() > 1e-6
    assert O.rotation_drift(fa) < 1e-12
    assert abs(np.linalg.det(fa[:9].reshape(3, 3)) - 1.0) <= 1e-12
    assert all(box[a] <= fa[9 + a] <= box[3 + a] for a in range(3))
    # Rotation-axis octant uniformity, chi^2 at the 1 % level (7 dof). The
    # axis of AngleAxisd(R) (angle in [0, pi]) has the signs of
    # (R21 - R12, R02 - R20, R10 - R01) = 2 sin(theta) axis.
    rng = O.SplitMix64(7)
    counts = np.zeros(8)
    n = 10000
    for _ in range(n):
        R = rng.random_lsh_frame(box)[:9].reshape(3, 3)
        ax = (R[2, 1] - R[1, 2], R[0, 2] - R[2, 0], R[1, 0] - R[0, 1])
        counts[(ax[0] > 0) | ((ax[1] > 0) << 1) | ((ax[2] > 0) << 2)] += 1
    chi2 = (((counts - n / 8) ** 2) / (n / 8)).sum()
    assert chi2 < 18.475


def test_lone_particle_keeps_self_only_list():  # :139-149
    s = random_cube_set(1, 1.0, 0.1, 20, 3)
    cfg = make_config()
    for p in range(5):
        O.update_neighbors(s, cfg, O.mix_seed(11, p), [0.0, 0.0, 0.0, 1.0, 1.0, 1.0])
    assert s.count[0] == 1 and s.idx[0, 0] == 0


def check_list_invariants(s):  # :39-51
    for i in range(s.n):
        nb = s.idx[i, : s.count[i]]
        assert len(set(nb.tolist())) == len(nb)
        assert i in nb
        assert s.count[i] <= s.k


def test_widely_separated_particles_pure_gn_updates():  # :151-181
    n = 100
    poses = np.tile(identity_pose(), (n, 1))
    poses[:, 9] = 10.0 * np.arange(n)
    s = Particles.from_poses(poses, 5)
    cfg = make_config(k_neighbors=5)
    bounds = [0.0, 0.0, 0.0, 1000.0, 1.0, 1.0]
    for p in range(5):
        O.update_neighbors(s, cfg, O.mix_seed(13, p), bounds)
    check_list_invariants(s)
    for i in range(n):
        for q in range(s.count[i]):
            if s.idx[i, q] != i:
                assert s.kval[i, q] < 1e-10
    rng = O.SplitMix64(15)
    steps = np.array([random_tangent(rng, 0.2, 0.3) for _ in range(n)])
    phis = O.compute_phis(s.poses, steps, s.idx, s.count, cfg)
    assert np.linalg.norm(phis - steps, axis=1).max() < 1e-9


def test_offer_known_answer_never_evicts_self():  # :183-202
    idx, kv = O.graph_offers(3, [(5, 0.5), (7, 0.2)])
    assert len(idx) == 3
    idx, kv = O.graph_offers(3, [(5, 0.5), (7, 0.2), (9, 0.4)])  # evicts 7 (weakest non-self)
    assert set(idx.tolist()) == {0, 5, 9}
    idx, kv = O.graph_offers(3, [(5, 0.5), (7, 0.2), (9, 0.4), (11, 0.1)])  # weaker than all: dropped
    assert set(idx.tolist()) == {0, 5, 9}
    idx, kv = O.graph_offers(3, [(5, 0.5), (7, 0.2), (9, 0.4), (11, 0.1), (5, 0.9)])  # duplicate: ignored
    assert len(idx) == 3 and set(idx.tolist()) == {0, 5, 9}
    idx, kv = O.graph_offers(3, [(5, 0.5), (7, 0.2), (9, 0.4), (11, 0.1), (5, 0.9), (13, 0.99)])
    assert (idx == 0).sum() == 1  # self survives even when every other entry is stronger
    assert kv[idx.tolist().index(0)] == 1.0


def test_iterative_search_approaches_brute_force_knn():  # :204-236
    k = 10
    s = random_cube_set(300, 8.0, 0.2, k, 17)
    cfg = make_config(k_neighbors=k)
    truth = O.brute_force_kernel_knn(s.poses, k, SR, ST)
    for p in range(10):
        O.update_neighbors(s, cfg, O.mix_seed(19, p), [0.0] * 3 + [8.0] * 3)
    check_list_invariants(s)
    slot_of_id = np.empty(s.n, np.int64)
    slot_of_id[s.id] = np.arange(s.n)
    hit = total = 0
    for orig in range(s.n):
        slot = slot_of_id[orig]
        got = {int(s.id[j]) for j in s.idx[slot, : s.count[slot]]}
        for want in truth[orig]:
            if want < 0:
                continue
            total += 1
            hit += int(want in got)
    assert hit / total > 0.6


def test_passes_deterministic_and_match_serial_twin():  # :238-263
    cfg = make_config()
    bounds = [0.0] * 3 + [6.0] * 3
    a = random_cube_set(500, 6.0, 0.3, 20, 23)
    b = random_cube_set(500, 6.0, 0.3, 20, 23)
    c = random_cube_set(500, 6.0, 0.3, 20, 23)
    for p in range(4):
        seed = O.mix_seed(29, p)
        O.update_neighbors(a, cfg, seed, bounds)
        O.update_neighbors(b, cfg, seed, bounds)
        O.update_neighbors(c, cfg, seed, bounds, serial=True)
    for x in (b, c):
        assert np.array_equal(a.id, x.id)
        assert np.array_equal(a.idx, x.idx)
        assert np.array_equal(a.kval, x.kval)
    assert np.array_equal(a.poses[:, 9:], c.poses[:, 9:])


def test_stats_are_coherent():  # :265-276
    s = random_cube_set(400, 5.0, 0.2, 20, 31)
    st = O.update_neighbors(s, make_config(), 37, [0.0] * 3 + [5.0] * 3)
    assert st["n_buckets"] >= 800
    assert st["buckets_used"] > 0
    assert st["overflow_dropped"] >= 0
    assert 0.0 <= st["mean_kernel"] <= 1.0


def apply(pose, x):
    return pose[:9].reshape(3, 3) @ x + pose[9:]


def skew(v):
    return np.array([[0.0, -v[2], v[1]], [v[2], 0.0, -v[0]], [-v[1], v[0], 0.0]])


def test_gicp_jacobian_matches_central_differences():  # test_gicp.cpp:104-128
    rng = O.SplitMix64(17)
    h = 1e-6
    for _ in range(20):
        pose = random_pose(rng, 2.5, 3.0)
        mu_s = np.array([rng.uniform_range(-2.0, 2.0) for _ in range(3)])
        mu_m = np.array([rng.uniform_range(-2.0, 2.0) for _ in range(3)])
        R = pose[:9].reshape(3, 3)
        jac = np.hstack([R @ skew(mu_s), -R])  # J = [R [mu_s]x | -R]
        for c in range(6):
            plus, minus = np.zeros(6), np.zeros(6)
            plus[c], minus[c] = h, -h
            ep = mu_m - apply(O.compose(pose, O.se3_exp(plus)[0]), mu_s)
            em = mu_m - apply(O.compose(pose, O.se3_exp(minus)[0]), mu_s)
            fd = (ep - em) / (2.0 * h)
            assert np.abs(jac[:, c] - fd).max() < 1e-5


def random_cloud(n, seed, sigma_iso):  # test_gicp.cpp:13-22
    rng = O.SplitMix64(seed)
    mu = np.array([[rng.uniform_range(0.0, 2.0) for _ in range(3)] for _ in range(n)])
    return mu, np.tile((sigma_iso * np.eye(3)).reshape(9), (n, 1))


def test_gicp_loglik_invariant_under_joint_rigid_transform():  # test_gicp.cpp:196-224
    rng = O.SplitMix64(31)
    map_mu, map_sig = random_cloud(100, 37, 1e-3)
    scan_mu, scan_sig = random_cloud(40, 41, 1e-3)
    pose = random_pose(rng, 0.5, 1.0)
    g = random_pose(rng, 2.0, 5.0)

    def pinned_loglik(mmu, msig, t):  # pinned correspondences k -> k % |map|
        R = t[:9].reshape(3, 3)
        ll = 0.0
        for k in range(len(scan_mu)):
            j = k % len(mmu)
            e = mmu[j] - apply(t, scan_mu[k])
            om = np.linalg.inv(msig[j].reshape(3, 3) + R @ scan_sig[k].reshape(3, 3) @ R.T)
            ll -= e @ om @ e
        return ll

    Rg = g[:9].reshape(3, 3)
    mmu_g = np.array([apply(g, m) for m in map_mu])
    msig_g = np.array([(Rg @ s.reshape(3, 3) @ Rg.T).reshape(9) for s in map_sig])
    a = pinned_loglik(map_mu, map_sig, pose)
    b = pinned_loglik(mmu_g, msig_g, O.compose(g, pose))
    assert abs(a - b) <= 1e-9 * abs(b)
