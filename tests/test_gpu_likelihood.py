"""GPU parity of K1/K2 (GICP likelihood + Gauss-Newton) against the CPU oracle.

Reference: gicp.cpp:11-137; pinned fixtures: test_parallel_consistency.cpp:31-95
(box room 8x6x3, density 60, NNF 0.2, 700 particles, seeds 3/5/7).

* exact mode (likelihood_mode=1) must equal the oracle bit for bit;
* fast mode (structured fp32 Woodbury algebra) must match n_matched exactly
  and ll/H/b/steps within the tolerances stated below.
"""
import numpy as np
import pytest

import oracle as O
from helpers import config, cube_set, room_scene
from paper_2404_16370_b200.api import FilterEngine, GaussianCloud

pytestmark = pytest.mark.gpu

# Fast-path tolerances (fp32 per-point algebra, fp32 per-lane accumulation).
TOL_LL = 2e-5      # |ll - ll_ref| / |ll_ref|
TOL_SYS = 2e-5     # ||H - H_ref||_F / ||H_ref||_F, same for b (normwise)
TOL_STEP = 1e-4    # ||(H_ref + lam I) step + b_ref|| / ||b_ref||  (backward error of the solve)


@pytest.fixture(scope="module")
def scene():
    rects, mapc, scan = room_scene()
    parts = cube_set(700, 7, 20)
    om = O.OracleMap(mapc.mu, mapc.sigma, mapc.bounds, 0.2, 0.5, 1.0)
    return mapc, scan, parts, om


def _engine(mapc, parts, mode):
    e = FilterEngine(mapc, config(nnf_resolution=0.2, likelihood_mode=mode))
    e.set_particles(parts)
    return e


def test_nnf_matches_oracle(scene):
    mapc, scan, parts, om = scene
    e = _engine(mapc, parts, 1)
    d, o, res, cells = e.nnf()
    d2, o2, c2 = om.nnf()
    assert np.array_equal(d, d2) and np.array_equal(o, o2) and np.array_equal(cells, c2)


def test_evaluate_all_exact_is_bitwise(scene):
    mapc, scan, parts, om = scene
    e = _engine(mapc, parts, 1)
    steps, ll, nm, H, b = e.evaluate_all(scan, want_system=True)
    s2, ll2, nm2, H2, b2 = O.evaluate_all(om, scan.mu, scan.sigma, parts.poses, config(), want_system=True)
    assert np.array_equal(nm, nm2)
    assert (nm > 0).sum() > 100
    assert np.array_equal(ll, ll2)
    m = nm > 0
    assert np.array_equal(H[m], H2[m])
    assert np.array_equal(b[m], b2[m])
    assert np.array_equal(steps, s2)


def test_evaluate_likelihoods_exact_is_bitwise(scene):
    mapc, scan, parts, om = scene
    e = _engine(mapc, parts, 1)
    ll, nm = e.evaluate_likelihoods(scan)
    ll2, nm2 = O.evaluate_likelihoods(om, scan.mu, scan.sigma, parts.poses, config())
    assert np.array_equal(nm, nm2)
    assert np.array_equal(ll, ll2)


def _lower(H):
    return np.tril(H)


def test_evaluate_all_fast_within_tolerance(scene):
    mapc, scan, parts, om = scene
    e = _engine(mapc, parts, 2)
    steps, ll, nm, H, b = e.evaluate_all(scan, want_system=True)
    s2, ll2, nm2, H2, b2 = O.evaluate_all(om, scan.mu, scan.sigma, parts.poses, config(), want_system=True)
    assert np.array_equal(nm, nm2)
    m = ll2 > -1e29
    assert m.sum() > 50
    assert np.array_equal(ll[~m], ll2[~m])
    rel_ll = np.abs(ll[m] - ll2[m]) / np.abs(ll2[m])
    k = nm2 > 0
    Hl, Hl2 = np.array([_lower(h) for h in H[k]]), np.array([_lower(h) for h in H2[k]])
    rel_H = np.linalg.norm((Hl - Hl2).reshape(k.sum(), -1), axis=1) / np.linalg.norm(Hl2.reshape(k.sum(), -1), axis=1)
    rel_b = np.linalg.norm(b[k] - b2[k], axis=1) / np.maximum(np.linalg.norm(b2[k], axis=1), 1e-300)
    print(f"fast GN: max rel ll {rel_ll.max():.2e}, H {rel_H.max():.2e}, b {rel_b.max():.2e}")
    assert rel_ll.max() < TOL_LL
    assert rel_H.max() < TOL_SYS
    assert rel_b.max() < TOL_SYS
    # Step: backward error against the oracle's own damped system, for
    # unclamped steps (clamping is a non-smooth projection).
    bad = 0
    for i in np.nonzero(k)[0]:
        Hs = H2[i]
        lam = 1e-3 * np.trace(Hs) / 6.0
        clamped = (np.abs(s2[i][:3]) >= 0.5).any() or (np.abs(s2[i][3:]) >= 1.0).any()
        if clamped:
            continue
        r = (Hs + lam * np.eye(6)) @ steps[i] + b2[i]
        if np.linalg.norm(r) > TOL_STEP * np.linalg.norm(b2[i]):
            bad += 1
    assert bad == 0


def test_evaluate_likelihoods_fast_within_tolerance(scene):
    mapc, scan, parts, om = scene
    e = _engine(mapc, parts, 2)
    ll, nm = e.evaluate_likelihoods(scan)
    ll2, nm2 = O.evaluate_likelihoods(om, scan.mu, scan.sigma, parts.poses, config())
    assert np.array_equal(nm, nm2)
    m = ll2 > -1e29
    assert np.array_equal(ll[~m], ll2[~m])
    rel = np.abs(ll[m] - ll2[m]) / np.abs(ll2[m])
    print(f"fast LL: max rel {rel.max():.2e}")
    assert rel.max() < TOL_LL


def test_unstructured_map_falls_back_to_exact(scene):
    """A map whose covariances are not plane-model cannot use the fast
    records; auto mode must use the exact kernels (and fast mode must refuse)."""
    mapc, scan, parts, om = scene
    rng = np.random.default_rng(0)
    sig = mapc.sigma.reshape(-1, 3, 3).copy()
    for i in range(len(sig)):
        d = np.diag(rng.uniform(1e-4, 3e-3, 3))
        sig[i] = d
    m2 = GaussianCloud(mapc.mu, sig.reshape(-1, 9), mapc.bounds)
    e = FilterEngine(m2, config(nnf_resolution=0.2, likelihood_mode=0))
    e.set_particles(parts)
    ll, nm = e.evaluate_likelihoods(scan)
    om2 = O.OracleMap(m2.mu, m2.sigma, m2.bounds, 0.2, 0.5, 1.0)
    ll2, nm2 = O.evaluate_likelihoods(om2, scan.mu, scan.sigma, parts.poses, config())
    assert np.array_equal(ll, ll2) and np.array_equal(nm, nm2)
    e2 = FilterEngine(m2, config(nnf_resolution=0.2, likelihood_mode=2))
    e2.set_particles(parts)
    with pytest.raises(ValueError):
        e2.evaluate_likelihoods(scan)


def test_empty_scan_rejected(scene):
    mapc, scan, parts, om = scene
    e = _engine(mapc, parts, 0)
    with pytest.raises(ValueError):
        e.evaluate_all(GaussianCloud(np.zeros((0, 3)), np.zeros((0, 9))))


@pytest.mark.parametrize("S", [1, 7, 33, 129, 1100])
def test_fast_paths_ragged_scan_sizes(scene, S):
    """Scan sizes off the kernels' step multiples (1 point, partial warps,
    one past a step, beyond the lane kernel's two-CTA limit) and particles far
    outside the map: n_matched exact, ll within tolerance, gating exact."""
    mapc, scan, parts, om = scene
    idx = np.arange(S) % len(scan)
    sc = GaussianCloud(scan.mu[idx], scan.sigma[idx])
    p = parts.copy() if hasattr(parts, "copy") else parts
    poses = p.poses.copy()
    poses[:50, 9] += 500.0  # every point out of bounds: n = 0, ll = -1e30
    from paper_2404_16370_b200.abi import Particles
    q = Particles.from_poses(poses, p.k)
    for gn in (False, True):
        e = _engine(mapc, q, 2)
        if gn:
            _, ll, nm = e.evaluate_all(sc)
            _, ll2, nm2 = O.evaluate_all(om, sc.mu, sc.sigma, poses, config())
        else:
            ll, nm = e.evaluate_likelihoods(sc)
            ll2, nm2 = O.evaluate_likelihoods(om, sc.mu, sc.sigma, poses, config())
        assert np.array_equal(nm, nm2)
        assert np.all(nm[:50] == 0) and np.all(ll[:50] == -1e30)
        m = ll2 > -1e29
        assert np.array_equal(ll[~m], ll2[~m])
        if m.any():
            assert np.all(np.abs(ll[m] - ll2[m]) <= TOL_LL * np.abs(ll2[m]))


@pytest.mark.parametrize("offset", [2.0e4, 3.0e6])
def test_fast_paths_far_from_origin(scene, offset):
    """The same room and particles translated far from the origin (e.g. a map
    in UTM coordinates): the reference's world-frame rounding grows with |t|,
    so the fast kernels must still pick the reference's cells (n_matched exact)
    — at 3e6 m every point takes the resolve path."""
    mapc, scan, parts, om = scene
    from paper_2404_16370_b200.abi import Particles
    m2 = GaussianCloud(mapc.mu + offset, mapc.sigma, mapc.bounds + offset)
    om2 = O.OracleMap(m2.mu, m2.sigma, m2.bounds, 0.2, 0.5, 1.0)
    poses = parts.poses.copy()
    poses[:, 9:] += offset
    q = Particles.from_poses(poses, parts.k)
    e = FilterEngine(m2, config(nnf_resolution=0.2, likelihood_mode=2))
    e.set_particles(q)
    ll, nm = e.evaluate_likelihoods(scan)
    ll2, nm2 = O.evaluate_likelihoods(om2, scan.mu, scan.sigma, poses, config())
    assert np.array_equal(nm, nm2) and (nm > 0).sum() > 100
    _, llg, nmg = e.evaluate_all(scan)
    _, llg2, nmg2 = O.evaluate_all(om2, scan.mu, scan.sigma, poses, config())
    assert np.array_equal(nmg, nmg2)
    m = ll2 > -1e29
    assert np.all(np.abs(ll[m] - ll2[m]) <= TOL_LL * np.abs(ll2[m]))


def test_fast_paths_points_on_cell_faces(scene):
    """Points placed on (or within 1e-15 .. 1e-4 voxel of) NNF cell faces: the
    scan is snapped to a lattice of res/4, rotations are exact multiples of
    90 degrees and translations are whole cells plus a small offset, so a
    quarter of the coordinates per axis land on a face. The fast kernels' cell
    decisions (K1's and K2's fixed-point split, K2a's fp32 count with its
    proven margin) must fall back to the reference-order transform there:
    n_matched exact for both passes, ll within tolerance (nnf.hpp:24-35)."""
    mapc, scan, parts, om = scene
    from paper_2404_16370_b200.abi import Particles
    e0 = FilterEngine(mapc, config(nnf_resolution=0.2, likelihood_mode=2))
    d, o, res, _ = e0.nnf()
    q = res / 4.0
    mu = np.round(scan.mu / q) * q
    sc = GaussianCloud(mu, scan.sigma)
    rots = [np.eye(3),
            np.array([[0., -1, 0], [1, 0, 0], [0, 0, 1]]),
            np.array([[-1., 0, 0], [0, -1, 0], [0, 0, 1]]),
            np.array([[1., 0, 0], [0, 0, -1], [0, 1, 0]]),
            np.array([[0., 0, 1], [0, 1, 0], [-1, 0, 0]])]
    deltas = [0.0, 1e-15, -1e-15, 1e-12, -1e-12, 1e-9, -1e-9, 2e-8, -2e-8, 6e-8, -6e-8, 1e-7, -1e-7,
              1e-6, -1e-6, 1e-5, -1e-5, 1e-4, -1e-4, 0.5]
    rng = np.random.default_rng(11)
    poses = []
    for R in rots:
        for dl in deltas:
            for _ in range(8):
                cell = np.array([rng.integers(int(0.2 * d[a]), int(0.8 * d[a])) for a in range(3)], float)
                t = np.asarray(o) + res * cell + dl * res
                poses.append(np.concatenate([R.reshape(-1), t]))
    poses = np.array(poses)
    e = FilterEngine(mapc, config(nnf_resolution=0.2, likelihood_mode=2))
    e.set_particles(Particles.from_poses(poses, 20))
    ll, nm = e.evaluate_likelihoods(sc)
    ll2, nm2 = O.evaluate_likelihoods(om, sc.mu, sc.sigma, poses, config())
    assert (nm2 > 0).sum() > 200
    assert np.array_equal(nm, nm2)
    m = ll2 > -1e29
    assert np.all(np.abs(ll[m] - ll2[m]) <= TOL_LL * np.abs(ll2[m]))
    _, llg, nmg = e.evaluate_all(sc)
    _, llg2, nmg2 = O.evaluate_all(om, sc.mu, sc.sigma, poses, config())
    assert np.array_equal(nmg, nmg2)
