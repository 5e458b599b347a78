"""Whole-step GPU parity: FilterEngine::step (filter.cpp:118-213) on the B200
against the oracle's FilterEngine, plus the reference's filter-level
behaviour tests (test_filter.cpp:136-304)."""
import math

import numpy as np
import pytest

import oracle as O
from paper_2404_16370_b200 import sim
from paper_2404_16370_b200.abi import identity_pose, make_config
from paper_2404_16370_b200.api import FilterEngine, GaussianCloud, make_scan_cloud

pytestmark = pytest.mark.gpu
I12 = identity_pose()


class SmallWorld:  # test_filter.cpp:21-37
    def __init__(self):
        self.rects = sim.box_room([10.0, 8.0, 3.0])
        self.map = sim.sample_world(self.rects, 60.0, 5)
        self.sensor = sim.sensor_spec(noise_sigma=0.0)

    def scan_at(self, pose, cfg, seed=9):
        pts, _ = sim.simulate_scan_points(self.rects, pose, self.sensor, seed)
        return make_scan_cloud(pts, cfg)


@pytest.fixture(scope="module")
def world():
    return SmallWorld()


def run_frames(world, cfg, n_frames, oracle=False, base_seed=100):
    eng = (O.FilterEngine(world.map.mu, world.map.sigma, cfg, world.map.bounds) if oracle
           else FilterEngine(world.map, cfg))
    eng.init_uniform(world.map.bounds)
    gt = I12.copy()
    gt[9:] = [5.0, 4.0, 1.5]
    delta = I12.copy()
    delta[9] = 0.05
    cov = np.diag([1e-4] * 6).reshape(36)
    frames = []
    for f in range(n_frames):
        gt = sim.compose(gt, delta)
        scan = world.scan_at(gt, cfg, base_seed + f)
        if oracle:
            frames.append(eng.step(scan.mu, scan.sigma, delta, cov, True))
        else:
            frames.append(eng.step(scan, delta, cov, True))
    return eng, frames


def test_step_exact_mode_matches_oracle(world):
    cfg = make_config(n_particles=500, seed=42, nnf_resolution=0.2, likelihood_mode=1)
    g, fg = run_frames(world, cfg, 6)
    r, fr = run_frames(world, cfg, 6, oracle=True)
    for a, b in zip(fg, fr):
        assert a["rep_id"] == b["rep_id"] and a["rep_index"] == b["rep_index"]
        assert a["observation_rejected"] == b["observation_rejected"]
        assert abs(a["mean_n_matched"] - b["mean_n_matched"]) == 0.0
        assert abs(a["rep_log_post"] - b["rep_log_post"]) < 1e-9
        assert np.abs(a["representative"] - b["representative"]).max() < 1e-9
        assert a["neighbor_stats"]["buckets_used"] == b["neighbor_stats"]["buckets_used"]
    pg, pr = g.particles(), r.particles()
    assert np.array_equal(pg.id, pr.id)
    assert np.array_equal(pg.idx, pr.idx) and np.array_equal(pg.count, pr.count)
    assert np.abs(pg.poses - pr.poses).max() < 1e-9
    assert np.abs(pg.log_post - pr.log_post).max() < 1e-9


def test_step_fast_mode_tracks_oracle(world):
    cfg = make_config(n_particles=500, seed=42, nnf_resolution=0.2, likelihood_mode=2)
    g, fg = run_frames(world, cfg, 6)
    r, fr = run_frames(world, cfg, 6, oracle=True)
    same = sum(a["rep_id"] == b["rep_id"] for a, b in zip(fg, fr))
    assert same >= 5
    pg, pr = g.particles(), r.particles()
    assert np.mean(pg.id == pr.id) > 0.99
    m = pg.id == pr.id
    assert np.median(np.abs(pg.poses[m] - pr.poses[m]).max(1)) < 1e-6


def test_replay_is_bit_identical(world):
    cfg = make_config(n_particles=500, seed=42, nnf_resolution=0.2)
    a, fa = run_frames(world, cfg, 5)
    b, fb = run_frames(world, cfg, 5)
    pa, pb = a.particles(), b.particles()
    assert np.array_equal(pa.poses, pb.poses) and np.array_equal(pa.log_post, pb.log_post)
    assert np.array_equal(pa.idx, pb.idx) and np.array_equal(pa.kval, pb.kval)
    for x, y in zip(fa, fb):
        assert x["rep_id"] == y["rep_id"] and x["rep_log_post"] == y["rep_log_post"]


def test_empty_scans_diffuse(world):
    cfg = make_config(n_particles=2000, seed=42, nnf_resolution=0.2)
    e = FilterEngine(world.map, cfg)
    e.init_uniform([4.0, 3.0, 1.0, 6.0, 5.0, 2.0])

    def spread():
        t = e.particles().poses[:, 9:]
        return np.mean(np.sum((t - t.mean(0)) ** 2, 1))

    prev = spread()
    for _ in range(8):
        res = e.step(None, valid=False)
        assert res["scan_empty"] == 1
        cur = spread()
        assert cur > prev
        prev = cur


def test_single_particle_tracks_truth():
    """test_filter.cpp:201-251."""
    rng = O.SplitMix64(55)
    pts = []
    for x in range(20):
        for y in range(16):
            for z in range(6):
                pts.append([0.5 * x + rng.uniform_range(-0.02, 0.02), 0.5 * y + rng.uniform_range(-0.02, 0.02),
                            0.5 * z + rng.uniform_range(-0.02, 0.02)])
    mu = np.array(pts)
    sig = np.tile((1e-4 * np.eye(3)).reshape(9), (len(mu), 1))
    mapc = GaussianCloud(mu, sig)
    cfg = make_config(n_particles=1, seed=42, nnf_resolution=0.1)
    e = FilterEngine(mapc, cfg)
    e.init_uniform([4.9, 3.9, 1.4, 5.1, 4.1, 1.6])
    gt = I12.copy()
    gt[9:] = [5.0, 4.0, 1.5]
    p = e.particles()
    p.poses[0] = gt
    e.set_particles(p)
    delta = O.compose(I12, I12)
    c, s = math.cos(0.01), math.sin(0.01)
    delta[:9] = [c, -s, 0, s, c, 0, 0, 0, 1]
    delta[9:] = [0.02, 0.01, 0.0]
    for f in range(60):
        gt = sim.compose(gt, delta)
        inv = sim.inverse(gt)
        sel = np.linalg.norm(mu - gt[9:], axis=1) < 4.0
        Ri = inv[:9].reshape(3, 3)
        smu = mu[sel] @ Ri.T + inv[9:]
        ssg = np.array([(Ri @ s_.reshape(3, 3) @ Ri.T).reshape(9) for s_ in sig[sel]])
        res = e.step(GaussianCloud(smu, ssg), delta, np.zeros(36), True)
        assert np.linalg.norm(res["representative"][9:] - gt[9:]) < 1e-3


def test_ids_fixed_and_timings(world):
    cfg = make_config(n_particles=3000, seed=42, nnf_resolution=0.2)
    e = FilterEngine(world.map, cfg)
    e.init_uniform(world.map.bounds)
    gt = I12.copy()
    gt[9:] = [5.0, 4.0, 1.5]
    delta = I12.copy()
    delta[9] = 0.05
    stage, total = 0.0, 0.0
    for f in range(5):
        gt = sim.compose(gt, delta)
        res = e.step(world.scan_at(gt, cfg, 700 + f), delta, np.diag([1e-4] * 6).reshape(36), True)
        assert res["n_particles"] == 3000
        assert np.array_equal(np.sort(e.particles().id), np.arange(3000))
        stage += sum(res[k] for k in ("predict_ms", "neighbor_ms", "likelihood_ms", "update_ms", "posterior_ms"))
        total += res["total_ms"]
    assert abs(stage - total) / total < 0.05


def test_rejected_observation_resets_uniformly(world):
    """posterior.cpp:29-33: when no particle matches, the Bayes update resets
    log_post to uniform and reports the observation rejected (decided on the
    device in the step); the following smoothing runs as usual."""
    for mode in (1, 2):
        cfg = make_config(n_particles=500, seed=42, nnf_resolution=0.2, likelihood_mode=mode)
        g = FilterEngine(world.map, cfg)
        r = O.FilterEngine(world.map.mu, world.map.sigma, cfg, world.map.bounds)
        g.init_uniform(world.map.bounds)
        r.init_uniform(world.map.bounds)
        gt = I12.copy()
        gt[9:] = [5.0, 4.0, 1.5]
        scan = world.scan_at(gt, cfg)
        far = GaussianCloud(scan.mu + 1000.0, scan.sigma)  # matches nothing anywhere
        cov = np.diag([1e-4] * 6).reshape(36)
        for sc in (scan, far, scan):
            a = g.step(sc, I12, cov, True)
            b = r.step(sc.mu, sc.sigma, I12, cov, True)
            assert a["observation_rejected"] == b["observation_rejected"]
            assert a["mean_n_matched"] == b["mean_n_matched"] or mode == 2
        assert a["observation_rejected"] == 0
        rej = g.step(far, I12, cov, True)
        assert rej["observation_rejected"] == 1 and rej["mean_n_matched"] == 0.0
        if mode == 1:
            r.step(far.mu, far.sigma, I12, cov, True)
            assert np.abs(g.particles().log_post - r.particles().log_post).max() < 1e-9


@pytest.mark.parametrize("k", [8, 32])
def test_step_exact_mode_other_list_sizes(world, k):
    """Whole steps with lists off the default 20 (generic reorder and
    smoothing kernels, the 8- / 32-slot neighbour-pass variants)."""
    cfg = make_config(n_particles=400, seed=7, nnf_resolution=0.2, likelihood_mode=1, k_neighbors=k)
    g, fg = run_frames(world, cfg, 4)
    r, fr = run_frames(world, cfg, 4, oracle=True)
    for a, b in zip(fg, fr):
        assert a["rep_id"] == b["rep_id"] and a["mean_n_matched"] == b["mean_n_matched"]
        assert abs(a["rep_log_post"] - b["rep_log_post"]) < 1e-9
    pg, pr = g.particles(), r.particles()
    assert np.array_equal(pg.id, pr.id)
    assert np.array_equal(pg.idx, pr.idx) and np.array_equal(pg.count, pr.count)
    assert np.array_equal(pg.kval, pr.kval)
    assert np.abs(pg.poses - pr.poses).max() < 1e-9
    assert np.abs(pg.log_post - pr.log_post).max() < 1e-9


def test_step_profile_counters_and_lazy_stage_times(world):
    """smcl_last_step_counts returns the step's counters without reading the
    per-kernel stage times; smcl_last_step_profile reads them from the step's
    events on demand (the same counters, stage times filled in)."""
    cfg = make_config(n_particles=2000, seed=3, nnf_resolution=0.2, likelihood_mode=2)
    eng, frames = run_frames(world, cfg, 3)
    c = eng.last_step_profile(times=False)
    p = eng.last_step_profile()
    S = c["ll_points"] // cfg.n_particles
    assert S > 0 and c["gn_points"] == S * cfg.n_particles * cfg.n_svgd_iters
    for k in ("gn_points", "ll_points", "gn_matched", "ll_matched", "kernel_launches", "fast_path"):
        assert c[k] == p[k]
    assert c["lsh_keys_ms"] == 0.0 and c["smooth_ms"] == 0.0  # not read
    assert p["lsh_keys_ms"] > 0.0 and p["smooth_ms"] > 0.0 and p["refresh_gather_ms"] > 0.0
    stages = sum(p[k] for k in ("predict_ms", "lsh_keys_ms", "sort_ms", "reorder_ms", "segments_ms",
                                "refresh_gather_ms", "nb_stats_ms", "gn_kernel_ms", "solve_ms", "svgd_ms",
                                "ll_kernel_ms", "bayes_ms", "smooth_ms"))
    assert abs(stages - p["total_ms"]) <= 0.05 * p["total_ms"] + 0.05
    assert abs(frames[-1]["total_ms"] - p["total_ms"]) < 1e-6
