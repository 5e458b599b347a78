"""The reference's LSH fixtures (proj/tests/test_neighbor_search.cpp) run on
the B200 and compared with the oracle bit for bit, plus the near-integer
stress test of the K3 hash guard (lsh.cu lsh_hash_hd):

* collision-trial poses (:65-107): GPU hashes == oracle hashes;
* lone particle (:139-149), widely separated particles (:151-181), kNN recall
  scene (:204-236), determinism scene (:238-263), stats scene (:265-276):
  GPU neighbour passes == oracle passes (ids, idx, float kval, count, stats);
* poses built so that every cell coordinate zeta lands within ~1e-15..1e-14
  of an integer: GPU hashes and neighbour lists == oracle (glibc) ones.
"""
import numpy as np
import pytest

import oracle as O
from helpers import random_cube_set, random_pose
from paper_2404_16370_b200.abi import Particles, identity_pose, make_config
from paper_2404_16370_b200.api import FilterEngine, GaussianCloud, lsh_hash

pytestmark = pytest.mark.gpu
SR, ST, ALPHA, NOISE = 5.0, 2.5, 0.1, 0.5


def dummy_map():
    rng = np.random.default_rng(0)
    mu = rng.uniform(0.0, 1.0, (64, 3))
    return GaussianCloud(mu, np.tile((1e-3 * np.eye(3)).reshape(9), (64, 1)))


def gpu_passes(parts, cfg, seeds, bounds):
    e = FilterEngine(dummy_map(), cfg)
    e.set_particles(parts)
    stats = [e.update_neighbors(s, bounds) for s in seeds]
    return e.particles(), stats


def oracle_passes(parts, cfg, seeds, bounds):
    p = parts.copy()
    stats = [O.update_neighbors(p, cfg, s, bounds) for s in seeds]
    return p, stats


def assert_same(g, o):
    for name in ("id", "idx", "kval", "count", "poses", "log_post"):
        assert np.array_equal(getattr(g, name), getattr(o, name)), name


def test_collision_trial_hashes_bitwise():  # :65-107 poses
    rng = O.SplitMix64(5)
    w = ALPHA * np.array([SR] * 3 + [ST] * 3)
    box = [-5.0] * 3 + [5.0] * 3
    for _ in range(2000):
        frame = rng.random_lsh_frame(box)
        noise = NOISE * rng.normal6()
        a = random_pose(rng, 1.5, 4.0)
        budget = rng.uniform_range(0.0, 0.1)
        dz = np.array([rng.uniform_range(-1.0, 1.0) for _ in range(6)])
        dz *= budget / np.abs(dz).sum()
        b = O.compose(a, O.se3_exp(dz / w)[0])
        c = a.copy()
        c[9:] += [50.0, -30.0, 40.0]
        got = lsh_hash(np.stack([a, b, c]), frame, noise, ALPHA, SR, ST)
        want = [O.lsh_hash(p, frame, noise, ALPHA, SR, ST) for p in (a, b, c)]
        assert [int(x) for x in got] == want


def test_lone_particle():  # :139-149
    s = random_cube_set(1, 1.0, 0.1, 20, 3)
    seeds = [O.mix_seed(11, p) for p in range(5)]
    g, _ = gpu_passes(s, make_config(), seeds, [0.0] * 3 + [1.0] * 3)
    o, _ = oracle_passes(s, make_config(), seeds, [0.0] * 3 + [1.0] * 3)
    assert_same(g, o)
    assert g.count[0] == 1 and g.idx[0, 0] == 0


def test_widely_separated():  # :151-181
    poses = np.tile(identity_pose(), (100, 1))
    poses[:, 9] = 10.0 * np.arange(100)
    s = Particles.from_poses(poses, 5)
    cfg = make_config(k_neighbors=5)
    seeds = [O.mix_seed(13, p) for p in range(5)]
    bounds = [0.0, 0.0, 0.0, 1000.0, 1.0, 1.0]
    g, _ = gpu_passes(s, cfg, seeds, bounds)
    o, _ = oracle_passes(s, cfg, seeds, bounds)
    assert_same(g, o)


def test_recall_scene_and_stats():  # :204-236, :265-276
    k = 10
    s = random_cube_set(300, 8.0, 0.2, k, 17)
    cfg = make_config(k_neighbors=k)
    seeds = [O.mix_seed(19, p) for p in range(10)]
    g, sg = gpu_passes(s, cfg, seeds, [0.0] * 3 + [8.0] * 3)
    o, so = oracle_passes(s, cfg, seeds, [0.0] * 3 + [8.0] * 3)
    assert_same(g, o)
    s2 = random_cube_set(400, 5.0, 0.2, 20, 31)
    g2, sg2 = gpu_passes(s2, make_config(), [37], [0.0] * 3 + [5.0] * 3)
    o2, so2 = oracle_passes(s2, make_config(), [37], [0.0] * 3 + [5.0] * 3)
    assert_same(g2, o2)
    for key in ("n_buckets", "buckets_used", "overflow_dropped"):
        assert sg2[0][key] == so2[0][key], key
    assert abs(sg2[0]["mean_kernel"] - so2[0]["mean_kernel"]) <= 1e-12


def test_determinism_scene():  # :238-263 (4 passes, 500 particles, default config)
    s = random_cube_set(500, 6.0, 0.3, 20, 23)
    seeds = [O.mix_seed(29, p) for p in range(4)]
    g, _ = gpu_passes(s, make_config(), seeds, [0.0] * 3 + [6.0] * 3)
    g2, _ = gpu_passes(s, make_config(), seeds, [0.0] * 3 + [6.0] * 3)
    o, _ = oracle_passes(s, make_config(), seeds, [0.0] * 3 + [6.0] * 3)
    assert_same(g, g2)
    assert_same(g, o)


def near_integer_poses(n, frame, noise, seed, spread=20):
    """Poses whose cell coordinates zeta = alpha W log(F^-1 T) + delta sit on
    integers up to the exp/log round trip (~1e-15..1e-14)."""
    rng = np.random.default_rng(seed)
    w = ALPHA * np.array([SR] * 3 + [ST] * 3)
    out = np.empty((n, 12))
    for i in range(n):
        while True:
            z = rng.integers(-spread, spread + 1, 6).astype(np.float64)
            d = (z - noise) / w
            if np.linalg.norm(d[:3]) < 3.0:  # rotation angle below pi
                break
        out[i] = O.compose(frame, O.se3_exp(d)[0])
    return out


def test_near_integer_zeta_hashes_bitwise():
    rng = O.SplitMix64(77)
    frame = rng.random_lsh_frame([-10.0] * 3 + [10.0] * 3)
    noise = NOISE * rng.normal6()
    poses = near_integer_poses(4000, frame, noise, 1)
    zeta = np.array([ALPHA * np.array([SR] * 3 + [ST] * 3) * O.se3_log(O.compose(O.inverse(frame), p))[0] + noise
                     for p in poses[:200]])
    assert np.abs(zeta - np.round(zeta)).max() < 1e-13  # the stress really is at the integers
    got = lsh_hash(poses, frame, noise, ALPHA, SR, ST)
    want = np.array([O.lsh_hash(p, frame, noise, ALPHA, SR, ST) for p in poses], np.uint64)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n", [512, 4096, 6000])
def test_near_integer_zeta_neighbour_pass_bitwise(n):
    """The product path: K3 keys (guarded, host rehash) -> sort -> lists.
    Up to kGuardListCap (4096) flags the host rehashes only the flagged
    particles; beyond, the whole shard."""
    cfg = make_config()
    bounds = [-10.0] * 3 + [10.0] * 3
    seed = O.mix_seed(91, 0)
    rng = O.SplitMix64(seed)  # the pass frame and noise, drawn as update_neighbors draws them
    frame = rng.random_lsh_frame(bounds)
    noise = cfg.lsh_noise_sigma * rng.normal6()
    s = Particles.from_poses(near_integer_poses(n, frame, noise, 2, spread=3), 20)
    e = FilterEngine(dummy_map(), cfg)
    e.set_particles(s)
    e.update_neighbors(seed, bounds)
    g = e.particles()
    prof = e.last_step_profile()
    o = s.copy()
    O.update_neighbors(o, cfg, seed, bounds)
    assert_same(g, o)
    print("guard: flagged", prof["hash_guard_flagged"], "replays", prof["hash_guard_replays"])
    assert prof["hash_guard_flagged"] > 0  # the stress really reaches the guard
