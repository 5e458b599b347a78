"""Full-size (BASELINE.json configs[2]: 1,048,576 particles x 512-pt scans)
checks through size-independent properties, plus oracle parity on a random
sample of the full-size particle set."""
import numpy as np
import pytest

import oracle as O
from paper_2404_16370_b200 import workload
from paper_2404_16370_b200.api import FilterEngine

pytestmark = pytest.mark.gpu
N = 1 << 20


@pytest.fixture(scope="module")
def run():
    wl = workload.build("global_init", n_particles=N, scan_points=512, n_frames=4)
    e = FilterEngine(wl.map, wl.cfg)
    e.init_uniform(wl.bounds)
    frames = []
    for f in range(3):
        d, c, v = wl.odometry[f]
        frames.append(e.step(wl.scans[f], d, c, v))
    return wl, e, frames, e.particles()


def test_particle_set_invariants(run):
    wl, e, frames, p = run
    K = p.k
    assert np.array_equal(np.sort(p.id), np.arange(N))  # no resampling: ids are a permutation
    assert p.count.min() >= 1 and p.count.max() <= K
    rows = np.arange(N)
    valid = np.arange(K)[None, :] < p.count[:, None]
    idx = np.where(valid, p.idx, -1)
    assert idx.max() < N and (idx[valid] >= 0).all()
    self_slot = (idx == rows[:, None])
    assert (self_slot.sum(1) == 1).all()  # self exactly once
    assert np.all(p.kval[self_slot] == 1.0)
    kv = p.kval[valid]
    assert kv.min() >= 0.0 and kv.max() <= 1.0
    srt = np.sort(idx, 1)  # no duplicates among the listed entries
    dup = (srt[:, 1:] == srt[:, :-1]) & (srt[:, 1:] >= 0)
    assert not dup.any()


def test_posterior_and_poses(run):
    wl, e, frames, p = run
    lp = p.log_post
    m = lp.max()
    assert abs(m + np.log(np.exp(lp - m).sum())) < 1e-9  # normalised (reduce.hpp order, fp64)
    assert lp.min() >= -80.0 - 1e-12
    R = p.poses[:, :9].reshape(-1, 3, 3)
    drift = np.abs(np.einsum("nji,njk->nik", R, R) - np.eye(3)).max()
    assert drift < 1e-6
    fr = frames[-1]
    assert fr["rep_log_post"] == m and fr["rep_index"] == int(np.argmax(lp))
    assert np.array_equal(fr["representative"], p.poses[fr["rep_index"]])
    assert fr["n_particles"] == N


def test_likelihood_parity_on_a_sample(run):
    wl, e, frames, p = run
    scan = wl.scans[3]
    steps, ll, nm = e.evaluate_all(scan)  # fast path on the full set
    rng = np.random.default_rng(5)
    sel = rng.choice(N, 4096, replace=False)
    cfg = wl.cfg
    om = O.OracleMap(wl.map.mu, wl.map.sigma, wl.map.bounds, cfg.nnf_resolution, cfg.nnf_padding,
                     cfg.nnf_max_query_dist)
    s2, ll2, nm2 = O.evaluate_all(om, scan.mu, scan.sigma, p.poses[sel], cfg)
    assert np.array_equal(nm[sel], nm2)
    g = ll2 > -1e29
    assert np.all(np.abs(ll[sel][g] - ll2[g]) <= 2e-5 * np.abs(ll2[g]))
