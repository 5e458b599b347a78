"""Shard-count invariance of the sharded engine.

G engines, each owning a contiguous 1/G of the particle indices and joined by
the in-process loopback all-gather (one host thread per engine), must produce
the bit-identical frame results and particle set of one unsharded engine:
every exchange point reproduces the single-engine order (global key sort,
reduce.hpp chunk order, lowest-index argmax ties). The reference's own
determinism contract is test_parallel_consistency.cpp:45-99 (thread-count
invariance); this is its multi-GPU analogue.
"""
import threading

import numpy as np
import pytest

from paper_2404_16370_b200 import sim
from paper_2404_16370_b200.abi import ALLTOALLV_FN, Particles, identity_pose, make_config
from paper_2404_16370_b200.api import FilterEngine, make_scan_cloud
from paper_2404_16370_b200.comm import LoopbackComms

pytestmark = pytest.mark.gpu
I12 = identity_pose()


@pytest.fixture(scope="module")
def world():
    rects = sim.box_room([10.0, 8.0, 3.0])
    mapc = sim.sample_world(rects, 60.0, 5)
    sensor = sim.sensor_spec(noise_sigma=0.0)
    return rects, mapc, sensor


def scans(world, cfg, n_frames):
    rects, _, sensor = world
    gt = I12.copy()
    gt[9:] = [5.0, 4.0, 1.5]
    delta = I12.copy()
    delta[9] = 0.05
    out = []
    for f in range(n_frames):
        gt = sim.compose(gt, delta)
        pts, _ = sim.simulate_scan_points(rects, gt, sensor, 100 + f)
        out.append(make_scan_cloud(pts, cfg))
    return out, delta, np.diag([1e-4] * 6).reshape(36)


def run_single(world, cfg, frames):
    scans_, delta, cov = frames
    eng = FilterEngine(world[1], cfg)
    eng.init_uniform(world[1].bounds)
    res = [eng.step(s, delta, cov, True) for s in scans_]
    return res, eng.particles()


def run_sharded(world, cfg, frames, G, alltoallv=True):
    scans_, delta, cov = frames
    comms = LoopbackComms(G)
    if not alltoallv:  # a communicator without alltoallv: the reorder all-gathers the state
        for r in range(G):
            comms[r].alltoallv = ALLTOALLV_FN()
    engines = [FilterEngine(world[1], cfg, comm=comms[r]) for r in range(G)]
    results = [None] * G
    errors = []

    def body(r):
        try:
            e = engines[r]
            e.init_uniform(world[1].bounds)
            results[r] = [e.step(s, delta, cov, True) for s in scans_]
        except Exception as ex:  # pragma: no cover - reported below
            errors.append(ex)

    th = [threading.Thread(target=body, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors
    parts = [e.particles() for e in engines]
    k = parts[0].k
    n = sum(p.n for p in parts)
    cat = Particles(n, k)
    for name in ("poses", "log_post", "id", "idx", "kval", "count"):
        getattr(cat, name)[...] = np.concatenate([getattr(p, name) for p in parts])
    for e in engines:
        e.close()
    comms.close()
    return results, cat


@pytest.mark.parametrize("G,mode,reorder,a2a", [(2, 2, 0, 1), (4, 2, 0, 1), (2, 1, 0, 1), (2, 2, 1, 1), (4, 2, 1, 1),
                                                (2, 1, 1, 1), (4, 2, 1, 0), (2, 1, 1, 0), (8, 2, 1, 1)])
def test_sharded_engine_is_bit_identical_to_single(world, G, mode, reorder, a2a):
    """reorder = 1: the LSH reorder migrates particle state across shards
    (particle_set.cpp:7-47 on the global order), by
    alltoallv of the migrating records (a2a = 1) or by all-gather (a2a = 0)."""
    n = max(16384 if mode == 2 else 8192, 4096 * G)
    cfg = make_config(n_particles=n, seed=7, nnf_resolution=0.2, likelihood_mode=mode, reorder_particles=reorder)
    frames = scans(world, cfg, 3)
    ref_res, ref_p = run_single(world, cfg, frames)
    sh_res, sh_p = run_sharded(world, cfg, frames, G, alltoallv=bool(a2a))
    for r in range(G):  # every rank reports the same global frame result
        for a, b in zip(sh_res[r], ref_res):
            assert a["rep_id"] == b["rep_id"] and a["rep_index"] == b["rep_index"]
            assert a["rep_log_post"] == b["rep_log_post"]
            assert a["mean_n_matched"] == b["mean_n_matched"]
            assert a["observation_rejected"] == b["observation_rejected"]
            assert np.array_equal(a["representative"], b["representative"])
            sa, sb = a["neighbor_stats"], b["neighbor_stats"]
            for key in ("n_buckets", "buckets_used", "overflow_dropped", "mean_kernel", "occupancy_hist"):
                assert sa[key] == sb[key], key
    for name in ("poses", "log_post", "id", "idx", "kval", "count"):
        assert np.array_equal(getattr(sh_p, name), getattr(ref_p, name)), name


def test_sharded_rejects_unaligned_shards(world):
    cfg = make_config(n_particles=4096 * 3, seed=1, reorder_particles=0)
    comms = LoopbackComms(2)
    e = FilterEngine(world[1], cfg, comm=comms[0])
    with pytest.raises(Exception):
        e.init_uniform(world[1].bounds)
    e.close()
    comms.close()


def test_sharded_profile_counts_all_shards_once(world):
    """bench.py's pp/step comes from the step profile: every rank reports the
    particle-point evaluations of ALL shards (gn_points + ll_points = N * (S_gn
    + S) for one SVGD iteration), so the whole-job value needs no world factor,
    and it equals one engine's count (bench.pp_per_step)."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location("bench", os.path.join(os.path.dirname(__file__), "..", "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    n, G = 8192, 2
    cfg = make_config(n_particles=n, seed=7, nnf_resolution=0.2, reorder_particles=1)
    scans_, delta, cov = scans(world, cfg, 1)
    single = FilterEngine(world[1], cfg)
    single.init_uniform(world[1].bounds)
    single.step(scans_[0], delta, cov, True)
    p1 = single.last_step_profile()
    single.close()
    comms = LoopbackComms(G)
    engines = [FilterEngine(world[1], cfg, comm=comms[r]) for r in range(G)]
    profs = [None] * G

    def body(r):
        engines[r].init_uniform(world[1].bounds)
        engines[r].step(scans_[0], delta, cov, True)
        profs[r] = engines[r].last_step_profile()

    th = [threading.Thread(target=body, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    S = len(scans_[0])
    for p in profs:
        assert p["gn_points"] == n * S and p["ll_points"] == n * S
        assert p["gn_points"] + p["ll_points"] == bench.pp_per_step(n, S, cfg)
    assert p1["gn_points"] + p1["ll_points"] == bench.pp_per_step(n, S, cfg)
    # matched counts are per shard: they add up to the single engine's
    assert sum(p["ll_matched"] for p in profs) == p1["ll_matched"]
    for e in engines:
        e.close()
    comms.close()
