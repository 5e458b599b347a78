"""Acceptance criteria C6-C8 of the reference (acceptance.cpp:291-380) run
through the GPU engine at (and beyond) the reference's scale: global
localization in the symmetric corridor, kidnap recovery after occlusions, and
the no-resampling invariant. The reference runs these at 1e5 particles on the
CPU (minutes per run); here C6 also runs at 1,048,576 particles."""
import numpy as np
import pytest

from paper_2404_16370_b200 import scenario as S
from paper_2404_16370_b200 import sim
from paper_2404_16370_b200.abi import make_config
from paper_2404_16370_b200.api import FilterEngine

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_particles", [100000, 1 << 20])
def test_c6_global_localization(n_particles, tmp_path):
    sc = sim.scenario_preset("corridor_easy", seed=1000)
    cfg = S.localization_config(2000, n_particles=n_particles)
    res = S.run_scenario(sc, cfg, out_dir=str(tmp_path / "c6"))
    rep = res.report
    print(f"C6 N={n_particles}: convergence_frame={rep.convergence_frame} "
          f"post_ate={rep.ate_rmse_post_convergence:.3f} mean_total_ms={rep.mean_times['total_ms']:.2f}")
    assert 0 <= rep.convergence_frame < 100
    assert 0.0 <= rep.ate_rmse_post_convergence <= 2.0 * cfg.nnf_resolution
    assert (tmp_path / "c6" / "report.txt").read_text().startswith("scenario: corridor_easy")
    assert len(S.read_tum(str(tmp_path / "c6" / "est.tum"))) == sc.n_frames


def test_c7_kidnap_recovery():
    sc = sim.scenario_preset("corridor_kidnap", seed=3000)
    cfg = S.localization_config(4000)
    res = S.run_scenario(sc, cfg)
    print(f"C7: recovery_frames={res.report.recovery_frames} convergence={res.report.convergence_frame}")
    assert len(res.report.recovery_frames) == 2
    assert all(r >= 0 for r in res.report.recovery_frames)
    assert any(fr["scan_empty"] for fr in res.frames)


def test_c8_no_resampling_invariant():
    sc = sim.scenario_preset("box_easy")
    sc.n_frames = 40
    sc.occlusions = [(15, 25)]
    cfg = make_config(n_particles=3000, nnf_resolution=0.2, seed=808)
    rects, mapc = sim.scenario_map(sc, cfg)
    e = FilterEngine(mapc, cfg)
    e.init_uniform(mapc.bounds)
    truth = sim.build_trajectory(sc)
    odo = sim.build_odometry(sc, truth)
    for f in range(sc.n_frames):
        d, c, v = odo[f]
        fr = e.step_points(sim.scan_points_for_frame(sc, rects, truth, f), d, c, v)
        assert fr["n_particles"] == 3000
        assert np.array_equal(np.sort(e.particles().id), np.arange(3000))


def test_c4_lsh_recall_at_20():
    """acceptance.cpp:169-220: 1,000 particles (rotations <= 0.2 rad, positions
    in a 10 m cube), default LSH, 10 passes: recall@20 against the brute-force
    kernel kNN >= 0.9, with the GPU neighbour pass."""
    import oracle as O
    from helpers import random_cube_set
    n, k = 1000, 20
    g = random_cube_set(n, 10.0, 0.2, k, 404)
    truth = O.brute_force_kernel_knn(g.poses, k)
    e = FilterEngine(None, make_config(k_neighbors=k))
    e.set_particles(g)
    for p in range(10):
        e.update_neighbors(O.mix_seed(405, p), [0, 0, 0, 10, 10, 10])
    got = e.particles()
    slot_of_id = np.empty(n, np.int64)
    slot_of_id[got.id] = np.arange(n)
    hit = total = 0
    for orig in range(n):
        s = slot_of_id[orig]
        have = {int(got.id[j]) for j in got.idx[s, : got.count[s]]}
        for want in truth[orig]:
            total += 1
            hit += int(want) in have
    print(f"C4: recall@20 = {hit / total:.4f}")
    assert hit / total >= 0.9


def test_outdoor_kidnap_1m_particles():
    """The paper's outdoor kidnap experiment at its scale (BASELINE configs[3]):
    1,048,576 particles on the builder-defined 280 x 200 x 30 m city map (NNF
    0.2 m, 2.2e8 cells built on the device), a 20-frame scan blackout during
    which the vehicle is teleported to another street. The filter (acceptance
    calibration) must localize globally, lose the pose during the blackout
    and re-localize right after it."""
    sc = sim.scenario_preset("outdoor_kidnap", seed=7)
    sc.sensor = sim.sensor_spec(n_azimuth=256, elevations_deg=list(np.linspace(-30.0, 30.0, 8)), max_range=60.0)
    cfg = S.localization_config(11, n_particles=1 << 20)
    cfg.nnf_resolution, cfg.nnf_max_query_dist, cfg.n_scan_max = 0.2, 2.0, 512
    res = S.run_scenario(sc, cfg)
    rep = res.report
    terr = rep.terr
    print(f"outdoor kidnap 1M: convergence={rep.convergence_frame} recovery={rep.recovery_frames} "
          f"mean_total_ms={rep.mean_times['total_ms']:.2f} final terr={terr[-10:].max():.3f}")
    assert 0 <= rep.convergence_frame < 20
    assert rep.recovery_frames and rep.recovery_frames[0] >= 0
    # Tracking after re-localization: 0.2 m NNF cells, 1-3 voxel errors. The
    # trajectory is chaotic in the fp32 rounding of the fast path (runs with
    # rounding-level code changes gave last-10-frame maxima of 0.15-0.55 m),
    # so the bound is on the median plus a loose cap.
    assert np.median(terr[-10:]) < 0.5 and terr[-10:].max() < 1.0
    assert terr[45] > 10.0  # the teleport inside the blackout really displaced the vehicle
