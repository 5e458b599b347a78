"""GPU map load: the engine builds the nearest-neighbour
field and the fast-map records on the device (kernels/map_build.cu).

The NNF must equal the host build (host/prep.cpp build_nnf_cells, itself pinned
to the oracle and to a brute-force nearest search in test_abi.py) bit for bit:
same reached cells (nnf.cpp:37-80), same nearest point, ties to the lower
index (point_grid.cpp:109-141). Cases: the bench's corridor map at 0.1 m, a
lattice cloud full of equidistant ties, caller bounds tighter than the points
(clamped cells), and a single-point map.
"""
import time

import numpy as np
import pytest

import oracle as O
from helpers import config
from paper_2404_16370_b200 import api, sim
from paper_2404_16370_b200.api import FilterEngine, GaussianCloud

pytestmark = pytest.mark.gpu


def _device_nnf(cloud, res, pad, maxq):
    e = FilterEngine(cloud, config(nnf_resolution=res, nnf_padding=pad, nnf_max_query_dist=maxq, n_particles=64))
    return e.nnf()


def _check(cloud, res, pad, maxq):
    d, o, r, cells = _device_nnf(cloud, res, pad, maxq)
    d2, o2, c2 = api.build_nnf(cloud, res, pad, maxq)
    assert np.array_equal(d, d2) and np.array_equal(o, o2) and r == res
    assert np.array_equal(cells, c2), f"{np.count_nonzero(cells != c2)} cells differ"
    return cells


def test_corridor_map_matches_host_build():
    sc = sim.scenario_preset("corridor_easy", seed=1)
    cfg = config(nnf_resolution=0.1)
    rects, mapc = sim.scenario_map(sc, cfg)
    t0 = time.perf_counter()
    cells = _check(mapc, 0.1, cfg.nnf_padding, cfg.nnf_max_query_dist)
    assert (cells >= 0).sum() > 100000
    print(f"corridor NNF {cells.size} cells, device engine setup + host check {time.perf_counter() - t0:.2f} s")


def test_lattice_ties_and_oracle():
    # Points on a 0.1 m lattice: many cell centres are equidistant to several points.
    g = np.arange(0.0, 1.01, 0.1)
    mu = np.stack(np.meshgrid(g, g, g[:4], indexing="ij"), -1).reshape(-1, 3)
    mu = np.concatenate([mu, mu[::7]])  # exact duplicates: the lower index must win
    sig = np.tile((1e-4 * np.eye(3)).reshape(9), (len(mu), 1))
    cloud = GaussianCloud(mu, sig)
    cells = _check(cloud, 0.05, 0.2, 0.3)
    om = O.OracleMap(mu, sig, cloud.bounds, 0.05, 0.2, 0.3)
    assert np.array_equal(cells, om.nnf()[2])


def test_bounds_tighter_than_points_and_tiny_maps():
    rng = np.random.default_rng(11)
    mu = rng.uniform(-1.0, 3.0, size=(400, 3))
    sig = np.tile((1e-4 * np.eye(3)).reshape(9), (400, 1))
    cloud = GaussianCloud(mu, sig, bounds=[0.0, 0.0, 0.0, 2.0, 2.0, 2.0])  # points outside are clamped
    _check(cloud, 0.1, 0.3, 0.5)
    one = GaussianCloud(np.array([[0.3, -0.2, 1.0]]), (1e-4 * np.eye(3)).reshape(1, 9))
    cells = _check(one, 0.1, 0.5, 1.0)
    assert set(np.unique(cells)) <= {-1, 0} and (cells == 0).sum() > 0


def test_fast_records_drive_the_same_likelihood():
    """Device-built records feed the fast path: n_matched equals the exact path."""
    from helpers import cube_set, room_scene
    rects, mapc, scan = room_scene()
    parts = cube_set(300, 7, 20)
    ef = FilterEngine(mapc, config(nnf_resolution=0.2, likelihood_mode=2))
    ex = FilterEngine(mapc, config(nnf_resolution=0.2, likelihood_mode=1))
    ef.set_particles(parts)
    ex.set_particles(parts)
    llf, nmf = ef.evaluate_likelihoods(scan)
    llx, nmx = ex.evaluate_likelihoods(scan)
    assert np.array_equal(nmf, nmx)
    m = llx > -1e29
    assert np.all(np.abs(llf[m] - llx[m]) <= 2e-5 * np.abs(llx[m]))
