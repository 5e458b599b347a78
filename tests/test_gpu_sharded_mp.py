"""Two processes, one sharded engine each: the engines are
joined by a torch.distributed gloo group (``TorchComm(staged=True)``: each
collective drains the engine stream and exchanges the bytes through host
memory, so no kernel ever waits on the other process) and must reproduce one
unsharded engine bit for bit, with and without the cross-shard reorder
(particle_set.cpp:7-47 over the global order, neighbor_search.cpp:119-125).
Both ranks share cuda:0 when only one GPU is visible."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N = 8192
FRAMES = 3


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(cfg):
    from paper_2404_16370_b200 import sim
    from paper_2404_16370_b200.abi import identity_pose
    from paper_2404_16370_b200.api import make_scan_cloud
    rects = sim.box_room([10.0, 8.0, 3.0])
    mapc = sim.sample_world(rects, 60.0, 5)
    sensor = sim.sensor_spec(noise_sigma=0.0)
    gt = identity_pose()
    gt[9:] = [5.0, 4.0, 1.5]
    delta = identity_pose()
    delta[9] = 0.05
    scans = []
    for f in range(FRAMES):
        gt = sim.compose(gt, delta)
        pts, _ = sim.simulate_scan_points(rects, gt, sensor, 100 + f)
        scans.append(make_scan_cloud(pts, cfg))
    return mapc, scans, delta, np.diag([1e-4] * 6).reshape(36)


def _summary(results, parts):
    keys = ("rep_id", "rep_index", "rep_log_post", "mean_n_matched", "observation_rejected")
    res = [{k: r[k] for k in keys} | {"representative": np.asarray(r["representative"]).copy()} for r in results]
    state = {k: np.asarray(getattr(parts, k)).copy() for k in ("poses", "log_post", "id", "idx", "kval", "count")}
    return res, state


def _rank(rank, world, port, reorder, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2404_16370_b200.abi import make_config
        from paper_2404_16370_b200.api import FilterEngine
        from paper_2404_16370_b200.comm import TorchComm
        dev = rank % torch.cuda.device_count()
        torch.cuda.set_device(dev)
        cfg = make_config(n_particles=N, seed=7, nnf_resolution=0.2, reorder_particles=reorder)
        mapc, scans, delta, cov = _inputs(cfg)
        tc = TorchComm(staged=True)
        e = FilterEngine(mapc, cfg, device=dev, comm=tc)
        e.init_uniform(mapc.bounds)
        results = [e.step(s, delta, cov, True) for s in scans]
        assert tc.error is None, tc.error
        out.put((rank, _summary(results, e.particles())))
        e.close()
    except Exception as ex:  # pragma: no cover - reported by the parent
        out.put((rank, repr(ex)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("reorder", [0, 1])
def test_two_process_sharded_engine_matches_single(reorder):
    from paper_2404_16370_b200.abi import make_config
    from paper_2404_16370_b200.api import FilterEngine
    cfg = make_config(n_particles=N, seed=7, nnf_resolution=0.2, reorder_particles=reorder)
    mapc, scans, delta, cov = _inputs(cfg)
    e = FilterEngine(mapc, cfg)
    e.init_uniform(mapc.bounds)
    ref_res, ref_state = _summary([e.step(s, delta, cov, True) for s in scans], e.particles())
    e.close()

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, 2, port, reorder, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=120)
    for r in range(2):
        assert not isinstance(got[r], str), got[r]
        res, _ = got[r]
        for a, b in zip(res, ref_res):  # every rank reports the global frame result
            for k in ("rep_id", "rep_index", "rep_log_post", "mean_n_matched", "observation_rejected"):
                assert a[k] == b[k], (r, k)
            assert np.array_equal(a["representative"], b["representative"])
    for k, v in ref_state.items():  # shards concatenate to the single engine's state
        assert np.array_equal(np.concatenate([got[0][1][k], got[1][1][k]]), v), k
