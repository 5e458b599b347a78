"""Python mirror of the reference ``steinmcl`` filter API over the C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/steinmcl/{filter,gicp,neighbor_search,svgd,posterior}.hpp;
every call runs the sm_100a kernels in libsmcl_gpu.so (no CPU fallback).
"""
import ctypes as C

import numpy as np

from . import _lib
from .abi import (Particles, SmclFrameResult, SmclNeighborStats, SmclStepProfile, cloud_struct, f64ptr, i32ptr,
                  make_config, odom_struct, u64ptr)

check = _lib.check


def _a(x, shape=None, dtype=np.float64):
    a = np.ascontiguousarray(x, dtype=dtype)
    return a if shape is None else a.reshape(shape)


class GaussianCloud:
    """gaussian_cloud.hpp:32-40: means, 3x3 covariances (row-major) and bounds."""

    def __init__(self, mu, sigma, bounds=None):
        self.mu = _a(mu, (-1, 3))
        self.sigma = _a(sigma, (-1, 9))
        if bounds is None and len(self.mu):
            bounds = np.concatenate([self.mu.min(0), self.mu.max(0)])
        self.bounds = None if bounds is None else _a(bounds, (6,))

    def __len__(self):
        return self.mu.shape[0]

    def empty(self):
        return len(self) == 0

    def struct(self):
        return cloud_struct(self.mu, self.sigma, self.bounds)


FilterConfig = make_config


class FilterEngine:
    """FilterEngine (filter.hpp:104-130) on one B200.

    ``map_cloud`` may be None for stage-only use (neighbour search, SVGD,
    posterior) on particles uploaded with ``set_particles``.

    ``comm`` (an ``SmclComm`` or an object with a ``.struct`` one, see
    ``comm.py``) makes this engine one shard of a particle set split across
    ranks; ``particles()`` / ``set_particles`` then move this rank's shard.
    """

    def __init__(self, map_cloud, cfg=None, device=0, comm=None):
        self.cfg = cfg if cfg is not None else make_config()
        self.h = C.c_void_p()
        if map_cloud is not None:
            self._map_c, self._map_keep = map_cloud.struct()
            mp = C.byref(self._map_c)
        else:
            mp = None
        self.comm = comm
        if comm is None:
            self.rank, self.world = 0, 1
            check(_lib.lib().smcl_create(mp, C.byref(self.cfg), device, C.byref(self.h)))
        else:
            cs = getattr(comm, "struct", comm)
            self.rank, self.world = cs.rank, cs.world
            check(_lib.lib().smcl_create_sharded(mp, C.byref(self.cfg), device, C.byref(cs), C.byref(self.h)))
        self.map = map_cloud

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            _lib.lib().smcl_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ engine
    def init_uniform(self, bounds):
        check(_lib.lib().smcl_init_uniform(self.h, f64ptr(_a(bounds, (6,)))))

    def init_uniform_seeded(self, n, bounds, full_rotation=True, seed=1):
        check(_lib.lib().smcl_init_uniform_seeded(self.h, n, f64ptr(_a(bounds, (6,))), int(full_rotation),
                                                  C.c_uint64(seed & (2**64 - 1))))

    def step(self, scan, delta=None, cov=None, valid=True):
        """FilterEngine::step(scan, odo) -> FrameResult as a dict."""
        if scan is None or len(scan) == 0:
            sc, keep = cloud_struct(np.zeros((0, 3)), np.zeros((0, 9)))
        else:
            sc, keep = scan.struct()
        o = odom_struct(delta, cov, valid)
        r = SmclFrameResult()
        check(_lib.lib().smcl_step(self.h, C.byref(sc), C.byref(o), C.byref(r)))
        del keep
        return r.to_dict()

    def scan_upload(self, slot, scan):
        """Stage a prepared scan into a device slot (no H2D inside step_slot)."""
        if scan is None or len(scan) == 0:
            sc, keep = cloud_struct(np.zeros((0, 3)), np.zeros((0, 9)))
        else:
            sc, keep = scan.struct()
        check(_lib.lib().smcl_scan_upload(self.h, slot, C.byref(sc)))
        del keep

    def step_slot(self, slot, delta=None, cov=None, valid=True):
        o = odom_struct(delta, cov, valid)
        r = SmclFrameResult()
        check(_lib.lib().smcl_step_slot(self.h, slot, C.byref(o), C.byref(r)))
        return r.to_dict()

    def scan_prepare(self, slot, points):
        """make_scan_cloud (filter.cpp:86-100) on the device, staged into a slot."""
        pts = _a(points, (-1, 3))
        check(_lib.lib().smcl_scan_prepare(self.h, slot, f64ptr(pts), pts.shape[0]))

    def scan_prepare_async(self, slot, points):
        """Queue make_scan_cloud for a slot on the engine's preparation stream
        (overlaps the step running on another slot); step_slot waits for it."""
        pts = _a(points, (-1, 3))
        check(_lib.lib().smcl_scan_prepare_async(self.h, slot, f64ptr(pts), pts.shape[0]))

    def scan_get(self, slot):
        """Prepared scan of a slot as a GaussianCloud."""
        n = C.c_int64()
        check(_lib.lib().smcl_scan_get(self.h, slot, None, None, C.byref(n)))
        mu, sg = np.empty((n.value, 3)), np.empty((n.value, 9))
        check(_lib.lib().smcl_scan_get(self.h, slot, f64ptr(mu), f64ptr(sg), C.byref(n)))
        return GaussianCloud(mu, sg)

    def step_points(self, points, delta=None, cov=None, valid=True):
        """Scenario-runner frame: make_scan_cloud + FilterEngine::step on raw points (device scan prep)."""
        pts = _a(points, (-1, 3))
        o = odom_struct(delta, cov, valid)
        r = SmclFrameResult()
        check(_lib.lib().smcl_step_points(self.h, f64ptr(pts), pts.shape[0], C.byref(o), C.byref(r)))
        return r.to_dict()

    def last_step_profile(self, times=True):
        """Profile of the last step; times=False skips the per-kernel stage
        times (read from CUDA events on demand) and returns the counters."""
        p = SmclStepProfile()
        fn = _lib.lib().smcl_last_step_profile if times else _lib.lib().smcl_last_step_counts
        check(fn(self.h, C.byref(p)))
        return p.to_dict()

    def timer_start(self):
        check(_lib.lib().smcl_timer_start(self.h))

    def timer_stop(self):
        ms = C.c_double()
        check(_lib.lib().smcl_timer_stop(self.h, C.byref(ms)))
        return ms.value

    def frame_index(self):
        return _lib.lib().smcl_frame_index(self.h)

    def num_particles(self):
        return _lib.lib().smcl_num_particles(self.h)

    def num_local_particles(self):
        """Particles held by this engine (its shard; all of them when unsharded)."""
        return self.num_particles() // self.world

    def particles(self):
        n = self.num_local_particles()
        p = Particles(n, self.cfg.k_neighbors)
        v = p.view()
        check(_lib.lib().smcl_get_particles(self.h, C.byref(v)))
        return p

    def set_particles(self, p):
        v = p.view()
        self.cfg.k_neighbors = p.k
        check(_lib.lib().smcl_set_particles(self.h, C.byref(v)))

    def nnf(self):
        dims = np.zeros(3, np.int32)
        origin = np.zeros(3)
        res = C.c_double()
        check(_lib.lib().smcl_get_nnf(self.h, i32ptr(dims), f64ptr(origin), C.byref(res), None))
        cells = np.empty(int(np.prod(dims.astype(np.int64))), np.int32)
        check(_lib.lib().smcl_get_nnf(self.h, i32ptr(dims), f64ptr(origin), C.byref(res), i32ptr(cells)))
        return dims, origin, res.value, cells

    # ------------------------------------------------------------ stages
    def predict(self, delta, cov, frame_seed):
        check(_lib.lib().smcl_predict(self.h, f64ptr(_a(delta, (12,))), f64ptr(_a(cov, (36,))),
                                      C.c_uint64(frame_seed & (2**64 - 1))))

    def update_neighbors(self, pass_seed, bounds):
        st = SmclNeighborStats()
        check(_lib.lib().smcl_update_neighbors(self.h, C.c_uint64(pass_seed & (2**64 - 1)),
                                               f64ptr(_a(bounds, (6,))), C.byref(st)))
        return st.to_dict()

    def evaluate_all(self, scan, want_system=False):
        n = self.num_local_particles()  # the ABI reads / writes this shard's rows
        sc, keep = scan.struct()
        steps, ll, nm = np.empty((n, 6)), np.empty(n), np.empty(n, np.int32)
        H = np.empty((n, 6, 6)) if want_system else None
        b = np.empty((n, 6)) if want_system else None
        check(_lib.lib().smcl_evaluate_all(self.h, C.byref(sc), f64ptr(steps), f64ptr(ll), i32ptr(nm),
                                           f64ptr(H) if want_system else None, f64ptr(b) if want_system else None))
        del keep
        return (steps, ll, nm, H, b) if want_system else (steps, ll, nm)

    def evaluate_likelihoods(self, scan):
        n = self.num_local_particles()  # the ABI reads / writes this shard's rows
        sc, keep = scan.struct()
        ll, nm = np.empty(n), np.empty(n, np.int32)
        check(_lib.lib().smcl_evaluate_likelihoods(self.h, C.byref(sc), f64ptr(ll), i32ptr(nm)))
        del keep
        return ll, nm

    def compute_phis(self, steps=None):
        n = self.num_local_particles()  # the ABI reads / writes this shard's rows
        out = np.empty((n, 6))
        sp = None if steps is None else f64ptr(_a(steps, (n, 6)))
        check(_lib.lib().smcl_compute_phis(self.h, sp, f64ptr(out)))
        return out

    def apply_updates(self, phis=None):
        n = self.num_local_particles()  # the ABI reads / writes this shard's rows
        pp = None if phis is None else f64ptr(_a(phis, (n, 6)))
        check(_lib.lib().smcl_apply_updates(self.h, pp))

    def bayes_update(self, ll=None, nm=None, beta=2.0, floor=-80.0):
        rej = C.c_int32()
        llp = None if ll is None else f64ptr(_a(ll))
        nmp = None if nm is None else i32ptr(_a(nm, None, np.int32))
        check(_lib.lib().smcl_bayes_update(self.h, llp, nmp, beta, floor, C.byref(rej)))
        return bool(rej.value)

    def normalize_log_post(self, floor=-80.0):
        check(_lib.lib().smcl_normalize_log_post(self.h, floor))

    def smooth(self, iters=10, floor=-80.0):
        check(_lib.lib().smcl_smooth(self.h, iters, floor))

    def representative(self):
        ix, val = C.c_int64(), C.c_double()
        pose = np.empty(12)
        check(_lib.lib().smcl_representative(self.h, C.byref(ix), f64ptr(pose), C.byref(val)))
        return ix.value, pose, val.value


# ---------------------------------------------------------------- batch device math
def se3_exp(xi):
    xi = _a(xi, (-1, 6))
    out = np.empty((xi.shape[0], 12))
    check(_lib.lib().smcl_se3_exp_batch(f64ptr(xi), xi.shape[0], f64ptr(out)))
    return out


def se3_log(poses):
    poses = _a(poses, (-1, 12))
    out = np.empty((poses.shape[0], 6))
    check(_lib.lib().smcl_se3_log_batch(f64ptr(poses), poses.shape[0], f64ptr(out)))
    return out


def kernel(a, b, sigma_r=5.0, sigma_t=2.5):
    a, b = _a(a, (-1, 12)), _a(b, (-1, 12))
    out = np.empty(a.shape[0])
    check(_lib.lib().smcl_kernel_batch(f64ptr(a), f64ptr(b), a.shape[0], sigma_r, sigma_t, f64ptr(out)))
    return out


def lsh_hash(poses, frame, noise, alpha=0.1, sigma_r=5.0, sigma_t=2.5):
    poses = _a(poses, (-1, 12))
    out = np.empty(poses.shape[0], np.uint64)
    check(_lib.lib().smcl_lsh_hash_batch(f64ptr(poses), poses.shape[0], f64ptr(_a(frame, (12,))),
                                         f64ptr(_a(noise, (6,))), alpha, sigma_r, sigma_t, u64ptr(out)))
    return out


def solve_step(H, b, lam, omega_max=0.5, v_max=1.0):
    H = _a(H, (-1, 36))
    n = H.shape[0]
    lam = _a(np.broadcast_to(np.asarray(lam, np.float64), (n,)))
    out = np.empty((n, 6))
    check(_lib.lib().smcl_solve_step_batch(f64ptr(H), f64ptr(_a(b, (n, 6))), f64ptr(lam), n, omega_max, v_max,
                                           f64ptr(out)))
    return out


# ---------------------------------------------------------------- host preparation
def estimate_covariances(points, k=10, eps=1e-3):
    p = _a(points, (-1, 3))
    out = np.empty((p.shape[0], 9))
    check(_lib.lib().smcl_estimate_covariances(f64ptr(p), p.shape[0], k, eps, f64ptr(out)))
    return out


def downsample_to(points, max_points, leaf):
    p = _a(points, (-1, 3))
    out = np.empty_like(p)
    n = C.c_int64()
    check(_lib.lib().smcl_downsample_to(f64ptr(p), p.shape[0], max_points, leaf, f64ptr(out), C.byref(n)))
    return out[: n.value].copy()


def make_scan_cloud(points, cfg=None):
    """filter.cpp:86-100 -> GaussianCloud (empty when too few points)."""
    cfg = cfg or make_config()
    p = _a(points, (-1, 3))
    m = max(p.shape[0], 1)
    mu, sg = np.empty((m, 3)), np.empty((m, 9))
    n = C.c_int64()
    check(_lib.lib().smcl_make_scan_cloud(f64ptr(p), p.shape[0], C.byref(cfg), f64ptr(mu), f64ptr(sg), C.byref(n)))
    n = n.value
    return GaussianCloud(mu[:n].copy(), sg[:n].copy())


def build_nnf(cloud, resolution, padding, max_query_dist=1.0):
    sc, keep = cloud.struct()
    dims = np.zeros(3, np.int32)
    origin = np.zeros(3)
    check(_lib.lib().smcl_build_nnf(C.byref(sc), resolution, padding, max_query_dist, i32ptr(dims), f64ptr(origin),
                                    None))
    cells = np.empty(int(np.prod(dims.astype(np.int64))), np.int32)
    check(_lib.lib().smcl_build_nnf(C.byref(sc), resolution, padding, max_query_dist, i32ptr(dims), f64ptr(origin),
                                    i32ptr(cells)))
    del keep
    return dims, origin, cells


def device_count():
    n = C.c_int()
    rc = _lib.lib().smcl_device_count(C.byref(n))
    return n.value if rc == 0 else 0
