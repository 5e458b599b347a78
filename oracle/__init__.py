"""ORACLE — test infrastructure only.

CPU restatement of the steinmcl reference hot path (/root/reference/proj),
compiled from oracle/src/*.cpp into oracle/build/libsmcl_oracle.so. Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package; the product (paper_2404_16370_b200) never does.

Parity status: pinned by the reference's own known-answer tests re-expressed in
tests/test_oracle_*.py (the reference ships no golden-vector files and cannot be
compiled here: it needs Eigen3, absent from the image). Ulp-level agreement with
an Eigen build is unpinned — see DESIGN.md.
"""
import ctypes as C
import os
import subprocess

import numpy as np

from paper_2404_16370_b200.abi import (SmclCloud, SmclConfig, SmclFrameResult, SmclNeighborStats, SmclOdom,
                                       SmclParticlesView, Particles, cloud_struct, f32ptr, f64ptr, i32ptr,
                                       make_config, odom_struct)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "build", "libsmcl_oracle.so")
_lib = None


def build():
    subprocess.check_call(["make", "-s", "-C", _HERE])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


def _declare(L):
    d, i32, i64, u64, vp = C.c_double, C.c_int32, C.c_int64, C.c_uint64, C.c_void_p
    P = C.POINTER
    sig = {
        "orc_last_error": (C.c_char_p, []),
        "orc_se3_exp": (None, [P(d), P(d)]),
        "orc_se3_log": (None, [P(d), P(d)]),
        "orc_compose": (None, [P(d), P(d), P(d)]),
        "orc_inverse": (None, [P(d), P(d)]),
        "orc_renormalize": (None, [P(d)]),
        "orc_rotation_drift": (d, [P(d)]),
        "orc_mix_seed": (u64, [u64, u64]),
        "orc_splitmix_next": (u64, [P(u64)]),
        "orc_normal6": (None, [P(u64), P(d)]),
        "orc_uniform01": (d, [P(u64)]),
        "orc_random_rotation": (None, [P(u64), P(d)]),
        "orc_kernel": (d, [P(d), P(d), d, d]),
        "orc_kernel_grad": (None, [P(d), P(d), d, d, P(d)]),
        "orc_lsh_hash": (u64, [P(d), P(d), P(d), d, d, d]),
        "orc_random_lsh_frame": (None, [P(u64), P(d), P(d)]),
        "orc_next_prime": (i32, [i32]),
        "orc_solve_step": (C.c_int, [P(d), P(d), d, d, d, P(d)]),
        "orc_covariance_sqrt": (None, [P(d), P(d)]),
        "orc_map_create": (vp, [P(SmclCloud), d, d, d]),
        "orc_map_destroy": (None, [vp]),
        "orc_map_nnf": (None, [vp, P(i32), P(d), P(i32)]),
        "orc_map_lookup": (i32, [vp, P(d)]),
        "orc_estimate_covariances": (C.c_int, [P(d), i64, C.c_int, d, P(d)]),
        "orc_downsample_to": (C.c_int, [P(d), i64, i64, d, P(d), P(i64)]),
        "orc_make_scan_cloud": (C.c_int, [P(d), i64, P(SmclConfig), P(d), P(d), P(i64)]),
        "orc_evaluate_all": (C.c_int, [vp, P(SmclCloud), P(d), i64, P(SmclConfig), P(d), P(d), P(i32), P(d),
                                       P(d), C.c_int]),
        "orc_evaluate_likelihoods": (C.c_int, [vp, P(SmclCloud), P(d), i64, P(SmclConfig), P(d), P(i32),
                                               C.c_int]),
        "orc_update_neighbors": (C.c_int, [P(SmclParticlesView), P(SmclConfig), u64, P(d), P(SmclNeighborStats),
                                           C.c_int]),
        "orc_brute_knn": (C.c_int, [P(d), i64, C.c_int, d, d, P(i32)]),
        "orc_compute_phis": (C.c_int, [P(d), P(d), P(i32), P(i32), i64, C.c_int, P(SmclConfig), P(d), C.c_int]),
        "orc_apply_updates": (C.c_int, [P(d), P(d), i64]),
        "orc_predict": (C.c_int, [P(d), i64, P(d), P(d), u64]),
        "orc_init_uniform": (C.c_int, [i64, C.c_int, P(d), C.c_int, u64, P(SmclParticlesView)]),
        "orc_normalize_log_post": (C.c_int, [P(d), i64, d]),
        "orc_bayes_update": (C.c_int, [P(d), P(d), P(i32), i64, d, d, P(i32)]),
        "orc_smooth": (C.c_int, [P(d), P(i32), P(C.c_float), P(i32), i64, C.c_int, C.c_int, d, C.c_int]),
        "orc_representative": (C.c_int, [P(d), i64, P(i64), P(d)]),
        "orc_engine_create": (vp, [P(SmclCloud), P(SmclConfig)]),
        "orc_engine_destroy": (None, [vp]),
        "orc_engine_init_uniform": (C.c_int, [vp, P(d)]),
        "orc_engine_step": (C.c_int, [vp, P(SmclCloud), P(SmclOdom), P(SmclFrameResult)]),
        "orc_engine_num_particles": (i64, [vp]),
        "orc_engine_get": (C.c_int, [vp, P(SmclParticlesView)]),
        "orc_engine_set": (C.c_int, [vp, P(SmclParticlesView)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


class OracleError(RuntimeError):
    pass


_EXC = {1: ValueError, 2: RuntimeError, 3: RuntimeError}


def _check(rc):
    if rc != 0:
        raise _EXC.get(rc, OracleError)(lib().orc_last_error().decode())


def _a(x, shape=None, dtype=np.float64):
    a = np.ascontiguousarray(x, dtype=dtype)
    return a if shape is None else a.reshape(shape)


# ---------------------------------------------------------------- primitives
def se3_exp(xi):
    xi = _a(xi, (-1, 6))
    out = np.empty((xi.shape[0], 12))
    for i in range(xi.shape[0]):
        lib().orc_se3_exp(f64ptr(xi[i]), f64ptr(out[i]))
    return out


def se3_log(poses):
    poses = _a(poses, (-1, 12))
    out = np.empty((poses.shape[0], 6))
    for i in range(poses.shape[0]):
        lib().orc_se3_log(f64ptr(poses[i]), f64ptr(out[i]))
    return out


def compose(a, b):
    a, b = _a(a, (12,)), _a(b, (12,))
    out = np.empty(12)
    lib().orc_compose(f64ptr(a), f64ptr(b), f64ptr(out))
    return out


def inverse(a):
    a = _a(a, (12,))
    out = np.empty(12)
    lib().orc_inverse(f64ptr(a), f64ptr(out))
    return out


def renormalize(p):
    p = _a(p, (12,)).copy()
    lib().orc_renormalize(f64ptr(p))
    return p


def rotation_drift(p):
    return lib().orc_rotation_drift(f64ptr(_a(p, (12,))))


def mix_seed(a, b, c=None):
    r = lib().orc_mix_seed(C.c_uint64(a & (2**64 - 1)), C.c_uint64(b & (2**64 - 1)))
    return r if c is None else lib().orc_mix_seed(C.c_uint64(r), C.c_uint64(c & (2**64 - 1)))


class SplitMix64:
    """rng.hpp:15-31 (drives the oracle's own generator)."""

    def __init__(self, seed):
        self.state = C.c_uint64(seed & (2**64 - 1))

    def __call__(self):
        return lib().orc_splitmix_next(C.byref(self.state))

    def uniform01(self):
        return lib().orc_uniform01(C.byref(self.state))

    def uniform_range(self, lo, hi):
        return lo + (hi - lo) * self.uniform01()

    def normal6(self):
        z = np.empty(6)
        lib().orc_normal6(C.byref(self.state), f64ptr(z))
        return z

    def normal01(self):
        # normal01 draws a pair and keeps z0 (rng.hpp:61-65): same stream use as normal6's first pair.
        st = self.state.value
        z = np.empty(6)
        tmp = C.c_uint64(st)
        lib().orc_normal6(C.byref(tmp), f64ptr(z))
        # normal6 consumed 6 draws; normal01 consumes 2.
        self.state = C.c_uint64((st + 2 * 0x9E3779B97F4A7C15) & (2**64 - 1))
        return z[0]

    def random_rotation(self):
        r = np.empty(9)
        lib().orc_random_rotation(C.byref(self.state), f64ptr(r))
        return r

    def random_lsh_frame(self, bounds):
        f = np.empty(12)
        b = _a(bounds, (6,))
        lib().orc_random_lsh_frame(C.byref(self.state), f64ptr(b), f64ptr(f))
        return f


def kernel(a, b, sigma_r=5.0, sigma_t=2.5):
    return lib().orc_kernel(f64ptr(_a(a, (12,))), f64ptr(_a(b, (12,))), sigma_r, sigma_t)


def kernel_grad(a, b, sigma_r=5.0, sigma_t=2.5):
    g = np.empty(6)
    lib().orc_kernel_grad(f64ptr(_a(a, (12,))), f64ptr(_a(b, (12,))), sigma_r, sigma_t, f64ptr(g))
    return g


def lsh_hash(pose, frame, noise, alpha=0.1, sigma_r=5.0, sigma_t=2.5):
    return lib().orc_lsh_hash(f64ptr(_a(pose, (12,))), f64ptr(_a(frame, (12,))), f64ptr(_a(noise, (6,))),
                              alpha, sigma_r, sigma_t)


def next_prime_at_least(n):
    return lib().orc_next_prime(n)


def solve_step(H, b, lam, omega_max=0.5, v_max=1.0):
    out = np.empty(6)
    _check(lib().orc_solve_step(f64ptr(_a(H, (36,))), f64ptr(_a(b, (6,))), lam, omega_max, v_max, f64ptr(out)))
    return out


def covariance_sqrt(cov):
    L = np.empty(36)
    lib().orc_covariance_sqrt(f64ptr(_a(cov, (36,))), f64ptr(L))
    return L.reshape(6, 6)


# ---------------------------------------------------------------- map / scan prep
class OracleMap:
    """GaussianCloud + NearestNeighborField (build_nnf, nnf.cpp:10-96)."""

    def __init__(self, mu, sigma, bounds=None, resolution=0.1, padding=0.5, max_query_dist=1.0):
        self._c, self._keep = cloud_struct(mu, sigma, bounds)
        self.h = lib().orc_map_create(C.byref(self._c), resolution, padding, max_query_dist)
        if not self.h:
            raise ValueError(lib().orc_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_map_destroy(self.h)
            self.h = None

    def nnf(self):
        dims = np.zeros(3, np.int32)
        origin = np.zeros(3)
        lib().orc_map_nnf(self.h, i32ptr(dims), f64ptr(origin), None)
        cells = np.empty(int(np.prod(dims.astype(np.int64))), np.int32)
        lib().orc_map_nnf(self.h, i32ptr(dims), f64ptr(origin), i32ptr(cells))
        return dims, origin, cells

    def lookup(self, p):
        return lib().orc_map_lookup(self.h, f64ptr(_a(p, (3,))))


def estimate_covariances(points, k=10, eps=1e-3):
    p = _a(points, (-1, 3))
    out = np.empty((p.shape[0], 9))
    _check(lib().orc_estimate_covariances(f64ptr(p), p.shape[0], k, eps, f64ptr(out)))
    return out


def downsample_to(points, max_points, leaf):
    p = _a(points, (-1, 3))
    out = np.empty_like(p)
    n = C.c_int64()
    _check(lib().orc_downsample_to(f64ptr(p), p.shape[0], max_points, leaf, f64ptr(out), C.byref(n)))
    return out[: n.value].copy()


def make_scan_cloud(points, cfg=None):
    cfg = cfg or make_config()
    p = _a(points, (-1, 3))
    mu = np.empty((max(p.shape[0], 1), 3))
    sg = np.empty((max(p.shape[0], 1), 9))
    n = C.c_int64()
    _check(lib().orc_make_scan_cloud(f64ptr(p), p.shape[0], C.byref(cfg), f64ptr(mu), f64ptr(sg), C.byref(n)))
    return mu[: n.value].copy(), sg[: n.value].copy()


# ---------------------------------------------------------------- GICP
def evaluate_all(omap, scan_mu, scan_sigma, poses, cfg=None, serial=False, want_system=False):
    cfg = cfg or make_config()
    sc, keep = cloud_struct(scan_mu, scan_sigma)
    poses = _a(poses, (-1, 12))
    n = poses.shape[0]
    steps, ll, nm = np.empty((n, 6)), np.empty(n), np.empty(n, np.int32)
    H = np.empty((n, 6, 6)) if want_system else None
    b = np.empty((n, 6)) if want_system else None
    _check(lib().orc_evaluate_all(omap.h, C.byref(sc), f64ptr(poses), n, C.byref(cfg), f64ptr(steps), f64ptr(ll),
                                  i32ptr(nm), f64ptr(H) if want_system else None,
                                  f64ptr(b) if want_system else None, int(serial)))
    del keep
    return (steps, ll, nm, H, b) if want_system else (steps, ll, nm)


def evaluate_likelihoods(omap, scan_mu, scan_sigma, poses, cfg=None, serial=False):
    cfg = cfg or make_config()
    sc, keep = cloud_struct(scan_mu, scan_sigma)
    poses = _a(poses, (-1, 12))
    n = poses.shape[0]
    ll, nm = np.empty(n), np.empty(n, np.int32)
    _check(lib().orc_evaluate_likelihoods(omap.h, C.byref(sc), f64ptr(poses), n, C.byref(cfg), f64ptr(ll),
                                          i32ptr(nm), int(serial)))
    del keep
    return ll, nm


# ---------------------------------------------------------------- particles
def update_neighbors(parts, cfg, pass_seed, bounds, serial=False):
    """In-place on a Particles object; returns NeighborStats as a dict."""
    v = parts.view()
    st = SmclNeighborStats()
    b = _a(bounds, (6,))
    _check(lib().orc_update_neighbors(C.byref(v), C.byref(cfg), C.c_uint64(pass_seed & (2**64 - 1)), f64ptr(b),
                                      C.byref(st), int(serial)))
    return st.to_dict()


def brute_force_kernel_knn(poses, k, sigma_r=5.0, sigma_t=2.5):
    poses = _a(poses, (-1, 12))
    out = np.full((poses.shape[0], k), -1, np.int32)
    _check(lib().orc_brute_knn(f64ptr(poses), poses.shape[0], k, sigma_r, sigma_t, i32ptr(out)))
    return out


def compute_phis(poses, steps, idx, count, cfg=None, serial=False):
    cfg = cfg or make_config()
    poses, steps = _a(poses, (-1, 12)), _a(steps, (-1, 6))
    n = poses.shape[0]
    idx = _a(idx, (n, -1), np.int32)
    count = _a(count, (n,), np.int32)
    out = np.empty((n, 6))
    _check(lib().orc_compute_phis(f64ptr(poses), f64ptr(steps), i32ptr(idx), i32ptr(count), n, idx.shape[1],
                                  C.byref(cfg), f64ptr(out), int(serial)))
    return out


def apply_updates(poses, phis):
    poses = _a(poses, (-1, 12)).copy()
    _check(lib().orc_apply_updates(f64ptr(poses), f64ptr(_a(phis, (-1, 6))), poses.shape[0]))
    return poses


def predict(poses, delta, cov, frame_seed):
    poses = _a(poses, (-1, 12)).copy()
    _check(lib().orc_predict(f64ptr(poses), poses.shape[0], f64ptr(_a(delta, (12,))), f64ptr(_a(cov, (36,))),
                             C.c_uint64(frame_seed & (2**64 - 1))))
    return poses


def init_uniform(n, k, bounds, full_rotation=True, seed=1):
    p = Particles(n, k)
    v = p.view()
    _check(lib().orc_init_uniform(n, k, f64ptr(_a(bounds, (6,))), int(full_rotation), C.c_uint64(seed), C.byref(v)))
    return p


# ---------------------------------------------------------------- posterior
def normalize_log_post(lp, floor=-80.0):
    lp = _a(lp).copy()
    _check(lib().orc_normalize_log_post(f64ptr(lp), lp.shape[0], floor))
    return lp


def bayes_update(lp, ll, nm, beta, floor=-80.0):
    lp = _a(lp).copy()
    rej = C.c_int32()
    _check(lib().orc_bayes_update(f64ptr(lp), f64ptr(_a(ll)), i32ptr(_a(nm, None, np.int32)), lp.shape[0], beta,
                                  floor, C.byref(rej)))
    return lp, bool(rej.value)


def smooth(lp, idx, kval, count, iters, floor=-80.0, serial=False):
    lp = _a(lp).copy()
    n = lp.shape[0]
    idx = _a(idx, (n, -1), np.int32)
    kval = _a(kval, (n, -1), np.float32)
    _check(lib().orc_smooth(f64ptr(lp), i32ptr(idx), f32ptr(kval), i32ptr(_a(count, (n,), np.int32)), n,
                            idx.shape[1], iters, floor, int(serial)))
    return lp


def representative(lp):
    idx, val = C.c_int64(), C.c_double()
    lp = _a(lp)
    _check(lib().orc_representative(f64ptr(lp), lp.shape[0], C.byref(idx), C.byref(val)))
    return idx.value, val.value


# ---------------------------------------------------------------- engine
class FilterEngine:
    """FilterEngine (filter.hpp:104-130) restated on the CPU."""

    def __init__(self, map_mu, map_sigma, cfg, bounds=None):
        self._c, self._keep = cloud_struct(map_mu, map_sigma, bounds)
        self.cfg = cfg
        self.h = lib().orc_engine_create(C.byref(self._c), C.byref(cfg))
        if not self.h:
            raise ValueError(lib().orc_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_engine_destroy(self.h)
            self.h = None

    def init_uniform(self, bounds):
        _check(lib().orc_engine_init_uniform(self.h, f64ptr(_a(bounds, (6,)))))

    def step(self, scan_mu, scan_sigma, delta=None, cov=None, valid=True):
        if scan_mu is None or len(scan_mu) == 0:
            sc, keep = cloud_struct(np.zeros((0, 3)), np.zeros((0, 9)))
        else:
            sc, keep = cloud_struct(scan_mu, scan_sigma)
        o = odom_struct(delta, cov, valid)
        r = SmclFrameResult()
        _check(lib().orc_engine_step(self.h, C.byref(sc), C.byref(o), C.byref(r)))
        del keep
        return r.to_dict()

    def particles(self):
        n = lib().orc_engine_num_particles(self.h)
        p = Particles(n, self.cfg.k_neighbors)
        v = p.view()
        _check(lib().orc_engine_get(self.h, C.byref(v)))
        return p

    def set_particles(self, p):
        v = p.view()
        _check(lib().orc_engine_set(self.h, C.byref(v)))
