"""ctypes mirror of the C ABI structs in include/smcl_gpu.h.

Pure type definitions shared by the product bindings (``_lib.py``) and the
test-side oracle wrapper, so both receive byte-identical inputs.
"""
import ctypes as C

import numpy as np

SMCL_OK, SMCL_EINVAL, SMCL_ERUNTIME, SMCL_ELOGIC, SMCL_ECUDA, SMCL_ENCCL = range(6)
SMCL_MAX_HIST = 1026

_f64p = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)


class SmclConfig(C.Structure):
    """FilterConfig (reference include/steinmcl/filter.hpp:17-51), flattened."""

    _fields_ = [
        ("n_particles", C.c_int32),
        ("k_neighbors", C.c_int32),
        ("sigma_r", C.c_double),
        ("sigma_t", C.c_double),
        ("repulsion_gain", C.c_double),
        ("lsh_alpha", C.c_double),
        ("lsh_noise_sigma", C.c_double),
        ("lsh_buckets_factor", C.c_double),
        ("lsh_n_buckets", C.c_int32),
        ("lsh_bucket_capacity", C.c_int32),
        ("reorder_particles", C.c_int32),
        ("smooth_iters", C.c_int32),
        ("nnf_resolution", C.c_double),
        ("nnf_max_query_dist", C.c_double),
        ("nnf_padding", C.c_double),
        ("beta", C.c_double),
        ("n_svgd_iters", C.c_int32),
        ("gn_scan_stride", C.c_int32),
        ("damping_scale", C.c_double),
        ("omega_max", C.c_double),
        ("v_max", C.c_double),
        ("min_match_fraction", C.c_double),
        ("miss_cost", C.c_double),
        ("log_post_floor", C.c_double),
        ("covariance_k", C.c_int32),
        ("n_scan_max", C.c_int32),
        ("epsilon_plane", C.c_double),
        ("scan_voxel_leaf", C.c_double),
        ("sensor_noise_sigma", C.c_double),
        ("diffusion_sigma_rot", C.c_double),
        ("diffusion_sigma_trans", C.c_double),
        ("full_rotation", C.c_int32),
        ("likelihood_mode", C.c_int32),
        ("seed", C.c_uint64),
    ]


# Reference defaults (filter.hpp:17-51, svgd.hpp:13-21, neighbor_search.hpp:13-21, gicp.hpp:45-57).
DEFAULT_CONFIG = dict(
    n_particles=10000, k_neighbors=20, sigma_r=5.0, sigma_t=2.5, repulsion_gain=1.0,
    lsh_alpha=0.1, lsh_noise_sigma=0.5, lsh_buckets_factor=2.0, lsh_n_buckets=0,
    lsh_bucket_capacity=64, reorder_particles=1, smooth_iters=10, nnf_resolution=0.1,
    nnf_max_query_dist=1.0, nnf_padding=0.5, beta=2.0, n_svgd_iters=1, gn_scan_stride=1,
    damping_scale=1e-3, omega_max=0.5, v_max=1.0, min_match_fraction=0.5, miss_cost=25.0,
    log_post_floor=-80.0, covariance_k=10, n_scan_max=1000, epsilon_plane=1e-3,
    scan_voxel_leaf=0.05, sensor_noise_sigma=0.01, diffusion_sigma_rot=0.02,
    diffusion_sigma_trans=0.5, full_rotation=1, likelihood_mode=0, seed=1,
)

# Desk-scale calibration, reference proj/configs/corridor.cfg:1-10.
CORRIDOR_CFG = dict(sigma_r=50.0, sigma_t=25.0, repulsion_gain=0.005, lsh_alpha=0.016, beta=5.0,
                    miss_cost=50.0, gn_scan_stride=2, nnf_resolution=0.1, nnf_max_query_dist=1.0)


def make_config(**overrides):
    d = dict(DEFAULT_CONFIG)
    for k, v in overrides.items():
        if k not in d:
            raise KeyError(f"unknown config key: {k}")
        d[k] = v
    c = SmclConfig()
    for k, v in d.items():
        if isinstance(v, bool):
            v = int(v)
        setattr(c, k, v)
    return c


class SmclCloud(C.Structure):
    _fields_ = [("n", C.c_int64), ("mu", _f64p), ("sigma", _f64p), ("bounds", _f64p)]


class SmclOdom(C.Structure):
    _fields_ = [("delta", C.c_double * 12), ("cov", C.c_double * 36), ("valid", C.c_int32)]


class SmclNeighborStats(C.Structure):
    _fields_ = [
        ("n_buckets", C.c_int64),
        ("buckets_used", C.c_int64),
        ("overflow_dropped", C.c_int64),
        ("mean_kernel", C.c_double),
        ("hist_len", C.c_int32),
        ("occupancy_hist", C.c_int64 * SMCL_MAX_HIST),
    ]

    def to_dict(self):
        return dict(n_buckets=self.n_buckets, buckets_used=self.buckets_used,
                    overflow_dropped=self.overflow_dropped, mean_kernel=self.mean_kernel,
                    occupancy_hist=list(self.occupancy_hist[: self.hist_len]))


class SmclFrameResult(C.Structure):
    _fields_ = [
        ("representative", C.c_double * 12),
        ("rep_log_post", C.c_double),
        ("rep_index", C.c_int64),
        ("rep_id", C.c_int32),
        ("scan_empty", C.c_int32),
        ("observation_rejected", C.c_int32),
        ("n_particles", C.c_int64),
        ("mean_n_matched", C.c_double),
        ("predict_ms", C.c_double),
        ("neighbor_ms", C.c_double),
        ("likelihood_ms", C.c_double),
        ("update_ms", C.c_double),
        ("posterior_ms", C.c_double),
        ("total_ms", C.c_double),
        ("neighbor_stats", SmclNeighborStats),
    ]

    def to_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k not in ("representative", "neighbor_stats")}
        d["representative"] = np.array(self.representative[:], dtype=np.float64)
        d["neighbor_stats"] = self.neighbor_stats.to_dict()
        return d


class SmclStepProfile(C.Structure):
    _fields_ = [(k, C.c_double) for k in (
        "predict_ms", "lsh_keys_ms", "sort_ms", "reorder_ms", "segments_ms", "refresh_gather_ms", "nb_stats_ms",
        "gn_kernel_ms", "solve_ms", "svgd_ms", "ll_kernel_ms", "bayes_ms", "smooth_ms", "rep_ms", "total_ms")] + [
        ("gn_points", C.c_int64), ("ll_points", C.c_int64), ("gn_matched", C.c_int64), ("ll_matched", C.c_int64),
        ("fast_path", C.c_int32), ("n_svgd_iters", C.c_int32), ("kernel_launches", C.c_int64),
        ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
        ("hash_guard_flagged", C.c_int64), ("hash_guard_replays", C.c_int64)]

    def to_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class SmclParticlesView(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("k", C.c_int32),
        ("poses", _f64p),
        ("log_post", _f64p),
        ("id", _i32p),
        ("idx", _i32p),
        ("kval", C.POINTER(C.c_float)),
        ("count", _i32p),
    ]


class SmclCorridorSpec(C.Structure):
    _fields_ = [
        ("corridor_length", C.c_double), ("corridor_width", C.c_double), ("height", C.c_double),
        ("n_rooms", C.c_int32), ("furniture", C.c_int32),
        ("room_width", C.c_double), ("room_depth", C.c_double), ("door_width", C.c_double),
        ("door_height", C.c_double),
    ]


class SmclSensorSpec(C.Structure):
    _fields_ = [
        ("n_azimuth", C.c_int32), ("n_elevations", C.c_int32), ("elevations_deg", C.c_double * 64),
        ("max_range", C.c_double), ("min_range", C.c_double), ("noise_sigma", C.c_double),
    ]


# int (*allgather)(void* ctx, const void* send, void* recv, uint64_t bytes, void* stream)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)
ALLTOALLV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.c_void_p,
                           C.POINTER(C.c_uint64), C.c_void_p)


class SmclComm(C.Structure):
    """smcl_comm: the collective backend of a sharded engine."""
    _fields_ = [("ctx", C.c_void_p), ("rank", C.c_int32), ("world", C.c_int32), ("allgather", ALLGATHER_FN),
                ("alltoallv", ALLTOALLV_FN)]


def f64ptr(a):
    return a.ctypes.data_as(_f64p)


def i32ptr(a):
    return a.ctypes.data_as(_i32p)


def f32ptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def u64ptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def cloud_struct(mu, sigma, bounds=None):
    """Build an SmclCloud over numpy arrays; returns (struct, keepalive)."""
    mu = np.ascontiguousarray(mu, dtype=np.float64).reshape(-1, 3)
    sigma = np.ascontiguousarray(sigma, dtype=np.float64).reshape(-1, 9)
    keep = [mu, sigma]
    b = None
    if bounds is not None:
        bounds = np.ascontiguousarray(bounds, dtype=np.float64).reshape(6)
        keep.append(bounds)
        b = f64ptr(bounds)
    c = SmclCloud(mu.shape[0], f64ptr(mu), f64ptr(sigma), b)
    return c, keep


class Particles:
    """Host-side ParticleSet (particle_set.hpp:16-27) as numpy SoA arrays."""

    def __init__(self, n, k):
        self.poses = np.zeros((n, 12), np.float64)
        self.log_post = np.zeros(n, np.float64)
        self.id = np.zeros(n, np.int32)
        self.idx = np.full((n, k), -1, np.int32)
        self.kval = np.zeros((n, k), np.float32)
        self.count = np.zeros(n, np.int32)

    @property
    def n(self):
        return self.poses.shape[0]

    @property
    def k(self):
        return self.idx.shape[1]

    @classmethod
    def from_poses(cls, poses, k):
        """Uniform posterior, id = index, self-only lists (NeighborGraph::init_self)."""
        poses = np.asarray(poses, np.float64).reshape(-1, 12)
        n = poses.shape[0]
        p = cls(n, k)
        p.poses[:] = poses
        p.log_post[:] = -np.log(float(n))
        p.id[:] = np.arange(n, dtype=np.int32)
        p.idx[:, 0] = np.arange(n, dtype=np.int32)
        p.kval[:, 0] = 1.0
        p.count[:] = 1
        return p

    def copy(self):
        q = Particles(self.n, self.k)
        for name in ("poses", "log_post", "id", "idx", "kval", "count"):
            getattr(q, name)[...] = getattr(self, name)
        return q

    def view(self):
        for name in ("poses", "log_post", "id", "idx", "kval", "count"):
            a = getattr(self, name)
            assert a.flags.c_contiguous
        return SmclParticlesView(self.n, self.k, f64ptr(self.poses), f64ptr(self.log_post), i32ptr(self.id),
                                 i32ptr(self.idx), f32ptr(self.kval), i32ptr(self.count))


def odom_struct(delta=None, cov=None, valid=True):
    """OdometryInput (filter.hpp:56-60); delta None = identity, cov None = zero."""
    o = SmclOdom()
    pose = identity_pose() if delta is None else np.ascontiguousarray(delta, np.float64).reshape(12)
    C.memmove(o.delta, pose.ctypes.data, 12 * 8)
    if cov is not None:  # a fresh structure is zero-filled
        c = np.ascontiguousarray(cov, np.float64).reshape(36)
        C.memmove(o.cov, c.ctypes.data, 36 * 8)
    o.valid = 1 if valid else 0
    return o


def identity_pose():
    p = np.zeros(12)
    p[[0, 4, 8]] = 1.0
    return p
