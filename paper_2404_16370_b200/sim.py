"""Synthetic workload generator (reference sim/world.cpp, sim/scenario.cpp).

Worlds, surface sampling and ray casting run in the product's host C++
(libsmcl_gpu.so); scenario scripting (trajectory, odometry, occlusions) is
plain numpy. These produce the seeded map/scan inputs used by tests and
bench.py; they are not part of the per-frame hot path.
"""
import ctypes as C
import math

import numpy as np

from . import _lib
from .abi import SmclCorridorSpec, SmclSensorSpec, f64ptr, identity_pose, make_config
from .api import GaussianCloud, make_scan_cloud

check = _lib.check
K_STREAM_SCAN, K_STREAM_ODOM, K_STREAM_MAP = 11, 12, 13  # scenario.cpp:16


def corridor_spec(**kw):
    s = SmclCorridorSpec()
    _lib.lib().smcl_sim_default_corridor(C.byref(s))
    for k, v in kw.items():
        setattr(s, k, v)
    return s


def sensor_spec(n_azimuth=16, elevations_deg=(-30.0, -10.0, 0.0, 10.0, 30.0), max_range=30.0, min_range=0.2,
                noise_sigma=0.01):
    s = SmclSensorSpec()
    s.n_azimuth = n_azimuth
    s.n_elevations = len(elevations_deg)
    for i, e in enumerate(elevations_deg):
        s.elevations_deg[i] = e
    s.max_range, s.min_range, s.noise_sigma = max_range, min_range, noise_sigma
    return s


def corridor_world(**kw):
    """world.cpp:77-133 -> (n, 9) rectangles (origin, edge_u, edge_v)."""
    spec = corridor_spec(**kw)
    n = C.c_int32()
    check(_lib.lib().smcl_sim_corridor_world(C.byref(spec), None, 0, C.byref(n)))
    out = np.empty((n.value, 9))
    check(_lib.lib().smcl_sim_corridor_world(C.byref(spec), f64ptr(out), n.value, C.byref(n)))
    return out


def box_room(size):
    size = np.ascontiguousarray(size, np.float64)
    n = C.c_int32()
    out = np.empty((6, 9))
    check(_lib.lib().smcl_sim_box_room(f64ptr(size), f64ptr(out), 6, C.byref(n)))
    return out


def _box_rects(x0, y0, z0, sx, sy, sz, floor=False):
    """Axis-aligned box as rectangles (4 walls + roof [+ floor])."""
    o = np.array([x0, y0, z0])
    ex, ey, ez = np.array([sx, 0, 0.0]), np.array([0, sy, 0.0]), np.array([0, 0, sz])
    faces = [(o, ex, ez), (o + ey, ex, ez), (o, ey, ez), (o + ex, ey, ez), (o + ez, ex, ey)]
    if floor:
        faces.append((o, ex, ey))
    return [np.concatenate(f) for f in faces]


def outdoor_world(size=(280.0, 200.0, 30.0), block=40.0, street=12.0, seed=7):
    """Builder-defined outdoor world for the kidnap configs (the
    reference has no outdoor preset): a ground plane of size[0] x size[1] m
    and a city grid of blocks (pitch `block`, streets `street` wide) holding
    one or two box buildings each, heights up to size[2]. Seeded; rects in the
    reference's (origin, edge_u, edge_v) form so sample_world / ray casting
    (world.cpp) consume them unchanged."""
    sx, sy, sz = size
    rng = np.random.default_rng(seed)
    rects = [np.concatenate([[0.0, 0.0, 0.0], [sx, 0.0, 0.0], [0.0, sy, 0.0]])]  # ground
    for bx in np.arange(street, sx - block / 2, block):
        for by in np.arange(street, sy - block / 2, block):
            w = block - street
            n_b = 1 + int(rng.integers(0, 2))
            for b in range(n_b):
                fx = rng.uniform(0.4, 0.9) * w / n_b
                fy = rng.uniform(0.5, 0.95) * w
                x0 = bx + b * w / n_b + rng.uniform(0.0, w / n_b - fx)
                y0 = by + rng.uniform(0.0, w - fy)
                h = rng.uniform(0.25, 1.0) * sz
                rects += _box_rects(x0, y0, 0.0, fx, fy, h)
    return np.array(rects)


def world_bounds(rects):
    r = np.asarray(rects).reshape(-1, 9)
    o, u, v = r[:, 0:3], r[:, 3:6], r[:, 6:9]
    corners = np.concatenate([o, o + u, o + v, o + u + v])
    return np.concatenate([corners.min(0), corners.max(0)])


def sample_world_points(rects, density, seed):
    rects = np.ascontiguousarray(rects, np.float64)
    n = C.c_int64()
    check(_lib.lib().smcl_sim_sample_world(f64ptr(rects), rects.shape[0], density, C.c_uint64(seed), 10, 1e-3, None,
                                           None, C.byref(n)))
    mu = np.empty((n.value, 3))
    check(_lib.lib().smcl_sim_sample_world(f64ptr(rects), rects.shape[0], density, C.c_uint64(seed), 10, 1e-3,
                                           f64ptr(mu), None, C.byref(n)))
    return mu


def sample_world(rects, density, seed, covariance_k=10, epsilon_plane=1e-3):
    """world.cpp:140-160 -> GaussianCloud with plane-model covariances."""
    rects = np.ascontiguousarray(rects, np.float64)
    n = C.c_int64()
    check(_lib.lib().smcl_sim_sample_world(f64ptr(rects), rects.shape[0], density, C.c_uint64(seed), covariance_k,
                                           epsilon_plane, None, None, C.byref(n)))
    mu, sg = np.empty((n.value, 3)), np.empty((n.value, 9))
    check(_lib.lib().smcl_sim_sample_world(f64ptr(rects), rects.shape[0], density, C.c_uint64(seed), covariance_k,
                                           epsilon_plane, f64ptr(mu), f64ptr(sg), C.byref(n)))
    return GaussianCloud(mu, sg)


def simulate_scan_points(rects, pose, sensor, rng_state):
    """world.cpp:162-181. rng_state: SplitMix64 state (int); returns (points, new_state)."""
    rects = np.ascontiguousarray(rects, np.float64)
    st = C.c_uint64(rng_state & (2**64 - 1))
    out = np.empty((sensor.n_azimuth * sensor.n_elevations, 3))
    n = C.c_int64()
    check(_lib.lib().smcl_sim_scan(f64ptr(rects), rects.shape[0], f64ptr(np.ascontiguousarray(pose, np.float64)),
                                   C.byref(sensor), C.byref(st), f64ptr(out), C.byref(n)))
    return out[: n.value].copy(), st.value


# ---------------------------------------------------------------- numpy SE3 helpers (input generation only)
_M64 = (1 << 64) - 1


def splitmix_next(state):
    state = (state + 0x9E3779B97F4A7C15) & _M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return state, z ^ (z >> 31)


def mix_seed(a, b, c=None):
    """rng.hpp:33-40."""
    s = (a ^ ((b + 0x9E3779B97F4A7C15 + ((a << 6) & _M64) + (a >> 2)) & _M64)) & _M64
    _, v = splitmix_next(s)
    return v if c is None else mix_seed(v, c)


def normal6(state):
    out = []
    for _ in range(3):
        state, a = splitmix_next(state)
        state, b = splitmix_next(state)
        u1 = 1.0 - (a >> 11) * 2.0**-53
        u2 = (b >> 11) * 2.0**-53
        r = math.sqrt(-2.0 * math.log(u1))
        ang = 2.0 * math.pi * u2
        out += [r * math.cos(ang), r * math.sin(ang)]
    return np.array(out), state


def skew(w):
    return np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])


def se3_exp(xi):
    w, v = np.asarray(xi[:3], float), np.asarray(xi[3:], float)
    th2 = float(w @ w)
    th = math.sqrt(th2)
    if th < 1e-4:
        a, b, c = 1 - th2 / 6 + th2 * th2 / 120, 0.5 - th2 / 24 + th2 * th2 / 720, 1 / 6 - th2 / 120 + th2 * th2 / 5040
    else:
        a, b, c = math.sin(th) / th, 2 * math.sin(0.5 * th) ** 2 / th2, (1 - math.sin(th) / th) / th2
    s = skew(w)
    R = np.eye(3) + a * s + b * (s @ s)
    t = (np.eye(3) + b * s + c * (s @ s)) @ v
    return pose_of(R, t)


def pose_of(R, t):
    p = np.empty(12)
    p[:9] = np.asarray(R).reshape(9)
    p[9:] = t
    return p


def compose(a, b):
    Ra, Rb = a[:9].reshape(3, 3), b[:9].reshape(3, 3)
    return pose_of(Ra @ Rb, Ra @ b[9:] + a[9:])


def inverse(a):
    R = a[:9].reshape(3, 3).T
    return pose_of(R, -(R @ a[9:]))


def yaw_rotation(yaw):
    c, s = math.cos(yaw), math.sin(yaw)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


# ---------------------------------------------------------------- scenarios (scenario.cpp)
class Scenario:
    def __init__(self, name, world_kind="corridor", n_frames=150, waypoints=(), occlusions=(), teleports=(),
                 box_size=(10.0, 10.0, 3.0), density=100.0, sensor=None, sensor_height=1.5, rate_hz=10.0, speed=1.0,
                 odom_sigma_rot=0.002, odom_sigma_trans=0.005, seed=1, corridor=None, outdoor=None):
        self.name, self.world_kind, self.n_frames = name, world_kind, n_frames
        self.waypoints = [np.array(w, float) for w in waypoints]
        self.occlusions, self.teleports = list(occlusions), list(teleports)
        self.box_size, self.density = np.array(box_size, float), density
        self.sensor = sensor if sensor is not None else sensor_spec()
        self.sensor_height, self.rate_hz, self.speed = sensor_height, rate_hz, speed
        self.odom_sigma_rot, self.odom_sigma_trans, self.seed = odom_sigma_rot, odom_sigma_trans, seed
        self.corridor = corridor or {}
        self.outdoor = outdoor or {}

    def build_world(self):
        if self.world_kind == "corridor":
            return corridor_world(**self.corridor)
        if self.world_kind == "box":
            return box_room(self.box_size)
        if self.world_kind == "outdoor":
            return outdoor_world(**self.outdoor)
        raise RuntimeError(f"unknown world kind: {self.world_kind}")

    def odom_cov(self):
        d = [self.odom_sigma_rot**2] * 3 + [self.odom_sigma_trans**2] * 3
        return np.diag(d).reshape(36)

    def is_occluded(self, f):
        return any(b <= f < e for b, e in self.occlusions)


def scenario_preset(name, **kw):
    """scenario.cpp:37-67."""
    if name == "corridor_easy":
        return Scenario(name, n_frames=150, waypoints=[(6.0, 1.5, 0.0), (2.0, 1.5, 0.0), (12.0, 1.5, 0.0)], **kw)
    if name == "corridor_kidnap":
        return Scenario(name, n_frames=440,
                        waypoints=[(5.0, 1.5, 0.0), (2.0, 1.5, 0.0), (8.0, 1.5, 0.0), (15.0, 5.5, 0.0),
                                   (15.0, 1.5, 0.0), (10.0, 1.5, 0.0), (35.0, 5.5, 0.0), (35.0, 1.5, 0.0),
                                   (38.5, 1.5, 0.0)],
                        occlusions=[(80, 180), (260, 360)],
                        teleports=[(130, (15.0, 5.5, 0.0)), (310, (35.0, 5.5, 0.0))], **kw)
    if name == "outdoor_kidnap":
        # configs[3]: drive along a street, scan blackout, teleport to another
        # street, recover (the corridor_kidnap pattern of scenario.cpp:47-58 on
        # the builder-defined outdoor world; 10 pts/m^2, 5 m/s).
        return Scenario(name, world_kind="outdoor", n_frames=90, density=10.0, speed=5.0, sensor_height=2.0,
                        waypoints=[(6.0, 6.0, 0.0), (120.0, 6.0, 0.0), (126.0, 126.0, 0.0), (250.0, 126.0, 0.0)],
                        occlusions=[(30, 50)], teleports=[(40, (126.0, 126.0, 0.0))], **kw)
    if name == "box_easy":
        return Scenario(name, world_kind="box", n_frames=60,
                        waypoints=[(3.0, 3.0, 0.0), (7.0, 3.0, 0.0), (7.0, 7.0, 0.0)], **kw)
    raise RuntimeError(f"unknown scenario preset: {name}")


def build_trajectory(sc):
    """scenario.cpp:183-243: frame-by-frame ground truth poses (12-vectors)."""
    dt = 1.0 / sc.rate_hz
    pos = sc.waypoints[0].copy()
    pos[2] = sc.sensor_height
    target = 1
    heading = np.array([1.0, 0.0, 0.0])
    if len(sc.waypoints) > 1:
        d = sc.waypoints[1] - sc.waypoints[0]
        d[2] = 0.0
        if np.linalg.norm(d) > 1e-9:
            heading = d / np.linalg.norm(d)
    traj = []
    for f in range(sc.n_frames):
        occluded = sc.is_occluded(f)
        for tf, tp in sc.teleports:
            if tf == f:
                pos[:2] = tp[:2]
                pos[2] = sc.sensor_height
                for wi, w in enumerate(sc.waypoints):
                    if np.linalg.norm(w[:2] - pos[:2]) < 0.5:
                        target = wi + 1
        if not occluded and target < len(sc.waypoints):
            budget = sc.speed * dt
            while budget > 1e-12 and target < len(sc.waypoints):
                goal = sc.waypoints[target].copy()
                goal[2] = sc.sensor_height
                to_goal = goal - pos
                dist = np.linalg.norm(to_goal)
                if dist < 1e-9:
                    target += 1
                    continue
                dirv = to_goal / dist
                heading = 0.7 * heading + 0.3 * dirv
                heading[2] = 0.0
                if np.linalg.norm(heading) < 1e-9:
                    heading = dirv
                heading = heading / np.linalg.norm(heading)
                step = min(dist, budget)
                pos = pos + step * dirv
                budget -= step
                if step >= dist - 1e-12:
                    target += 1
        traj.append(pose_of(yaw_rotation(math.atan2(heading[1], heading[0])), pos.copy()))
    return traj


def build_odometry(sc, truth):
    """scenario.cpp:245-275 -> list of (delta, cov36, valid)."""
    out = []
    sigma = np.array([sc.odom_sigma_rot] * 3 + [sc.odom_sigma_trans] * 3)
    for f in range(len(truth)):
        if sc.is_occluded(f):
            out.append((identity_pose(), np.zeros(36), False))
            continue
        dgt = identity_pose() if f == 0 else compose(inverse(truth[f - 1]), truth[f])
        z, _ = normal6(mix_seed(sc.seed, K_STREAM_ODOM, f))
        out.append((compose(dgt, se3_exp(sigma * z)), sc.odom_cov(), True))
    return out


def scan_points_for_frame(sc, rects, truth, f):
    if sc.is_occluded(f):
        return np.zeros((0, 3))
    pts, _ = simulate_scan_points(rects, truth[f], sc.sensor, mix_seed(sc.seed, K_STREAM_SCAN, f))
    return pts


def scan_for_frame(sc, rects, truth, f, cfg=None):
    return make_scan_cloud(scan_points_for_frame(sc, rects, truth, f), cfg or make_config())


def scenario_map(sc, cfg=None):
    cfg = cfg or make_config()
    rects = sc.build_world()
    return rects, sample_world(rects, sc.density, mix_seed(sc.seed, K_STREAM_MAP), cfg.covariance_k,
                               cfg.epsilon_plane)
